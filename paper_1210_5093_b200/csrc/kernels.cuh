// kernels.cuh -- device-side data structures and launchers of the B200 path.
//
// Pipeline of one call:
//   1. converge_kernel  (only when I_max > kLanes): one warp per execution
//      sub-chunk runs all |I_sigma| lanes in lock-step over the first bytes and
//      merges lanes that reach the same state until <= kLanes survive.
//   2. lanes_kernel: one thread per execution sub-chunk carries its (<= kLanes)
//      lanes in registers through the rest of the sub-chunk (Alg.MatchingInitialStates
//      lines 17-19), merging converged lanes and dropping lanes in
//      absorbing states.
//   3. tree_kernel: one launch composing the sub-chunk maps into the
//      reporting chunk maps and those into the final state and its accept bit
//      (Eq.MapReduction P:819-830 hierarchically -- the on-GPU analog of the
//      two-tier merge of Fig.Merge -- with a last-arriver-continues rule per
//      tree node instead of barriers; Alg.seqmatch l.4-6 at the root).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dfa {

constexpr int kLanes = 8;          // register lanes per thread in lanes_kernel
constexpr int kConvergeLA = 4;     // lanes per thread per batch in converge_kernel's wide phase
constexpr uint32_t kSubWindow = 16;
constexpr uint32_t kNoWarpGroup = 0xFFFFFFFFu;  // lanes_kernel g_log: per-sub-chunk maps

struct DevTables {
    const uint32_t *image;      // smem image of the transition table (32-bit words)
    uint32_t image_words;
    const uint16_t *gtable;     // [nq][256] byte-indexed table (global)
    const uint8_t *byte_class;  // [256]
    const uint16_t *dom_list;   // [(nclass+1) * rs] internal I_sigma, ascending, rows padded 0xFFFF
    const uint16_t *dom_size;   // [nclass+1]
    const uint16_t *rank;       // [(nclass+1) * nq] index in dom_list or 0xFFFF
    const uint8_t *rank8;       // same as uint8 (0xFF = none) when imax < 255, else null
    const uint32_t *dead_bits;  // internal Z
    const uint32_t *absorb_bits;
    const uint32_t *accept_bits;
    const uint16_t *xlat;       // [nclass * imax_user]
    const uint16_t *ixlat;      // [nclass * rs]: user index of internal entry j, or 0xFFFF
    const uint16_t *dom_user_size; // [nclass]
    const uint32_t *dead_user_bits; // user Z (reading R1) over the user states
    const uint32_t *sticky_bits;    // states kept by every byte that is not a universal kill byte
    // two-symbol initial sets (Eq.istatesm with r = 2) for the converge stage:
    // dom2[(c1 * nclass + c2) * dom2_stride + e] = state | rank in I_c2 << 16, ascending, of
    // delta(I_c1, c2) \ Z; null when not built (small I_max, Alg.2 ablation, table too large)
    const uint32_t *dom2;
    const uint16_t *dom2_size;
    uint32_t dom2_stride;
    uint32_t nq, nclass, start_dom, imax, imax_user;
    uint32_t nq_user, ns;       // user |Q| and |Sigma|
    uint32_t rs;                // map row stride: imax rounded up to 8 (16-byte rows)
    uint32_t has_dead;          // internal Z non-empty
    uint32_t has_absorb;        // some state absorbs every byte
    uint32_t has_sticky;        // some non-absorbing state is sticky (lanes_kernel parks it)
    uint32_t stride, win_base, win_w;
    int mode;
    uint32_t q0, poison;
};

struct Plan {
    uint64_t n;
    uint32_t P;
    uint32_t m0, m;          // sub-chunks in chunk 0 / in every chunk k >= 1
    uint64_t NS;             // m0 + (P-1) m
    const uint64_t *bounds;  // device [P+1]
    uint32_t first_dom;      // domain of sub-chunk 0: start_dom ({q0}) or a lookahead class
    uint64_t in_addr;        // device address of the input (split alignment)
    uint32_t indep;          // batch: every chunk is an independent input matched from q0
    unsigned long long *work; // DFA_OPT_COUNT_WORK: [0] converge, [1] lanes lane-steps; else null
    uint32_t keep_amap;      // factored composition: lanes_kernel leaves the converge maps coded
    uint32_t use_dom2;       // converge_kernel starts internal sub-chunks from the two-symbol sets
    const void *tmap;        // device CUtensorMap of the input for TMA staging (run_lanes_tma), else null
    uint32_t magic_m0, magic_m; // min(floor(2^32 / m0), 2^32 - 1), same for m: exact 32-bit division on the device
};
inline uint32_t plan_magic(uint32_t d) { return d <= 1 ? 0xFFFFFFFFu : (uint32_t)((1ull << 32) / d); }

// Fused composition tail of lanes_kernel (grouped path, one execution sub-chunk
// per thread, so CTA b holds the contiguous leaves [b LPC, (b+1) LPC)): each CTA
// composes its own leaves per reporting chunk (Eq.MapReduction), chunks that
// straddle CTAs are finished by the last CTA to arrive (acq_rel counters), and
// the last CTA overall folds the CTA maps into the final state (Eq.SeqReduction,
// Alg.seqmatch l.4-6).  Replaces leaf_fold_kernel + compose8_kernel.
struct Fuse {
    uint32_t on;             // 1: the tail runs (then leaf_rows/leaf_dom are not written)
    uint32_t rows;           // 1: reporting rows are wanted (rep_rows and the API outputs)
    uint32_t L0, L;          // leaves of chunk 0 / of every chunk k >= 1
    uint32_t P;
    uint16_t *rep_rows, *rep_doms;     // [P][8] rank-space reporting maps, their domains
    uint16_t *user_rows, *user_row0, *e0;
    uint16_t *part_rows, *part_doms;   // [P + grid] partial maps of straddling chunks, slot k + b
    uint32_t *chunk_cnt;               // [P] arrival counters, reset by the last arriver
    uint16_t *cta_rows, *cta_doms;     // [grid] CTA maps
    uint32_t *ticket;
    uint16_t *final2;
    uint16_t *starts;        // [P] true chunk starts (optional; then every segment map is
    uint16_t *cta_code;      //  published and the last CTA writes each CTA's start code)
    uint32_t info_off;       // (set by launch_lanes) shared-memory offset of the tail's info area
};

struct DevStatus {
    uint32_t err;            // 0 ok, 5 bad symbol, 8 internal
    uint32_t final_state;
    uint32_t accept;
    uint32_t pad;            // factored composition: bit 0 = some chunk node is FULL (no group links)
};

struct Shape {
    uint64_t f, m, S;        // segment 0 holds f maps, segments 1..S-1 hold m maps
    uint32_t G;              // max maps per group
    __host__ __device__ uint64_t groups() const {
        uint64_t gf = (f + G - 1) / G;
        uint64_t gm = S > 1 ? (m + G - 1) / G : 0;
        return gf + (S - 1) * gm;
    }
};

// Composition tree (Eq.MapReduction applied hierarchically, the on-GPU analog
// of the paper's two-tier merge, Fig.Merge): level 0 = the sub-chunk maps
// (leaves), level L >= 1 groups <= G consecutive level L-1 nodes that lie in
// the same reporting chunk, up to one node per reporting chunk (rep_level),
// then groups reporting chunk nodes up to the single root (final state).
constexpr int kMaxLevels = 24;
struct TreeLevel {            // all 32-bit: node counts stay far below 2^32
    uint32_t f, m, S, G;     // shape of level L-1 (segment 0: f nodes, others m) and group size
    uint32_t gf, gm;         // groups of segment 0 / of every other segment
    uint32_t nodes;          // node count of this level
    uint32_t off;            // offset of this level's nodes in rows/doms/counters
};
struct Tree {
    uint32_t nlevels;        // levels 1..nlevels
    uint32_t rep_level;      // its nodes are the reporting chunks 0..P-1
    uint32_t F;              // staging capacity (children per node) of a warp
    uint32_t lrs;            // log2 of the shared-memory row stride (>= T.rs)
    int rank_smem;           // uint8 rank table staged in shared memory
    int root_final;          // the top level is the root: write the final state
    TreeLevel lv[kMaxLevels + 1];
    // leaves (lanes kernel output)
    const uint16_t *amap, *sfin;
    uint32_t sk;
    const uint16_t *dom_of;
    // factored composition (fwalk_kernel / fexpand_kernel): survivor counts of the leaves,
    // per node value count (bit 15: FULL) and first leaf, full rows of the reporting chunks
    const uint8_t *leaf_nv;
    uint16_t *node_nv;
    uint32_t *node_fl;
    uint16_t *rep_full;
    uint16_t *clinks;        // [ceil(P/8)][8] fchunk_kernel: links composed per group of 8 chunks (or null)
    // nodes
    uint16_t *rows, *doms;
    uint32_t *counters;
    // outputs
    uint16_t *user_rows, *e0, *dev_final;
    uint16_t *user_row0;     // optional API row of reporting chunk 0 (segment maps)
    uint16_t *seg_row;       // optional: the root map (the whole input over chunk 0's domain), user order
    DevStatus *status;
};

struct LaunchCfg {
    int sms;
    cudaStream_t stream;
};

// launchers (return cudaError_t of the launch)
cudaError_t launch_converge(const DevTables &T, const Plan &p, const uint8_t *in, uint16_t *surv,
                            uint8_t *surv_n, uint64_t *surv_pos, uint16_t *amap, uint32_t cap, int warps_per_cta,
                            int grid, cudaStream_t s);
int converge_smem_bytes(const DevTables &T, int warps_per_cta);
cudaError_t launch_lanes(const DevTables &T, const Plan &p, const uint8_t *in, const uint16_t *surv,
                         const uint8_t *surv_n, const uint64_t *surv_pos, uint16_t *sfin, uint32_t sk,
                         uint16_t *dom_of, int convergence, uint16_t *amap, uint32_t g_log,
                         uint16_t *leaf_rows, uint16_t *leaf_dom, DevStatus *status, uint32_t cap, int threads,
                         int grid, cudaStream_t s, const Fuse &fz);
int fused_tail_smem_bytes(int threads, uint32_t g_log, int grid);
cudaError_t launch_fused_starts(const DevTables &T, const Plan &p, const Fuse &fz, const uint8_t *in, uint32_t lpc,
                                uint32_t g_log, int grid, cudaStream_t s);
int lanes_smem_bytes(const DevTables &T);
bool lanes_tma_available(const DevTables &T, int threads, int optin_smem);
int lanes_occupancy(const DevTables &T, int threads);
int converge_occupancy(const DevTables &T, int warps_per_cta);
cudaError_t launch_tree(const DevTables &T, const Tree &tr, int grid, int smem_bytes, cudaStream_t s);
cudaError_t launch_walk(const DevTables &T, const Tree &tr, uint32_t L, int sms, cudaStream_t s);
cudaError_t launch_fwalk(const DevTables &T, const Tree &tr, uint32_t L, int sms, cudaStream_t s);
cudaError_t launch_fexpand(const DevTables &T, const Tree &tr, uint32_t L, int sms, cudaStream_t s);
uint32_t fchunk_cap(); // most leaves per reporting chunk fchunk_kernel takes
cudaError_t launch_fchunk(const DevTables &T, const Tree &tr, int sms, cudaStream_t s);
uint32_t ffold_cap();  // most nodes ffold_kernel stages in shared memory
cudaError_t launch_ffold(const DevTables &T, const Tree &tr, uint32_t Ls, cudaStream_t s);
cudaError_t launch_lookahead(const DevTables &T, const uint8_t *in, const uint64_t *bounds, uint32_t P, uint32_t r,
                             const uint16_t *maps, uint16_t *doms_out, uint16_t *sizes_out, uint16_t *maps_out,
                             DevStatus *st, int sms, cudaStream_t s);
cudaError_t launch_leaf_fold(const uint16_t *in_rows, const uint16_t *in_dom, uint32_t L0, uint32_t L, uint32_t P,
                             uint16_t *out_rows, uint16_t *out_dom, int sms, cudaStream_t s);
cudaError_t launch_compose8(const DevTables &T, const uint16_t *leaves, const uint16_t *leaf_dom, uint32_t L0,
                            uint32_t L, uint32_t P, uint32_t cpc, uint16_t *rep_rows, uint16_t *rep_doms,
                            uint16_t *user_rows, uint16_t *user_row0, uint16_t *e0, uint16_t *cta_rows,
                            uint16_t *cta_doms, uint32_t *ticket, DevStatus *st, uint16_t *dev_final,
                            uint16_t *cta_start, uint16_t *starts, uint16_t *seg_row, cudaStream_t s);
size_t fold_rows_fixed_bytes(const DevTables &T);
cudaError_t launch_fold_rows(const DevTables &T, const uint16_t *rows, const uint16_t *doms, uint32_t P,
                             uint32_t per_cta, uint16_t *cta_rows, uint16_t *cta_doms, uint32_t *ticket,
                             DevStatus *st, uint16_t *dev_final, uint16_t *seg_row, cudaStream_t s);
int tree_slice_bytes(const DevTables &T, uint32_t F);
uint32_t tree_lrs(const DevTables &T);
int tree_fixed_bytes(const DevTables &T, int rank_smem);
const void *tree_fn();
cudaError_t launch_starts(const DevTables &T, const Plan &p, const uint16_t *row0, const uint16_t *rows,
                          const uint16_t *dom, uint16_t *starts, DevStatus *st, cudaStream_t s);
cudaError_t setup_kernel_attributes(const DevTables &T);
cudaError_t launch_batch_out(const DevTables &T, const uint16_t *rep_rows, uint32_t rs, const int32_t *kidx,
                             const uint64_t *offsets, uint64_t data_len, uint32_t count, uint16_t *dev_final,
                             uint8_t *dev_accept, DevStatus *st, cudaStream_t s);
cudaError_t launch_fold_segments(const DevTables &T, const uint16_t *rows, const uint8_t *lookahead, uint32_t G,
                                 DevStatus *st, uint16_t *dev_final, cudaStream_t s);
int probe_dynamic_smem_base(uint32_t *dev_scratch);

// Match kernels of one table layout (MODE = TableMode), one translation unit
// each (kernels_m<MODE>.cu); nullptr where a layout has no such kernel.
template <int MODE> void *lanes_entry(bool sticky, bool count, bool tma);
template <int MODE> void *ceiling_entry();
template <int MODE> void *converge_entry(bool id8);
#define DFA_DECLARE_MODE_ENTRIES(M)                  \
    template <> void *lanes_entry<M>(bool sticky, bool count, bool tma); \
    template <> void *ceiling_entry<M>();            \
    template <> void *converge_entry<M>(bool id8);
DFA_DECLARE_MODE_ENTRIES(1) DFA_DECLARE_MODE_ENTRIES(2) DFA_DECLARE_MODE_ENTRIES(3)
DFA_DECLARE_MODE_ENTRIES(4) DFA_DECLARE_MODE_ENTRIES(5) DFA_DECLARE_MODE_ENTRIES(6)
DFA_DECLARE_MODE_ENTRIES(7) DFA_DECLARE_MODE_ENTRIES(8) DFA_DECLARE_MODE_ENTRIES(9)
#undef DFA_DECLARE_MODE_ENTRIES
int ceiling_occupancy(const DevTables &T, int threads);
cudaError_t launch_ceiling(const DevTables &T, const uint8_t *in, uint64_t per, uint16_t *out, int threads, int grid,
                           cudaStream_t s);

} // namespace dfa
