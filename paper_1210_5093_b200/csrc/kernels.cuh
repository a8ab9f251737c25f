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
//   3. compose_kernel: tree composition of sub-chunk maps into the reporting
//      chunk maps, then of those into the final state (Eq.MapReduction,
//      P:819-830, applied hierarchically: the on-GPU analog of Fig.Merge).
//   4. finalize_kernel: final state, accept bit (Alg.seqmatch l.4-6), errors.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace dfa {

constexpr int kLanes = 8;          // register lanes per thread in lanes_kernel
constexpr int kConvergeLA = 8;     // lanes per thread per pass in converge_kernel
constexpr uint32_t kSubWindow = 16;

struct DevTables {
    const uint32_t *image;      // smem image of the transition table (32-bit words)
    uint32_t image_words;
    const uint16_t *gtable;     // [nq][256] byte-indexed table (global)
    const uint8_t *byte_class;  // [256]
    const uint16_t *dom_list;   // [(nclass+1) * imax] internal I_sigma, ascending
    const uint16_t *dom_size;   // [nclass+1]
    const uint16_t *rank;       // [(nclass+1) * nq] index in dom_list or 0xFFFF
    const uint32_t *dead_bits;  // internal Z
    const uint32_t *absorb_bits;
    const uint32_t *accept_bits;
    const uint16_t *xlat;       // [nclass * imax_user]
    const uint16_t *dom_user_size; // [nclass]
    uint32_t nq, nclass, start_dom, imax, imax_user;
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
};

struct DevStatus {
    uint32_t err;            // 0 ok, 5 bad symbol, 8 internal
    uint32_t final_state;
    uint32_t accept;
    uint32_t pad;
};

struct LevelIn {
    int kind;                // 0: sub-chunk maps (amap/sfin), 1: rows
    const uint16_t *amap;    // kind 0, may be null
    const uint16_t *sfin;
    uint32_t sk;             // sfin row stride
    const uint16_t *row0, *rows;
    const uint16_t *dom;
};

struct LevelOut {
    uint16_t *row0, *rows;   // internal rows; row(g) = g ? rows + (g-1)*imax : row0
    uint16_t *dom;
    uint16_t *user_rows;     // optional API rows (k >= 1) in the user's domain order
    uint16_t *e0;            // optional chunk-0 end state
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

struct LaunchCfg {
    int sms;
    cudaStream_t stream;
};

// launchers (return cudaError_t of the launch)
cudaError_t launch_converge(const DevTables &T, const Plan &p, const uint8_t *in, uint16_t *surv,
                            uint8_t *surv_n, uint64_t *surv_pos, uint16_t *amap, int warps_per_cta,
                            int grid, cudaStream_t s);
int converge_smem_bytes(const DevTables &T, int warps_per_cta);
cudaError_t launch_lanes(const DevTables &T, const Plan &p, const uint8_t *in, const uint16_t *surv,
                         const uint8_t *surv_n, const uint64_t *surv_pos, uint16_t *sfin, uint32_t sk,
                         uint16_t *dom_of, int convergence, int threads, int grid, cudaStream_t s);
int lanes_smem_bytes(const DevTables &T);
int lanes_occupancy(const DevTables &T, int threads);
int converge_occupancy(const DevTables &T, int warps_per_cta);
cudaError_t launch_compose(const DevTables &T, const LevelIn &in, const LevelOut &out, const Shape &sh,
                           DevStatus *st, int grid, cudaStream_t s);
int compose_smem_bytes(const DevTables &T, uint32_t G);
cudaError_t launch_finalize(const DevTables &T, const uint16_t *final_row, DevStatus *st,
                            uint16_t *dev_final, cudaStream_t s);
cudaError_t launch_starts(const DevTables &T, const Plan &p, const uint16_t *row0, const uint16_t *rows,
                          const uint16_t *dom, uint16_t *starts, DevStatus *st, cudaStream_t s);
cudaError_t setup_kernel_attributes(const DevTables &T);
int probe_dynamic_smem_base(uint32_t *dev_scratch);

} // namespace dfa
