// prep.h -- host preprocessing of a DFA for the B200 matching path.
//
// Everything here runs once per DFA at dfa_create (the paper computes I_max
// "online for every matching run" but notes it is a static property that can
// be computed offline).  Product code: shares nothing with
// oracle/.
#pragma once
#include <cstdint>
#include <string>
#include <vector>

namespace dfa {

constexpr uint16_t kNone = 0xFFFF;     // "no state" / map padding (reading R6)
constexpr uint16_t kSurvBase = 0xFF00; // amap code: survivor index (internal)
constexpr uint32_t kMaxStates = 65000; // leaves room for kSurvBase codes

enum TableMode : int {
    kIdentU8 = 1,   // smem, row = 256 byte columns, uint8 entries
    kIdentU16 = 2,  // smem, row = 256 byte columns, uint16 entries
    kWindowU8 = 3,  // smem, row = W window columns + 1 default column, uint8
    kWindowU16 = 4, // same, uint16
    kPacked9 = 5,   // smem, 256 columns of 9-bit states, 3 per 32-bit word
    kGlobalU16 = 6, // global memory [nq][256] uint16 through the read-only path
    // IdentU8 replicated in shared memory: copy g (of R) confined to banks
    // g*32/R .. (g+1)*32/R - 1, lane l of a warp reads copy l % R, so a warp's
    // gather conflicts only within groups of 32/R lanes.
    // The host image is the IdentU8 image; the lanes kernel expands it.
    kRepU8x8 = 7,   // R = 8 (|Q| <= ~110: |Q| * 2 KB)
    kRepU8x4 = 8,   // R = 4 (|Q| * 1 KB)
    // IdentU8 with rows padded to kPadStride = 260 bytes: entry (s, b) in bank
    // (s_enc + b/4) mod 32, so lanes in different states that read the same
    // byte (Zipf text; the converge kernel's lanes, which all step one byte)
    // fall into different banks.  Address s_enc * 260 + b: one IMAD.
    kIdentU8P = 9
};
constexpr uint32_t kPadStride = 260;

#ifdef __CUDACC__
#define DFA_HD __host__ __device__
#else
#define DFA_HD
#endif
DFA_HD constexpr uint32_t rep_log_of(int mode) { return mode == kRepU8x8 ? 3u : mode == kRepU8x4 ? 2u : 0u; }
// lanes_kernel CTA size bound per layout.  rep8_u8 (one 131+ KB CTA per SM) runs
// 640 threads: 102 registers (no spills) and longer sub-chunks, so fewer initial
// I_sigma lane-steps; measured on Random 1868 GB/s vs 1746 at 1024 threads (sweep
// 512..1024 in DESIGN.md section 4).  packed9 (176 KB, Worst) is bounded at 704
// threads for 88 registers with its sub-chunk count unchanged (6.80 vs 6.99 ms).
// Every other layout: 1024 (64 registers).
#ifndef DFA_WIN16_MAX_THREADS
#define DFA_WIN16_MAX_THREADS 896   // window_u16 (Protein) CTA bound: 73 registers; run at 768 threads behind the
                                    // converge stage (plan_split), 1.624 ms vs 1.691 at 1024 threads / 64 registers
#endif
#ifndef DFA_PACKED9_MAX_THREADS
#define DFA_PACKED9_MAX_THREADS 704  // packed9 (Worst) CTA bound; -D for the register-budget experiment
#endif
#ifndef DFA_PAD_MAX_THREADS
#define DFA_PAD_MAX_THREADS 768     // ident_u8_pad (Keyword) CTA bound: fewer, longer sub-chunks (6 instead of 9 per
                                    // chunk at P = 16384): 0.425 ms vs 0.442 at 1024 threads (sweep in DESIGN.md section 11)
#endif
DFA_HD constexpr int lanes_max_threads(int mode) {
    return mode == kRepU8x8 ? 640 : mode == kIdentU8P ? DFA_PAD_MAX_THREADS : mode == kPacked9 ? DFA_PACKED9_MAX_THREADS : mode == kWindowU16 ? DFA_WIN16_MAX_THREADS : 1024;
}

struct Prep {
    // user view
    uint32_t nq_user = 0, ns = 0;
    uint16_t q0 = 0;
    // internal automaton: user states + (if ns < 256) one poison state that
    // absorbs every byte >= ns (reading R12: bad symbols are detected without a
    // per-byte check).  Internal table is byte-indexed over all 256 bytes.
    uint32_t nq = 0;
    uint16_t poison = kNone;
    std::vector<uint16_t> full;      // [nq][256]
    std::vector<uint8_t> accepting;  // [nq]
    std::vector<uint8_t> dead;       // [nq] internal Z: absorbing over all 256 bytes, not accepting
    std::vector<uint8_t> dead_user;  // [nq] user Z over Sigma (reading R1); == dead if no poison
    std::vector<uint8_t> absorbing;  // [nq] delta(q,.) == q
    // column classes over the 256 bytes (north_star "byte-class alphabet compression")
    std::vector<uint8_t> byte_class; // [256]
    std::vector<uint16_t> class_rep; // representative byte per class
    uint32_t nclass = 0;
    uint32_t start_dom = 0;          // domain id of the {q0} domain = nclass
    // initial-state sets I_sigma = delta(Q, sigma) \ Z per class, ascending
    // (Eq.istates P:946-951 with Alg.MatchingInitialStates line 5).
    // dom_user uses the user's Z (what the API reports); dom uses the internal
    // Z, a superset when a poison state exists (user error states must keep
    // being tracked, since a later byte >= |Sigma| still leaves them).
    std::vector<std::vector<uint16_t>> dom;      // [nclass + 1], last = {q0}
    std::vector<std::vector<uint16_t>> dom_user; // [nclass]
    std::vector<std::vector<uint16_t>> xlat;     // [nclass]: dom_user[c][j] == dom[c][xlat[c][j]]
    uint32_t imax_user = 0;          // Eq.MaxIstates over valid symbols
    uint32_t imax = 1;               // internal row stride (>= 1)
    uint32_t imax_user_stride = 1;   // max(1, imax_user): API map row stride
    uint32_t num_dead_user = 0, num_absorbing_user = 0;
    uint16_t first_dead_user = kNone;
    uint32_t nclass_user = 0;        // classes containing a valid symbol
    bool full_domain = false;        // Alg.2 ablation: dom[c] = Q \ Z for every class
    // device table layout
    int mode = 0;
    uint32_t stride = 0;             // entries per row (u8/u16) or words per row (packed9)
    uint32_t win_base = 0, win_w = 0;
    std::vector<uint32_t> image;     // smem image (32-bit words), empty for global
};

// Validates and analyses; returns 0 or a dfa_status code.
// u8_state_limit: largest internal |Q| for the IdentU8 layout (256 minus the
// shared-address bias of the table, see Tab<kIdentU8> in kernels.cu).
int prepare(const uint16_t *table, uint32_t nq, uint32_t ns, uint16_t q0,
            const uint8_t *accept_bitmap, uint32_t smem_budget, uint32_t u8_state_limit, Prep &out,
            bool full_domain = false, uint32_t rep_budget = 0, int forced_mode = 0);

// Exact c-form partition (header dfa.h), 128-bit integer arithmetic.
uint64_t cform_bound(uint64_t n, uint32_t P, uint64_t c_num, uint64_t c_den, uint32_t k);

} // namespace dfa
