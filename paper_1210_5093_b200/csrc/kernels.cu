// kernels.cu -- sm_100a kernels of the speculative chunked DFA membership test.
//
// Paper: Ko, Jung, Han, Burgstaller, arXiv:1210.5093.  The paper's
// kernels are a scalar C loop (Listing Cmatching) and an 8-way
// AVX2 gather loop (Listing AVX2matching) over a flattened table
// (SBase, Fig.SBaseExample).  Here the same transition step
// s <- delta(s, x[i]) is a shared-memory gather (LDS) per lane; a warp issues
// 32 of them per instruction where AVX2 issued 8.  No tensor cores: the path
// is a dependent gather chain, not a contraction.
#include "kernels.cuh"
#include "prep.h"

// Translation units: kernels.cu (DFA_TU_MAIN: composition kernels, launchers) and
// kernels_m<MODE>.cu (DFA_TU_MODE = MODE: the match kernels of one table layout).
#if !defined(DFA_TU_MODE)
#define DFA_TU_MAIN 1
#endif

#include <cuda_runtime.h>
#include <algorithm>
#include <type_traits>
#include <utility>
#include <cstdint>

// DFA_CHECKED (the bounds-checked build, tools/checked_run.sh): every table lookup,
// data-dependent index and input read is range-checked on the device; a violation
// traps.  compute-sanitizer is not available on the B200 pool
// (DESIGN.md section 5), this is the memory-safety evidence instead.  Compiles to
// nothing in the production build.
#ifdef DFA_CHECKED
// a failed check executes the trap instruction (the launch fails with an illegal-instruction
// error at the next synchronisation); no call, so the checked build compiles like the product
#define DFA_CHECK(cond, what)                       \
    do {                                            \
        if (__builtin_expect(!(cond), 0)) asm volatile("trap;"); \
    } while (0)
#else
#define DFA_CHECK(cond, what) \
    do {                      \
    } while (0)
#endif

namespace dfa {

namespace {

constexpr uint32_t kDone = 0xFFu;
constexpr uint32_t kNoGroup = 0xFFFFFFFFu;

#ifdef DFA_TREE_TIMING
__device__ unsigned long long g_tree_t[32];  // debug phase timestamps (tools/*_timing.py)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif

// Programmatic dependent launch (sm_90+): a kernel launched with
// launch_pdl may start while its predecessor drains; it stages what does not
// depend on it, then waits here for the predecessor's completion and memory.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ bool test_bit(const uint32_t *bits, uint32_t q) {
    return (bits[q >> 5] >> (q & 31)) & 1u;
}

struct U8x32 { uint4 lo, hi; };

// One full 32-byte sector per thread and request (sm_100 256-bit load).
__device__ __forceinline__ U8x32 ldg32(const void *p) {
    U8x32 v;
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v.lo.x), "=r"(v.lo.y), "=r"(v.lo.z), "=r"(v.lo.w), "=r"(v.hi.x), "=r"(v.hi.y), "=r"(v.hi.z),
                   "=r"(v.hi.w)
                 : "l"(p));
    return v;
}

__device__ __forceinline__ uint4 ldg16(const uint4 *p) {
    uint4 v;
    asm volatile("ld.global.nc.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p));
    return v;
}

// Execution sub-chunk i -> [start, end): reporting chunk k is [b_k, b_{k+1})
// (Eq.StartPosition/EndPosition, half-open, reading R5), split into m_k equal
// parts (m_0 = m0, m_k = m for k >= 1).
// Internal split points (j > 0) are moved down to a 32-byte aligned address
// when the parts are long enough, so that a sub-chunk is whole 32-byte sectors
// except at reporting-chunk bounds; the split is internal, results unchanged.
// n / d for 32-bit n with the plan's magic = min(floor(2^32 / d), 2^32 - 1): the estimate
// umulhi(n, magic) is floor(n / d) or one less, one correction makes it exact.
__device__ __forceinline__ uint32_t udiv_magic(uint32_t n, uint32_t d, uint32_t magic) {
    const uint32_t q = __umulhi(n, magic);
    return n - q * d >= d ? q + 1u : q;
}

// sub-chunk i -> its reporting chunk k, its index j in the chunk and the chunk's split mk
__device__ __forceinline__ void sub_locate(const Plan &p, uint64_t i, uint64_t &k, uint64_t &j, uint64_t &mk) {
    if (i < p.m0) { k = 0; j = i; mk = p.m0; return; }
    mk = p.m;
    const uint64_t t = i - p.m0;
    if ((t >> 32) == 0) {
        const uint32_t q = udiv_magic((uint32_t)t, p.m, p.magic_m);
        k = 1ull + q;
        j = (uint32_t)t - q * p.m;
    } else {
        k = 1 + t / p.m;
        j = t % p.m;
    }
}

// [b0 + floor(len j / mk), b0 + floor(len (j+1) / mk)) with internal split points moved down
// to a 32-byte aligned address.  Exact: len = q mk + r gives floor(len j / mk) = q j +
// floor(r j / mk), all 32-bit when len < 2^32 and mk <= 2^16 (r j < mk^2).
__device__ __forceinline__ void split_range(const Plan &p, uint64_t b0, uint64_t len, uint64_t j, uint64_t mk,
                                            uint64_t &s, uint64_t &e) {
    uint64_t o0, o1;
    if ((len >> 32) == 0 && mk <= 65536u) {
        const uint32_t d = (uint32_t)mk, magic = mk == p.m ? p.magic_m : p.magic_m0, jj = (uint32_t)j;
        const uint32_t q = udiv_magic((uint32_t)len, d, magic), r = (uint32_t)len - q * d;
        o0 = (uint64_t)q * jj + udiv_magic(r * jj, d, magic);
        o1 = (uint64_t)q * (jj + 1u) + udiv_magic(r * (jj + 1u), d, magic);
    } else {
        o0 = len * j / mk;
        o1 = len * (j + 1) / mk;
    }
    s = b0 + o0;
    e = b0 + o1;
    if (len >= 64 * mk) {
        if (j != 0) s -= (p.in_addr + s) & 31u;
        if (j + 1 != mk) e -= (p.in_addr + e) & 31u;
    }
}

// sub-chunk i's reporting chunk k (its bounds are p.bounds[k], p.bounds[k+1])
__device__ __forceinline__ uint64_t sub_chunk_of(const Plan &p, uint64_t i) {
    uint64_t k, j, mk;
    sub_locate(p, i, k, j, mk);
    return k;
}
// sub_range with the chunk's bounds already loaded (b0, b1 = bounds of sub_chunk_of(i))
__device__ __forceinline__ void sub_range_b(const Plan &p, uint64_t i, uint64_t &b0, uint64_t b1, uint64_t &s,
                                            uint64_t &e, uint64_t &j) {
    uint64_t k, mk;
    sub_locate(p, i, k, j, mk);
    if (p.indep) {
        b0 = min(b0, p.n);
        b1 = min(max(b1, b0), p.n);
    }
    DFA_CHECK(b0 <= b1 && b1 <= p.n, "chunk bounds out of order or past n");
    split_range(p, b0, b1 - b0, j, mk, s, e);
    DFA_CHECK(b0 <= s && s <= e && e <= b1, "sub-chunk outside its chunk");
}

__device__ __forceinline__ void sub_range(const Plan &p, uint64_t i, uint64_t &s, uint64_t &e) {
    uint64_t k, j, mk;
    sub_locate(p, i, k, j, mk);
    uint64_t b0 = p.bounds[k], b1 = p.bounds[k + 1];
    if (p.indep) {  // caller-given batch offsets: clamp (batch_out_kernel flags bad ones)
        b0 = min(b0, p.n);
        b1 = min(max(b1, b0), p.n);
    }
    split_range(p, b0, b1 - b0, j, mk, s, e);
}

// Reverse lookahead: the domain of sub-chunk i is I_sigma with
// sigma the byte before it; the very first sub-chunk starts from {q0}.
__device__ __forceinline__ bool chunk_first_sub(const Plan &p, uint64_t i) {
    uint64_t k, j, mk;
    sub_locate(p, i, k, j, mk);
    return j == 0;
}

__device__ __forceinline__ uint32_t sub_domain(const DevTables &T, const Plan &p, const uint8_t *in, uint64_t i,
                                               uint64_t start) {
    DFA_CHECK(i < p.NS, "sub-chunk index past NS");
    if (i == 0) return p.first_dom;
    if (p.indep && chunk_first_sub(p, i)) return T.start_dom;  // batch: every input starts at q0
    DFA_CHECK(start >= 1 && start <= p.n, "lookahead byte before the input");
    return (uint32_t)T.byte_class[__ldg(in + start - 1)];
}

// ---------------------------------------------------------------------------
// Transition step per table layout.  wprep: per 32-bit input word (window
// modes map 4 bytes to 4 columns with two SIMD ops); bprep: per byte, shared
// by all lanes of a thread; look: per lane, one shared-memory load.
// ---------------------------------------------------------------------------
// prmt.b32 with sign-replicate selector nibbles (0xC -> 0x00 for a byte < 0x80);
// __byte_perm keeps only the low three bits of each nibble.
__device__ __forceinline__ uint32_t prmt_s(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r;
    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel));
    return r;
}

template <int MODE>
__host__ __device__ constexpr bool is_rep() { return rep_log_of(MODE) != 0; }

// Words of the table image as laid out in shared memory (R copies for the
// replicated modes).
template <int MODE>
__device__ __forceinline__ uint32_t smem_words(const DevTables &T) {
    if constexpr (MODE == kIdentU8P) return T.image_words / 64u * (kPadStride / 4u);
    else return T.image_words << rep_log_of(MODE);
}

template <int MODE>
struct Tab {
    const uint8_t *t8;
    const uint16_t *t16;
    const uint32_t *t32;
    const uint16_t *g;
    uint32_t stride, base4, w4, base, w;
    uint32_t lo4, hi4;  // window modes: column bits / window-tag bits of every byte
    uint32_t tb;      // shared-space address of the table
    uint32_t rowb;    // bytes per table row
    // IdentU8: the table sits at a 256-aligned shared address A = bias*256 and
    // holds encoded states s + bias, so the shared address of entry (s, b) is
    // exactly (s_enc << 8) | b -- one PRMT builds it from the state and the
    // input word ("we only add the current state's offset to the
    // current input symbol"), with no base add.  Other modes: bias = 0 and
    // one IMAD per lane (state * row bytes + per-byte column address).
    uint32_t bias;
    // Replicated modes (R = 2^LR copies): the copy of lane l is g = l % R, and
    // the shared address of entry (s, b) in it is
    //   (s_enc << (8 + LR)) + K(b),  K(b) = (b & (2^M - 1)) | g << M | (b >> M) << 7,
    // M = 7 - LR: each 128-byte bank row holds R slices of 2^M bytes, slice g
    // in banks g*32/R .. (g+1)*32/R - 1.  G = g << M in every byte.
    static constexpr uint32_t LR = rep_log_of(MODE);
    static constexpr uint32_t M = 7u - LR;
    uint32_t G;

    struct Pre { uint32_t a, sh; };

    __device__ __forceinline__ void init(const DevTables &T, const void *table_smem) {
        t8 = reinterpret_cast<const uint8_t *>(table_smem);
        t16 = reinterpret_cast<const uint16_t *>(table_smem);
        t32 = reinterpret_cast<const uint32_t *>(table_smem);
        g = T.gtable;
        stride = T.stride;
        base = T.win_base;
        w = T.win_w;
        base4 = T.win_base * 0x01010101u;
        w4 = T.win_w * 0x01010101u;
        tb = (uint32_t)__cvta_generic_to_shared(table_smem);
        bias = MODE == kIdentU8 ? (tb >> 8) : is_rep<MODE>() ? (tb >> (8 + LR)) : MODE == kIdentU8P ? tb / kPadStride : 0u;
        lo4 = (T.win_w - 1u) * 0x01010101u;
        hi4 = (~(T.win_w - 1u) & 0xFFu) * 0x01010101u;
        G = is_rep<MODE>() ? (((threadIdx.x & 31u) & ((1u << LR) - 1u)) << M) * 0x01010101u : 0u;
        rowb = MODE == kIdentU16 ? 512u : MODE == kWindowU8 ? T.stride : MODE == kWindowU16 ? 2u * T.stride
             : MODE == kPacked9 ? 4u * T.stride : 0u;
        // WindowU16: the table starts at a multiple of the row size and holds
        // s + bias, so s_enc * rowb is the row's shared address (no base add)
        if (MODE == kWindowU16) bias = tb / rowb;
#ifdef DFA_CHECKED
        tlim = smem_words<MODE>(T) * 4u;
        glim = T.nq * 256u;
#endif
    }
    __device__ __forceinline__ uint32_t enc(uint32_t s) const { return s + bias; }
    __device__ __forceinline__ uint32_t dec(uint32_t s) const { return s - bias; }
#ifdef DFA_CHECKED
    uint32_t tlim, glim;  // table bytes in shared memory / entries of the global table
#endif
    __device__ __forceinline__ uint32_t lds_u8(uint32_t addr) const {
        DFA_CHECK(addr - tb < tlim, "u8 table lookup outside the shared-memory table");
        uint32_t r;
        asm volatile("ld.shared.u8 %0, [%1];" : "=r"(r) : "r"(addr));
        return r;
    }
    __device__ __forceinline__ uint32_t lds_u16(uint32_t addr) const {
        DFA_CHECK(addr - tb < tlim && !(addr & 1u), "u16 table lookup outside the shared-memory table");
        uint32_t r;
        asm volatile("ld.shared.u16 %0, [%1];" : "=r"(r) : "r"(addr));
        return r;
    }
    __device__ __forceinline__ uint32_t lds_u32(uint32_t addr) const {
        DFA_CHECK(addr - tb < tlim && !(addr & 3u), "u32 table lookup outside the shared-memory table");
        uint32_t r;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(addr));
        return r;
    }
    __device__ __forceinline__ uint32_t ldg_tab(uint32_t idx) const {
        DFA_CHECK(idx < glim, "global table lookup out of range");
        return __ldg(g + idx);
    }
    // replicated modes: K(b) of a raw byte
    __device__ __forceinline__ uint32_t rep_k(uint32_t b) const {
        return (b & ((1u << M) - 1u)) | (G & 0xFFu) | ((b >> M) << 7);
    }
    __device__ __forceinline__ auto wprep(uint32_t x) const {
        if constexpr (MODE == kWindowU8 || MODE == kWindowU16) return __vminu4(__vsub4(x, base4), w4);
        else if constexpr (is_rep<MODE>()) {
            // per byte: y = low M bits | g << M | bit M << 7, z = b >> (M + 1)
            constexpr uint32_t lo = ((1u << M) - 1u) * 0x01010101u, bm = (1u << M) * 0x01010101u;
            constexpr uint32_t zm = ((1u << (7u - M)) - 1u) * 0x01010101u;
            return make_uint2((x & lo) | ((x & bm) << (7u - M)) | G, (x >> (M + 1u)) & zm);
        } else return x;
    }
    // per input byte, shared by all lanes of the thread: the column's address
    // PX: byte k by one PRMT (lanes_kernel: one instruction less on two bytes of four);
    // converge_kernel keeps shift + mask (the PRMT form spills at its 64 registers)
    template <bool PX = true, class X>
    __device__ __forceinline__ Pre bprep(X xw, int k) const {
        if constexpr (is_rep<MODE>()) {
            return {prmt_s(xw.x, xw.y, 0xCC00u | ((4u + k) << 4) | (uint32_t)k), 0u};
        } else {
        const uint32_t x = xw;
        const uint32_t c = PX ? __byte_perm(x, 0u, 0x4440u | (uint32_t)k) : (x >> (8 * k)) & 0xFFu;
        if constexpr (MODE == kIdentU16) return {tb + 2u * c, 0u};
        else if constexpr (MODE == kWindowU8) return {tb + c, 0u};
        else if constexpr (MODE == kWindowU16) return {2u * c, 0u};
        else if constexpr (MODE == kPacked9) {
            const uint32_t wc = (c * 171u) >> 9;  // c / 3 for c < 256
            return {tb + 4u * wc, (c - 3u * wc) * 9u};
        } else return {c, 0u};
        }
    }
    template <class X>
    __device__ __forceinline__ uint32_t look(uint32_t s, X x, int k, Pre p) const {
        if constexpr (is_rep<MODE>()) return lds_u8((s << (8 + LR)) + p.a);
        else if constexpr (MODE == kIdentU8P) return lds_u8(s * kPadStride + p.a);
        else if constexpr (MODE == kIdentU8) return lds_u8(__byte_perm(x, s, 0x6540 + k));
        else if constexpr (MODE == kIdentU16 || MODE == kWindowU16) return lds_u16(s * rowb + p.a);
        else if constexpr (MODE == kWindowU8) return lds_u8(s * rowb + p.a);
        else if constexpr (MODE == kPacked9) return (lds_u32(s * rowb + p.a) >> p.sh) & 511u;
        else return ldg_tab((s << 8) + p.a);
    }
    // per raw byte b, shared by all lanes stepping on it (scalar paths)
    __device__ __forceinline__ Pre bpre(uint32_t b) const {
        if constexpr (is_rep<MODE>()) return {rep_k(b), 0u};
        else if constexpr (MODE == kIdentU8 || MODE == kIdentU8P || MODE == kGlobalU16) return {b, 0u};
        else if constexpr (MODE == kIdentU16) return {tb + 2u * b, 0u};
        else if constexpr (MODE == kWindowU8 || MODE == kWindowU16) {
            const uint32_t c = min((b - base) & 0xFFu, w);
            return {MODE == kWindowU16 ? 2u * c : tb + c, 0u};
        } else {
            const uint32_t wc = (b * 171u) >> 9;
            return {tb + 4u * wc, (b - 3u * wc) * 9u};
        }
    }
    __device__ __forceinline__ uint32_t look_pre(uint32_t s, Pre p) const {
        if constexpr (is_rep<MODE>()) return lds_u8((s << (8 + LR)) + p.a);
        else if constexpr (MODE == kIdentU8P) return lds_u8(s * kPadStride + p.a);
        else if constexpr (MODE == kIdentU8) return lds_u8((s << 8) | p.a);
        else if constexpr (MODE == kIdentU16 || MODE == kWindowU16) return lds_u16(s * rowb + p.a);
        else if constexpr (MODE == kWindowU8) return lds_u8(s * rowb + p.a);
        else if constexpr (MODE == kPacked9) return (lds_u32(s * rowb + p.a) >> p.sh) & 511u;
        else return ldg_tab((s << 8) + p.a);
    }
    // scalar step on an encoded state and a raw byte
    __device__ __forceinline__ uint32_t look_byte(uint32_t s, uint32_t b) const {
        if constexpr (is_rep<MODE>()) return lds_u8((s << (8 + LR)) + rep_k(b));
        else if constexpr (MODE == kIdentU8P) return lds_u8(s * kPadStride + b);
        else if constexpr (MODE == kIdentU8) return lds_u8((s << 8) | b);
        else if constexpr (MODE == kIdentU16) return t16[(s << 8) | b];
        else if constexpr (MODE == kWindowU8 || MODE == kWindowU16) {
            uint32_t c = min((b - base) & 0xFFu, w);
            if constexpr (MODE == kWindowU8) return t8[s * stride + c];
            else return lds_u16(s * rowb + 2u * c);
        } else if constexpr (MODE == kPacked9) {
            return (t32[s * stride + b / 3u] >> ((b % 3u) * 9u)) & 511u;
        } else return ldg_tab((s << 8) + b);
    }
};

// Shared-memory layout: [pad to a 256-aligned shared address][table image]
// [absorbing-state bitmap][kernel scratch].  Returns the table pointer.
// IdentU8 entries are stored biased by the table's shared address >> 8.
template <int MODE>
__device__ __forceinline__ uint8_t *load_tables(const DevTables &T, uint4 *smem, uint32_t bits_words_n) {
    constexpr uint32_t LR = rep_log_of(MODE);
    constexpr uint32_t AL = 256u << LR;  // table alignment: (s_enc << (8 + LR)) is a row address
    constexpr bool PAD = MODE == kIdentU8P;
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(smem);
    // IdentU8P: s_enc * 260 is a row address, so the table starts at a multiple of 260
    constexpr bool WIN16 = MODE == kWindowU16;
    const uint32_t rowb = 2u * T.stride;  // WindowU16 row bytes (4-byte multiple: odd word count)
    const uint32_t tb = PAD ? (sb + kPadStride - 1u) / kPadStride * kPadStride
                      : WIN16 ? (sb + rowb - 1u) / rowb * rowb : (sb + AL - 1u) & ~(AL - 1u);
    uint8_t *tab = reinterpret_cast<uint8_t *>(smem) + (tb - sb);
    const uint32_t bias2 = WIN16 ? (tb / rowb) * 0x00010001u : 0u;
    const uint32_t bias4 = PAD ? (tb / kPadStride) * 0x01010101u
                         : (MODE == kIdentU8 || LR) ? (tb >> (8 + LR)) * 0x01010101u : 0u;
    const uint4 *src = reinterpret_cast<const uint4 *>(T.image);
    uint4 *dst = reinterpret_cast<uint4 *>(tab);
    for (uint32_t i = threadIdx.x; i < T.image_words / 4; i += blockDim.x) {
        uint4 v = __ldg(src + i);
        if (MODE == kIdentU8 || LR || PAD) {
            v.x = __vadd4(v.x, bias4); v.y = __vadd4(v.y, bias4);
            v.z = __vadd4(v.z, bias4); v.w = __vadd4(v.w, bias4);
        }
        if constexpr (WIN16) {
            // u16 entries + bias; rows are 4-byte multiples, the image 16-byte chunks
            // are not row aligned: store as words
            uint32_t *d32 = reinterpret_cast<uint32_t *>(tab) + 4u * i;
            d32[0] = v.x + bias2; d32[1] = v.y + bias2; d32[2] = v.z + bias2; d32[3] = v.w + bias2;
        } else if constexpr (PAD) {
            // bytes 16j..16j+15 of row s -> s*260 + 16j (4-byte aligned)
            uint32_t *d32 = reinterpret_cast<uint32_t *>(tab) + (i >> 4) * (kPadStride / 4u) + (i & 15u) * 4u;
            d32[0] = v.x; d32[1] = v.y; d32[2] = v.z; d32[3] = v.w;
        } else if constexpr (LR != 0) {
            // bytes 16j..16j+15 of row s -> R copies at (s << (8+LR)) + K(16j)
            constexpr uint32_t M = 7u - LR;
            const uint32_t s = i >> 4, j = i & 15u;
            const uint32_t off = (s << (8 + LR)) | ((16u * j) & ((1u << M) - 1u)) | (((16u * j) >> M) << 7);
#pragma unroll
            for (uint32_t g = 0; g < (1u << LR); g++) dst[(off | (g << M)) >> 4] = v;
        } else {
            dst[i] = v;
        }
    }
    uint32_t *w = reinterpret_cast<uint32_t *>(tab) + smem_words<MODE>(T);
    for (uint32_t i = threadIdx.x; i < bits_words_n; i += blockDim.x) w[i] = __ldg(T.absorb_bits + i);
    return tab;
}

__device__ __forceinline__ uint32_t bits_words(uint32_t nq) { return ((nq + 31) / 32 + 3) & ~3u; }

// converge_kernel scratch per warp: pool_s, pool_id, link (u16 x I_max rounded to 8)
// and first (u8 per state when lane ids fit a byte, else u16), 16-byte multiple
__host__ __device__ __forceinline__ uint32_t converge_scratch_bytes(uint32_t imax, uint32_t nq) {
    const uint32_t ip = (imax + 7u) & ~7u;
    return (6u * ip + (imax <= 254u ? nq : 2u * nq) + 15u) & ~15u;
}

// DFA_OPT_COUNT_WORK: a warp's executed lane-steps into one 64-bit counter
// (called by every thread of the warp at kernel end).
__device__ __forceinline__ void add_work(unsigned long long *ctr, uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o /= 2) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(ctr, (unsigned long long)v);
}

// ---------------------------------------------------------------------------
// lanes_kernel: one thread per execution sub-chunk, <= kLanes lanes in registers.
// ---------------------------------------------------------------------------
// Lanes l >= nlive of a thread do not load: a warp gather in which only some
// threads still carry a second lane costs wavefronts for those threads only.
template <int B, int MODE, bool PX = true, int N>
__device__ __forceinline__ void block16(const Tab<MODE> &tab, uint4 v, uint32_t (&st)[N], uint32_t nlive) {
    static_assert(B <= N, "block16: more lanes than state registers");
    const uint32_t wds[4] = {v.x, v.y, v.z, v.w};
    bool act[B];
#pragma unroll
    for (int l = 0; l < B; l++) act[l] = l == 0 || (uint32_t)l < nlive;
    if constexpr (MODE == kWindowU16) {
        // All 16 bytes inside the aligned window [base, base + W): the column is
        // the byte's low bits, no clamp (residue text: always).  u16 entries and
        // W <= 128, so 2 * column fits the byte lane.
        const uint32_t out = ((v.x ^ tab.base4) | (v.y ^ tab.base4) | (v.z ^ tab.base4) | (v.w ^ tab.base4)) & tab.hi4;
        if (out == 0) {
#pragma unroll
            for (int wi = 0; wi < 4; wi++) {
                const uint32_t xd = (wds[wi] & tab.lo4) << 1;
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const uint32_t a = PX ? __byte_perm(xd, 0u, 0x4440u | (uint32_t)k) : (xd >> (8 * k)) & 0xFFu;
#pragma unroll
                    for (int l = 0; l < B; l++)
                        if (act[l]) st[l] = tab.lds_u16(st[l] * tab.rowb + a);
                }
            }
            return;
        }
    }
#pragma unroll
    for (int wi = 0; wi < 4; wi++) {
        const auto x = tab.wprep(wds[wi]);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const typename Tab<MODE>::Pre c = tab.template bprep<PX>(x, k);
#pragma unroll
            for (int l = 0; l < B; l++)
                if (act[l]) st[l] = tab.look(st[l], x, k, c);
        }
    }
}

// A lane whose slot is `slot` finished: write its final state for every
// original lane it carries (own[r] == slot).
__device__ __forceinline__ void finish_slot(uint32_t slot, uint32_t state, uint32_t (&own)[kLanes],
                                            uint32_t (&fin)[kLanes]) {
#pragma unroll
    for (int r = 0; r < kLanes; r++)
        if (own[r] == slot) { fin[r] = state; own[r] = kDone; }
}

// Merge converged lanes, retire absorbing ones, compact.  B = the
// warp's maximum live-lane count (compile time): the pair tests and the
// compaction cost O(B^2), not O(kLanes^2).
// Sticky-lane suspension: a state A is sticky when every byte either keeps A
// or is a universal kill byte (every state -> Z; e.g. a motif-found state
// over residues, foreign bytes -> the dead sink).  While another lane of the
// thread stays live, a lane in A is parked (Pend: A, the original lanes it
// carries, the 32-byte-aligned offset where it was parked): a kill byte would
// also kill the live lane, so A survives exactly while some live lane does.
// If all live lanes end, the parked lanes resume from the parking offset.
constexpr uint32_t kNoPend = 0xFFFFFFFFu;

template <int B>
__device__ __forceinline__ void checkpoint(const uint32_t *absorb, bool has_absorb, uint32_t bias,
                                           uint32_t (&st)[kLanes],
                                           uint32_t (&own)[kLanes], uint32_t &nlive, uint32_t (&fin)[kLanes],
                                           const uint32_t *sticky, bool suspend, uint32_t &pend,
                                           uint32_t &pend_off, uint32_t cur_off) {
    const uint32_t full = (1u << nlive) - 1u;
    uint32_t lm = full;
    if (nlive == 1) {
        if (has_absorb && test_bit(absorb, st[0] - bias)) { finish_slot(0, st[0] - bias, own, fin); lm = 0; }
    } else {
#pragma unroll
        for (int l = 0; l < B; l++)
            if (has_absorb && ((lm >> l) & 1u) && test_bit(absorb, st[l] - bias)) {
                finish_slot(l, st[l] - bias, own, fin);
                lm &= ~(1u << l);
            }
#pragma unroll
        for (int a = 0; a < B - 1; a++)
#pragma unroll
            for (int b = a + 1; b < B; b++)
                if (((lm >> a) & (lm >> b) & 1u) && st[a] == st[b]) {
                    lm &= ~(1u << b);
#pragma unroll
                    for (int r = 0; r < kLanes; r++)
                        if (own[r] == (uint32_t)b) own[r] = a;
                }
        if (suspend) {
            uint32_t pstate = pend == kNoPend ? kNone : (pend & 0xFFFFu), sm = 0;
#pragma unroll
            for (int l = 0; l < B; l++) {
                if (!((lm >> l) & 1u)) continue;
                const uint32_t q = st[l] - bias;
                if (!test_bit(sticky, q)) continue;
                if (pstate == kNone) pstate = q;
                if (q == pstate) sm |= 1u << l;
            }
            if (sm && sm != lm) {  // keep at least one live lane as the witness
                uint32_t mask = pend == kNoPend ? 0u : (pend >> 16);
#pragma unroll
                for (int l = 0; l < B; l++) {
                    if (!((sm >> l) & 1u)) continue;
#pragma unroll
                    for (int r = 0; r < kLanes; r++)
                        if (own[r] == (uint32_t)l) { mask |= 1u << r; own[r] = kDone; }
                }
                if (pend == kNoPend) pend_off = cur_off;
                pend = pstate | (mask << 16);
                lm &= ~sm;
            }
        }
    }
    if (lm == full) return;
    uint32_t pc[B];
#pragma unroll
    for (int s = 0; s < B; s++) pc[s] = __popc(lm & ((1u << s) - 1u));
    // ns[t] = st[s] for the live slot s of rank t (branch-free masks keep
    // everything in registers: no dynamically indexed array)
    uint32_t ns[B];
#pragma unroll
    for (int t = 0; t < B; t++) {
        uint32_t v = 0, any = 0;
#pragma unroll
        for (int s = t; s < B; s++) {
            const uint32_t hit = 0u - (uint32_t)((((lm >> s) & 1u) != 0) & (pc[s] == (uint32_t)t));
            v |= st[s] & hit;
            any |= hit;
        }
        ns[t] = v | (bias & ~any);  // unused slots keep a valid (encoded) state id
    }
#pragma unroll
    for (int t = 0; t < B; t++) st[t] = ns[t];
#pragma unroll
    for (int r = 0; r < kLanes; r++)
        if (own[r] != kDone) own[r] = __popc(lm & ((1u << own[r]) - 1u));
    nlive = __popc(lm);
}

// 16 bytes on B lanes, then (convergence on) the checkpoint; true = all lanes done.
template <int B, int MODE>
__device__ __forceinline__ bool block_step(const Tab<MODE> &tab, uint4 v, const uint32_t *absorb, bool has_absorb,
                                           uint32_t (&st)[kLanes], uint32_t (&own)[kLanes], uint32_t &nlive,
                                           uint32_t (&fin)[kLanes], int convergence, bool tick,
                                           const uint32_t *sticky, bool suspend, uint32_t &pend, uint32_t &pend_off,
                                           uint32_t cur_off) {
    block16<B, MODE>(tab, v, st, nlive);
    if (!convergence) return false;
    if (B > 1 && nlive > 1) {
        checkpoint<B>(absorb, has_absorb, tab.bias, st, own, nlive, fin, sticky, suspend, pend, pend_off, cur_off);
        return nlive == 0;
    }
    if (has_absorb && tick && nlive == 1 && test_bit(absorb, st[0] - tab.bias)) {
        finish_slot(0, st[0] - tab.bias, own, fin);  // the lane is done
        return true;
    }
    return false;
}

template <int MODE>
__device__ __forceinline__ void step_scalar(const Tab<MODE> &tab, uint32_t b, uint32_t (&st)[kLanes],
                                            uint32_t nlive) {
    const typename Tab<MODE>::Pre pb = tab.bpre(b);
#pragma unroll
    for (int l = 0; l < kLanes; l++)
        if ((uint32_t)l < nlive) st[l] = tab.look_pre(st[l], pb);
}

// Parked lanes resume as one live slot (the state's encoding) carrying them.
__device__ __forceinline__ void resume_pend(uint32_t &pend, uint32_t bias, uint32_t (&st)[kLanes],
                                            uint32_t (&own)[kLanes], uint32_t &nlive) {
    const uint32_t mask = pend >> 16, q = pend & 0xFFFFu;
#pragma unroll
    for (int l = 0; l < kLanes; l++)
        if ((uint32_t)l == nlive) st[l] = q + bias;
#pragma unroll
    for (int r = 0; r < kLanes; r++)
        if ((mask >> r) & 1u) own[r] = nlive;
    nlive++;
    pend = kNoPend;
}

template <int MODE, bool STICKY, bool COUNT>
__device__ __forceinline__ void run_lanes(const Tab<MODE> &tab, const uint32_t *absorb, bool has_absorb,
                                          const uint32_t *sticky, const uint32_t *deadb,
                                          const uint8_t *in, uint64_t pos,
                          uint64_t end, uint32_t (&st)[kLanes], uint32_t (&own)[kLanes], uint32_t nl,
                          int convergence, uint32_t (&fin)[kLanes], uint32_t &wk) {
    uint32_t nlive = nl;
    const uint8_t *s0 = in + pos;
    const uint8_t *ptr = s0;
    const uint8_t *endp = in + end;
    uint32_t pend = kNoPend, pend_off = 0;
    const bool susp = STICKY && convergence;
    // head: up to 31 bytes until 32-byte alignment
    while (ptr < endp && (reinterpret_cast<uintptr_t>(ptr) & 31u)) {
        if constexpr (COUNT) wk += nlive;
        step_scalar(tab, *ptr++, st, nlive);
    }
    for (;;) {
        bool restart = false;
        const uint32_t nblk = (uint32_t)((uint64_t)(endp - ptr) >> 5);  // sub-chunks < 128 GiB
        if (nblk) {
            DFA_CHECK(ptr + 32 * (uint64_t)nblk <= endp && !(reinterpret_cast<uintptr_t>(ptr) & 31u),
                      "sub-chunk block loads past its end or misaligned");
            U8x32 cur = ldg32(ptr);
            const uint8_t *nptr = ptr + 32;
            for (uint32_t bi = 0; bi < nblk && !restart; bi++, nptr += 32) {
                U8x32 nxt = cur;
                if (bi + 1 < nblk) nxt = ldg32(nptr);
#pragma unroll
                for (int half = 0; half < 2; half++) {
                    const uint4 v = half ? cur.hi : cur.lo;
                    // the warp steps max(live lanes) lanes (exact, 1..8): lanes converge fast
                    const bool tick = half && (bi & 1);
                    const bool sp = susp && half;
                    const uint32_t co = (uint32_t)(nptr - s0);
                    if constexpr (COUNT) wk += 16u * max(nlive, 1u);  // block16: lane 0 always steps
                    bool done;
                    switch (__reduce_max_sync(__activemask(), nlive)) {
                    case 0:
                    case 1: done = block_step<1>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, sticky, sp, pend, pend_off, co); break;
                    case 2: done = block_step<2>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, sticky, sp, pend, pend_off, co); break;
                    case 3: done = block_step<3>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, sticky, sp, pend, pend_off, co); break;
                    case 4: done = block_step<4>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, sticky, sp, pend, pend_off, co); break;
                    case 5: done = block_step<5>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, sticky, sp, pend, pend_off, co); break;
                    case 6: done = block_step<6>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, sticky, sp, pend, pend_off, co); break;
                    case 7: done = block_step<7>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, sticky, sp, pend, pend_off, co); break;
                    default: done = block_step<8>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, sticky, sp, pend, pend_off, co); break;
                    }
                    if (done) {
                        if (pend == kNoPend) return;
                        restart = true;  // no live witness left: the parked lanes resume
                        break;
                    }
                }
                cur = nxt;
            }
            if (!restart) ptr += (uint64_t)nblk * 32;
        }
        if (!restart) {
            while (ptr < endp) {
                if constexpr (COUNT) wk += nlive;
                step_scalar(tab, *ptr++, st, nlive);
            }
            if (pend == kNoPend) break;
            bool alive = false;  // a live, non-error lane witnesses that no kill byte came
#pragma unroll
            for (int l = 0; l < kLanes; l++)
                if ((uint32_t)l < nlive && !test_bit(deadb, st[l] - tab.bias)) alive = true;
            if (alive) {
                const uint32_t mask = pend >> 16, q = pend & 0xFFFFu;
#pragma unroll
                for (int r = 0; r < kLanes; r++)
                    if ((mask >> r) & 1u) fin[r] = q;
                break;
            }
        }
        ptr = s0 + pend_off;
        resume_pend(pend, tab.bias, st, own, nlive);
    }
    // remaining lanes: final state of the slot that carries them
#pragma unroll
    for (int r = 0; r < kLanes; r++) {
        if ((uint32_t)r >= nl || own[r] == kDone) continue;
        uint32_t v = 0;
#pragma unroll
        for (int l = 0; l < kLanes; l++) v |= st[l] & (0u - (uint32_t)(own[r] == (uint32_t)l));
        fin[r] = v - tab.bias;
    }
}

// ---------------------------------------------------------------------------
// TMA input staging (a.4, north_star): run_lanes with the sub-chunk's 32-byte
// blocks brought into shared memory by cp.async.bulk.tensor ... tile::gather4
// instead of per-thread global loads.  The input is a 2-D tensor of overlapping
// rows (row r = bytes [32 r, 32 r + 64) from a 32-byte aligned base), so every
// lane's aligned position is a row; per warp and stage eight ops fetch 64 bytes
// for each of the 32 lanes into the warp's ring (2 stages x 32 x 64 B, SWIZZLE_64B:
// each lane's 16-byte reads are conflict-free), one mbarrier per (warp, stage),
// no CTA-wide synchronisation.  Every lane of the warp takes part in the issue
// and the waits for max-over-lanes stages; a lane past its own range, or done,
// idles.  Measured on the match step alone (tools/tma_gather4_bench.cu): rep8_u8 at
// 640 threads 2754 vs 2351 GB/s for the register loads; in this kernel (Random):
// 0.1398 vs 0.1316 ms -- every gather4 op takes its operands from uniform registers,
// so the eight ops of a warp-stage are issued one lane at a time (~100 instructions
// per 64 bytes per lane-row, +41 % instructions overall).  Opt-in (DFA_OPT_TMA_INPUT).
// ---------------------------------------------------------------------------
constexpr uint32_t kTmaW = 64, kTmaStages = 2;
__host__ __device__ __forceinline__ uint32_t tma_ring_bytes(uint32_t warps) {
    return 1024u + warps * (kTmaStages * 32u * kTmaW) + warps * (kTmaStages * 8u);
}

template <int MODE>
__device__ __forceinline__ void run_lanes_tma(const Tab<MODE> &tab, const uint32_t *absorb, bool has_absorb,
                                              const uint8_t *in, uint64_t pos, uint64_t end, uint64_t n,
                                              const void *tmap, uint32_t ring, uint32_t bars,
                                              uint32_t (&st)[kLanes], uint32_t (&own)[kLanes], uint32_t nl,
                                              int convergence, uint32_t (&fin)[kLanes], uint32_t &phase) {
    const uint32_t lane = threadIdx.x & 31;
    uint32_t nlive = nl;
    const uint8_t *ptr = in + pos;
    const uint8_t *endp = in + end;
    uint32_t pend = kNoPend, pend_off = 0;
    bool live = nl != 0;
    // head: up to 31 bytes until 32-byte alignment
    while (ptr < endp && (reinterpret_cast<uintptr_t>(ptr) & 31u)) step_scalar(tab, *ptr++, st, nlive);
    // staged blocks: whole 32-byte blocks of the sub-chunk whose 64-byte row lies inside the input
    const uintptr_t base = reinterpret_cast<uintptr_t>(in) & ~(uintptr_t)31;
    const uintptr_t lim = reinterpret_cast<uintptr_t>(in) + n;  // rows must end at or before lim
    uint32_t nblk = live && ptr < endp ? (uint32_t)((uint64_t)(endp - ptr) >> 5) : 0u;
    while (nblk && reinterpret_cast<uintptr_t>(ptr) + 32ull * (nblk - 1) + kTmaW > lim) nblk--;
    const uint32_t nst = (nblk + 1) >> 1;
    const uint32_t wst = __reduce_max_sync(0xffffffffu, nst);
    const uint32_t row0 = nblk ? (uint32_t)((reinterpret_cast<uintptr_t>(ptr) - base) >> 5) : 0u;
    uint32_t r[4];
#pragma unroll
    for (int j = 0; j < 4; j++) r[j] = __shfl_sync(0xffffffffu, row0, 4 * (lane & 7) + j);
    auto issue = [&](uint32_t stg, uint32_t k) {
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(bars + 8 * k), "r"(32u * kTmaW) : "memory");
        __syncwarp();
        if (lane < 8) {
            const uint32_t adv = stg * (kTmaW / 32u);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // the lanes' reads of this stage, then the copy
            asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                         :: "r"(ring + k * 32u * kTmaW + lane * 4u * kTmaW), "l"(tmap), "r"(0), "r"(r[0] + adv), "r"(r[1] + adv),
                            "r"(r[2] + adv), "r"(r[3] + adv), "r"(bars + 8 * k) : "memory");
        }
    };
    for (uint32_t k = 0; k < kTmaStages; k++) if (k < wst) issue(k, k);
    for (uint32_t stg = 0; stg < wst; stg++) {
        const uint32_t k = stg % kTmaStages;
        // (phase: completed uses of each stage's barrier so far in this kernel, one bit per stage)
        const uint32_t par = (phase >> k) & 1u;
        uint32_t done = 0, spins = 0;
        while (!done) {
            asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                         : "=r"(done) : "r"(bars + 8 * k), "r"(par) : "memory");
            if (!done && ++spins > (1u << 26)) asm volatile("trap;");  // never hang the GPU on a lost copy
        }
        phase ^= 1u << k;
        uint4 q[kTmaW / 16];
        const uint32_t rb = ring + k * 32u * kTmaW + lane * kTmaW;
#pragma unroll
        for (int j = 0; j < (int)(kTmaW / 16); j++) {
            uint32_t a = rb + 16 * j;
            a ^= ((a >> 7) & 3u) << 4;  // SWIZZLE_64B
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q[j].x), "=r"(q[j].y), "=r"(q[j].z), "=r"(q[j].w) : "r"(a));
        }
        __syncwarp();
        if (stg + kTmaStages < wst) issue(stg + kTmaStages, k);
        if (live && stg < nst) {
            // the two 32-byte blocks of the stage, one copy of the step code (as run_lanes)
#pragma unroll 1
            for (uint32_t bb = 0; bb < 2 && live; bb++) {
                const uint32_t bi = 2 * stg + bb;
                if (bi >= nblk) break;  // the odd last block: first half of the stage only
                const uint4 blo = bb ? q[2] : q[0], bhi = bb ? q[3] : q[1];
#pragma unroll
                for (int half = 0; half < 2; half++) {
                    const uint4 v = half ? bhi : blo;
                    const bool tick = half && (bi & 1);
                    bool fin_all;
                    switch (__reduce_max_sync(__activemask(), nlive)) {
                    case 0:
                    case 1: fin_all = block_step<1>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, nullptr, false, pend, pend_off, 0u); break;
                    case 2: fin_all = block_step<2>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, nullptr, false, pend, pend_off, 0u); break;
                    case 3: fin_all = block_step<3>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, nullptr, false, pend, pend_off, 0u); break;
                    case 4: fin_all = block_step<4>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, nullptr, false, pend, pend_off, 0u); break;
                    case 5: fin_all = block_step<5>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, nullptr, false, pend, pend_off, 0u); break;
                    case 6: fin_all = block_step<6>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, nullptr, false, pend, pend_off, 0u); break;
                    case 7: fin_all = block_step<7>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, nullptr, false, pend, pend_off, 0u); break;
                    default: fin_all = block_step<8>(tab, v, absorb, has_absorb, st, own, nlive, fin, convergence, tick, nullptr, false, pend, pend_off, 0u); break;
                    }
                    if (fin_all) { live = false; break; }
                }
            }
        }
    }
    if (!live) return;
    ptr += (uint64_t)nblk * 32;
    while (ptr < endp) step_scalar(tab, *ptr++, st, nlive);
    // remaining lanes: final state of the slot that carries them
#pragma unroll
    for (int rr = 0; rr < kLanes; rr++) {
        if ((uint32_t)rr >= nl || own[rr] == kDone) continue;
        uint32_t v = 0;
#pragma unroll
        for (int l = 0; l < kLanes; l++) v |= st[l] & (0u - (uint32_t)(own[rr] == (uint32_t)l));
        fin[rr] = v - tab.bias;
    }
}

// Rank-space maps (maps of <= 8 entries, the grouped path): an entry is either
// a rank code kRank + r = "the r-th state of the NEXT sub-chunk's domain" or
// an absolute state (error states, which no later byte leaves, and
// the final states of the input's last sub-chunk); kNone pads.  Composing
// L_j o L_i is then a pure gather, L_i[x] <- L_j[r] (Eq.MapReduction), with no
// table lookup: the rank was taken once, where the state was produced.
constexpr uint32_t kRank = 0xFF00u;
__device__ __forceinline__ bool is_rank(uint32_t v) { return v - kRank < (uint32_t)kLanes; }

// Warp-level composition of g = 2^g_log consecutive sub-chunk maps (aligned
// groups of lanes, one sub-chunk each): in round r, lane t (t % 2^(r+1) == 0)
// absorbs the map of lane t + 2^r, L_t <- L_{t+2^r} o L_t, with the partner's
// map taken by shuffles.
__device__ __forceinline__ void warp_compose(uint32_t mask, uint32_t g_log, uint32_t (&fin)[kLanes]) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint32_t r = 0; r < g_log; r++) {
        const uint32_t step = 1u << r;
        uint32_t pm[kLanes];
#pragma unroll
        for (int e = 0; e < kLanes; e++) pm[e] = __shfl_down_sync(mask, fin[e], step);
        if ((lane & ((2u << r) - 1)) != 0) continue;
#pragma unroll
        for (int j = 0; j < kLanes; j++) {
            const uint32_t rr = fin[j] - kRank;
            if (rr >= (uint32_t)kLanes) continue;
            uint32_t v = 0;
#pragma unroll
            for (int e = 0; e < kLanes; e++) v |= pm[e] & (0u - (uint32_t)(rr == (uint32_t)e));
            fin[j] = v;
        }
    }
}

// One lane's view of a map: entry v (j = lane & 7), the map's domain (its
// first sub-chunk's, replicated over the 8 lanes), ok = the map exists.
struct LMap {
    uint32_t v, dom, ok;
};

// Tree step over the 4 maps of a warp: group g (g % 2gs == 0) <- group g+gs o g.
__device__ __forceinline__ void lmap_merge(LMap &m, uint32_t gs) {
    const uint32_t lane = threadIdx.x & 31, g = lane >> 3;
    const uint32_t sb = ((g + gs) & 3) * 8;
    const uint32_t bdom = __shfl_sync(0xffffffffu, m.dom, sb);
    const uint32_t bok = __shfl_sync(0xffffffffu, m.ok, sb);
    const bool lead = (g & (2 * gs - 1)) == 0 && bok;
    const uint32_t rr = m.v - kRank;
    const bool take = lead && (!m.ok || rr < (uint32_t)kLanes);
    const uint32_t nv = __shfl_sync(0xffffffffu, m.v, sb + (m.ok ? (rr & 7u) : (lane & 7u)));
    if (take) m.v = nv;
    if (lead && !m.ok) { m.dom = bdom; m.ok = 1; }
}

// Tree fold of the n >= 1 maps (rows, doms) in shared memory: each level,
// warp w folds maps 4w..4w+3 into slot w of the other buffer (trows/tdoms,
// >= ceil(n/4) slots; the two alternate).  Result in warp 0, lanes 0..7.
__device__ __forceinline__ LMap cta_tree_fold(uint16_t *rows, uint16_t *doms, uint16_t *trows, uint16_t *tdoms,
                                              uint32_t n) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t g = lane >> 3, j = lane & 7;
    LMap m{kNone, 0, 0};
    for (;;) {
        const uint32_t groups = (n + 3) / 4;
#pragma unroll 1
        for (uint32_t w = warp; w < groups; w += nw) {
            const uint32_t r = 4 * w + g;
            m.ok = r < n;
            m.v = m.ok ? rows[r * 8 + j] : (uint32_t)kNone;
            m.dom = m.ok ? doms[r] : 0u;
            lmap_merge(m, 1);
            lmap_merge(m, 2);
            if (groups > 1) {
                if (lane < 8) trows[w * 8 + j] = (uint16_t)m.v;
                if (lane == 0) tdoms[w] = (uint16_t)m.dom;
            }
        }
        if (groups == 1) break;
        n = groups;
        uint16_t *t = rows; rows = trows; trows = t;
        t = doms; doms = tdoms; tdoms = t;
        __syncthreads();
    }
    return m;
}

// ---------------------------------------------------------------------------
// Fused composition tail (struct Fuse in kernels.cuh).
// ---------------------------------------------------------------------------
// Reporting chunk k's map, 8-lane group view (lane gb + j holds entry j, domain d0):
// the rank-space row and domain, and the API outputs -- the user-order row with states
// (rank codes decoded through the next chunk's I_sigma nd, sigma = the byte before
// b_{k+1}), chunk 0's e0 / user row.  Every lane of the warp calls (has = this group's).
__device__ __forceinline__ void emit_chunk(const DevTables &T, const Fuse &fz, bool has, uint32_t k, uint32_t d0,
                                           uint32_t nd, uint32_t av) {
    const uint32_t lane = threadIdx.x & 31, j = lane & 7, gb = lane & ~7u;
    // independent loads first: the decode row, the user-order translation
    const uint32_t dl = has && k + 1 < fz.P ? (uint32_t)__ldg(T.dom_list + (uint64_t)nd * T.rs + j) : kNone;
    uint32_t du = 0, xl = j;
    if (has && d0 < T.nclass) {
        du = T.dom_user_size[d0];
        xl = j < T.imax_user ? T.xlat[(uint64_t)d0 * T.imax_user + j] : 0u;
    } else if (has) {
        du = d0 == T.start_dom ? 1u : 0u;
    }
    if (has) {
        fz.rep_rows[(uint64_t)k * 8 + j] = (uint16_t)av;
        if (j == 0) fz.rep_doms[k] = (uint16_t)d0;
    }
    const uint32_t rr = av - kRank;
    const uint32_t dv = __shfl_sync(0xffffffffu, dl, gb + (rr & 7u));
    const uint32_t sv = rr < (uint32_t)kLanes ? dv : av;
    if (has && fz.e0 && k == 0 && j == 0) fz.e0[0] = (uint16_t)sv;
    uint16_t *urow = nullptr;
    if (has && fz.user_rows && k > 0) urow = fz.user_rows + (uint64_t)(k - 1) * T.imax_user;
    else if (has && fz.user_row0 && k == 0) urow = fz.user_row0;
    const uint32_t v = __shfl_sync(0xffffffffu, sv, gb + (xl & 7u));
    if (urow && j < T.imax_user) urow[j] = (uint16_t)(j < du ? v : kNone);
}

// Group-sequential fold (compose8's chunk phase): group g of the warp folds its n maps
// rows[0..n) (u16 rows of 8, in order); returns entry j of the composition.  Every lane
// of the warp calls; groups may have different n (0 = none).
__device__ __forceinline__ uint32_t group_fold(const uint16_t *rows, uint32_t n, bool cg) {
    const uint32_t lane = threadIdx.x & 31, j = lane & 7, gb = lane & ~7u;
    const uint32_t nmax = __reduce_max_sync(0xffffffffu, n);
    uint32_t av = kNone, aok = 0;
#pragma unroll 1
    for (uint32_t t0 = 0; t0 < nmax; t0 += 8) {
        uint32_t lv[8];
#pragma unroll
        for (int q = 0; q < 8; q++)
            lv[q] = t0 + q < n ? (uint32_t)(cg ? __ldcg(rows + (uint64_t)(t0 + q) * 8 + j) : rows[(t0 + q) * 8 + j])
                               : (uint32_t)kNone;
#pragma unroll
        for (int q = 0; q < 8; q++) {
            const bool bok = t0 + q < n;
            const uint32_t rr = av - kRank;
            const bool take = bok && (!aok || rr < (uint32_t)kLanes);
            const uint32_t nv = __shfl_sync(0xffffffffu, lv[q], gb + (aok ? (rr & 7u) : j));
            if (take) av = nv;
            aok |= bok;
        }
    }
    return av;
}

// Segment geometry of the fused tail: CTA b holds leaves [l0, l0 + nl), which lie in
// reporting chunks ka..ka+nseg-1 (a "segment" = one chunk's leaves inside this CTA).
// (32-bit: the fused path has one sub-chunk per thread of one wave, NS < 2^21)
struct TailGeom {
    uint32_t LPC, nl, ka, nseg, l0;
};
__device__ __forceinline__ uint32_t fuse_chunk_of(const Fuse &fz, uint32_t l) {
    return l < fz.L0 ? 0u : 1u + (l - fz.L0) / fz.L;
}
__device__ __forceinline__ uint32_t fuse_first_leaf(const Fuse &fz, uint32_t k) {
    return k == 0 ? 0u : fz.L0 + (k - 1) * fz.L;
}
__device__ __forceinline__ TailGeom tail_geom(const Plan &p, const Fuse &fz, uint32_t g_log) {
    TailGeom g;
    g.LPC = blockDim.x >> g_log;
    const uint32_t NL = (uint32_t)(p.NS >> g_log);
    g.l0 = blockIdx.x * g.LPC;
    g.nl = min(g.LPC, NL > g.l0 ? NL - g.l0 : 0u);
    g.ka = g.nl ? fuse_chunk_of(fz, g.l0) : 0;
    g.nseg = g.nl ? fuse_chunk_of(fz, g.l0 + g.nl - 1) - g.ka + 1 : 0;
    return g;
}
// Tail shared-memory layout for N = max(leaves per CTA, grid) maps: [rows N][segs N]
// [parts N][scratch N/4+1] (uint4 each), [segment info N] (uint2), then u16 [ldom N]
// [sdom N][pdom N][scratch N/4+1].
struct TailSmem {
    uint16_t *rows, *segs, *prow, *scr, *ldom, *sdom, *pdom, *sdoms;
    uint2 *sinfo;
    __device__ __forceinline__ TailSmem(uint4 *smem, uint32_t N) {
        const uint32_t ns = N / 4 + 1;
        rows = reinterpret_cast<uint16_t *>(smem);
        segs = reinterpret_cast<uint16_t *>(smem + N);
        prow = reinterpret_cast<uint16_t *>(smem + 2 * N);
        scr = reinterpret_cast<uint16_t *>(smem + 3 * N);
        sinfo = reinterpret_cast<uint2 *>(smem + 3 * N + ns);
        ldom = reinterpret_cast<uint16_t *>(sinfo + N);
        sdom = ldom + N;
        pdom = sdom + N;
        sdoms = pdom + N;
    }
};
// segment info: x = a | n << 11 | whole << 22 | big << 23 (a, n <= 1024), y = b_lo | nparts << 16
constexpr uint32_t kSegWhole = 1u << 22, kSegBig = 1u << 23;
// At kernel start (latency hidden by the match loop): the decode domain of each segment's
// chunk -- I_sigma of the byte before b_{k+1} -- into the tail's info area.
__device__ __forceinline__ void tail_prefetch(const DevTables &T, const Plan &p, const Fuse &fz, const uint8_t *in,
                                              uint4 *smem, uint32_t g_log) {
    const TailGeom g = tail_geom(p, fz, g_log);
    uint16_t *info = reinterpret_cast<uint16_t *>(reinterpret_cast<uint8_t *>(smem) + fz.info_off);
    for (uint32_t t = threadIdx.x; t < g.nseg; t += blockDim.x) {
        const uint32_t k = g.ka + t;
        info[t] = k + 1 < fz.P ? (uint16_t)T.byte_class[__ldg(in + p.bounds[k + 1] - 1)] : (uint16_t)0;
    }
}

// The tail proper (every thread of the CTA; the CTA's matching is done).  Shared memory
// is the table's (no longer read), laid out as TailSmem; the info area follows it.
__device__ __forceinline__ void fused_tail(const DevTables &T, const Plan &p, const Fuse &fz, uint4 *smem,
                                           uint32_t g_log, const uint16_t *leaf_rows, const uint16_t *leaf_dom,
                                           DevStatus *status) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const uint32_t j = lane & 7, grp = lane >> 3;
    const TailGeom g = tail_geom(p, fz, g_log);
    const uint32_t LPC = g.LPC, nl = g.nl, ka = g.ka, nseg = g.nseg, l0 = g.l0;
    TailSmem S(smem, max(LPC, gridDim.x));
    const uint16_t *info = reinterpret_cast<const uint16_t *>(reinterpret_cast<const uint8_t *>(smem) + fz.info_off);
    // (no static __shared__ in the lanes kernel: it would move the table's shared address,
    // which the IdentU8 state bias is derived from)
    uint32_t &s_last = *reinterpret_cast<uint32_t *>(reinterpret_cast<uint8_t *>(smem) + fz.info_off + ((2u * LPC + 7u) & ~3u));
    __syncthreads();  // every warp is past its match loop (its leaves are written): the table's space is free
#ifdef DFA_TREE_TIMING
    const unsigned long long t_tail0 = gtimer();
#endif
    for (uint32_t t = threadIdx.x; t < nl; t += blockDim.x) {
        reinterpret_cast<uint4 *>(S.rows)[t] = __ldcg(reinterpret_cast<const uint4 *>(leaf_rows) + l0 + t);
        S.ldom[t] = __ldcg(leaf_dom + l0 + t);
    }
    // segment geometry, once per segment: leaves [a, a + n) of the CTA, whole chunk or
    // straddling (parts b_lo .. b_lo + nparts - 1), big = the CTA-wide pass
    for (uint32_t t = threadIdx.x; t < nseg; t += blockDim.x) {
        const uint32_t k = ka + t;
        const uint32_t f = fuse_first_leaf(fz, k), e = fuse_first_leaf(fz, k + 1);
        const uint32_t a = max(f, l0) - l0, n = min(e, l0 + nl) - l0 - a;
        const bool whole = f >= l0 && e <= l0 + nl;
        const uint32_t b_lo = f / LPC, np = (e - 1) / LPC - b_lo + 1;
        const bool big = n > 64 || (!whole && np > 8);
        S.sinfo[t] = make_uint2(a | n << 11 | (whole ? kSegWhole : 0u) | (big ? kSegBig : 0u), b_lo | np << 16);
    }
    __syncthreads();
#ifdef DFA_TREE_TIMING
    if (threadIdx.x == 0) atomicMax(&g_tree_t[11], gtimer());
    if (threadIdx.x == 0) atomicMax(&g_tree_t[13], gtimer() - t_tail0);  // staging + geometry, per CTA
#endif
    // segment sgi = chunk ka + sgi: a chunk wholly in this CTA yields its reporting row here,
    // a straddling chunk publishes this CTA's part (slot k + b) and the last CTA to arrive
    // folds the parts in order.  Short segments (<= 64 leaves, <= 8 parts): an 8-lane group
    // each, sequential folds.
    for (uint32_t s0 = warp * 4; s0 < nseg; s0 += nw * 4) {
        const uint32_t sgi = s0 + grp, k = ka + sgi;
        const uint2 si = sgi < nseg ? S.sinfo[sgi] : make_uint2(0u, 0u);
        const uint32_t a = si.x & 2047u, n = (si.x >> 11) & 2047u, b_lo = si.y & 0xFFFFu, nparts = si.y >> 16;
        const bool whole = (si.x & kSegWhole) != 0;
        const bool has = sgi < nseg && !(si.x & kSegBig);  // big: the CTA-wide pass below
        const uint32_t av = group_fold(S.rows + a * 8, has ? n : 0u, false);
        const uint32_t d = has ? S.ldom[a] : 0u;
        if (has) {
            S.segs[sgi * 8 + j] = (uint16_t)av;
            if (j == 0) S.sdom[sgi] = (uint16_t)d;
            if (fz.starts) fz.part_rows[((uint64_t)k + blockIdx.x) * 8 + j] = (uint16_t)av;  // starts walk
        }
        if (!fz.rows) continue;
        const bool part = has && !whole;
        if (part) {
            fz.part_rows[((uint64_t)k + blockIdx.x) * 8 + j] = (uint16_t)av;
            if (j == 0) fz.part_doms[k + blockIdx.x] = (uint16_t)d;
        }
        __syncwarp();
        uint32_t prev = 0;
        if (part && j == 0)
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(fz.chunk_cnt + k) : "memory");
        prev = __shfl_sync(0xffffffffu, prev, lane & ~7u);
        const bool last = part && prev + 1 == nparts;
        if (last && j == 0) fz.chunk_cnt[k] = 0;  // every part has arrived: reset for the next launch
        const uint32_t pv = group_fold(fz.part_rows + ((uint64_t)k + b_lo) * 8, last ? nparts : 0u, true);
        const bool out = (has && whole) || last;
        const uint32_t od = last ? (uint32_t)__ldcg(fz.part_doms + k + b_lo) : d;
        emit_chunk(T, fz, out, k, od, out ? (uint32_t)info[sgi] : 0u, last ? pv : av);
    }
#ifdef DFA_TREE_TIMING
    if (lane == 0) atomicMax(&g_tree_t[18], gtimer() - t_tail0);  // short-segment phase, per warp
#endif
    // big segments (a chunk of > 64 leaves here, or one spanning > 8 CTAs; at most a few
    // per CTA): the whole CTA folds each, and the parts when it arrives last
    for (uint32_t sgi = 0; sgi < nseg; sgi++) {
        const uint2 si = S.sinfo[sgi];
        if (!(si.x & kSegBig)) continue;  // (uniform over the CTA)
        const uint32_t k = ka + sgi;
        const uint32_t a = si.x & 2047u, n = (si.x >> 11) & 2047u, b_lo = si.y & 0xFFFFu, nparts = si.y >> 16;
        const bool whole = (si.x & kSegWhole) != 0;
        __syncthreads();
        const uint32_t d = S.ldom[a];
        const LMap m = cta_tree_fold(S.rows + a * 8, S.ldom + a, S.scr, S.sdoms, n);
        if (warp == 0) {
            if (lane < 8) {
                S.segs[sgi * 8 + j] = (uint16_t)m.v;
                if (fz.starts || (fz.rows && !whole)) fz.part_rows[((uint64_t)k + blockIdx.x) * 8 + j] = (uint16_t)m.v;
            }
            if (lane == 0) {
                S.sdom[sgi] = (uint16_t)d;
                s_last = 0;
                if (fz.rows && !whole) {
                    fz.part_doms[k + blockIdx.x] = (uint16_t)d;
                    uint32_t prev;
                    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(fz.chunk_cnt + k) : "memory");
                    if (prev + 1 == nparts) {
                        fz.chunk_cnt[k] = 0;
                        s_last = 1;
                    }
                }
            }
            if (fz.rows && whole) emit_chunk(T, fz, grp == 0, k, d, info[sgi], m.v);
        }
        __syncthreads();
        if (!s_last) continue;
        for (uint32_t t = threadIdx.x; t < nparts; t += blockDim.x) {
            reinterpret_cast<uint4 *>(S.prow)[t] = __ldcg(reinterpret_cast<const uint4 *>(fz.part_rows) + k + b_lo + t);
            S.pdom[t] = __ldcg(fz.part_doms + k + b_lo + t);
        }
        __syncthreads();
        const uint32_t pd = S.pdom[0];
        const LMap pm = cta_tree_fold(S.prow, S.pdom, S.scr, S.sdoms, nparts);
        if (warp == 0) emit_chunk(T, fz, grp == 0, k, pd, info[sgi], pm.v);
    }
    __syncthreads();
#ifdef DFA_TREE_TIMING
    if (threadIdx.x == 0) atomicMax(&g_tree_t[12], gtimer());
    if (threadIdx.x == 0) atomicMax(&g_tree_t[17], gtimer() - t_tail0);  // whole chunk phase, per CTA
#endif
    // the CTA map: its segment maps in order
    LMap cm{kNone, 0, 0};
    if (nseg > 1) cm = cta_tree_fold(S.segs, S.sdom, S.scr, S.sdoms, nseg);
    else cm.v = j < 8 ? S.segs[j] : kNone;
    if (warp == 0) {
        if (lane < 8) fz.cta_rows[(uint64_t)blockIdx.x * 8 + j] = (uint16_t)cm.v;
        if (lane == 0) fz.cta_doms[blockIdx.x] = S.sdom[0];
        __syncwarp();
        if (lane == 0) {
            uint32_t prev;
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(fz.ticket) : "memory");
            s_last = prev + 1 == gridDim.x;
            if (s_last) atomicExch(fz.ticket, 0u);  // every CTA has its ticket: reset for the next launch
        }
    }
    __syncthreads();
#ifdef DFA_TREE_TIMING
    if (threadIdx.x == 0) atomicMax(&g_tree_t[16], gtimer());
#endif
    if (!s_last) return;
    // last CTA: the CTA maps staged in shared memory and folded by the whole CTA
    const uint32_t G = gridDim.x;
    for (uint32_t b = threadIdx.x; b < G; b += blockDim.x) {
        reinterpret_cast<uint4 *>(S.rows)[b] = __ldcg(reinterpret_cast<const uint4 *>(fz.cta_rows) + b);
        S.ldom[b] = __ldcg(fz.cta_doms + b);
    }
    __syncthreads();
    if (fz.starts && threadIdx.x == 0) {
        // rank code of the state at every CTA's first leaf: the prefix of Eq.SeqReduction
        // over the CTA maps (the input's first state is rank 0 of {q0})
        uint32_t code = kRank;
        for (uint32_t b = 0; b < G; b++) {
            fz.cta_code[b] = (uint16_t)code;
            if (is_rank(code)) code = S.rows[b * 8 + (code - kRank)];
        }
    }
    __syncthreads();
    LMap fm{kNone, 0, 0};
    if (G > 1) fm = cta_tree_fold(S.rows, S.ldom, S.scr, S.sdoms, G);
    else fm.v = j < 8 ? S.rows[j] : kNone;
    if (threadIdx.x == 0) {
        const uint32_t fs = fm.v;  // absolute: the input's last sub-chunk ends in states
        if (fs == T.poison) atomicMax(&status->err, 5u);
        if (is_rank(fs)) atomicMax(&status->err, 8u);
        status->final_state = fs;
        status->accept = fs < T.nq ? (uint32_t)test_bit(T.accept_bits, fs) : 0u;
        if (fz.final2) {
            fz.final2[0] = (uint16_t)fs;
            fz.final2[1] = (uint16_t)status->accept;
        }
#ifdef DFA_TREE_TIMING
        atomicMax(&g_tree_t[19], gtimer());
#endif
    }
}

// COUNT: the DFA_OPT_COUNT_WORK instantiation (a live counter register would make the
// timed kernel spill, so counting is a separate instantiation)
template <int MODE, bool STICKY, bool COUNT, bool TMA>
__global__ void __launch_bounds__(lanes_max_threads(MODE), 1) lanes_kernel(DevTables T, Plan p, const uint8_t *__restrict__ in,
                                                    const uint16_t *__restrict__ surv,
                                                    const uint8_t *__restrict__ surv_n,
                                                    const uint64_t *__restrict__ surv_pos,
                                                    uint16_t *__restrict__ sfin, uint32_t sk,
                                                    uint16_t *__restrict__ dom_of, int convergence,
                                                    uint16_t *__restrict__ amap, uint32_t g_log,
                                                    uint16_t *__restrict__ leaf_rows, uint16_t *__restrict__ leaf_dom,
                                                    DevStatus *status, uint32_t cap, Fuse fz) {
    pdl_trigger();  // one wave: the composition kernels may take SMs as CTAs retire
#ifdef DFA_TREE_TIMING
    if (threadIdx.x == 0) atomicMin(&g_tree_t[25], gtimer());
#endif
    extern __shared__ uint4 smem4[];
    uint8_t *tsm = load_tables<MODE>(T, smem4, bits_words(T.nq));
    // sticky and error-state bitmaps after the absorbing one (sticky variant only)
    const uint32_t bw = bits_words(T.nq);
    uint32_t *sticky_s = reinterpret_cast<uint32_t *>(tsm) + smem_words<MODE>(T) + bw;
    uint32_t *dead_s = sticky_s + bw;
    if (STICKY) {
        for (uint32_t i = threadIdx.x; i < bw; i += blockDim.x) {
            sticky_s[i] = __ldg(T.sticky_bits + i);
            dead_s[i] = __ldg(T.dead_bits + i);
        }
    }
    __syncthreads();
#ifdef DFA_TREE_TIMING
    if (threadIdx.x == 0) atomicMax(&g_tree_t[26], gtimer());
#endif
    Tab<MODE> tab;
    tab.init(T, tsm);
    const uint32_t *absorb = reinterpret_cast<const uint32_t *>(tsm) + smem_words<MODE>(T);
    uint64_t work = 0;  // executed lane-steps of this thread (DFA_OPT_COUNT_WORK)
    if (fz.on && fz.rows) tail_prefetch(T, p, fz, in, smem4, g_log);
    // TMA input staging: the warp's ring and barriers after the bitmaps; whole warps enter the
    // loop (lanes past NS idle through the warp-collective copy issue and waits)
    uint32_t tma_ring = 0, tma_bars = 0, tma_phase = 0;
    if constexpr (TMA) {
        const uint32_t after = (uint32_t)__cvta_generic_to_shared(absorb + bw);
        const uint32_t nwarps = blockDim.x >> 5, warp = threadIdx.x >> 5;
        const uint32_t ring0 = (after + 1023u) & ~1023u;
        tma_ring = ring0 + warp * (kTmaStages * 32u * kTmaW);
        tma_bars = ring0 + nwarps * (kTmaStages * 32u * kTmaW) + warp * (kTmaStages * 8u);
        if ((threadIdx.x & 31) == 0) {
#pragma unroll
            for (uint32_t k = 0; k < kTmaStages; k++) asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(tma_bars + 8 * k));
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        }
        __syncwarp();
    }
    const uint64_t ns_loop = TMA ? (p.NS + 31) & ~31ull : p.NS;

    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ns_loop;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if constexpr (TMA) {
            if (i >= p.NS) {  // an idle lane of the last warp
                uint32_t st0[kLanes], own0[kLanes], fin0[kLanes];
#pragma unroll
                for (int l = 0; l < kLanes; l++) { st0[l] = tab.enc(0); own0[l] = kDone; fin0[l] = kNone; }
                run_lanes_tma<MODE>(tab, absorb, T.has_absorb != 0, in, 0, 0, p.n, p.tmap, tma_ring, tma_bars, st0, own0, 0u,
                                    convergence, fin0, tma_phase);
                continue;
            }
        }
        uint64_t start, end;
        sub_range(p, i, start, end);
        const uint32_t dom = sub_domain(T, p, in, i, start);
        DFA_CHECK(dom <= T.nclass && start <= end && end <= p.n, "lanes kernel: domain id or sub-chunk range");
        // the next sub-chunk's domain (its sigma = this sub-chunk's last byte), loaded now
        // beside this one's so that the epilogue's rank conversion waits for one load only
        const bool to_rank = g_log != kNoGroup && i + 1 < p.NS && !(p.indep && chunk_first_sub(p, i + 1));
        const uint32_t nd_pre = to_rank ? (uint32_t)T.byte_class[__ldg(in + end - 1)] : 0u;
        dom_of[i] = (uint16_t)dom;
        uint32_t u;
        uint64_t pos;
        if (surv) { u = surv_n[i]; pos = surv_pos[i]; }
        else { u = T.dom_size[dom]; pos = start; }
        DFA_CHECK(u <= (surv ? (uint32_t)kLanes : T.imax) && pos >= start && pos <= end, "lanes kernel: lane count or start");
        // the grouped (rank-space) epilogue: convert, compose the warp's groups, write leaves
        auto grouped_epilogue = [&](uint32_t (&fin)[kLanes]) {
            const uint64_t wbase = i & ~31ull;
            const uint32_t mask = wbase + 32 <= p.NS ? 0xffffffffu : ((1u << (uint32_t)(p.NS - wbase)) - 1u);
            // rank space: final states as ranks in the next sub-chunk's domain
            // I_sigma, sigma = this sub-chunk's last byte (absolute for error
            // states and for the input's last sub-chunk)
            if (to_rank) {
                // rank = position in the next domain's row (<= 8 entries, one 16-byte load)
                const uint4 nr = __ldg(reinterpret_cast<const uint4 *>(T.dom_list + (uint64_t)nd_pre * 8));
                const uint32_t w[4] = {nr.x, nr.y, nr.z, nr.w};
#pragma unroll
                for (int l = 0; l < kLanes; l++) {
                    if ((uint32_t)l >= u) continue;
                    uint32_t rr = kNone;
#pragma unroll
                    for (int e = 0; e < kLanes; e++)
                        if (((w[e >> 1] >> (16 * (e & 1))) & 0xFFFFu) == fin[l]) rr = e;
                    if (rr != kNone) fin[l] = kRank + rr;
                    else if (!(T.has_dead && test_bit(T.dead_bits, fin[l]))) atomicMax(&status->err, 8u);
                }
            }
            __syncwarp(mask);
            warp_compose(mask, g_log, fin);
#ifdef DFA_TREE_TIMING
            if ((threadIdx.x & 31) == 0) atomicMax(&g_tree_t[28], gtimer());
#endif
            if (((threadIdx.x & 31) & ((1u << g_log) - 1)) == 0) {
                const uint64_t leaf = i >> g_log;
                uint4 v;
                v.x = (fin[0] & 0xFFFFu) | (fin[1] << 16);
                v.y = (fin[2] & 0xFFFFu) | (fin[3] << 16);
                v.z = (fin[4] & 0xFFFFu) | (fin[5] << 16);
                v.w = (fin[6] & 0xFFFFu) | (fin[7] << 16);
                // (the fused tail reads its CTA's leaves back: holding them in registers
                // across the grid-stride loop made the match loop spill)
                reinterpret_cast<uint4 *>(leaf_rows)[leaf] = v;
                leaf_dom[leaf] = (uint16_t)dom;
            }
        };
        // grouped with cap = 8 (u <= 8): one pass, the map stays in registers and every
        // thread of the warp reaches the epilogue's shuffles (also u = 0); otherwise
        // passes of <= cap lanes whose finals go through sfin
        const bool single = g_log != kNoGroup && cap >= (uint32_t)kLanes;
        for (uint32_t pass = 0;; pass++) {
            const uint32_t nl = u > pass * cap ? min(cap, u - pass * cap) : 0u;
            uint32_t st[kLanes], own[kLanes], fin[kLanes];
            uint32_t dw[4] = {0, 0, 0, 0};
            if (single && !surv) {  // rows of stride 8 when rs == 8: the domain in one 16-byte load
                const uint4 r4 = __ldg(reinterpret_cast<const uint4 *>(T.dom_list + (uint64_t)dom * 8));
                dw[0] = r4.x; dw[1] = r4.y; dw[2] = r4.z; dw[3] = r4.w;
            }
#pragma unroll
            for (int l = 0; l < kLanes; l++) {
                const uint32_t r = pass * cap + l;
                if ((uint32_t)l < nl) {
                    const uint32_t q = single && !surv ? (dw[l >> 1] >> (16 * (l & 1))) & 0xFFFFu
                                                      : (surv ? surv[i * kLanes + r] : T.dom_list[(uint64_t)dom * T.rs + r]);
                    st[l] = tab.enc(q);
                    own[l] = l;
                } else {
                    st[l] = tab.enc(0);
                    own[l] = kDone;
                }
                fin[l] = kNone;
            }
            uint32_t wk = 0;
            if constexpr (TMA)
                run_lanes_tma<MODE>(tab, absorb, T.has_absorb != 0, in, pos, end, p.n, p.tmap, tma_ring, tma_bars, st, own, nl,
                                    convergence, fin, tma_phase);
            else if (nl) run_lanes<MODE, STICKY, COUNT>(tab, absorb, T.has_absorb != 0, sticky_s, dead_s, in, pos, end, st, own, nl,
                                            convergence, fin, wk);
            work += wk;
#ifdef DFA_TREE_TIMING
            if ((threadIdx.x & 31) == 0) atomicMax(&g_tree_t[27], gtimer());
#endif
            if (single) {
                grouped_epilogue(fin);
                break;
            }
#pragma unroll
            for (int l = 0; l < kLanes; l++)
                if ((uint32_t)l < nl) sfin[i * sk + pass * cap + l] = (uint16_t)fin[l];
            if ((pass + 1) * cap >= u) break;
        }
        if (g_log != kNoGroup && !single) {
            uint32_t fin[kLanes];
#pragma unroll
            for (int e = 0; e < kLanes; e++) fin[e] = (uint32_t)e < u ? sfin[i * sk + e] : (uint32_t)kNone;
            grouped_epilogue(fin);
        }
        if (surv && !p.keep_amap) {
            // resolve this sub-chunk's converge_kernel map in place: survivor code
            // kSurvBase + e -> final state of survivor e (this thread just wrote them)
            uint32_t fin[kLanes];
#pragma unroll
            for (int e = 0; e < kLanes; e++) fin[e] = (uint32_t)e < u ? sfin[i * sk + e] : 0u;
            const uint32_t du = T.dom_size[dom];
            uint4 *row = reinterpret_cast<uint4 *>(amap + i * T.rs);
            for (uint32_t k = 0; k * 8 < du; k++) {
                uint4 v = row[k];
                uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int h = 0; h < 8; h++) {
                    uint32_t a = (w[h >> 1] >> (16 * (h & 1))) & 0xFFFFu;
                    if (a >= kSurvBase && a != kNone) {
                        uint32_t f = 0;
#pragma unroll
                        for (int e = 0; e < kLanes; e++) f |= fin[e] & (0u - (uint32_t)(a - kSurvBase == (uint32_t)e));
                        a = f;
                    }
                    w[h >> 1] = (w[h >> 1] & ~(0xFFFFu << (16 * (h & 1)))) | (a << (16 * (h & 1)));
                }
                row[k] = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
    }
#ifdef DFA_TREE_TIMING
    if ((threadIdx.x & 31) == 0) atomicMax(&g_tree_t[29], gtimer());
#endif
    if constexpr (COUNT) add_work(p.work + 1, work);
    if (fz.on) fused_tail(T, p, fz, smem4, g_log, leaf_rows, leaf_dom, status);
}

// ---------------------------------------------------------------------------
// ceiling_kernel (dfa_gather_ceiling, a measurement aid): the lanes kernel's
// match step alone -- one lane per thread from q0 over `per` bytes, the same
// table layout, 32-byte loads and 16-byte block step, no domains, convergence
// checkpoints, maps or composition.  Its rate is the practical ceiling of the
// layout on this input; out[t] = delta-hat(q0, in[t*per .. (t+1)*per)).
// ---------------------------------------------------------------------------
template <int MODE>
__global__ void __launch_bounds__(1024, 1) ceiling_kernel(DevTables T, const uint8_t *__restrict__ in, uint64_t per,
                                                          uint16_t *__restrict__ out) {
    extern __shared__ uint4 smem4[];
    uint8_t *tsm = load_tables<MODE>(T, smem4, bits_words(T.nq));
    __syncthreads();
    Tab<MODE> tab;
    tab.init(T, tsm);
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint8_t *p = in + tid * per;
    uint32_t st[kLanes];
#pragma unroll
    for (int l = 0; l < kLanes; l++) st[l] = tab.enc(l == 0 ? T.q0 : 0u);
    const uint64_t nblk = per >> 5;
    if (nblk) {
        U8x32 cur = ldg32(p);
        for (uint64_t bi = 0; bi < nblk; bi++) {
            U8x32 nxt = cur;
            if (bi + 1 < nblk) nxt = ldg32(p + 32 * (bi + 1));
            block16<1, MODE>(tab, cur.lo, st, 1u);
            block16<1, MODE>(tab, cur.hi, st, 1u);
            cur = nxt;
        }
    }
    out[tid] = (uint16_t)(st[0] - tab.bias);
}

// ---------------------------------------------------------------------------
// converge_kernel: one warp per sub-chunk, all |I_sigma| lanes in lock-step
// (the lanes of Alg.MatchingInitialStates line 17 for one chunk) over 16-byte
// windows until <= cap (<= kLanes) distinct live states remain.
//   Wide phase (more than 32 lanes): every thread steps ceil(lanes/32) lanes
//   held in registers; after a window, lanes in equal states are merged from the
//   registers (a lane claims first[state], the claim that survives the warp
//   barrier leads, the others link to it), lanes in absorbing states retire
//   (P:450-454), the leaders are compacted into the pool.
//   Narrow phase (<= 32 lanes): one lane per thread, state and lane id in
//   registers, no compaction (a warp step costs the same for 9 or 32 lanes);
//   after each window the distinct live states are counted (match.any) and the
//   stage ends at <= cap.
// Output: survivors (states + position for lanes_kernel) and amap[i][j] = final
// state of initial lane j, or kSurvBase + survivor index.
// Scratch per warp: pool_s, pool_id, link (u16 x I_max each) and first (one
// entry per state: u8 when I_max <= 254, else u16).  link[id] = final state,
// survivor code, or kParent + leader id (needs |Q| <= kParent: converge_ok).
// ---------------------------------------------------------------------------
constexpr uint32_t kParent = 0x8000u;

template <int MODE, bool ID8>
__global__ void __launch_bounds__(1024, 1) converge_kernel(DevTables T, Plan p, const uint8_t *__restrict__ in,
                                                       uint16_t *__restrict__ surv, uint8_t *__restrict__ surv_n,
                                                       uint64_t *__restrict__ surv_pos,
                                                       uint16_t *__restrict__ amap, uint32_t cap) {
    extern __shared__ uint4 smem4[];
    const uint32_t bw = bits_words(T.nq);
    uint8_t *tsm = load_tables<MODE>(T, smem4, bw);
    Tab<MODE> tab;
    tab.init(T, tsm);
    const uint32_t *absorb = reinterpret_cast<const uint32_t *>(tsm) + smem_words<MODE>(T);
    const bool has_absorb = T.has_absorb != 0;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ltmask = (1u << lane) - 1u;
    const uint32_t ip = (T.imax + 7u) & ~7u;
    using FirstT = typename std::conditional<ID8, uint8_t, uint16_t>::type;  // lane ids fit a byte (I_max <= 254)
    constexpr uint32_t kFirstNone = ID8 ? 0xFFu : 0xFFFFu;
    uint8_t *scr = reinterpret_cast<uint8_t *>(const_cast<uint32_t *>(absorb) + bw) +
                   (size_t)warp * converge_scratch_bytes(T.imax, T.nq);
    uint16_t *pool_s = reinterpret_cast<uint16_t *>(scr), *pool_id = pool_s + ip, *link = pool_id + ip;
    FirstT *first = reinterpret_cast<FirstT *>(link + ip);
    for (uint32_t q = lane; q < T.nq; q += 32) first[q] = (FirstT)kFirstNone;
    __syncthreads();

    const uint64_t warps_total = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint64_t work = 0;  // lane-steps of this warp (counted on lane 0; DFA_OPT_COUNT_WORK)
    // The stage is latency-bound (a few windows per sub-chunk, each a dependent chain):
    // the next sub-chunk's bounds are loaded one iteration ahead, and the first 512 bytes
    // of a sub-chunk are fetched at once (one 16-byte block per lane) before its domain
    // is looked up, so the windows take their bytes by shuffle instead of a load each.
    uint64_t i = (uint64_t)blockIdx.x * (blockDim.x >> 5) + warp;
    uint64_t nb0 = 0, nb1 = 0;
    if (i < p.NS) {
        const uint64_t k = sub_chunk_of(p, i);
        nb0 = p.bounds[k];
        nb1 = p.bounds[k + 1];
    }
    for (; i < p.NS; i += warps_total) {
        uint64_t start, end, jsub, cb0 = nb0;
        sub_range_b(p, i, cb0, nb1, start, end, jsub);
        if (i + warps_total < p.NS) {
            const uint64_t k = sub_chunk_of(p, i + warps_total);
            nb0 = p.bounds[k];
            nb1 = p.bounds[k + 1];
        }
        const uint64_t ab0 = start - ((reinterpret_cast<uintptr_t>(in) + start) & 15u);
        const uint64_t pb = ab0 + 16ull * lane;
        const uint4 pre = pb + 16 <= p.n ? ldg16(reinterpret_cast<const uint4 *>(in + pb)) : make_uint4(0, 0, 0, 0);
        // (the byte two before the sub-chunk is loaded beside the one before it: one latency, not two)
        const bool two = p.use_dom2 && T.dom2 && jsub != 0 && start >= cb0 + 2;
        const uint32_t c1 = two ? (uint32_t)T.byte_class[__ldg(in + start - 2)] : 0u;
        const uint32_t dom = sub_domain(T, p, in, i, start);
        const uint32_t u = T.dom_size[dom];
        const uint16_t *dl = T.dom_list + (uint64_t)dom * T.rs;
        DFA_CHECK(dom <= T.nclass && u <= T.imax && start <= end && end <= p.n, "converge: domain or sub-chunk range");
        uint32_t np = u;
        uint64_t pos = start;
        bool fresh = true;  // the pool is still the domain list itself: entry e = (dl[e], id e)
        // An internal sub-chunk (not a reporting chunk's first: those report over all of
        // I_sigma) starts from the two-symbol set I_{s1 s2} = delta(I_s1, s2) \ Z of the two
        // bytes before it, a subset of I_s2 that holds every state the run can be in
        // (Eq.istatesm, Lemma 1): fewer lanes (Worst 165 of 240, Protein 25 of 77).  Lane ids
        // stay ranks in I_s2, so the map and the composition do not change; the entries of
        // unreachable ranks are kNone and never looked up.
        const uint32_t *dl2 = nullptr;
        if (two) {
            const uint32_t pair = c1 * T.nclass + dom;
            dl2 = T.dom2 + (uint64_t)pair * T.dom2_stride;
            np = T.dom2_size[pair];
            DFA_CHECK(dom < T.nclass && np <= u, "converge: two-symbol set");
            for (uint32_t j = lane; j < u; j += 32) link[j] = kNone;
            __syncwarp();
        }
        // window [pos, min(next 16-byte boundary of the address, end)): bytes k0..k1-1 of v
        uint4 v;
        uint32_t k0, k1;
        uint64_t abase;
        auto fetch_window = [&]() {
            abase = pos - ((reinterpret_cast<uintptr_t>(in) + pos) & 15u);
            k0 = (uint32_t)(pos - abase);
            k1 = (uint32_t)(end - abase < 16 ? end - abase : 16);
            const uint64_t wi = (abase - ab0) >> 4;  // (uniform over the warp)
            if (abase + 16 <= p.n && wi < 32) {
                v.x = __shfl_sync(0xffffffffu, pre.x, (uint32_t)wi);
                v.y = __shfl_sync(0xffffffffu, pre.y, (uint32_t)wi);
                v.z = __shfl_sync(0xffffffffu, pre.z, (uint32_t)wi);
                v.w = __shfl_sync(0xffffffffu, pre.w, (uint32_t)wi);
            } else if (abase + 16 <= p.n && abase <= pos) {
                v = ldg16(reinterpret_cast<const uint4 *>(in + abase));
            } else {  // last partial block of the input: byte loads, never past n
                uint32_t wv[4] = {0, 0, 0, 0};
                for (uint32_t k = k0; k < k1; k++) wv[k >> 2] |= (uint32_t)__ldg(in + abase + k) << (8 * (k & 3));
                v = make_uint4(wv[0], wv[1], wv[2], wv[3]);
            }
        };
        // ---- wide phase
        while (np > 32 && np > cap && pos < end) {
            fetch_window();
            uint32_t np_new = 0;
            for (uint32_t base = 0; base < np; base += 32 * kConvergeLA) {
                uint32_t s[kConvergeLA], id[kConvergeLA];
#pragma unroll
                for (int l = 0; l < kConvergeLA; l++) {
                    const uint32_t e = base + lane + 32 * l;
                    uint32_t q = 0;
                    id[l] = e;
                    if (e < np) {
                        if (!fresh) { q = pool_s[e]; id[l] = pool_id[e]; }
                        else if (dl2) { const uint32_t w = __ldg(dl2 + e); q = w & 0xFFFFu; id[l] = w >> 16; }
                        else q = __ldg(dl + e);
                    }
                    DFA_CHECK(q < T.nq && (e >= np || id[l] < T.imax), "converge: pool entry");
                    s[l] = tab.enc(q);
                }
                const uint32_t rows = min((uint32_t)kConvergeLA, (np - base + 31u) / 32u);  // (uniform)
                if (k0 == 0 && k1 == 16) {
                    // a full aligned window: the match kernel's 16-byte step (static byte
                    // selection, per-word column preparation) on B = ceil(lanes left / 32)
                    // lanes per thread
                    const uint32_t nact = np > base + lane ? min((uint32_t)kConvergeLA, (np - base - lane + 31u) / 32u) : 0u;
                    // (three step variants only: the stage is instruction-fetch bound with
                    // eight, Worst: stall no_instruction 4.2 per issue)
                    switch (rows) {
                    case 1: block16<1, MODE, false>(tab, v, s, nact); break;
                    case 2: block16<2, MODE, false>(tab, v, s, nact); break;
                    default: block16<kConvergeLA, MODE, false>(tab, v, s, nact); break;
                    }
                } else {
                    for (uint32_t k = k0; k < k1; k++) {
                        const uint32_t wsel = k >> 2;
                        const uint32_t word = wsel == 0 ? v.x : wsel == 1 ? v.y : wsel == 2 ? v.z : v.w;
                        const uint32_t b = (word >> (8 * (k & 3))) & 0xFFu;
                        const typename Tab<MODE>::Pre pbk = tab.bpre(b);
#pragma unroll
                        for (int l = 0; l < kConvergeLA; l++) s[l] = tab.look_pre(s[l], pbk);
                    }
                }
                // merge from the registers.  A: absorbed lanes retire; a live lane whose
                // state has no leader yet claims it (any claim may win: all claimants are
                // in that state; a leader of an earlier batch stays)
                uint32_t live = 0;
#pragma unroll
                for (int l = 0; l < kConvergeLA; l++) {
                    const uint32_t e = base + lane + 32 * l;
                    s[l] = tab.dec(s[l]);
                    if (e >= np) continue;
                    DFA_CHECK(s[l] < T.nq, "converge: state id past |Q|");
                    if (has_absorb && test_bit(absorb, s[l])) { link[id[l]] = (uint16_t)s[l]; continue; }
                    live |= 1u << l;
                    if (first[s[l]] == kFirstNone) first[s[l]] = (FirstT)id[l];
                }
                __syncwarp();
                // B: the surviving claim leads; the others link to it; leaders are compacted
#pragma unroll
                for (int l = 0; l < kConvergeLA; l++) {
                    if ((uint32_t)l >= rows) break;
                    bool lead = false;
                    if (live & (1u << l)) {
                        const uint32_t w = first[s[l]];
                        lead = w == id[l];
                        if (!lead) link[id[l]] = (uint16_t)(kParent + w);
                    }
                    const uint32_t mask = __ballot_sync(0xffffffffu, lead);
                    if (lead) {
                        const uint32_t off = np_new + __popc(mask & ltmask);
                        pool_s[off] = (uint16_t)s[l];
                        pool_id[off] = (uint16_t)id[l];
                    }
                    np_new += __popc(mask);
                }
                __syncwarp();
            }
            if (lane == 0) work += (uint64_t)(k1 - k0) * np;
            for (uint32_t e = lane; e < np_new; e += 32) first[pool_s[e]] = (FirstT)kFirstNone;
            np = np_new;
            fresh = false;
            pos = abase + k1;
            __syncwarp();
        }
        if (np <= 32) {
            // ---- narrow phase
            const bool act = lane < np;
            uint32_t st1[kLanes];
            uint32_t id = lane;
            {
                uint32_t q = 0;
                if (act) {
                    if (!fresh) { q = pool_s[lane]; id = pool_id[lane]; }
                    else if (dl2) { const uint32_t w = __ldg(dl2 + lane); q = w & 0xFFFFu; id = w >> 16; }
                    else q = __ldg(dl + lane);
                }
                st1[0] = tab.enc(q);
            }
            uint32_t sd, peers, leadmask, nd;
            bool absorbed, lead;
            for (;;) {
                sd = tab.dec(st1[0]);
                DFA_CHECK(sd < T.nq, "converge: state id past |Q|");
                absorbed = act && has_absorb && test_bit(absorb, sd);
                const uint32_t key = act && !absorbed ? sd : (0x10000u | lane);
                peers = __match_any_sync(0xffffffffu, key);
                lead = act && !absorbed && (uint32_t)(__ffs(peers) - 1) == lane;
                leadmask = __ballot_sync(0xffffffffu, lead);
                nd = __popc(leadmask);
                if (nd <= cap || pos >= end) break;
                fetch_window();
                if (act) {
                    if (k0 == 0 && k1 == 16) block16<1, MODE, false>(tab, v, st1, 1u);
                    else
                        for (uint32_t k = k0; k < k1; k++) {
                            const uint32_t wsel = k >> 2;
                            const uint32_t word = wsel == 0 ? v.x : wsel == 1 ? v.y : wsel == 2 ? v.z : v.w;
                            st1[0] = tab.look_pre(st1[0], tab.bpre((word >> (8 * (k & 3))) & 0xFFu));
                        }
                }
                if (lane == 0) work += (uint64_t)(k1 - k0) * np;
                pos = abase + k1;
            }
            // equal states share their leader's survivor slot; at the sub-chunk's end the
            // lanes keep their states
            const uint32_t slot = __popc(leadmask & ltmask);
            const uint32_t lslot = __shfl_sync(0xffffffffu, slot, (uint32_t)(__ffs(peers) - 1));
            const bool more = pos < end;
            if (act) {
                DFA_CHECK(id < T.imax && (!more || absorbed || lslot < (uint32_t)kLanes), "converge: lane id or survivor slot");
                link[id] = (uint16_t)(absorbed || !more ? sd : kSurvBase + lslot);
                if (lead && more) surv[i * kLanes + slot] = (uint16_t)sd;
            }
            if (lane == 0) { surv_n[i] = (uint8_t)(more ? nd : 0u); surv_pos[i] = more ? pos : end; }
        } else {
            // the sub-chunk ended with more than 32 lanes: its map is the lanes' states
            for (uint32_t e = lane; e < np; e += 32) {
                if (!fresh) link[pool_id[e]] = pool_s[e];
                else if (dl2) { const uint32_t w = __ldg(dl2 + e); link[w >> 16] = (uint16_t)w; }
                else link[e] = __ldg(dl + e);
            }
            if (lane == 0) { surv_n[i] = 0; surv_pos[i] = end; }
        }
        __syncwarp();
        for (uint32_t j = lane; j < u; j += 32) {
            uint32_t r = link[j];
            while (r - kParent < (uint32_t)kSurvBase - kParent) {
                DFA_CHECK(r - kParent < T.imax, "converge: parent link");
                r = link[r - kParent];
            }
            amap[i * T.rs + j] = (uint16_t)r;
        }
        __syncwarp();
    }
    if (p.work) add_work(p.work, work);
}

#ifdef DFA_TU_MAIN  // composition, batch, lookahead, starts kernels: main translation unit only
// ---------------------------------------------------------------------------
// tree_kernel: the composition tree of Tree (kernels.cuh) in one launch.  Warps
// take level-1 nodes; a warp that finishes a node bumps its parent's arrival
// counter and, if it was the last child, processes the parent too (no warp
// ever waits for another).  A node stages its <= F children's maps in the
// warp's shared-memory slice, then pushes every entry of the first child's
// map through the others: L_{i,j}[q] = L_j[rank_j(L_i[q])] (Eq.MapReduction,
// P:819-830); error states map to themselves (reading R1).
// Counters are never reset: a node is complete when its count reaches a
// multiple of its child count (calls on a stream do not overlap).
// ---------------------------------------------------------------------------

__device__ __forceinline__ void group_range(const TreeLevel &lv, uint32_t g, uint32_t &st, uint32_t &en) {
    if (g < lv.gf) { st = g * lv.G; en = min(lv.f, st + lv.G); return; }
    const uint32_t t = g - lv.gf, seg = t / lv.gm, r = t - seg * lv.gm;
    const uint32_t base = lv.f + seg * lv.m;
    st = base + r * lv.G;
    en = min(base + lv.m, st + lv.G);
}

__device__ __forceinline__ uint32_t parent_of(const TreeLevel &lv, uint32_t c) {
    if (c < lv.f) return c / lv.G;
    const uint32_t t = c - lv.f, seg = t / lv.m;
    return lv.gf + seg * lv.gm + (t - seg * lv.m) / lv.G;
}

__device__ __forceinline__ const uint4 *tree_child_row(const Tree &tr, const DevTables &T, uint32_t Lc, uint32_t c) {
    const uint16_t *p = Lc == 0 ? (tr.amap ? tr.amap + (uint64_t)c * T.rs : tr.sfin + (uint64_t)c * tr.sk)
                                : tr.rows + (uint64_t)(tr.lv[Lc].off + c) * T.rs;
    return reinterpret_cast<const uint4 *>(p);
}

__device__ __forceinline__ uint32_t tree_child_dom(const Tree &tr, uint32_t Lc, uint32_t c) {
    return Lc == 0 ? tr.dom_of[c] : __ldcg(tr.doms + tr.lv[Lc].off + c);
}

// One round of the pairwise composition of maps stored in shared memory
// (row c at st + (c << lrs), domain dch[c]): map a = p * 2^(lstep+1) absorbs
// map b = a + 2^lstep, L_a <- L_b o L_a (Eq.MapReduction).  Tasks (pair,
// entry) are spread over nthr threads and batched U deep so that the U
// dependent load chains (row entry -> rank -> row entry) overlap.  Tasks of a
// round read b rows and write a rows only, so batching is race-free.
template <int U>
__device__ __forceinline__ void pairwise_round(const DevTables &T, const uint8_t *rank8, const uint32_t *dead,
                                               const uint16_t *dsz, const uint16_t *dch, uint16_t *st,
                                               uint32_t lrs, uint32_t lstep, uint32_t npairs, uint32_t tid,
                                               uint32_t nthr, DevStatus *status) {
    const uint32_t rsp = 1u << lrs, ntasks = npairs << lrs;
    for (uint32_t t0 = tid; t0 < ntasks; t0 += nthr * U) {
        uint32_t dst[U], s[U], d[U];
        bool ok[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            const uint32_t t = t0 + q * nthr;
            const uint32_t p = t >> lrs, j = t & (rsp - 1);
            const uint32_t a = p << (lstep + 1), b = a + (1u << lstep);
            ok[q] = t < ntasks && j < dsz[dch[a]];
            dst[q] = (a << lrs) + j;
            s[q] = ok[q] ? st[dst[q]] : 0u;
            d[q] = ok[q] ? ((uint32_t)dch[b] | (b << 16)) : 0u;
            if (ok[q] && T.has_dead && test_bit(dead, s[q])) ok[q] = false;
        }
        uint32_t r[U];
#pragma unroll
        for (int q = 0; q < U; q++) {
            if (!ok[q]) { r[q] = 0; continue; }
            const uint32_t db = d[q] & 0xFFFFu;
            uint32_t v;
            if (rank8) { v = rank8[db * T.nq + s[q]]; v = v == 0xFFu ? kNone : v; }
            else v = __ldg(T.rank + (uint64_t)db * T.nq + s[q]);
            if (v == kNone) { atomicMax(&status->err, 8u); v = 0; }
            r[q] = v;
        }
        uint32_t out[U];
#pragma unroll
        for (int q = 0; q < U; q++) out[q] = ok[q] ? st[((d[q] >> 16) << lrs) + r[q]] : 0u;
#pragma unroll
        for (int q = 0; q < U; q++)
            if (ok[q]) st[dst[q]] = (uint16_t)out[q];
    }
}

// L_a[j] <- L_b[rank_b(L_a[j])]; error states stay
__device__ __forceinline__ void tree_compose_entry(const DevTables &T, const Tree &tr, const uint32_t *dead,
                                                   const uint8_t *rank8, uint16_t *st, uint32_t lrs, uint32_t a,
                                                   uint32_t b, uint32_t j, uint32_t db) {
    const uint32_t s = st[(a << lrs) + j];
    if (T.has_dead && test_bit(dead, s)) return;
    uint32_t r;
    if (rank8) { r = rank8[db * T.nq + s]; r = r == 0xFFu ? kNone : r; }
    else r = __ldg(T.rank + (uint64_t)db * T.nq + s);
    if (r == kNone) { atomicMax(&tr.status->err, 8u); r = 0; }
    DFA_CHECK(r < T.rs && s < T.nq, "tree: rank past the row");
    st[(a << lrs) + j] = st[(b << lrs) + r];
}

__global__ void __launch_bounds__(256) tree_kernel(DevTables T, Tree tr) {
    extern __shared__ uint4 smem4[];
#ifdef DFA_TREE_TIMING
    if (threadIdx.x == 0) atomicMin(&g_tree_t[0], gtimer());
#endif
    // shared: [rank table u8 (optional)][dom sizes u16][error-state bits][warp slices].
    // The walk must not depend on L1: every acquire invalidates it.
    uint8_t *sb = reinterpret_cast<uint8_t *>(smem4);
    const uint32_t rank_bytes = tr.rank_smem ? (((T.nclass + 1) * T.nq + 15) & ~15u) : 0u;
    const uint8_t *rank8 = tr.rank_smem ? sb : T.rank8;
    if (tr.rank_smem) {
        const uint4 *src = reinterpret_cast<const uint4 *>(T.rank8);
        for (uint32_t i = threadIdx.x; i < rank_bytes / 16; i += blockDim.x)
            reinterpret_cast<uint4 *>(sb)[i] = __ldg(src + i);
    }
    uint16_t *dsz = reinterpret_cast<uint16_t *>(sb + rank_bytes);
    const uint32_t dsz_bytes = ((T.nclass + 1) * 2 + 15) & ~15u;
    uint32_t *dead = reinterpret_cast<uint32_t *>(sb + rank_bytes + dsz_bytes);
    const uint32_t dead_words = ((T.nq + 31) / 32 + 3) & ~3u;
    for (uint32_t i = threadIdx.x; i <= T.nclass; i += blockDim.x) dsz[i] = T.dom_size[i];
    for (uint32_t i = threadIdx.x; i < dead_words; i += blockDim.x) dead[i] = __ldg(T.dead_bits + i);
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const uint32_t lrs = tr.lrs, rsp = 1u << lrs;     // shared row stride (power of two)
    const uint32_t q4 = T.rs >> 3;                     // 16-byte pieces of a global row
    uint32_t lq = 0;
    while ((1u << lq) < q4) lq++;                      // pieces per row rounded to a power of two
    uint16_t *slice = reinterpret_cast<uint16_t *>(sb + rank_bytes + dsz_bytes + dead_words * 4) +
                      (size_t)warp * ((tr.F << lrs) + ((tr.F + 7) & ~7u) + rsp);
    uint16_t *st = slice, *dch = slice + (tr.F << lrs), *row = dch + ((tr.F + 7) & ~7u);

    for (uint32_t g1 = blockIdx.x * nwarps + warp; g1 < tr.lv[1].nodes; g1 += gridDim.x * nwarps) {
        uint32_t L = 1;
        uint32_t node = g1;
        for (;;) {
            // ---- process node (L, node): stage children (doms, 16-byte row pieces)
            const TreeLevel lv = tr.lv[L];
            uint32_t c0, c1;
            group_range(lv, node, c0, c1);
            const uint32_t nc = c1 - c0;
            for (uint32_t t = lane; t < nc; t += 32) dch[t] = (uint16_t)tree_child_dom(tr, L - 1, c0 + t);
            for (uint32_t t = lane; t < (nc << lq); t += 32) {
                const uint32_t c = t >> lq, k = t & ((1u << lq) - 1);
                if (k < q4)
                    reinterpret_cast<uint4 *>(st + (c << lrs))[k] = __ldcg(tree_child_row(tr, T, L - 1, c0 + c) + k);
            }
            __syncwarp();
            // pairwise tree over the children in the warp: in round `step`, map a
            // (a = 0, 2step, ...) absorbs map a+step: L_a <- L_{a+step} o L_a
            for (uint32_t step = 1; step < nc; step *= 2) {
                const uint32_t npairs = (nc - step + 2 * step - 1) / (2 * step);
                if (lrs <= 4) {
                    // short rows: (pair, entry) tasks packed across the lanes, 4 deep
                    uint32_t lstep = 0;
                    while ((1u << lstep) < step) lstep++;
                    pairwise_round<4>(T, rank8, dead, dsz, dch, st, lrs, lstep, npairs, lane, 32, tr.status);
                } else {
                    // long rows: lanes over the valid entries of one pair at a time
                    for (uint32_t p = 0; p < npairs; p++) {
                        const uint32_t a = p * 2 * step, b = a + step, ua = dsz[dch[a]], db = dch[b];
                        for (uint32_t j = lane; j < ua; j += 32) tree_compose_entry(T, tr, dead, rank8, st, lrs, a, b, j, db);
                    }
                }
                __syncwarp();
            }
            const uint32_t d0 = dch[0];
            const uint32_t u = dsz[d0];
            for (uint32_t j = lane; j < T.rs; j += 32) row[j] = j < u ? st[j] : kNone;
            __syncwarp();
            uint16_t *orow = tr.rows + (uint64_t)(lv.off + node) * T.rs;
            for (uint32_t t = lane; t < q4; t += 32)
                reinterpret_cast<uint4 *>(orow)[t] = reinterpret_cast<const uint4 *>(row)[t];
            if (lane == 0) tr.doms[lv.off + node] = (uint16_t)d0;
            if (L == tr.rep_level) {
                // reporting chunk k = node: API row in the user's I_sigma order
                if (tr.user_rows && node > 0) {
                    const uint32_t du = d0 < T.nclass ? T.dom_user_size[d0] : 0;
                    uint16_t *urow = tr.user_rows + (uint64_t)(node - 1) * T.imax_user;
                    for (uint32_t j = lane; j < T.imax_user; j += 32)
                        urow[j] = j < du ? row[T.xlat[(uint64_t)d0 * T.imax_user + j]] : kNone;
                }
                if (tr.e0 && node == 0 && lane == 0) tr.e0[0] = row[0];
                if (tr.user_row0 && node == 0) {
                    const uint32_t du = d0 < T.nclass ? T.dom_user_size[d0] : (d0 == T.start_dom ? 1u : 0u);
                    for (uint32_t j = lane; j < T.imax_user; j += 32)
                        tr.user_row0[j] = j < du ? row[d0 < T.nclass ? T.xlat[(uint64_t)d0 * T.imax_user + j] : j]
                                                 : kNone;
                }
            }
#ifdef DFA_TREE_TIMING
            if (lane == 0) atomicMax(&g_tree_t[L], gtimer());
#endif
            if (L == tr.nlevels) {
                // root: Alg.seqmatch lines 4-6 on delta-hat(q0, x) (unless fold_rows_kernel follows)
                if (tr.seg_row && tr.root_final && node == 0) {
                    // the segment map: the root's row over chunk 0's domain, in the user's order
                    const uint32_t du = d0 < T.nclass ? T.dom_user_size[d0] : (d0 == T.start_dom ? 1u : 0u);
                    for (uint32_t j = lane; j < T.imax_user; j += 32)
                        tr.seg_row[j] = j < du ? row[d0 < T.nclass ? T.xlat[(uint64_t)d0 * T.imax_user + j] : j] : kNone;
                }
                if (lane == 0 && tr.root_final && node == 0) {
                    const uint32_t fs = row[0];
                    DevStatus *S = tr.status;
                    if (fs == T.poison) atomicMax(&S->err, 5u);
                    S->final_state = fs;
                    S->accept = fs < T.nq ? (uint32_t)test_bit(T.accept_bits, fs) : 0u;
                    if (tr.dev_final) {
                        tr.dev_final[0] = (uint16_t)fs;
                        tr.dev_final[1] = (uint16_t)S->accept;
                    }
                }
                __syncwarp();
                break;
            }
            // ---- hand the result to the parent; continue with it if last to arrive
            const TreeLevel &up = tr.lv[L + 1];
            const uint32_t parent = parent_of(up, node);
            uint32_t p0, p1;
            group_range(up, parent, p0, p1);
            const uint32_t nchild = p1 - p0;
            __syncwarp();
            uint32_t prev = 0;
            if (lane == 0) {
                // release: this node's row (written by all lanes, ordered by the
                // syncwarp) before the count; acquire: the siblings' rows after it.
                // A release/acquire RMW, not fence.sc: thousands of warps do this.
                asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                             : "=r"(prev) : "l"(tr.counters + up.off + parent) : "memory");
            }
            prev = __shfl_sync(0xffffffffu, prev, 0);
            if ((prev + 1) % nchild != 0) break;
            L++;
            node = parent;
        }
    }
}

// ---------------------------------------------------------------------------
// walk_kernel: one level of the same composition tree for long rows (large
// I_max), one thread per (node, entry): the entry is pushed through the node's
// children in order, each step one rank lookup and one row lookup
// (Eq.MapReduction / Eq.SeqReduction).  One launch per level; the
// chains are short (the host picks small fan-ins) and there are
// nodes * I_max independent ones, so the level is latency-hidden by numbers.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) walk_kernel(DevTables T, Tree tr, uint32_t L) {
    const TreeLevel lv = tr.lv[L];
    const uint64_t total = (uint64_t)lv.nodes * T.rs;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t node = (uint32_t)(t / T.rs), j = (uint32_t)(t - (uint64_t)node * T.rs);
        uint32_t c0, c1;
        group_range(lv, node, c0, c1);
        const uint32_t d0 = tree_child_dom(tr, L - 1, c0);
        const uint32_t u = T.dom_size[d0];
        uint32_t s = kNone;
        if (j < u) {
            s = reinterpret_cast<const uint16_t *>(tree_child_row(tr, T, L - 1, c0))[j];
            for (uint32_t c = c0 + 1; c < c1; c++) {
                if (T.has_dead && test_bit(T.dead_bits, s)) continue;
                const uint32_t d = tree_child_dom(tr, L - 1, c);
                uint32_t r;
                if (T.rank8) { r = __ldg(T.rank8 + (uint64_t)d * T.nq + s); r = r == 0xFFu ? kNone : r; }
                else r = __ldg(T.rank + (uint64_t)d * T.nq + s);
                if (r == kNone) { atomicMax(&tr.status->err, 8u); s = 0; break; }
                DFA_CHECK(r < T.rs && d <= T.nclass, "walk: rank past the row");
                s = reinterpret_cast<const uint16_t *>(tree_child_row(tr, T, L - 1, c))[r];
            }
        }
        tr.rows[(uint64_t)(lv.off + node) * T.rs + j] = (uint16_t)s;
        if (j == 0) tr.doms[lv.off + node] = (uint16_t)d0;
        if (L == tr.rep_level) {
            if (tr.user_rows && node > 0 && j < T.imax_user) {
                // API row: user entry ju = internal entry xlat[ju]; padding 0xFFFF
                const uint32_t du = d0 < T.nclass ? T.dom_user_size[d0] : 0;
                uint16_t *urow = tr.user_rows + (uint64_t)(node - 1) * T.imax_user;
                if (j >= du) urow[j] = kNone;
            }
            if (tr.user_rows && node > 0 && j < u && d0 < T.nclass) {
                const uint32_t ju = T.ixlat[(uint64_t)d0 * T.rs + j];
                if (ju != kNone) tr.user_rows[(uint64_t)(node - 1) * T.imax_user + ju] = (uint16_t)s;
            }
            if (tr.e0 && node == 0 && j == 0) tr.e0[0] = (uint16_t)s;
            if (tr.user_row0 && node == 0) {
                const uint32_t du = d0 < T.nclass ? T.dom_user_size[d0] : (d0 == T.start_dom ? 1u : 0u);
                if (j < T.imax_user && j >= du) tr.user_row0[j] = kNone;
                if (j < u) {
                    const uint32_t ju = d0 < T.nclass ? T.ixlat[(uint64_t)d0 * T.rs + j] : j;
                    if (ju != kNone) tr.user_row0[ju] = (uint16_t)s;
                }
            }
        }
        if (tr.seg_row && L == tr.nlevels && node == 0) {
            // the segment map: the root's row over chunk 0's domain, in the user's order
            const uint32_t du = d0 < T.nclass ? T.dom_user_size[d0] : (d0 == T.start_dom ? 1u : 0u);
            if (j < T.imax_user && j >= du) tr.seg_row[j] = kNone;
            if (j < u) {
                const uint32_t ju = d0 < T.nclass ? T.ixlat[(uint64_t)d0 * T.rs + j] : j;
                if (ju != kNone) tr.seg_row[ju] = (uint16_t)s;
            }
        }
        if (L == tr.nlevels && node == 0 && j == 0) {
            DevStatus *S = tr.status;
            if (s == T.poison) atomicMax(&S->err, 5u);
            S->final_state = s;
            S->accept = s < T.nq ? (uint32_t)test_bit(T.accept_bits, s) : 0u;
            if (tr.dev_final) {
                tr.dev_final[0] = (uint16_t)s;
                tr.dev_final[1] = (uint16_t)S->accept;
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Factored composition for long rows behind the converge stage (I_max > kLanes):
// a sub-chunk's map is its converge map amap (I_sigma -> absorbed state or
// survivor code) followed by the <= kLanes survivor finals of lanes_kernel, so
// every composed node is "the first leaf's amap, then nv values":
//   FACT node: row[j] = amap_f[j] < kSurvBase ? amap_f[j] : vals[amap_f[j] - kSurvBase]
//   FULL node: row[j] = vals[j]   (first leaf ended inside converge_kernel with
//                                  all-absolute amap: vals = that row pushed on)
// Composing a node costs nv (<= 8) chains instead of I_max (Eq.MapReduction,
// P:819-830, on the image of the first map only); full rows are written for the
// reporting chunks and the root alone (fexpand_kernel).
// ---------------------------------------------------------------------------
struct FNode {
    const uint16_t *vals;
    uint32_t nv, full, fl, dom;
};

__device__ __forceinline__ FNode fnode(const DevTables &T, const Tree &tr, uint32_t Lc, uint32_t c) {
    FNode n;
    if (Lc == 0) {
        n.nv = tr.leaf_nv[c];
        n.fl = c;
        n.dom = tr.dom_of[c];
        n.full = n.nv == 0;  // no survivor codes: the converge map holds final states only
        if (n.full) { n.vals = tr.amap + (uint64_t)c * T.rs; n.nv = T.dom_size[n.dom]; }
        else n.vals = tr.sfin + (uint64_t)c * tr.sk;
    } else {
        const uint32_t idx = tr.lv[Lc].off + c;
        const uint32_t w = tr.node_nv[idx];
        n.nv = w & 0x7FFFu;
        n.full = w >> 15;
        n.fl = tr.node_fl[idx];
        n.dom = tr.doms[idx];
        n.vals = tr.rows + (uint64_t)idx * T.rs;
    }
    DFA_CHECK(n.dom <= T.nclass && n.nv <= T.rs, "fnode: domain or value count");
    return n;
}

// state s entering node B -> state leaving it (error states pass)
__device__ __forceinline__ uint32_t fapply(const DevTables &T, const Tree &tr, const FNode &B, uint32_t s) {
    if (s == kNone) return s;  // (an unreachable rank of a FULL node behind a two-symbol start)
    if (T.has_dead && test_bit(T.dead_bits, s)) return s;
    uint32_t r;
    if (T.rank8) { r = __ldg(T.rank8 + (uint64_t)B.dom * T.nq + s); r = r == 0xFFu ? kNone : r; }
    else r = __ldg(T.rank + (uint64_t)B.dom * T.nq + s);
    if (r == kNone) { atomicMax(&tr.status->err, 8u); return 0; }
    DFA_CHECK(r < T.rs, "fapply: rank past the row");
    if (B.full) return B.vals[r];
    const uint32_t c = tr.amap[(uint64_t)B.fl * T.rs + r];
    if (c < kSurvBase) return c;
    DFA_CHECK(c - kSurvBase < B.nv, "fapply: survivor code past the node's values");
    return B.vals[c - kSurvBase];
}

// entry j of a node's full row
__device__ __forceinline__ uint32_t frow(const DevTables &T, const Tree &tr, const FNode &N, uint32_t j) {
    if (N.full) return N.vals[j];
    const uint32_t c = tr.amap[(uint64_t)N.fl * T.rs + j];
    return c < kSurvBase ? c : N.vals[c - kSurvBase];
}

// one level: 8 threads per node, thread e pushes value e (e + 8, ...) of the first child
// through the node's other children
__global__ void __launch_bounds__(256) fwalk_kernel(DevTables T, Tree tr, uint32_t L) {
    pdl_trigger();
    pdl_wait();
    const TreeLevel lv = tr.lv[L];
    const uint64_t total = (uint64_t)lv.nodes * 8;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t node = (uint32_t)(t >> 3), e0 = (uint32_t)t & 7u;
        uint32_t c0, c1;
        group_range(lv, node, c0, c1);
        const FNode A = fnode(T, tr, L - 1, c0);
        const uint32_t idx = lv.off + node;
        uint16_t *out = tr.rows + (uint64_t)idx * T.rs;
        for (uint32_t e = e0; e < A.nv; e += 8) {
            uint32_t s = A.vals[e];
            for (uint32_t c = c0 + 1; c < c1; c++) s = fapply(T, tr, fnode(T, tr, L - 1, c), s);
            out[e] = (uint16_t)s;
        }
        if (e0 == 0) {
            tr.node_nv[idx] = (uint16_t)(A.nv | (A.full << 15));
            tr.node_fl[idx] = A.fl;
            tr.doms[idx] = (uint16_t)A.dom;
        }
    }
}

// full rows of level L's nodes: the reporting chunks (internal rows for starts/batch, API
// rows in the user's order, e0) and the root (final state, accept, segment row)
// the root's outputs for entry j of its row (value s): segment row, final state, accept bit
__device__ __forceinline__ void froot_out(const DevTables &T, const Tree &tr, uint32_t d0, uint32_t u, uint32_t j,
                                          uint32_t s) {
    if (tr.seg_row) {
        // the segment map: the root's row over chunk 0's domain, in the user's order
        const uint32_t du = d0 < T.nclass ? T.dom_user_size[d0] : (d0 == T.start_dom ? 1u : 0u);
        if (j < T.imax_user && j >= du) tr.seg_row[j] = kNone;
        if (j < u) {
            const uint32_t ju = d0 < T.nclass ? T.ixlat[(uint64_t)d0 * T.rs + j] : j;
            if (ju != kNone) tr.seg_row[ju] = (uint16_t)s;
        }
    }
    if (j == 0) {
        DevStatus *S = tr.status;
        if (s == T.poison) atomicMax(&S->err, 5u);
        S->final_state = s;
        S->accept = s < T.nq ? (uint32_t)test_bit(T.accept_bits, s) : 0u;
        if (tr.dev_final) {
            tr.dev_final[0] = (uint16_t)s;
            tr.dev_final[1] = (uint16_t)S->accept;
        }
    }
}

__global__ void __launch_bounds__(256) fexpand_kernel(DevTables T, Tree tr, uint32_t L) {
    pdl_trigger();
    pdl_wait();
    const TreeLevel lv = tr.lv[L];
    const bool rep = L == tr.rep_level, root = L == tr.nlevels && tr.root_final;
    const uint64_t total = (uint64_t)(rep ? lv.nodes : 1u) * T.rs;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total;
         t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t node = (uint32_t)(t / T.rs), j = (uint32_t)(t - (uint64_t)node * T.rs);
        const FNode N = fnode(T, tr, L, node);
        const uint32_t d0 = N.dom, u = T.dom_size[d0];
        const uint32_t s = j < u ? frow(T, tr, N, j) : (uint32_t)kNone;
        if (rep) {
            tr.rep_full[(uint64_t)node * T.rs + j] = (uint16_t)s;
            if (tr.user_rows && node > 0 && j < T.imax_user) {
                // API row: user entry ju = internal entry xlat[ju]; padding 0xFFFF
                const uint32_t du = d0 < T.nclass ? T.dom_user_size[d0] : 0;
                if (j >= du) tr.user_rows[(uint64_t)(node - 1) * T.imax_user + j] = kNone;
            }
            if (tr.user_rows && node > 0 && j < u && d0 < T.nclass) {
                const uint32_t ju = T.ixlat[(uint64_t)d0 * T.rs + j];
                if (ju != kNone) tr.user_rows[(uint64_t)(node - 1) * T.imax_user + ju] = (uint16_t)s;
            }
            if (tr.e0 && node == 0 && j == 0) tr.e0[0] = (uint16_t)s;
            if (tr.user_row0 && node == 0) {
                const uint32_t du = d0 < T.nclass ? T.dom_user_size[d0] : (d0 == T.start_dom ? 1u : 0u);
                if (j < T.imax_user && j >= du) tr.user_row0[j] = kNone;
                if (j < u) {
                    const uint32_t ju = d0 < T.nclass ? T.ixlat[(uint64_t)d0 * T.rs + j] : j;
                    if (ju != kNone) tr.user_row0[ju] = (uint16_t)s;
                }
            }
        }
        if (root && node == 0) froot_out(T, tr, d0, u, j, s);
    }
}

// link values: state sv leaving a FACT node re-coded into the next FACT node's code space
// (its first leaf nfl, domain nd): the next node's converge code amap[rank(sv)], or sv itself
// for an error state.  U independent chains per thread, each stage's loads issued together
// (the kernels that use it are latency-bound on these dependent L2 loads).
template <int U>
__device__ __forceinline__ void flink_batch(const DevTables &T, const Tree &tr, const bool (&ok)[U],
                                            const uint32_t (&sv)[U], const uint32_t (&nd)[U],
                                            const uint32_t (&nfl)[U], uint32_t (&c)[U]) {
    bool lk[U];
    uint32_t r[U];
#pragma unroll
    for (int u = 0; u < U; u++) lk[u] = ok[u] && !(T.has_dead && test_bit(T.dead_bits, sv[u]));
#pragma unroll
    for (int u = 0; u < U; u++) {
        r[u] = 0;
        if (!lk[u]) continue;
        if (T.rank8) { r[u] = __ldg(T.rank8 + (uint64_t)nd[u] * T.nq + sv[u]); r[u] = r[u] == 0xFFu ? (uint32_t)kNone : r[u]; }
        else r[u] = __ldg(T.rank + (uint64_t)nd[u] * T.nq + sv[u]);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
        c[u] = sv[u];
        if (!lk[u]) continue;
        if (r[u] == kNone) { atomicMax(&tr.status->err, 8u); r[u] = 0; }
        DFA_CHECK(r[u] < T.rs, "flink: rank past the row");
        c[u] = tr.amap[(uint64_t)nfl[u] * T.rs + r[u]];
    }
}

// fchunk_kernel: the levels up to the reporting chunks in one launch, a warp per chunk of
// n <= 64 leaves.  No FULL leaf (the common case): every survivor final of leaf i is
// re-coded into leaf i+1's code space (link_i[e] = amap_{i+1}[rank_{i+1}(sfin_i[e])], the
// last leaf keeps its states), all in parallel; the chunk's map is then a pairwise gather
// between 8-entry rows in the warp's shared memory.  Otherwise: value e of the first leaf
// is pushed through the leaves in order (fapply).  Writes the chunk's node like fwalk_kernel.
constexpr uint32_t kChunkLeaves = 64;
__global__ void __launch_bounds__(256) fchunk_kernel(DevTables T, Tree tr) {
    __shared__ uint16_t Ls[8][kChunkLeaves * 8];
    __shared__ uint16_t doms[8][kChunkLeaves];
    __shared__ uint8_t nvs[8][kChunkLeaves];
    pdl_trigger();
    pdl_wait();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const TreeLevel l1 = tr.lv[1];
    const uint32_t P = tr.lv[tr.rep_level].nodes, roff = tr.lv[tr.rep_level].off;
    uint16_t *Lw = Ls[warp], *dw = doms[warp];
    uint8_t *nw = nvs[warp];
    // chunk k's values re-coded into chunk k+1's code space (the last chunk keeps its states),
    // composed over the CTA's group of 8 chunks -> clinks[g]: ffold_kernel then folds P / 8
    // rows with no lookups.  A FULL chunk or successor sets the status flag instead.
    __shared__ uint16_t CL[8][8];
    const uint32_t G = (P + 7) / 8;
    for (uint32_t g = blockIdx.x; g < G; g += gridDim.x) {
      const uint32_t k = g * 8 + warp;
      if (k < P) {
        const uint32_t c0 = k == 0 ? 0u : l1.f + (k - 1) * l1.m, n = k == 0 ? l1.f : l1.m;
        bool full = false;
        for (uint32_t i = lane; i < n; i += 32) {
            const uint32_t nv = tr.leaf_nv[c0 + i], d = tr.dom_of[c0 + i];
            nw[i] = (uint8_t)nv;
            dw[i] = (uint16_t)d;
            full |= nv == 0 && T.dom_size[d] != 0;
        }
        full = __any_sync(0xffffffffu, full);
        __syncwarp();
        const uint32_t idx = roff + k;
        uint16_t *out = tr.rows + (uint64_t)idx * T.rs;
        if (!full) {
            constexpr int U = 8;
            for (uint32_t t0 = lane; t0 < n * 8; t0 += 32 * U) {
                bool has[U], ok[U];
                uint32_t sv[U], nd[U], nfl[U], c[U];
#pragma unroll
                for (int u = 0; u < U; u++) {
                    const uint32_t t = t0 + 32 * u, i = t >> 3, e = t & 7u;
                    has[u] = t < n * 8 && e < nw[i];
                    ok[u] = has[u] && i + 1 < n;  // (the chunk's last leaf keeps its states)
                    sv[u] = has[u] ? (uint32_t)tr.sfin[(uint64_t)(c0 + i) * tr.sk + e] : 0u;
                    nd[u] = ok[u] ? (uint32_t)dw[i + 1] : 0u;
                    nfl[u] = c0 + i + 1;
                }
                flink_batch<U>(T, tr, ok, sv, nd, nfl, c);
#pragma unroll
                for (int u = 0; u < U; u++) {
                    DFA_CHECK(!ok[u] || c[u] < kSurvBase || c[u] - kSurvBase < nw[((t0 + 32 * u) >> 3) + 1], "fchunk: link code");
                    if (has[u]) Lw[t0 + 32 * u] = (uint16_t)c[u];
                }
            }
            __syncwarp();
            for (uint32_t stride = 1; stride < n; stride *= 2) {
                const uint32_t pairs = (n + stride - 1) / (2 * stride);
                for (uint32_t t = lane; t < pairs * 8; t += 32) {
                    const uint32_t a = (t >> 3) * 2 * stride, b = a + stride;
                    if (b >= n) continue;
                    const uint32_t c = Lw[a * 8 + (t & 7u)];
                    if (c >= kSurvBase && c != kNone && (t & 7u) < nw[a]) Lw[a * 8 + (t & 7u)] = Lw[b * 8 + (c - kSurvBase)];
                }
                __syncwarp();
            }
            if (lane < nw[0]) out[lane] = Lw[lane];
            if (lane == 0) {
                tr.node_nv[idx] = nw[0];
                tr.node_fl[idx] = c0;
                tr.doms[idx] = dw[0];
            }
            if (tr.clinks && lane < 8) {
                const bool ok1[1] = {lane < nw[0] && k + 1 < P};
                const uint32_t sv1[1] = {lane < nw[0] ? (uint32_t)Lw[lane] : (uint32_t)kNone};
                uint32_t nd1[1] = {0}, c1[1];
                const uint32_t nfl1[1] = {c0 + n};
                if (k + 1 < P) {
                    nd1[0] = tr.dom_of[c0 + n];
                    if (tr.leaf_nv[c0 + n] == 0 && T.dom_size[nd1[0]] != 0) atomicOr(&tr.status->pad, 1u);  // FULL successor
                }
                flink_batch<1>(T, tr, ok1, sv1, nd1, nfl1, c1);
                CL[warp][lane] = (uint16_t)c1[0];
            }
        } else {
            if (tr.clinks && lane == 0) atomicOr(&tr.status->pad, 1u);
            const FNode A = fnode(T, tr, 0, c0);
            for (uint32_t e = lane; e < A.nv; e += 32) {
                uint32_t sv = A.vals[e];
                for (uint32_t c = c0 + 1; c < c0 + n; c++) sv = fapply(T, tr, fnode(T, tr, 0, c), sv);
                out[e] = (uint16_t)sv;
            }
            if (lane == 0) {
                tr.node_nv[idx] = (uint16_t)(A.nv | (A.full << 15));
                tr.node_fl[idx] = A.fl;
                tr.doms[idx] = (uint16_t)A.dom;
            }
        }
        __syncwarp();
      }
      if (tr.clinks) {
        __syncthreads();
        if (warp == 0 && lane < 8) {
            const uint32_t cnt = min(8u, P - g * 8);
            uint32_t c = CL[0][lane];
            for (uint32_t w = 1; w < cnt && c >= kSurvBase && c != kNone; w++) c = CL[w][c - kSurvBase];
            tr.clinks[(uint64_t)g * 8 + lane] = (uint16_t)c;
        }
        __syncthreads();
      }
    }
}

// ffold_kernel: every level above Ls in one CTA (no launch per level): the N <= kFoldCap
// nodes of level Ls are staged in shared memory (8 values each; FULL nodes keep their rows
// in global memory) and folded in place with fan-in 4 -- node a absorbs a + s, a + 2s,
// a + 3s at stride s = 1, 4, 16, ... (Eq.SeqReduction as a tree of Eq.MapReduction) -- then
// the root's row gives the final state, accept bit and segment row (Alg.seqmatch l.4-6).
constexpr uint32_t kFoldCap = 8192;
__host__ __device__ __forceinline__ uint32_t ffold_smem_bytes(uint32_t N) { return N * 24u + 16u; }

__global__ void __launch_bounds__(1024) ffold_kernel(DevTables T, Tree tr, uint32_t Ls) {
    extern __shared__ uint4 smem4[];
    pdl_wait();
    const uint32_t N = tr.lv[Ls].nodes, off = tr.lv[Ls].off;
    uint16_t *vals = reinterpret_cast<uint16_t *>(smem4);          // [N][8]
    // pairwise gather fold of M link rows in shared memory (row a absorbs row a + stride)
    auto fold_rounds = [&](uint32_t M) {
        for (uint64_t stride = 1; stride < M; stride *= 2) {
            const uint64_t pairs = (M + stride - 1) / (2 * stride);  // rows a = 2 stride g with a + stride < M
            for (uint64_t t = threadIdx.x; t < pairs * 8; t += blockDim.x) {
                const uint64_t a = (t >> 3) * 2 * stride, b = a + stride;
                if (b >= M) continue;
                const uint32_t c = vals[a * 8 + (t & 7u)];
                if (c >= kSurvBase && c != kNone) vals[a * 8 + (t & 7u)] = vals[b * 8 + (c - kSurvBase)];
            }
            __syncthreads();
        }
    };
    if (tr.clinks && Ls == tr.rep_level && tr.status->pad == 0) {
        // fchunk_kernel left the links composed per group of 8 chunks: fold those rows
        const uint32_t G = (N + 7) / 8;
        for (uint32_t i = threadIdx.x; i < G; i += blockDim.x)
            reinterpret_cast<uint4 *>(vals)[i] = reinterpret_cast<const uint4 *>(tr.clinks)[i];
        __syncthreads();
        fold_rounds(G);
        FNode R = fnode(T, tr, Ls, 0);
        R.vals = vals;
        const uint32_t u = T.dom_size[R.dom];
        for (uint32_t j = threadIdx.x; j < T.rs; j += blockDim.x)
            froot_out(T, tr, R.dom, u, j, j < u ? frow(T, tr, R, j) : (uint32_t)kNone);
        return;
    }
    uint32_t *fl = reinterpret_cast<uint32_t *>(vals + (size_t)N * 8);  // [N]
    uint16_t *dom = reinterpret_cast<uint16_t *>(fl + N);          // [N]
    uint16_t *nvf = dom + N;                                       // [N] value count | FULL << 15
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) {
        nvf[i] = tr.node_nv[off + i];
        fl[i] = tr.node_fl[off + i];
        dom[i] = tr.doms[off + i];
        reinterpret_cast<uint4 *>(vals)[i] = *reinterpret_cast<const uint4 *>(tr.rows + (uint64_t)(off + i) * T.rs);
    }
    __syncthreads();
    auto node = [&](uint32_t c) {
        FNode n;
        const uint32_t w = nvf[c];
        n.nv = w & 0x7FFFu;
        n.full = w >> 15;
        n.fl = fl[c];
        n.dom = dom[c];
        n.vals = n.full ? tr.rows + (uint64_t)(off + c) * T.rs : vals + (size_t)c * 8;
        DFA_CHECK(n.full || n.nv <= 8u, "ffold: factored node with more than 8 values");
        return n;
    };
    // No FULL node (the common case): every node's values are first re-coded into the next
    // node's code space -- link_k[e] = amap_{k+1}[rank_{k+1}(vals_k[e])], all N x 8 lookups
    // in parallel -- then Eq.MapReduction is a gather between 8-entry rows in shared memory
    // (absolute values pass: error and absorbing states), pairwise, log2 N rounds.
    bool any_full = false;
    for (uint32_t i = threadIdx.x; i < N; i += blockDim.x) any_full |= (nvf[i] >> 15) != 0;
    if (!__syncthreads_or(any_full)) {
        constexpr int U = 8;
        for (uint32_t t0 = threadIdx.x; t0 < (N - 1) * 8; t0 += blockDim.x * U) {
            bool ok[U];
            uint32_t sv[U], nd[U], nfl[U], c[U];
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t t = t0 + blockDim.x * u, k = t >> 3;
                ok[u] = t < (N - 1) * 8 && (t & 7u) < (nvf[k] & 0x7FFFu);
                sv[u] = ok[u] ? (uint32_t)vals[t] : 0u;
                nd[u] = ok[u] ? (uint32_t)dom[k + 1] : 0u;
                nfl[u] = ok[u] ? fl[k + 1] : 0u;
            }
            flink_batch<U>(T, tr, ok, sv, nd, nfl, c);
#pragma unroll
            for (int u = 0; u < U; u++) {
                const uint32_t t = t0 + blockDim.x * u;
                DFA_CHECK(!ok[u] || c[u] < kSurvBase || c[u] - kSurvBase < (nvf[(t >> 3) + 1] & 0x7FFFu), "ffold: link code");
                if (t < (N - 1) * 8) vals[t] = ok[u] ? (uint16_t)c[u] : kNone;  // (unused entries: never followed)
            }
        }
        __syncthreads();
        fold_rounds(N);
    } else
    for (uint64_t stride = 1; stride < N; stride *= 4) {
        const uint32_t ngroups = (uint32_t)((N + 4 * stride - 1) / (4 * stride));
        for (uint32_t g = threadIdx.x >> 3; g < ngroups; g += blockDim.x >> 3) {
            const uint32_t a = (uint32_t)(g * 4 * stride);
            const FNode A = node(a);
            uint16_t *av = const_cast<uint16_t *>(A.vals);
            for (uint32_t e = threadIdx.x & 7u; e < A.nv; e += 8) {
                uint32_t s = av[e];
                for (uint32_t q = 1; q < 4; q++) {
                    const uint64_t c = a + q * stride;
                    if (c >= N) break;
                    s = fapply(T, tr, node((uint32_t)c), s);
                }
                av[e] = (uint16_t)s;
            }
        }
        __syncthreads();
    }
    const FNode R = node(0);
    const uint32_t u = T.dom_size[R.dom];
    for (uint32_t j = threadIdx.x; j < T.rs; j += blockDim.x)
        froot_out(T, tr, R.dom, u, j, j < u ? frow(T, tr, R, j) : (uint32_t)kNone);
}


cudaError_t launch_walk_level(const DevTables &T, const Tree &tr, uint32_t L, int sms, cudaStream_t s) {
    const uint64_t total = (uint64_t)tr.lv[L].nodes * T.rs;
    const uint64_t grid = std::min<uint64_t>((total + 255) / 256, (uint64_t)sms * 16);
    walk_kernel<<<(unsigned)std::max<uint64_t>(grid, 1), 256, 0, s>>>(T, tr, L);
    return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// fold_rows_kernel: the top of the composition tree for short rows -- P
// reporting-chunk rows (internal order, stride rs) composed into the final
// state (Eq.SeqReduction as a tree of Eq.MapReduction).  CTA b stages up to
// `per_cta` consecutive rows in shared memory and composes them pairwise with
// all its threads; the last CTA to finish (acq_rel ticket) composes the CTA
// maps the same way and applies Alg.seqmatch l.4-6.
// ---------------------------------------------------------------------------
__device__ void cta_pairwise(const DevTables &T, const uint8_t *rank8, const uint32_t *dead, const uint16_t *dsz,
                             uint16_t *st, const uint16_t *dch, uint32_t nc, uint32_t lrs, DevStatus *status) {
    for (uint32_t lstep = 0; (1u << lstep) < nc; lstep++) {
        const uint32_t step = 1u << lstep;
        const uint32_t npairs = (nc - step + 2 * step - 1) >> (lstep + 1);
        pairwise_round<4>(T, rank8, dead, dsz, dch, st, lrs, lstep, npairs, threadIdx.x, blockDim.x, status);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(1024) fold_rows_kernel(DevTables T, const uint16_t *rows, const uint16_t *doms,
                                                         uint32_t P, uint32_t per_cta, uint32_t lrs,
                                                         uint16_t *cta_rows, uint16_t *cta_doms,
                                                         uint32_t *ticket, DevStatus *status,
                                                         uint16_t *dev_final, uint16_t *seg_row) {
    extern __shared__ uint4 smem4[];
    const uint32_t q4 = T.rs >> 3;
    // shared: [rank table u8][error bits][dom sizes][child doms][rows]
    uint8_t *rank8 = reinterpret_cast<uint8_t *>(smem4);
    const uint32_t rank_bytes = T.rank8 ? (((T.nclass + 1) * T.nq + 15) & ~15u) : 0u;
    uint32_t *dead = reinterpret_cast<uint32_t *>(rank8 + rank_bytes);
    const uint32_t dead_words = ((T.nq + 31) / 32 + 3) & ~3u;
    uint16_t *dsz = reinterpret_cast<uint16_t *>(dead + dead_words);
    const uint32_t dsz_n = (T.nclass + 1 + 7) & ~7u;
    uint16_t *dch = dsz + dsz_n;
    uint16_t *st = dch + ((per_cta + 7) & ~7u);
#ifdef DFA_TREE_TIMING
    if (threadIdx.x == 0) atomicMin(&g_tree_t[20], gtimer());
#endif
    for (uint32_t i = threadIdx.x; i < rank_bytes / 16; i += blockDim.x)
        reinterpret_cast<uint4 *>(rank8)[i] = __ldg(reinterpret_cast<const uint4 *>(T.rank8) + i);
    for (uint32_t i = threadIdx.x; i < dead_words; i += blockDim.x) dead[i] = __ldg(T.dead_bits + i);
    for (uint32_t i = threadIdx.x; i <= T.nclass; i += blockDim.x) dsz[i] = T.dom_size[i];
    const uint32_t r0 = blockIdx.x * per_cta, nc = min(per_cta, P - r0);
    for (uint32_t t = threadIdx.x; t < nc; t += blockDim.x) dch[t] = doms[r0 + t];
    for (uint32_t t = threadIdx.x; t < nc * q4; t += blockDim.x) {
        const uint32_t c = t / q4, k = t - c * q4;
        reinterpret_cast<uint4 *>(st + (c << lrs))[k] =
            __ldcg(reinterpret_cast<const uint4 *>(rows + (uint64_t)(r0 + c) * T.rs) + k);
    }
    __syncthreads();
#ifdef DFA_TREE_TIMING
    if (threadIdx.x == 0) atomicMax(&g_tree_t[21], gtimer());
#endif
    cta_pairwise(T, T.rank8 ? rank8 : nullptr, dead, dsz, st, dch, nc, lrs, status);
#ifdef DFA_TREE_TIMING
    if (threadIdx.x == 0) atomicMax(&g_tree_t[22], gtimer());
#endif

    // publish this CTA's map, take a ticket; the last CTA folds the CTA maps
    for (uint32_t t = threadIdx.x; t < q4; t += blockDim.x)
        reinterpret_cast<uint4 *>(cta_rows + (uint64_t)blockIdx.x * T.rs)[t] = reinterpret_cast<const uint4 *>(st)[t];
    if (threadIdx.x == 0) cta_doms[blockIdx.x] = dch[0];
    __syncthreads();
    __shared__ uint32_t last;
    if (threadIdx.x == 0) {
        uint32_t prev;
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(ticket) : "memory");
        last = prev + 1 == gridDim.x;
        if (last) atomicExch(ticket, 0u);  // every CTA has its ticket: reset for the next launch
    }
    __syncthreads();
    if (!last) return;
#ifdef DFA_TREE_TIMING
    if (threadIdx.x == 0) atomicMax(&g_tree_t[23], gtimer());
#endif
    const uint32_t G = gridDim.x;
    if (G > 1) {
        for (uint32_t t = threadIdx.x; t < G; t += blockDim.x) dch[t] = __ldcg(cta_doms + t);
        for (uint32_t t = threadIdx.x; t < G * q4; t += blockDim.x) {
            const uint32_t c = t / q4, k = t - c * q4;
            reinterpret_cast<uint4 *>(st + (c << lrs))[k] =
                __ldcg(reinterpret_cast<const uint4 *>(cta_rows + (uint64_t)c * T.rs) + k);
        }
        __syncthreads();
        cta_pairwise(T, T.rank8 ? rank8 : nullptr, dead, dsz, st, dch, G, lrs, status);
    }
#ifdef DFA_TREE_TIMING
    if (threadIdx.x == 0) atomicMax(&g_tree_t[24], gtimer());
#endif

    if (seg_row) {
        // the segment map: the folded row over the first chunk's domain, in the user's order
        const uint32_t d0 = dch[0];
        const uint32_t du = d0 < T.nclass ? T.dom_user_size[d0] : (d0 == T.start_dom ? 1u : 0u);
        for (uint32_t j = threadIdx.x; j < T.imax_user; j += blockDim.x)
            seg_row[j] = j < du ? st[d0 < T.nclass ? T.xlat[(uint64_t)d0 * T.imax_user + j] : j] : kNone;
    }
    if (threadIdx.x == 0) {
        const uint32_t fs = st[0];
        if (fs == T.poison) atomicMax(&status->err, 5u);
        status->final_state = fs;
        status->accept = fs < T.nq ? (uint32_t)test_bit(T.accept_bits, fs) : 0u;
        if (dev_final) {
            dev_final[0] = (uint16_t)fs;
            dev_final[1] = (uint16_t)status->accept;
        }
    }
}

// ---------------------------------------------------------------------------
// Composition of rank-space maps with <= 8 entries (the grouped path; see
// kRank): the reporting-chunk maps from the group leaves, the fold of the
// reporting maps into the final state, and the chunk starts.  Entry per lane:
// a warp holds 4 maps, lane 8g + j = entry j of map g, so composing two maps
// is one shuffle per lane (Eq.MapReduction) -- no table lookups at all.
// ---------------------------------------------------------------------------
// A rank-space entry as a state: rank codes index the next map's domain nd.
__device__ __forceinline__ uint32_t decode_entry(const DevTables &T, uint32_t v, uint32_t nd) {
    return is_rank(v) ? (uint32_t)__ldg(T.dom_list + (uint64_t)nd * T.rs + (v - kRank)) : v;
}

// leaf_fold_kernel: one level of leaf reduction for long chunks: the leaves of
// every chunk (chunk 0: L0, others L) in aligned runs of 32, each run folded
// by one warp (lane = leaf, shuffle butterfly) into one leaf of the output
// (chunk 0: ceil(L0/32), others ceil(L/32)).  Launched dependent.
__global__ void __launch_bounds__(256) leaf_fold_kernel(const uint16_t *in_rows, const uint16_t *in_dom, uint32_t L0,
                                                        uint32_t L, uint32_t P, uint16_t *out_rows,
                                                        uint16_t *out_dom) {
    pdl_trigger();
    pdl_wait();
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t L0n = (L0 + 31) / 32, Ln = (L + 31) / 32;
    const uint64_t total = (uint64_t)L0n + (uint64_t)(P - 1) * Ln;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t o = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); o < total; o += nwarps) {
        uint64_t a, e;
        if (o < L0n) { a = o * 32; e = L0; }
        else {
            const uint64_t k = 1 + (o - L0n) / Ln, idx = (o - L0n) % Ln;
            const uint64_t ck = (uint64_t)L0 + (k - 1) * L;
            a = ck + idx * 32;
            e = ck + L;
        }
        const uint64_t leaf = a + lane;
        const bool valid = leaf < e;
        uint32_t fin[kLanes], dom = 0;
        if (valid) {
            const uint4 v = __ldcg(reinterpret_cast<const uint4 *>(in_rows) + leaf);
            fin[0] = v.x & 0xFFFFu; fin[1] = v.x >> 16; fin[2] = v.y & 0xFFFFu; fin[3] = v.y >> 16;
            fin[4] = v.z & 0xFFFFu; fin[5] = v.z >> 16; fin[6] = v.w & 0xFFFFu; fin[7] = v.w >> 16;
            dom = __ldcg(in_dom + leaf);
        } else {
#pragma unroll
            for (int q = 0; q < kLanes; q++) fin[q] = kNone;
        }
#pragma unroll
        for (uint32_t step = 1; step < 32; step *= 2) {
            uint32_t pm[kLanes];
#pragma unroll
            for (int q = 0; q < kLanes; q++) pm[q] = __shfl_down_sync(0xffffffffu, fin[q], step);
            const bool pv = __shfl_down_sync(0xffffffffu, valid, step);
            if ((lane & (2 * step - 1)) != 0 || !pv || lane + step >= 32) continue;
#pragma unroll
            for (int q = 0; q < kLanes; q++) {
                const uint32_t rr = fin[q] - kRank;
                if (rr >= (uint32_t)kLanes) continue;
                uint32_t v = 0;
#pragma unroll
                for (int t = 0; t < kLanes; t++) v |= pm[t] & (0u - (uint32_t)(rr == (uint32_t)t));
                fin[q] = v;
            }
        }
        if (lane == 0) {
            uint4 v;
            v.x = (fin[0] & 0xFFFFu) | (fin[1] << 16);
            v.y = (fin[2] & 0xFFFFu) | (fin[3] << 16);
            v.z = (fin[4] & 0xFFFFu) | (fin[5] << 16);
            v.w = (fin[6] & 0xFFFFu) | (fin[7] << 16);
            reinterpret_cast<uint4 *>(out_rows)[o] = v;
            out_dom[o] = (uint16_t)dom;
        }
    }
}

// starts8_kernel: true start of every reporting chunk (optional output): CTA b
// walks its compose8 chunks from the rank code cta_start[b].  Launched dependent.
__global__ void __launch_bounds__(256) starts8_kernel(DevTables T, const uint16_t *rep_rows, const uint16_t *rep_doms,
                                                     uint32_t P, uint32_t cpc, const uint16_t *cta_start,
                                                     uint16_t *starts) {
    __shared__ __align__(16) uint16_t srow[1024 * 8];
    __shared__ uint16_t sdom[1024];
    pdl_wait();
    const uint32_t c0 = blockIdx.x * cpc, c1 = min(P, c0 + cpc), n = c1 - c0;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        reinterpret_cast<uint4 *>(srow)[i] = __ldcg(reinterpret_cast<const uint4 *>(rep_rows) + c0 + i);
        sdom[i] = __ldcg(rep_doms + c0 + i);
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    uint32_t code = __ldcg(cta_start + blockIdx.x);
    for (uint32_t i = 0; i < n; i++) {
        starts[c0 + i] = (uint16_t)decode_entry(T, code, sdom[i]);
        if (is_rank(code)) code = srow[i * 8 + (code - kRank)];
    }
}

// compose8_kernel: the whole composition for rank-space maps, one launch
// (dependent, PDL).  CTA b owns reporting chunks [b cpc, (b+1) cpc): a warp per
// chunk folds the chunk's group leaves (chunk 0: L0 leaves, others L) into the
// reporting map (internal row, API row in the user's order with states, chunk
// 0's user row, e0); the CTA folds its chunk maps (Eq.SeqReduction), the last
// CTA (acq_rel ticket) folds the CTA maps and applies Alg.seqmatch lines 4-6.
__global__ void __launch_bounds__(1024) compose8_kernel(DevTables T, const uint16_t *leaves, const uint16_t *leaf_dom,
                                                        uint32_t L0, uint32_t L, uint32_t P, uint32_t cpc,
                                                        uint16_t *rep_rows, uint16_t *rep_doms, uint16_t *user_rows,
                                                        uint16_t *user_row0, uint16_t *e0, uint16_t *cta_rows,
                                                        uint16_t *cta_doms, uint32_t *ticket, DevStatus *status,
                                                        uint16_t *dev_final, uint16_t *cta_start, uint16_t *seg_row) {
#ifdef DFA_TREE_TIMING
    if (threadIdx.x == 0) atomicMin(&g_tree_t[10], gtimer());
#endif
    pdl_trigger();
    pdl_wait();
#ifdef DFA_TREE_TIMING
    if (threadIdx.x == 0) atomicMax(&g_tree_t[11], gtimer());
#endif
    __shared__ __align__(16) uint16_t crow[1024 * 8];
    __shared__ __align__(16) uint16_t trow[256 * 8];
    __shared__ uint16_t cdom[1024], tdom[256];
    __shared__ uint32_t last;
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5, j = lane & 7;
    const uint32_t c0 = blockIdx.x * cpc, c1 = min(P, c0 + cpc);
    const uint32_t g = lane >> 3, gb = lane & ~7u;
    // chunk phase: each warp takes 4 chunks at a time, one per 8-lane group,
    // and folds the chunk's leaves in order (group-local shuffles)
#pragma unroll 1
    for (uint32_t kb = c0 + warp * 4; kb < c1; kb += nw * 4) {
        const uint32_t k = kb + g;
        const bool has = k < c1;
        const uint32_t a = k == 0 ? 0u : L0 + (k - 1) * L, b = L0 + k * L;
        const uint32_t nk = has ? b - a : 0u;
        DFA_CHECK(!has || (a <= b && b <= L0 + (uint64_t)(P - 1) * L), "compose8: leaf range past the leaves");
        // the next chunk's domain (its first leaf's) decodes this chunk's rank codes
        const uint32_t nd = has && k + 1 < P ? (uint32_t)__ldcg(leaf_dom + b) : 0u;
        const uint32_t d0 = has ? (uint32_t)__ldcg(leaf_dom + a) : 0u;
        const uint32_t nmax = __reduce_max_sync(0xffffffffu, nk);
        uint32_t av = kNone, aok = 0;
        uint32_t dl = kNone, xl = 0, du = 0;
#pragma unroll 1
        for (uint32_t t0 = 0; t0 < nmax; t0 += 16) {
            uint32_t lv[16];
#pragma unroll
            for (int q = 0; q < 16; q++)
                lv[q] = t0 + q < nk ? (uint32_t)__ldcg(leaves + (uint64_t)(a + t0 + q) * 8 + j) : kNone;
            if (t0 == 0 && has) {
                // decode and user-order rows, loaded while the leaves are in flight
                if (k + 1 < P) dl = __ldg(T.dom_list + (uint64_t)nd * T.rs + j);
                if (d0 < T.nclass) {
                    du = T.dom_user_size[d0];
                    if (j < T.imax_user) xl = T.xlat[(uint64_t)d0 * T.imax_user + j];
                } else {
                    du = d0 == T.start_dom ? 1u : 0u;
                    xl = j;
                }
            }
#pragma unroll
            for (int q = 0; q < 16; q++) {
                const bool bok = t0 + q < nk;
                const uint32_t rr = av - kRank;
                const bool take = bok && (!aok || rr < (uint32_t)kLanes);
                const uint32_t nv = __shfl_sync(0xffffffffu, lv[q], gb + (aok ? (rr & 7u) : j));
                if (take) av = nv;
                aok |= bok;
            }
        }
        if (has) {
            rep_rows[(uint64_t)k * 8 + j] = (uint16_t)av;
            crow[(k - c0) * 8 + j] = (uint16_t)av;
            if (j == 0) {
                rep_doms[k] = (uint16_t)d0;
                cdom[k - c0] = (uint16_t)d0;
            }
        }
        // the map with states: rank codes through the next domain's list
        const uint32_t rr = av - kRank;
        const uint32_t dv = __shfl_sync(0xffffffffu, dl, gb + (rr & 7u));
        const uint32_t sv = rr < (uint32_t)kLanes ? dv : av;
        if (e0 && has && k == 0 && j == 0) e0[0] = (uint16_t)sv;
        uint16_t *urow = nullptr;
        if (has && user_rows && k > 0) urow = user_rows + (uint64_t)(k - 1) * T.imax_user;
        else if (has && user_row0 && k == 0) urow = user_row0;
        // user row: imax_user <= 8 entries (rs == 8), lane j of the group writes entry j
        const uint32_t v = __shfl_sync(0xffffffffu, sv, gb + (xl & 7u));
        if (urow && j < T.imax_user) urow[j] = (uint16_t)(j < du ? v : kNone);
    }
    __syncthreads();
#ifdef DFA_TREE_TIMING
    unsigned long long tc0 = gtimer();
    if (threadIdx.x == 0) atomicMax(&g_tree_t[12], tc0);
#endif
    // CTA fold of its chunk maps (shared memory), then the last CTA
    const uint32_t n = c1 - c0;
    LMap acc = cta_tree_fold(crow, cdom, trow, tdom, n);
#ifdef DFA_TREE_TIMING
    unsigned long long tc1 = gtimer();
    if (threadIdx.x == 0) atomicMax(&g_tree_t[20], tc1 - tc0);
#endif
    if (gridDim.x > 1) {
        if (warp == 0) {
            if (lane < 8) cta_rows[(uint64_t)blockIdx.x * 8 + j] = (uint16_t)acc.v;
            if (lane == 0) cta_doms[blockIdx.x] = (uint16_t)acc.dom;
            __syncwarp();
            if (lane == 0) {
                uint32_t prev;
                asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;" : "=r"(prev) : "l"(ticket) : "memory");
                last = prev + 1 == gridDim.x;
                if (last) atomicExch(ticket, 0u);  // every CTA has its ticket: reset for the next launch
            }
        }
        __syncthreads();
#ifdef DFA_TREE_TIMING
        unsigned long long tc2 = gtimer();
        if (threadIdx.x == 0) atomicMax(&g_tree_t[16], tc2);
        if (threadIdx.x == 0) atomicMax(&g_tree_t[21], tc2 - tc1);
#endif
        if (!last) return;
        for (uint32_t i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
            reinterpret_cast<uint4 *>(crow)[i] = __ldcg(reinterpret_cast<const uint4 *>(cta_rows) + i);
            cdom[i] = __ldcg(cta_doms + i);
        }
        __syncthreads();
        if (cta_start && threadIdx.x == 0) {
            // rank code of every CTA's first chunk start: the prefix of
            // Eq.SeqReduction over the CTA maps (chunk 0 starts at rank 0 of {q0})
            uint32_t code = kRank;
            for (uint32_t i = 0; i < gridDim.x; i++) {
                cta_start[i] = (uint16_t)code;
                if (is_rank(code)) code = crow[i * 8 + (code - kRank)];
            }
        }
        acc = cta_tree_fold(crow, cdom, trow, tdom, gridDim.x);
#ifdef DFA_TREE_TIMING
        if (threadIdx.x == 0) atomicMax(&g_tree_t[22], gtimer() - tc2);
#endif
    }
    if (cta_start && gridDim.x == 1 && threadIdx.x == 0) cta_start[0] = (uint16_t)kRank;
    if (seg_row && warp == 0) {
        // the segment map: the fold of every chunk map over chunk 0's domain (absolute states:
        // the input's last sub-chunk ends in states), in the user's order
        const uint32_t d0 = __shfl_sync(0xffffffffu, acc.dom, 0);
        uint32_t du, xl;
        if (d0 < T.nclass) {
            du = T.dom_user_size[d0];
            xl = j < T.imax_user ? T.xlat[(uint64_t)d0 * T.imax_user + j] : 0u;
        } else {
            du = d0 == T.start_dom ? 1u : 0u;
            xl = j;
        }
        const uint32_t v = __shfl_sync(0xffffffffu, acc.v, xl & 7u);
        if (lane < 8 && j < T.imax_user) seg_row[j] = (uint16_t)(j < du ? v : kNone);
    }
    if (threadIdx.x == 0) {
        const uint32_t fs = acc.v;  // absolute: the input's last sub-chunk ends in states
        if (fs == T.poison) atomicMax(&status->err, 5u);
        if (is_rank(fs)) atomicMax(&status->err, 8u);
        status->final_state = fs;
        status->accept = fs < T.nq ? (uint32_t)test_bit(T.accept_bits, fs) : 0u;
        if (dev_final) {
            dev_final[0] = (uint16_t)fs;
            dev_final[1] = (uint16_t)status->accept;
        }
#ifdef DFA_TREE_TIMING
        atomicMax(&g_tree_t[19], gtimer());
#endif
    }
}

// ---------------------------------------------------------------------------
// batch_out_kernel (dfa_match_batch): input j's final state is entry 0 of its
// reporting map over {q0} (absolute: its last sub-chunk ends in states); empty
// inputs (kidx < 0) end in q0.
// ---------------------------------------------------------------------------
__global__ void batch_out_kernel(DevTables T, const uint16_t *rep_rows, uint32_t rs, const int32_t *kidx,
                                 const uint64_t *offsets, uint64_t data_len, uint32_t count, uint16_t *dev_final,
                                 uint8_t *dev_accept, DevStatus *status) {
    pdl_wait();
    for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < count; j += gridDim.x * blockDim.x) {
        if (offsets && (offsets[j + 1] < offsets[j] || offsets[j + 1] > data_len))
            atomicMax(&status->err, 1u);  // DFA_ERR_ARG: decreasing offsets or past data_len
        const int32_t k = kidx ? kidx[j] : (int32_t)j;
        DFA_CHECK(k < (int32_t)count, "batch_out: input index past the batch");
        uint32_t q = k < 0 ? T.q0 : rep_rows[(uint64_t)k * rs];
        if (q >= T.nq || is_rank(q)) { atomicMax(&status->err, 8u); q = T.q0; }
        if (q == T.poison) atomicMax(&status->err, 5u);
        dev_final[j] = (uint16_t)q;
        dev_accept[j] = (uint8_t)test_bit(T.accept_bits, q);
    }
}

// ---------------------------------------------------------------------------
// fold_segments_kernel: the top of the multi-GPU merge (the
// master step of Fig.Merge): segment g's map is a row over the
// user's I_sigma of lookahead byte lookahead[g] (segment 0: over {q0});
// Eq.SeqReduction over the G rows, then Alg.seqmatch l.4-6.
// ---------------------------------------------------------------------------
__global__ void fold_segments_kernel(DevTables T, const uint16_t *rows, const uint8_t *lookahead, uint32_t G,
                                     DevStatus *status, uint16_t *dev_final) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    uint32_t s = rows[0];
    for (uint32_t g = 1; g < G; g++) {
        // error states pass through: the internal Z (poison included) and the
        // user's Z, whose states are absorbing over Sigma but not over bytes >= |Sigma|
        if (s == kNone || test_bit(T.dead_bits, s) || (s < T.nq_user && test_bit(T.dead_user_bits, s))) continue;
        const uint32_t d = T.byte_class[lookahead[g]];
        const uint32_t r = T.rank[(uint64_t)d * T.nq + s];
        const uint32_t ju = r == kNone ? kNone : T.ixlat[(uint64_t)d * T.rs + r];
        if (ju == kNone) { atomicMax(&status->err, 8u); break; }
        DFA_CHECK(ju < T.imax_user && d < T.nclass, "fold_segments: user index past the row");
        s = rows[(uint64_t)g * T.imax_user + ju];
    }
    uint32_t err = status->err;
    if (s == T.poison) err = max(err, 5u);
    status->err = err;
    status->final_state = s;
    status->accept = s < T.nq ? (uint32_t)test_bit(T.accept_bits, s) : 0u;
    if (dev_final) {
        dev_final[0] = (uint16_t)s;
        dev_final[1] = (uint16_t)status->accept;
    }
}

// ---------------------------------------------------------------------------
// lookahead_kernel (N1): the chunk maps restricted to r reverse lookahead
// symbols (Sec. "Multiple Reverse Lookahead Symbols").  A warp
// per chunk k >= 1: the image of the user states Q under the L = min(r, b_k)
// bytes before b_k (Eq.istatesm, O(L |Q|) table reads) marks a bitmap; the
// chunk's I_sigma (sigma = x[b_k - 1]) is then walked in its ascending order
// and the marked states kept with their map entries (Lemma 1: the r-symbol
// set is a subset of I_sigma), compacted with ballots.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) lookahead_kernel(DevTables T, const uint8_t *in, const uint64_t *bounds,
                                                        uint32_t P, uint32_t r, const uint16_t *maps,
                                                        uint16_t *doms_out, uint16_t *sizes_out, uint16_t *maps_out,
                                                        DevStatus *status) {
    extern __shared__ uint32_t lbm[];
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t bw = (T.nq_user + 31) / 32;
    uint32_t *bm = lbm + warp * bw;
    const uint32_t imu = T.imax_user;
    const uint32_t nwarps = gridDim.x * (blockDim.x >> 5);
    for (uint32_t k = 1 + blockIdx.x * (blockDim.x >> 5) + warp; k < P; k += nwarps) {
        const uint64_t b = bounds[k];
        const uint32_t L = (uint64_t)r < b ? r : (uint32_t)b;
        const uint8_t *sy = in + (b - L);
        for (uint32_t i = lane; i < bw; i += 32) bm[i] = 0;
        if (lane < L && sy[lane] >= T.ns) atomicMax(&status->err, 5u);
        __syncwarp();
        for (uint32_t q = lane; q < T.nq_user; q += 32) {
            uint32_t st = q;
            for (uint32_t i = 0; i < L; i++) st = __ldg(T.gtable + (uint64_t)st * 256 + sy[i]);
            if (st < T.nq_user && !test_bit(T.dead_user_bits, st)) atomicOr(&bm[st >> 5], 1u << (st & 31));
        }
        __syncwarp();
        const uint32_t c = T.byte_class[sy[L - 1]];
        const uint32_t du = c < T.nclass ? T.dom_user_size[c] : 0u;
        uint16_t *dout = doms_out + (uint64_t)(k - 1) * imu, *mout = maps_out + (uint64_t)(k - 1) * imu;
        const uint16_t *min_ = maps + (uint64_t)(k - 1) * imu;
        uint32_t count = 0;
        for (uint32_t j0 = 0; j0 < du; j0 += 32) {
            const uint32_t j = j0 + lane;
            uint32_t st = 0;
            bool keep = false;
            if (j < du) {
                st = T.dom_list[(uint64_t)c * T.rs + T.xlat[(uint64_t)c * imu + j]];
                keep = (bm[st >> 5] >> (st & 31)) & 1u;
            }
            const uint32_t mask = __ballot_sync(0xffffffffu, keep);
            if (keep) {
                const uint32_t pos = count + __popc(mask & ((1u << lane) - 1u));
                dout[pos] = (uint16_t)st;
                mout[pos] = min_[j];
            }
            count += __popc(mask);
        }
        for (uint32_t i = count + lane; i < imu; i += 32) {
            dout[i] = kNone;
            mout[i] = kNone;
        }
        if (lane == 0) sizes_out[k - 1] = (uint16_t)count;
        __syncwarp();
    }
}

// ---------------------------------------------------------------------------
// starts_kernel (optional output): true initial state of every reporting
// chunk, the prefix of Eq.SeqReduction.  One CTA: the rank table (when it
// fits) and blocks of rows are staged in shared memory by all threads, one
// thread walks the P - 1 dependent steps.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512) starts_kernel(DevTables T, Plan p, const uint16_t *row0, const uint16_t *rows,
                                                     const uint16_t *dom, uint16_t *starts, DevStatus *status,
                                                     uint32_t rank_mode, uint32_t blk) {
    extern __shared__ __align__(16) uint8_t ssm[];
    // rank_mode: 0 = global rank, 1 = rank8 in smem, 2 = rank u16 in smem
    const uint32_t nr = (T.nclass + 1) * T.nq;
    const uint32_t rbytes = rank_mode == 1 ? ((nr + 15) & ~15u) : rank_mode == 2 ? ((nr * 2 + 15) & ~15u) : 0u;
    if (rank_mode == 1) for (uint32_t i = threadIdx.x; i < nr; i += blockDim.x) ssm[i] = __ldg(T.rank8 + i);
    if (rank_mode == 2)
        for (uint32_t i = threadIdx.x; i < nr; i += blockDim.x) reinterpret_cast<uint16_t *>(ssm)[i] = __ldg(T.rank + i);
    uint16_t *srow = reinterpret_cast<uint16_t *>(ssm + rbytes);
    uint16_t *sdom = srow + (size_t)blk * T.rs;
    pdl_wait();
    __shared__ uint32_t carry;
    if (threadIdx.x == 0) {
        starts[0] = (uint16_t)T.q0;
        carry = p.P > 1 ? row0[0] : 0u;
    }
    for (uint32_t k0 = 1; k0 < p.P; k0 += blk) {
        const uint32_t n = min(blk, p.P - k0);
        __syncthreads();
        const uint32_t q = T.rs / 8;  // uint4 per row
        for (uint32_t i = threadIdx.x; i < n * q; i += blockDim.x)
            reinterpret_cast<uint4 *>(srow)[i] = __ldcg(reinterpret_cast<const uint4 *>(rows + (uint64_t)(k0 - 1) * T.rs) + i);
        for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) sdom[i] = __ldcg(dom + k0 + i);
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t st = carry;
            for (uint32_t i = 0; i < n; i++) {
                starts[k0 + i] = (uint16_t)st;
                if (T.has_dead && test_bit(T.dead_bits, st)) continue;
                const uint64_t ri = (uint64_t)sdom[i] * T.nq + st;
                uint32_t r = rank_mode == 1 ? ssm[ri] : rank_mode == 2 ? reinterpret_cast<const uint16_t *>(ssm)[ri]
                                                                       : __ldg(T.rank + ri);
                if (rank_mode == 1 && r == 0xFFu) r = kNone;
                if (r == kNone) { atomicMax(&status->err, 8u); break; }
                st = srow[(size_t)i * T.rs + r];
            }
            carry = st;
        }
    }
}

#endif  // DFA_TU_MAIN

} // namespace

// Per-layout kernel entry points, defined in the translation unit of that
// layout (kernels_m<MODE>.cu): the template kernels of every layout compile in
// parallel, and the main unit dispatches through these.
#ifdef DFA_TU_MODE
template <int M>
void *converge_or_null(bool id8) {
    // the converge kernel runs the byte-table modes on the padded copy (converge_fn)
    if constexpr (M == kIdentU8 || M == kRepU8x8 || M == kRepU8x4) return nullptr;
    else return id8 ? (void *)converge_kernel<M, true> : (void *)converge_kernel<M, false>;
}
template <int M>
void *lanes_tma_or_null() {
    // TMA input staging is built for the replicated layout (one 640-thread CTA per SM: few
    // warps, where it pays)
    if constexpr (M == kRepU8x8) return (void *)lanes_kernel<M, false, false, true>;
    else return nullptr;
}
#define DFA_DEFINE_MODE_ENTRIES(M)                                                                      \
    template <> void *lanes_entry<M>(bool sticky, bool count, bool tma) {                               \
        if (tma) return lanes_tma_or_null<M>();                                                         \
        return count ? (sticky ? (void *)lanes_kernel<M, true, true, false> : (void *)lanes_kernel<M, false, true, false>) \
                     : (sticky ? (void *)lanes_kernel<M, true, false, false> : (void *)lanes_kernel<M, false, false, false>); \
    }                                                                                                   \
    template <> void *ceiling_entry<M>() { return (void *)ceiling_kernel<M>; }                          \
    template <> void *converge_entry<M>(bool id8) { return converge_or_null<M>(id8); }
#if DFA_TU_MODE == 0
DFA_DEFINE_MODE_ENTRIES(kIdentU8)
DFA_DEFINE_MODE_ENTRIES(kIdentU16)
DFA_DEFINE_MODE_ENTRIES(kWindowU8)
DFA_DEFINE_MODE_ENTRIES(kWindowU16)
DFA_DEFINE_MODE_ENTRIES(kPacked9)
DFA_DEFINE_MODE_ENTRIES(kGlobalU16)
DFA_DEFINE_MODE_ENTRIES(kRepU8x8)
DFA_DEFINE_MODE_ENTRIES(kRepU8x4)
DFA_DEFINE_MODE_ENTRIES(kIdentU8P)
#else
DFA_DEFINE_MODE_ENTRIES(DFA_TU_MODE)
#endif
#endif  // DFA_TU_MODE

#ifdef DFA_TU_MAIN
namespace {

void *ceiling_fn(int mode) {
    switch (mode) {
    case kIdentU8: return ceiling_entry<kIdentU8>();
    case kRepU8x8: return ceiling_entry<kRepU8x8>();
    case kRepU8x4: return ceiling_entry<kRepU8x4>();
    case kIdentU8P: return ceiling_entry<kIdentU8P>();
    case kIdentU16: return ceiling_entry<kIdentU16>();
    case kWindowU8: return ceiling_entry<kWindowU8>();
    case kWindowU16: return ceiling_entry<kWindowU16>();
    case kPacked9: return ceiling_entry<kPacked9>();
    default: return ceiling_entry<kGlobalU16>();
    }
}

void *lanes_fn(const DevTables &T, bool count = false, bool tma = false) {
    const bool st = T.has_sticky != 0;
    switch (T.mode) {
    case kIdentU8: return lanes_entry<kIdentU8>(st, count, tma);
    case kRepU8x8: return lanes_entry<kRepU8x8>(st, count, tma);
    case kRepU8x4: return lanes_entry<kRepU8x4>(st, count, tma);
    case kIdentU8P: return lanes_entry<kIdentU8P>(st, count, tma);
    case kIdentU16: return lanes_entry<kIdentU16>(st, count, tma);
    case kWindowU8: return lanes_entry<kWindowU8>(st, count, tma);
    case kWindowU16: return lanes_entry<kWindowU16>(st, count, tma);
    case kPacked9: return lanes_entry<kPacked9>(st, count, tma);
    default: return lanes_entry<kGlobalU16>(st, count, tma);
    }
}
// The converge kernel steps all lanes of one sub-chunk on the same byte (a
// warp per sub-chunk): with 256-byte rows they would all read one bank, so
// every byte-table mode converges on the padded single copy of the same image.
void *converge_fn(const DevTables &T) {
    const bool id8 = T.imax <= 254u;  // lane ids fit a byte (converge_scratch_bytes)
    switch (T.mode) {
    case kIdentU8:
    case kIdentU8P:
    case kRepU8x8:
    case kRepU8x4: return converge_entry<kIdentU8P>(id8);
    case kIdentU16: return converge_entry<kIdentU16>(id8);
    case kWindowU8: return converge_entry<kWindowU8>(id8);
    case kWindowU16: return converge_entry<kWindowU16>(id8);
    case kPacked9: return converge_entry<kPacked9>(id8);
    default: return converge_entry<kGlobalU16>(id8);
    }
}

int bits_words_host(uint32_t nq) { return (int)((((nq + 31) / 32) + 3) & ~3u); }

} // namespace

__global__ void probe_smem_kernel(uint32_t *out) {
    extern __shared__ uint4 smem4[];
    if (threadIdx.x == 0) *out = (uint32_t)__cvta_generic_to_shared(smem4);
}

// Shared-space address at which dynamic shared memory starts (the IdentU8
// table bias of Tab<kIdentU8> is that address rounded up to 256, >> 8).
int probe_dynamic_smem_base(uint32_t *dev_scratch) {
    probe_smem_kernel<<<1, 32, 256>>>(dev_scratch);
    uint32_t v = 0;
    if (cudaMemcpy(&v, dev_scratch, 4, cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    return (int)v;
}

// shared-memory bytes of the table as a kernel lays it out (plus alignment pad)
static int table_smem_bytes(const DevTables &T, int mode) {
    if (mode == kIdentU8P) return (int)(kPadStride + T.image_words / 64 * kPadStride);
    const uint32_t lr = rep_log_of(mode);
    return (int)((256u << lr) + (T.image_words << lr) * 4);
}
static bool is_u8_mode(int mode) { return mode == kIdentU8 || mode == kIdentU8P || mode == kRepU8x8 || mode == kRepU8x4; }

int lanes_smem_bytes(const DevTables &T) {
    return table_smem_bytes(T, T.mode) + (T.has_sticky ? 3 : 1) * bits_words_host(T.nq) * 4;
}

int converge_smem_bytes(const DevTables &T, int warps_per_cta) {
    return table_smem_bytes(T, is_u8_mode(T.mode) ? kIdentU8P : T.mode) + bits_words_host(T.nq) * 4 +
           warps_per_cta * (int)converge_scratch_bytes(T.imax, T.nq);
}

uint32_t tree_lrs(const DevTables &T) {
    uint32_t l = 3;
    while ((1u << l) < T.rs) l++;
    return l;
}
int tree_slice_bytes(const DevTables &T, uint32_t F) {
    const uint32_t rsp = 1u << tree_lrs(T);
    return (int)((F * rsp + ((F + 7) & ~7u) + rsp) * 2);
}
int tree_fixed_bytes(const DevTables &T, int rank_smem) {
    const uint32_t rank_bytes = rank_smem ? (((T.nclass + 1) * T.nq + 15) & ~15u) : 0u;
    const uint32_t dsz_bytes = ((T.nclass + 1) * 2 + 15) & ~15u;
    const uint32_t dead_words = ((T.nq + 31) / 32 + 3) & ~3u;
    return (int)(rank_bytes + dsz_bytes + dead_words * 4);
}

cudaError_t setup_kernel_attributes(const DevTables &T) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    // both lanes kernel variants: DFA_OPT_STICKY_PARKING switches between them
    DevTables T2 = T;
    for (uint32_t v = 0; v < 4; v++) {
        T2.has_sticky = v & 1;
        cudaError_t e = cudaFuncSetAttribute(lanes_fn(T2, v >= 2), cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
        if (e != cudaSuccess) return e;
    }
    cudaError_t e;
    if (void *ft = lanes_fn(T, false, true)) {
        e = cudaFuncSetAttribute(ft, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
        if (e != cudaSuccess) return e;
    }
    e = cudaFuncSetAttribute(converge_fn(T), cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(ceiling_fn(T.mode), cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute((void *)fold_rows_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute((void *)lookahead_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 8 * 8192);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute((void *)starts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - 1024);
    if (e != cudaSuccess) return e;

    e = cudaFuncSetAttribute((void *)ffold_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)ffold_smem_bytes(kFoldCap));
    if (e != cudaSuccess) return e;
    return cudaFuncSetAttribute((void *)tree_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, optin);
}

int lanes_occupancy(const DevTables &T, int threads) {
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, lanes_fn(T), threads, lanes_smem_bytes(T));
    return blocks;
}

int converge_occupancy(const DevTables &T, int warps_per_cta) {
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, converge_fn(T), warps_per_cta * 32,
                                                  converge_smem_bytes(T, warps_per_cta));
    return blocks;
}

cudaError_t launch_converge(const DevTables &T, const Plan &p, const uint8_t *in, uint16_t *surv, uint8_t *surv_n,
                            uint64_t *surv_pos, uint16_t *amap, uint32_t cap, int warps_per_cta, int grid,
                            cudaStream_t s) {
    void *args[] = {(void *)&T, (void *)&p, (void *)&in, (void *)&surv, (void *)&surv_n, (void *)&surv_pos,
                    (void *)&amap, (void *)&cap};
    return cudaLaunchKernel(converge_fn(T), dim3(grid), dim3(warps_per_cta * 32), args,
                            converge_smem_bytes(T, warps_per_cta), s);
}

// tail area (leaves, segment maps, their domains; or the last CTA's CTA maps and warp
// results), rounded to 16 bytes: the info area (decode domains, s_last) follows
int fused_tail_smem_bytes(int threads, uint32_t g_log, int grid) {
    const int N = std::max(threads >> g_log, grid), ns = N / 4 + 1;
    return ((3 * N + ns) * 16 + N * 8 + (3 * N + ns) * 2 + 15) & ~15;  // TailSmem
}
int fused_info_bytes(int threads, uint32_t g_log) { return 2 * (threads >> g_log) + 16; }

// fused_starts_kernel: true start of every reporting chunk for the fused tail.  CTA b
// stages the segment maps of lanes-CTA b (slots k + b, k = its chunks) and walks them
// from its start code (rank codes decode through I_sigma of the byte before b_k).
__global__ void __launch_bounds__(128) fused_starts_kernel(DevTables T, Plan p, Fuse fz, const uint8_t *in,
                                                           uint32_t lpc, uint32_t g_log) {
    __shared__ uint4 seg[1024];
    pdl_wait();
    const uint64_t NL = p.NS >> g_log, l0 = (uint64_t)blockIdx.x * lpc;
    if (l0 >= NL) return;
    const uint64_t l1 = min(NL, l0 + lpc);
    auto chunk_of = [&](uint64_t l) -> uint32_t {
        return l < fz.L0 ? 0u : (uint32_t)(1 + (l - fz.L0) / fz.L);
    };
    const uint32_t ka = chunk_of(l0), kb = chunk_of(l1 - 1);
    for (uint32_t t = threadIdx.x; t <= kb - ka; t += blockDim.x)
        seg[t] = __ldcg(reinterpret_cast<const uint4 *>(fz.part_rows) + ka + t + blockIdx.x);
    __syncthreads();
    if (threadIdx.x != 0) return;
    uint32_t code = __ldcg(fz.cta_code + blockIdx.x);
    for (uint32_t k = ka; k <= kb; k++) {
        const uint64_t f = k == 0 ? 0 : (uint64_t)fz.L0 + (uint64_t)(k - 1) * fz.L;
        if (f >= l0) {
            const uint32_t d = k == 0 ? p.first_dom : (uint32_t)T.byte_class[__ldg(in + p.bounds[k] - 1)];
            fz.starts[k] = (uint16_t)(is_rank(code) ? __ldg(T.dom_list + (uint64_t)d * T.rs + (code - kRank)) : code);
        }
        if (is_rank(code)) code = reinterpret_cast<const uint16_t *>(seg + (k - ka))[code - kRank];
    }
}

cudaError_t launch_lanes(const DevTables &T, const Plan &p, const uint8_t *in, const uint16_t *surv,
                         const uint8_t *surv_n, const uint64_t *surv_pos, uint16_t *sfin, uint32_t sk,
                         uint16_t *dom_of, int convergence, uint16_t *amap, uint32_t g_log,
                         uint16_t *leaf_rows, uint16_t *leaf_dom, DevStatus *status, uint32_t cap, int threads,
                         int grid, cudaStream_t s, const Fuse &fz) {
    void *args[] = {(void *)&T, (void *)&p, (void *)&in, (void *)&surv, (void *)&surv_n, (void *)&surv_pos,
                    (void *)&sfin, (void *)&sk, (void *)&dom_of, (void *)&convergence, (void *)&amap,
                    (void *)&g_log, (void *)&leaf_rows, (void *)&leaf_dom, (void *)&status, (void *)&cap,
                    (void *)&fz};
    int smem = lanes_smem_bytes(T);
    const bool tma = p.tmap != nullptr;
    if (tma) smem += (int)tma_ring_bytes((uint32_t)threads / 32u);
    Fuse f2 = fz;
    if (fz.on) {
        // info area after both the table image and the tail area (it is written at kernel start)
        f2.info_off = (uint32_t)((std::max(smem, fused_tail_smem_bytes(threads, g_log, grid)) + 15) & ~15);
        smem = (int)f2.info_off + fused_info_bytes(threads, g_log);
    }
    args[16] = (void *)&f2;
    return cudaLaunchKernel(lanes_fn(T, p.work != nullptr, tma), dim3(grid), dim3(threads), args, smem, s);
}

// TMA input staging available for this layout and CTA size (the ring must fit beside the table)
bool lanes_tma_available(const DevTables &T, int threads, int optin_smem) {
    return lanes_fn(T, false, true) != nullptr && !T.has_sticky &&
           lanes_smem_bytes(T) + (int)tma_ring_bytes((uint32_t)threads / 32u) <= optin_smem;
}

const void *tree_fn() { return (const void *)tree_kernel; }

int ceiling_occupancy(const DevTables &T, int threads) {
    int blocks = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, ceiling_fn(T.mode), threads, lanes_smem_bytes(T));
    return blocks;
}

cudaError_t launch_ceiling(const DevTables &T, const uint8_t *in, uint64_t per, uint16_t *out, int threads, int grid,
                           cudaStream_t s) {
    void *args[] = {(void *)&T, (void *)&in, (void *)&per, (void *)&out};
    return cudaLaunchKernel(ceiling_fn(T.mode), dim3(grid), dim3(threads), args, lanes_smem_bytes(T), s);
}

#ifdef DFA_TREE_TIMING
extern "C" int dfa_debug_tree_timing(unsigned long long *out, int reset) {
    if (cudaMemcpyFromSymbol(out, g_tree_t, sizeof(unsigned long long) * 32) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long init[32];
        init[0] = ~0ull;
        init[20] = ~0ull;
        for (int i = 1; i < 32; i++) init[i] = (i == 10 || i == 14 || i == 25) ? ~0ull : 0;
        cudaMemcpyToSymbol(g_tree_t, init, sizeof(init));
    }
    return 0;
}
#endif

cudaError_t launch_fold_segments(const DevTables &T, const uint16_t *rows, const uint8_t *lookahead, uint32_t G,
                                 DevStatus *st, uint16_t *dev_final, cudaStream_t s) {
    fold_segments_kernel<<<1, 32, 0, s>>>(T, rows, lookahead, G, st, dev_final);
    return cudaGetLastError();
}

size_t fold_rows_fixed_bytes(const DevTables &T) {
    const size_t rank_bytes = T.rank8 ? (((T.nclass + 1) * T.nq + 15) & ~15u) : 0u;
    const size_t dead_words = ((T.nq + 31) / 32 + 3) & ~3u;
    return rank_bytes + dead_words * 4 + ((T.nclass + 1 + 7) & ~7u) * 2;
}

cudaError_t launch_fold_rows(const DevTables &T, const uint16_t *rows, const uint16_t *doms, uint32_t P,
                             uint32_t per_cta, uint16_t *cta_rows, uint16_t *cta_doms, uint32_t *ticket,
                             DevStatus *st, uint16_t *dev_final, uint16_t *seg_row, cudaStream_t s) {
    const uint32_t lrs = tree_lrs(T);
    const uint32_t grid = (P + per_cta - 1) / per_cta;
    const size_t smem = fold_rows_fixed_bytes(T) + ((per_cta + 7) & ~7u) * 2 + ((size_t)per_cta << lrs) * 2;
    fold_rows_kernel<<<grid, 256, smem, s>>>(T, rows, doms, P, per_cta, lrs, cta_rows, cta_doms, ticket, st,
                                              dev_final, seg_row);
    return cudaGetLastError();
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*k)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, k, std::forward<Args>(args)...);
}

cudaError_t launch_fused_starts(const DevTables &T, const Plan &p, const Fuse &fz, const uint8_t *in, uint32_t lpc,
                                uint32_t g_log, int grid, cudaStream_t s) {
    return launch_pdl(fused_starts_kernel, dim3(grid), dim3(128), 0, s, T, p, fz, in, lpc, g_log);
}

cudaError_t launch_batch_out(const DevTables &T, const uint16_t *rep_rows, uint32_t rs, const int32_t *kidx,
                             const uint64_t *offsets, uint64_t data_len, uint32_t count, uint16_t *dev_final,
                             uint8_t *dev_accept, DevStatus *st, cudaStream_t s) {
    const uint32_t grid = std::min<uint32_t>((count + 255) / 256, 1024);
    return launch_pdl(batch_out_kernel, dim3(std::max<uint32_t>(grid, 1)), dim3(256), 0, s, T, rep_rows, rs, kidx,
                      offsets, data_len, count, dev_final, dev_accept, st);
}

cudaError_t launch_leaf_fold(const uint16_t *in_rows, const uint16_t *in_dom, uint32_t L0, uint32_t L, uint32_t P,
                             uint16_t *out_rows, uint16_t *out_dom, int sms, cudaStream_t s) {
    const uint64_t total = (uint64_t)(L0 + 31) / 32 + (uint64_t)(P - 1) * ((L + 31) / 32);
    const uint32_t grid = (uint32_t)std::min<uint64_t>((total + 7) / 8, (uint64_t)sms * 8);
    return launch_pdl(leaf_fold_kernel, dim3(grid), dim3(256), 0, s, in_rows, in_dom, L0, L, P, out_rows, out_dom);
}

cudaError_t launch_compose8(const DevTables &T, const uint16_t *leaves, const uint16_t *leaf_dom, uint32_t L0,
                            uint32_t L, uint32_t P, uint32_t cpc, uint16_t *rep_rows, uint16_t *rep_doms,
                            uint16_t *user_rows, uint16_t *user_row0, uint16_t *e0, uint16_t *cta_rows,
                            uint16_t *cta_doms, uint32_t *ticket, DevStatus *st, uint16_t *dev_final,
                            uint16_t *cta_start, uint16_t *starts, uint16_t *seg_row, cudaStream_t s) {
    // 4 chunks per warp per round: about one round per SM-resident CTA, cpc <= 1024
    const uint32_t warps = std::min<uint32_t>(32, std::max<uint32_t>(1, (cpc + 3) / 4));
    const uint32_t grid = (P + cpc - 1) / cpc;
    cudaError_t e = launch_pdl(compose8_kernel, dim3(grid), dim3(warps * 32), 0, s, T, leaves, leaf_dom, L0, L, P, cpc,
                               rep_rows, rep_doms, user_rows, user_row0, e0, cta_rows, cta_doms, ticket, st,
                               dev_final, starts ? cta_start : nullptr, seg_row);
    if (e != cudaSuccess || !starts) return e;
    return launch_pdl(starts8_kernel, dim3(grid), dim3(256), 0, s, T, (const uint16_t *)rep_rows,
                      (const uint16_t *)rep_doms, P, cpc, (const uint16_t *)cta_start, starts);
}

cudaError_t launch_lookahead(const DevTables &T, const uint8_t *in, const uint64_t *bounds, uint32_t P, uint32_t r,
                             const uint16_t *maps, uint16_t *doms_out, uint16_t *sizes_out, uint16_t *maps_out,
                             DevStatus *st, int sms, cudaStream_t s) {
    if (P < 2) return cudaSuccess;
    const uint32_t smem = 8 * ((T.nq_user + 31) / 32) * 4;
    const uint32_t grid = std::min<uint32_t>((P - 1 + 7) / 8, (uint32_t)sms * 8);
    lookahead_kernel<<<grid, 256, smem, s>>>(T, in, bounds, P, r, maps, doms_out, sizes_out, maps_out, st);
    return cudaGetLastError();
}

cudaError_t launch_walk(const DevTables &T, const Tree &tr, uint32_t L, int sms, cudaStream_t s) {
    return launch_walk_level(T, tr, L, sms, s);
}
cudaError_t launch_fwalk(const DevTables &T, const Tree &tr, uint32_t L, int sms, cudaStream_t s) {
    const uint64_t total = (uint64_t)tr.lv[L].nodes * 8;
    const uint64_t grid = std::min<uint64_t>((total + 255) / 256, (uint64_t)sms * 16);
    return launch_pdl(fwalk_kernel, dim3((unsigned)std::max<uint64_t>(grid, 1)), dim3(256), 0, s, T, tr, L);
}
cudaError_t launch_fexpand(const DevTables &T, const Tree &tr, uint32_t L, int sms, cudaStream_t s) {
    const uint64_t total = (uint64_t)(L == tr.rep_level ? tr.lv[L].nodes : 1u) * T.rs;
    const uint64_t grid = std::min<uint64_t>((total + 255) / 256, (uint64_t)sms * 16);
    return launch_pdl(fexpand_kernel, dim3((unsigned)std::max<uint64_t>(grid, 1)), dim3(256), 0, s, T, tr, L);
}
uint32_t ffold_cap() { return kFoldCap; }
uint32_t fchunk_cap() { return kChunkLeaves; }
cudaError_t launch_fchunk(const DevTables &T, const Tree &tr, int sms, cudaStream_t s) {
    const uint32_t P = tr.lv[tr.rep_level].nodes;
    const uint32_t grid = std::max<uint32_t>(1, std::min<uint32_t>((P + 7) / 8, (uint32_t)sms * 8));
    return launch_pdl(fchunk_kernel, dim3(grid), dim3(256), 0, s, T, tr);
}
cudaError_t launch_ffold(const DevTables &T, const Tree &tr, uint32_t Ls, cudaStream_t s) {
    return launch_pdl(ffold_kernel, dim3(1), dim3(1024), ffold_smem_bytes(tr.lv[Ls].nodes), s, T, tr, Ls);
}

cudaError_t launch_tree(const DevTables &T, const Tree &tr, int grid, int smem_bytes, cudaStream_t s) {
    tree_kernel<<<grid, 256, smem_bytes, s>>>(T, tr);
    return cudaGetLastError();
}

cudaError_t launch_starts(const DevTables &T, const Plan &p, const uint16_t *row0, const uint16_t *rows,
                          const uint16_t *dom, uint16_t *starts, DevStatus *st, cudaStream_t s) {
    int dev = 0, optin = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const uint64_t nr = (uint64_t)(T.nclass + 1) * T.nq;
    const uint64_t budget = (uint64_t)optin - 1024;
    const uint64_t row_budget = 48 * 1024;
    uint32_t mode = 0;
    uint64_t rb = 0;
    if (T.rank8 && ((nr + 15) & ~15ull) + row_budget <= budget) { mode = 1; rb = (nr + 15) & ~15ull; }
    else if (((nr * 2 + 15) & ~15ull) + row_budget <= budget) { mode = 2; rb = (nr * 2 + 15) & ~15ull; }
    const uint32_t blk = (uint32_t)std::max<uint64_t>(1, std::min<uint64_t>(1024, row_budget / (T.rs * 2 + 2)));
    const size_t smem = rb + (size_t)blk * T.rs * 2 + (size_t)blk * 2 + 16;
    return launch_pdl(starts_kernel, dim3(1), dim3(512), smem, s, T, p, row0, rows, dom, starts, st, mode, blk);
}

#endif  // DFA_TU_MAIN

} // namespace dfa
