// lds_gather_bench.cu -- micro-benchmark of the lanes kernel's hot step
// s <- T[s][b] on B200 shared memory, one lane per thread, for table layouts
// that trade shared-memory capacity for bank-conflict degree.
// Not part of the library; results go to profiles/.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ldsb tools/lds_gather_bench.cu -lcuda
//   ./ldsb [MiB]
//
// Layouts (random DFA over 256 byte columns; each thread runs its own
// contiguous sub-chunk with 32-byte loads, as lanes_kernel does):
//   0 ident_u8   one copy, address (s<<8)|b            -> ~3.5 wavefronts / warp LDS
//   1 rep8_u8    8 copies, copy g in banks 4g..4g+3   -> ~2.96
//   2 rep16_p6   16 copies in bank pairs, 6-bit entries 5 per word (|Q| <= 65)
//   3 rep16_u8   16 copies in bank pairs, u8 (|Q| <= 56; run with 32 states)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda.h>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t lds_u8(uint32_t a) { uint32_t r; asm volatile("ld.shared.u8 %0, [%1];" : "=r"(r) : "r"(a)); return r; }
// prmt with sign-replicate selectors (bit 3 of a nibble): 0xC -> 0x00 for a byte < 0x80.
// (__byte_perm keeps only the low 3 bits of each selector nibble.)
__device__ __forceinline__ uint32_t prmt(uint32_t a, uint32_t b, uint32_t sel) {
    uint32_t r; asm("prmt.b32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(b), "r"(sel)); return r;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) { uint32_t r; asm volatile("ld.shared.u32 %0, [%1];" : "=r"(r) : "r"(a)); return r; }

// one 32-byte sector per thread; cache qualifiers per layout under test
template <int L>
__device__ __forceinline__ void load8(uint32_t (&r)[8], const uint8_t *q) {
    if (L == 6 || L == 7)
        asm volatile("ld.global.nc.L1::no_allocate.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "l"(q));
    else if (L == 5)
        asm volatile("ld.global.nc.L2::256B.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "l"(q));
    else
        asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]) : "l"(q));
}

template <int L, int ILP>
__global__ void __launch_bounds__(1024, 1) gather(const uint8_t *img, uint32_t img_bytes, uint32_t align,
                                                  const uint8_t *in, uint64_t per_thread, uint32_t *out) {
    extern __shared__ uint4 sm[];
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t base = (sb + align - 1) & ~(align - 1);
    uint8_t *tab = reinterpret_cast<uint8_t *>(sm) + (base - sb);
    const int shift = (L == 0 || L == 5 || L == 6) ? 8 : L == 1 ? 11 : L == 3 ? 12 : 0;
    const uint32_t bias = shift ? (base >> shift) : 0u, bias4 = bias * 0x01010101u;
    for (uint32_t i = threadIdx.x; i < img_bytes / 16; i += blockDim.x) {
        uint4 v = reinterpret_cast<const uint4 *>(img)[i];
        v.x = __vadd4(v.x, bias4); v.y = __vadd4(v.y, bias4); v.z = __vadd4(v.z, bias4); v.w = __vadd4(v.w, bias4);
        reinterpret_cast<uint4 *>(tab)[i] = v;
    }
    __syncthreads();
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    // ILP independent chains per thread: chain c runs sub-chunk tid*ILP + c
    const uint64_t per = per_thread / ILP;
    const uint8_t *p = in + (uint64_t)tid * per_thread;
    const uint32_t lane = threadIdx.x & 31;
    uint32_t s[ILP];
    uint32_t g4 = 0, g3 = 0;
#pragma unroll
    for (int c = 0; c < ILP; c++) {
        if (L == 0 || L == 5 || L == 6) s[c] = (base >> 8);
        if (L == 4 || L == 7) s[c] = 0;
        if (L == 1) s[c] = base >> 11;
        if (L == 2) s[c] = 0;
        if (L == 3) s[c] = base >> 12;
    }
    if (L == 1) g4 = ((lane & 7) << 4) * 0x01010101u;
    if (L == 2) g3 = base + ((lane & 15) << 3);
    if (L == 3) g3 = ((lane & 15) << 3) * 0x01010101u;
    uint32_t nx[ILP][8];
#pragma unroll
    for (int c = 0; c < ILP; c++) load8<L>(nx[c], p + c * per);
    for (uint64_t o = 0; o < per; o += 32) {
        uint32_t w[ILP][8];
#pragma unroll
        for (int c = 0; c < ILP; c++)
#pragma unroll
            for (int q = 0; q < 8; q++) w[c][q] = nx[c][q];
        if (o + 32 < per)  // register double buffer: the next sector is in flight
#pragma unroll
            for (int c = 0; c < ILP; c++) load8<L>(nx[c], p + c * per + o + 32);
#pragma unroll
        for (int q = 0; q < 8; q++) {
#pragma unroll
            for (int k = 0; k < 4; k++) {
#pragma unroll
                for (int c = 0; c < ILP; c++) {
                    const uint32_t x = w[c][q];
                    if (L == 0 || L == 5 || L == 6) {
                        s[c] = lds_u8(__byte_perm(x, s[c], 0x6540 + k));
                    } else if (L == 4 || L == 7) {
                        s[c] = (s[c] * 3u) ^ (x >> (8 * k));
                    } else if (L == 1) {
                        const uint32_t y = (x & 0x0F0F0F0Fu) | ((x & 0x10101010u) << 3) | g4;
                        const uint32_t z = (x >> 5) & 0x07070707u;
                        s[c] = lds_u8((s[c] << 11) + prmt(y, z, 0xCC00 | ((4 + k) << 4) | k));
                    } else if (L == 2) {
                        const uint32_t b = (x >> (8 * k)) & 0xFFu;
                        const uint32_t kb = ((b >> 1) << 7) + ((b & 1u) << 2) + g3;
                        const uint32_t G = (s[c] * 205u) >> 10;
                        const uint32_t sh = 6u * (s[c] - 5u * G);
                        s[c] = (lds_u32((G << 14) + kb) >> sh) & 63u;
                    } else {
                        const uint32_t y = (x & 0x07070707u) | g3 | ((x & 0x08080808u) << 4);
                        const uint32_t z = (x >> 4) & 0x0F0F0F0Fu;
                        s[c] = lds_u8((s[c] << 12) + prmt(y, z, 0xCC00 | ((4 + k) << 4) | k));
                    }
                }
            }
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int c = 0; c < ILP; c++) r = r * 131u + (s[c] - bias);
    out[tid] = ILP == 1 ? s[0] - bias : r;
}


// Input staged by per-thread 1-D bulk copies (cp.async.bulk, the TMA engine)
// into a shared-memory ring instead of register loads: S stages of CH bytes per
// thread, slot pitch CH + 16 (conflict-free LDS.128 read-back), one mbarrier per
// thread and stage.  L = 0 (ident_u8) or 1 (rep8_u8) table layout.
template <int L, int CH, int S>
__global__ void __launch_bounds__(1024, 1) gather_tma(const uint8_t *img, uint32_t img_bytes, uint32_t align,
                                                      const uint8_t *in, uint64_t per_thread, uint32_t *out) {
    extern __shared__ uint4 sm[];
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t base = (sb + align - 1) & ~(align - 1);
    uint8_t *tab = reinterpret_cast<uint8_t *>(sm) + (base - sb);
    const int shift = L == 0 ? 8 : 11;
    const uint32_t bias = base >> shift, bias4 = bias * 0x01010101u;
    for (uint32_t i = threadIdx.x; i < img_bytes / 16; i += blockDim.x) {
        uint4 v = reinterpret_cast<const uint4 *>(img)[i];
        v.x = __vadd4(v.x, bias4); v.y = __vadd4(v.y, bias4); v.z = __vadd4(v.z, bias4); v.w = __vadd4(v.w, bias4);
        reinterpret_cast<uint4 *>(tab)[i] = v;
    }
    constexpr uint32_t PITCH = CH + 16;
    uint8_t *ring = tab + ((img_bytes + 127) & ~127u);
    uint64_t *bars = reinterpret_cast<uint64_t *>(ring + (size_t)blockDim.x * S * PITCH);
    const uint32_t t = threadIdx.x;
    const uint32_t my_slot0 = (uint32_t)__cvta_generic_to_shared(ring) + t * S * PITCH;
    const uint32_t my_bar0 = (uint32_t)__cvta_generic_to_shared(bars) + t * S * 8;
#pragma unroll
    for (int k = 0; k < S; k++) asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(my_bar0 + 8 * k));
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint8_t *p = in + (uint64_t)tid * per_thread;
    const uint32_t lane = t & 31;
    uint32_t s = L == 0 ? (base >> 8) : (base >> 11);
    const uint32_t g4 = L == 1 ? ((lane & 7) << 4) * 0x01010101u : 0u;
    auto issue = [&](uint64_t off, int k) {
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(my_bar0 + 8 * k), "r"((uint32_t)CH) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(my_slot0 + k * PITCH), "l"(p + off), "r"((uint32_t)CH), "r"(my_bar0 + 8 * k) : "memory");
    };
    const uint64_t nblk = per_thread / CH;
#pragma unroll
    for (int k = 0; k < S; k++) if ((uint64_t)k < nblk) issue((uint64_t)k * CH, k);
    uint32_t phase = 0;
    for (uint64_t bi = 0; bi < nblk; bi++) {
        const int k = (int)(bi % S);
        const uint32_t bar = my_bar0 + 8 * k;
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                         : "=r"(done) : "r"(bar), "r"((phase >> k) & 1u) : "memory");
        phase ^= 1u << k;
        uint4 q[CH / 16];
#pragma unroll
        for (int j = 0; j < CH / 16; j++)
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q[j].x), "=r"(q[j].y), "=r"(q[j].z), "=r"(q[j].w)
                         : "r"(my_slot0 + k * PITCH + 16 * j));
        if (bi + S < nblk) issue((bi + S) * CH, k);  // the slot is in registers now
#pragma unroll
        for (int j = 0; j < CH / 16; j++) {
            const uint32_t w4[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
            for (int wq = 0; wq < 4; wq++) {
                const uint32_t x = w4[wq];
                if (L == 0) {
#pragma unroll
                    for (int kk = 0; kk < 4; kk++) s = lds_u8(__byte_perm(x, s, 0x6540 + kk));
                } else {
                    const uint32_t y = (x & 0x0F0F0F0Fu) | ((x & 0x10101010u) << 3) | g4;
                    const uint32_t z = (x >> 5) & 0x07070707u;
#pragma unroll
                    for (int kk = 0; kk < 4; kk++) s = lds_u8((s << 11) + prmt(y, z, 0xCC00 | ((4 + kk) << 4) | kk));
                }
            }
        }
    }
    out[tid] = s - bias;
}

// Input staged CTA-cooperatively by 2-D tensor-map copies (cp.async.bulk.tensor.2d,
// TMA): thread t's sub-chunk is row t of a [rows][per] byte matrix (a uniform stride),
// one stage = a box of CH bytes x 256 rows per TMA op (4 ops for the CTA's 1024 rows),
// full/empty mbarriers per stage, S stages; each thread reads its CH bytes back with
// 16-byte shared loads.  L = 0 (ident_u8) or 1 (rep8_u8).
template <int L, int CH, int S>
__global__ void __launch_bounds__(1024, 1) gather_tma2d(const __grid_constant__ CUtensorMap tmap, const uint8_t *img,
                                                        uint32_t img_bytes, uint32_t align, uint64_t per,
                                                        uint32_t *out) {
    extern __shared__ uint4 sm[];
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t base = (sb + align - 1) & ~(align - 1);
    uint8_t *tab = reinterpret_cast<uint8_t *>(sm) + (base - sb);
    const int shift = L == 0 ? 8 : 11;
    const uint32_t bias = base >> shift, bias4 = bias * 0x01010101u;
    for (uint32_t i = threadIdx.x; i < img_bytes / 16; i += blockDim.x) {
        uint4 v = reinterpret_cast<const uint4 *>(img)[i];
        v.x = __vadd4(v.x, bias4); v.y = __vadd4(v.y, bias4); v.z = __vadd4(v.z, bias4); v.w = __vadd4(v.w, bias4);
        reinterpret_cast<uint4 *>(tab)[i] = v;
    }
    const uint32_t T = blockDim.x;
    uint8_t *ring = tab + ((img_bytes + 1023) & ~1023u);                 // [S][T][CH], 1 KB aligned
    uint64_t *bars = reinterpret_cast<uint64_t *>(ring + (size_t)S * T * CH);  // full[S], empty[S]
    const uint32_t ring_s = (uint32_t)__cvta_generic_to_shared(ring), bar_s = (uint32_t)__cvta_generic_to_shared(bars);
    const uint32_t t = threadIdx.x, lane = t & 31;
    if (t == 0) {
#pragma unroll
        for (int k = 0; k < S; k++) {
            asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(bar_s + 8 * k));
            asm volatile("mbarrier.init.shared.b64 [%0], %1;" :: "r"(bar_s + 8 * (S + k)), "r"(T));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    const uint32_t row0 = blockIdx.x * T;
    auto issue = [&](uint64_t bi, int k) {  // thread 0: stage k <- bytes [bi CH, (bi+1) CH) of all rows
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(bar_s + 8 * k), "r"(T * (uint32_t)CH) : "memory");
        for (uint32_t q = 0; q < T / 256; q++)
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         :: "r"(ring_s + (uint32_t)(k * T * CH) + q * 256 * CH), "l"(&tmap), "r"((int)(bi * CH)),
                            "r"((int)(row0 + q * 256)), "r"(bar_s + 8 * k) : "memory");
    };
    const uint64_t nblk = per / CH;
    if (t == 0)
        for (int k = 0; k < S; k++) if ((uint64_t)k < nblk) issue(k, k);
    uint32_t s = L == 0 ? (base >> 8) : (base >> 11);
    const uint32_t g4 = L == 1 ? ((lane & 7) << 4) * 0x01010101u : 0u;
    for (uint64_t bi = 0; bi < nblk; bi++) {
        const int k = (int)(bi % S);
        const uint32_t par = (uint32_t)((bi / S) & 1);
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                         : "=r"(done) : "r"(bar_s + 8 * k), "r"(par) : "memory");
        uint4 q[CH / 16];
#pragma unroll
        for (int j = 0; j < CH / 16; j++)
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q[j].x), "=r"(q[j].y), "=r"(q[j].z), "=r"(q[j].w)
                         : "r"(ring_s + (uint32_t)(k * T * CH) + t * CH + 16 * j));
        asm volatile("mbarrier.arrive.shared.b64 _, [%0];" :: "r"(bar_s + 8 * (S + k)) : "memory");
        if (t == 0 && bi + S < nblk) {  // the stage is free once every thread has read it
            uint32_t e = 0;
            while (!e)
                asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                             : "=r"(e) : "r"(bar_s + 8 * (S + k)), "r"(par) : "memory");
            issue(bi + S, k);
        }
#pragma unroll
        for (int j = 0; j < CH / 16; j++) {
            const uint32_t w4[4] = {q[j].x, q[j].y, q[j].z, q[j].w};
#pragma unroll
            for (int wq = 0; wq < 4; wq++) {
                const uint32_t x = w4[wq];
                if (L == 0) {
#pragma unroll
                    for (int kk = 0; kk < 4; kk++) s = lds_u8(__byte_perm(x, s, 0x6540 + kk));
                } else {
                    const uint32_t y = (x & 0x0F0F0F0Fu) | ((x & 0x10101010u) << 3) | g4;
                    const uint32_t z = (x >> 5) & 0x07070707u;
#pragma unroll
                    for (int kk = 0; kk < 4; kk++) s = lds_u8((s << 11) + prmt(y, z, 0xCC00 | ((4 + kk) << 4) | kk));
                }
            }
        }
    }
    out[blockIdx.x * T + t] = s - bias;
}

static uint64_t rng = 88172645463325252ull;
static uint32_t nxt() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return (uint32_t)rng; }

int main(int argc, char **argv) {
    const uint64_t n = (uint64_t)(argc > 1 ? atoi(argv[1]) : 256) << 20;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::vector<uint8_t> hin(n);
    for (uint64_t i = 0; i < n; i += 4) { uint32_t v = nxt(); memcpy(&hin[i], &v, 4); }
    uint8_t *din; uint32_t *dout;
    CK(cudaMalloc(&din, n));
    CK(cudaMemcpy(din, hin.data(), n, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dout, 4u << 20));
    const int order[][2] = {{0, 1}, {1, 1}, {2, 1}, {3, 1}, {4, 1}, {5, 1}, {6, 1}, {7, 1}};
    for (auto &oi : order) {
        const int L = oi[0], ILP = oi[1];
        const int nq = L == 3 ? 32 : 64;
        const int Li = (L == 5 || L == 6) ? 0 : L;  // image layout
        std::vector<uint8_t> delta(nq * 256);
        for (auto &d : delta) d = nxt() % nq;
        uint32_t bytes = 0, align = 0;
        std::vector<uint8_t> img;
        // images are position independent except for the encoded-state bias,
        // which the kernel adds via its base address: store raw states here and
        // bias them below where the layout needs it
        if (L == 4 || L == 7) { bytes = 16; align = 16; img.assign(bytes, 0); }
        if (Li == 0) { bytes = nq * 256; align = 256; img.assign(bytes, 0);
            for (int s = 0; s < nq; s++) for (int b = 0; b < 256; b++) img[s * 256 + b] = delta[s * 256 + b]; }
        if (Li == 1) { bytes = nq * 2048; align = 2048; img.assign(bytes, 0);
            for (int g = 0; g < 8; g++) for (int s = 0; s < nq; s++) for (int b = 0; b < 256; b++)
                img[(s << 11) | (((b >> 5) & 7) << 8) | (((b >> 4) & 1) << 7) | (g << 4) | (b & 15)] = delta[s * 256 + b]; }
        if (Li == 2) { bytes = 13 << 14; align = 16; img.assign(bytes, 0);
            for (int g = 0; g < 16; g++) for (int s = 0; s < nq; s++) for (int b = 0; b < 256; b++) {
                uint32_t G = s / 5, j = s % 5, a = (G << 14) + ((b >> 1) << 7) + (g << 3) + ((b & 1) << 2);
                uint32_t v; memcpy(&v, &img[a], 4); v |= (uint32_t)delta[s * 256 + b] << (6 * j); memcpy(&img[a], &v, 4); } }
        if (Li == 3) { bytes = nq << 12; align = 4096; img.assign(bytes, 0);
            for (int g = 0; g < 16; g++) for (int s = 0; s < nq; s++) for (int b = 0; b < 256; b++)
                img[(s << 12) + ((b >> 3) << 7) + (g << 3) + (((b >> 2) & 1) << 2) + (b & 3)] = delta[s * 256 + b]; }
        uint8_t *dimg; CK(cudaMalloc(&dimg, bytes + 16));
        CK(cudaMemcpy(dimg, img.data(), bytes, cudaMemcpyHostToDevice));
        const int threads = 1024, smem = bytes + align + 16;
        const int grid = sms;
        const uint64_t per = (n / ((uint64_t)grid * threads)) & ~(32ull * ILP - 1);
        auto launch = [&]() {
            void (*f)(const uint8_t *, uint32_t, uint32_t, const uint8_t *, uint64_t, uint32_t *) = nullptr;
#define PICK(l, i) if (L == l && ILP == i) f = gather<l, i>;
            PICK(0, 1) PICK(1, 1) PICK(2, 1) PICK(3, 1) PICK(0, 2) PICK(1, 2) PICK(3, 2) PICK(4, 1) PICK(5, 1) PICK(4, 2) PICK(6, 1) PICK(7, 1)
            CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
            f<<<grid, threads, smem>>>(dimg, bytes, align, din, per, dout);
        };
        launch();
        CK(cudaDeviceSynchronize());
        // check three threads' final states against a host run
        std::vector<uint32_t> got(grid * threads);
        CK(cudaMemcpy(got.data(), dout, got.size() * 4, cudaMemcpyDeviceToHost));
        int bad = 0;
        for (uint32_t t : {0u, 777u, (uint32_t)(grid * threads - 1)}) {
            uint32_t r = 0;
            for (int c = 0; c < ILP; c++) {
                uint32_t hs = 0;
                for (uint64_t i = 0; i < per / ILP; i++) {
                    const uint32_t b = hin[t * per + c * (per / ILP) + i];
                    if (L == 4 || L == 7) {  // kernel: s = s*3 ^ (x >> 8k), x = the 4-byte word holding b
                        uint32_t x; memcpy(&x, &hin[t * per + c * (per / ILP) + (i & ~3ull)], 4);
                        hs = (hs * 3u) ^ (x >> (8 * (i & 3)));
                    } else hs = delta[hs * 256 + b];
                }
                r = r * 131u + hs;
            }
            bad += got[t] != r;
        }
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        const int reps = 20;
        cudaEventRecord(a);
        for (int r = 0; r < reps; r++) launch();
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b);
        ms /= reps;
        const double bytes_done = (double)per * grid * threads;
        printf("{\"layout\": %d, \"ilp\": %d, \"name\": \"%s\", \"states\": %d, \"smem_table_bytes\": %u, \"ms\": %.4f, \"GBps\": %.1f, "
               "\"lookups_per_clk_per_sm_at_1965\": %.2f, \"check\": \"%s\"}\n",
               L, ILP, L == 0 ? "ident_u8" : L == 1 ? "rep8_u8" : L == 2 ? "rep16_p6" : L == 3 ? "rep16_u8" : L == 4 ? "load_only" : L == 5 ? "ident_u8_L2pf256" : L == 6 ? "ident_u8_L1noalloc" : "load_only_L1noalloc", nq, bytes, ms,
               bytes_done / ms / 1e6, bytes_done / (ms * 1e-3) / sms / 1.965e9, bad ? "FAIL" : "ok");
        CK(cudaFree(dimg));
    }
    // TMA-staged input (layouts 0 and 1, CH bytes per stage, S stages)
    for (int L = 0; L < 2; L++) {
        const int nq = 64;
        std::vector<uint8_t> delta(nq * 256);
        for (auto &d : delta) d = nxt() % nq;
        uint32_t bytes, align;
        std::vector<uint8_t> img;
        if (L == 0) { bytes = nq * 256; align = 256; img.assign(bytes, 0);
            for (int s = 0; s < nq; s++) for (int b = 0; b < 256; b++) img[s * 256 + b] = delta[s * 256 + b]; }
        else { bytes = nq * 2048; align = 2048; img.assign(bytes, 0);
            for (int g = 0; g < 8; g++) for (int s = 0; s < nq; s++) for (int b = 0; b < 256; b++)
                img[(s << 11) | (((b >> 5) & 7) << 8) | (((b >> 4) & 1) << 7) | (g << 4) | (b & 15)] = delta[s * 256 + b]; }
        uint8_t *dimg; CK(cudaMalloc(&dimg, bytes + 16));
        CK(cudaMemcpy(dimg, img.data(), bytes, cudaMemcpyHostToDevice));
        for (int variant = 0; variant < 3; variant++) {
            const int CHv = variant == 0 ? 32 : variant == 1 ? 64 : 32, Sv = variant == 2 ? 3 : 2;
            void (*f)(const uint8_t *, uint32_t, uint32_t, const uint8_t *, uint64_t, uint32_t *) =
                L == 0 ? (variant == 0 ? gather_tma<0, 32, 2> : variant == 1 ? gather_tma<0, 64, 2> : gather_tma<0, 32, 3>)
                       : (variant == 0 ? gather_tma<1, 32, 2> : variant == 1 ? gather_tma<1, 64, 2> : gather_tma<1, 32, 3>);
            const int threads = 1024, grid = sms;
            const size_t smem = align + ((bytes + 127) & ~127u) + (size_t)threads * Sv * (CHv + 16) + threads * Sv * 8 + 64;
            if (smem > 232448) { printf("{\"tma\": 1, \"layout\": %d, \"skip\": \"smem %zu\"}\n", L, smem); continue; }
            CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
            const uint64_t per = (n / ((uint64_t)grid * threads)) & ~(uint64_t)(CHv - 1);
            f<<<grid, threads, smem>>>(dimg, bytes, align, din, per, dout);
            CK(cudaDeviceSynchronize());
            std::vector<uint32_t> got(grid * threads);
            CK(cudaMemcpy(got.data(), dout, got.size() * 4, cudaMemcpyDeviceToHost));
            int bad = 0;
            for (uint32_t t : {0u, 777u, (uint32_t)(grid * threads - 1)}) {
                uint32_t hs = 0;
                for (uint64_t i = 0; i < per; i++) hs = delta[hs * 256 + hin[t * per + i]];
                bad += got[t] != hs;
            }
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            for (int r = 0; r < 20; r++) f<<<grid, threads, smem>>>(dimg, bytes, align, din, per, dout);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b);
            ms /= 20;
            const double bytes_done = (double)per * grid * threads;
            printf("{\"tma\": 1, \"layout\": %d, \"name\": \"%s_tma\", \"stage_bytes\": %d, \"stages\": %d, \"ms\": %.4f, "
                   "\"GBps\": %.1f, \"lookups_per_clk_per_sm_at_1965\": %.2f, \"check\": \"%s\"}\n",
                   L, L == 0 ? "ident_u8" : "rep8_u8", CHv, Sv, ms, bytes_done / ms / 1e6,
                   bytes_done / (ms * 1e-3) / sms / 1.965e9, bad ? "FAIL" : "ok");
        }
        CK(cudaFree(dimg));
    }
    // CTA-cooperative 2-D tensor-map staging (uniform sub-chunk stride)
    for (int L = 0; L < 2; L++) {
        const int nq = 64;
        std::vector<uint8_t> delta(nq * 256);
        for (auto &d : delta) d = nxt() % nq;
        uint32_t bytes, align;
        std::vector<uint8_t> img;
        if (L == 0) { bytes = nq * 256; align = 256; img.assign(bytes, 0);
            for (int s = 0; s < nq; s++) for (int b = 0; b < 256; b++) img[s * 256 + b] = delta[s * 256 + b]; }
        else { bytes = nq * 2048; align = 2048; img.assign(bytes, 0);
            for (int g = 0; g < 8; g++) for (int s = 0; s < nq; s++) for (int b = 0; b < 256; b++)
                img[(s << 11) | (((b >> 5) & 7) << 8) | (((b >> 4) & 1) << 7) | (g << 4) | (b & 15)] = delta[s * 256 + b]; }
        uint8_t *dimg; CK(cudaMalloc(&dimg, bytes + 16));
        CK(cudaMemcpy(dimg, img.data(), bytes, cudaMemcpyHostToDevice));
        for (int variant = 0; variant < 4; variant++) {
            const int CHv = (variant & 1) ? 64 : 32, Sv = (variant & 2) ? 4 : 2;
            void (*f)(const CUtensorMap, const uint8_t *, uint32_t, uint32_t, uint64_t, uint32_t *) =
                L == 0 ? (variant == 0 ? gather_tma2d<0, 32, 2> : variant == 1 ? gather_tma2d<0, 64, 2>
                          : variant == 2 ? gather_tma2d<0, 32, 4> : gather_tma2d<0, 64, 4>)
                       : (variant == 0 ? gather_tma2d<1, 32, 2> : variant == 1 ? gather_tma2d<1, 64, 2>
                          : variant == 2 ? gather_tma2d<1, 32, 4> : gather_tma2d<1, 64, 4>);
            const int threads = 1024, grid = sms;
            const size_t smem = align + ((bytes + 1023) & ~1023u) + (size_t)threads * Sv * CHv + 2 * Sv * 8 + 64;
            if (smem > 232448) { printf("{\"tma2d\": 1, \"layout\": %d, \"stage_bytes\": %d, \"stages\": %d, \"skip\": \"smem %zu\"}\n", L, CHv, Sv, smem); continue; }
            CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
            const uint64_t per = (n / ((uint64_t)grid * threads)) & ~(uint64_t)(CHv - 1);
            CUtensorMap tm;
            const cuuint64_t dims[2] = {(cuuint64_t)per, (cuuint64_t)grid * threads};
            const cuuint64_t strides[1] = {(cuuint64_t)per};
            const cuuint32_t box[2] = {(cuuint32_t)CHv, 256}, estr[2] = {1, 1};
            CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, din, dims, strides, box, estr,
                                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (cr != CUDA_SUCCESS) { printf("{\"tma2d\": 1, \"error\": \"cuTensorMapEncodeTiled %d\"}\n", (int)cr); continue; }
            f<<<grid, threads, smem>>>(tm, dimg, bytes, align, per, dout);
            CK(cudaDeviceSynchronize());
            std::vector<uint32_t> got(grid * threads);
            CK(cudaMemcpy(got.data(), dout, got.size() * 4, cudaMemcpyDeviceToHost));
            int bad = 0;
            for (uint32_t t : {0u, 777u, (uint32_t)(grid * threads - 1)}) {
                uint32_t hs = 0;
                for (uint64_t i = 0; i < per; i++) hs = delta[hs * 256 + hin[t * per + i]];
                bad += got[t] != hs;
            }
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            for (int r = 0; r < 20; r++) f<<<grid, threads, smem>>>(tm, dimg, bytes, align, per, dout);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b);
            ms /= 20;
            const double bytes_done = (double)per * grid * threads;
            printf("{\"tma2d\": 1, \"layout\": %d, \"name\": \"%s_tma2d\", \"stage_bytes\": %d, \"stages\": %d, \"ms\": %.4f, "
                   "\"GBps\": %.1f, \"lookups_per_clk_per_sm_at_1965\": %.2f, \"check\": \"%s\"}\n",
                   L, L == 0 ? "ident_u8" : "rep8_u8", CHv, Sv, ms, bytes_done / ms / 1e6,
                   bytes_done / (ms * 1e-3) / sms / 1.965e9, bad ? "FAIL" : "ok");
        }
        CK(cudaFree(dimg));
    }
    return 0;
}
