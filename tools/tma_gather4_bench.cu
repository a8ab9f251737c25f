// Input staging by TMA gather4 (cp.async.bulk.tensor.2d ... tile::gather4, sm_100a) against the
// production path's 32-byte register loads, on the match step alone (ident_u8 layout, 64
// states, one lane per thread, thread t streams bytes [t per, (t+1) per)).
// gather4 variant: the input is a 2-D tensor of overlapping rows (row r = bytes [32 r, 32 r + W)),
// so any 32-byte aligned address is a row; per warp and stage eight ops fetch four lanes' rows
// each (W bytes per lane) into the warp's ring; one mbarrier per (warp, stage); the matching
// swizzle mode makes every lane's 16-byte reads conflict-free.  No CTA-wide synchronisation.
// Prints one JSON line per variant.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("{\"error\": \"%s line %d\"}\n", cudaGetErrorString(e_), __LINE__); return 1; } } while (0)

__device__ __forceinline__ uint32_t lds_u8(uint32_t a) { uint32_t r; asm volatile("ld.shared.u8 %0, [%1];" : "=r"(r) : "r"(a)); return r; }

// TAB 0: ident_u8 (64 states, state register holds s + table >> 8); TAB 1: packed9 (512 states,
// rows of 87 words, three 9-bit entries per word; the Worst layout), tb = table's shared address
template <int TAB>
__device__ __forceinline__ uint32_t step16(uint32_t s, uint4 q, uint32_t tb) {
    const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
    for (int wq = 0; wq < 4; wq++)
#pragma unroll
        for (int kk = 0; kk < 4; kk++) {
            if (TAB == 0) s = lds_u8(__byte_perm(w4[wq], s, 0x6540 + kk));
            else if (TAB == 2) {
                // rep8_u8: copy g = lane % 8 in banks 4g..4g+3; state register holds s + table >> 11
                const uint32_t x = w4[wq], g4 = ((threadIdx.x & 7u) << 4) * 0x01010101u;
                const uint32_t y = (x & 0x0F0F0F0Fu) | ((x & 0x10101010u) << 3) | g4, z = (x >> 5) & 0x07070707u;
                uint32_t sel;
                asm("prmt.b32 %0, %1, %2, %3;" : "=r"(sel) : "r"(y), "r"(z), "r"(0xCC00u | ((4u + kk) << 4) | (uint32_t)kk));
                s = lds_u8((s << 11) + sel);
            } else {
                const uint32_t c = (w4[wq] >> (8 * kk)) & 0xFFu, wc = (c * 171u) >> 9;
                uint32_t v;
                asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(s * 348u + tb + 4u * wc));
                s = (v >> ((c - 3u * wc) * 9u)) & 511u;
            }
        }
    return s;
}

template <int TAB>
__device__ __forceinline__ uint32_t load_table(uint8_t *sm, const uint8_t *img, uint32_t img_bytes) {
    const uint32_t sb = (uint32_t)__cvta_generic_to_shared(sm);
    const uint32_t base = TAB == 2 ? (sb + 2047) & ~2047u : (sb + 255) & ~255u;
    uint8_t *tab = sm + (base - sb);
    const uint32_t bias4 = TAB == 0 ? (base >> 8) * 0x01010101u : TAB == 2 ? (base >> 11) * 0x01010101u : 0u;
    for (uint32_t i = threadIdx.x; i < img_bytes / 16; i += blockDim.x) {
        uint4 v = reinterpret_cast<const uint4 *>(img)[i];
        v.x = __vadd4(v.x, bias4); v.y = __vadd4(v.y, bias4); v.z = __vadd4(v.z, bias4); v.w = __vadd4(v.w, bias4);
        reinterpret_cast<uint4 *>(tab)[i] = v;
    }
    return base;
}

// baseline: 32-byte loads, double-buffered in registers
template <int TAB>
__global__ void __launch_bounds__(1024, 1) gather_ldg(const uint8_t *img, uint32_t img_bytes, uint32_t pad, const uint8_t *in,
                                                      uint64_t per, uint32_t *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t base = load_table<TAB>(sm, img, img_bytes);
    __syncthreads();
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint8_t *p = in + tid * per;
    uint32_t s = TAB == 0 ? base >> 8 : TAB == 2 ? base >> 11 : 0u;
    uint4 lo, hi;
    asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(lo.x), "=r"(lo.y), "=r"(lo.z), "=r"(lo.w), "=r"(hi.x), "=r"(hi.y), "=r"(hi.z), "=r"(hi.w) : "l"(p));
    for (uint64_t bi = 0; bi < per / 32; bi++) {
        uint4 nlo = lo, nhi = hi;
        if (bi + 1 < per / 32)
            asm volatile("ld.global.nc.v8.u32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];" : "=r"(nlo.x), "=r"(nlo.y), "=r"(nlo.z), "=r"(nlo.w), "=r"(nhi.x), "=r"(nhi.y), "=r"(nhi.z), "=r"(nhi.w) : "l"(p + 32 * (bi + 1)));
        s = step16<TAB>(s, lo, base);
        s = step16<TAB>(s, hi, base);
        lo = nlo; hi = nhi;
    }
    out[tid] = s - (TAB == 0 ? base >> 8 : TAB == 2 ? base >> 11 : 0u);
}

// W bytes per lane and stage, S stages, swizzle SW (0 none, else matching W: 32/64/128)
template <int W, int S, int SW, int TAB>
__global__ void __launch_bounds__(1024, 1) gather_g4(const __grid_constant__ CUtensorMap tmap, const uint8_t *img,
                                                     uint32_t img_bytes, uint32_t pad, uint64_t per, uint32_t *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    const uint32_t base = load_table<TAB>(sm, img, img_bytes);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    // [table + pad][rings: warp x S x (32 rows x W)], 1 KB aligned; [barriers]
    const uint32_t ring0 = (base + img_bytes + pad + 1023u) & ~1023u;
    const uint32_t ring = ring0 + warp * (S * 32 * W);
    const uint32_t bars = ring0 + nw * (S * 32 * W) + warp * (S * 8);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < S; k++) asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(bars + 8 * k));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    __syncthreads();
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t row0 = (uint32_t)(tid * per / 32);        // this lane's first row (32-byte pitch)
    // issuing lane q < 8 fetches the rows of lanes 4q .. 4q+3
    uint32_t r[4];
#pragma unroll
    for (int j = 0; j < 4; j++) r[j] = __shfl_sync(0xffffffffu, row0, 4 * (lane & 7) + j);
    const uint64_t nblk = per / W;
    auto issue = [&](uint64_t bi, int k) {
        if (lane == 0) asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(bars + 8 * k), "r"(32 * W) : "memory");
        __syncwarp();
        if (lane < 8) {
            const uint32_t adv = (uint32_t)bi * (W / 32);
            asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                         :: "r"(ring + k * 32 * W + lane * 4 * W), "l"(&tmap), "r"(0), "r"(r[0] + adv), "r"(r[1] + adv),
                            "r"(r[2] + adv), "r"(r[3] + adv), "r"(bars + 8 * k) : "memory");
        }
    };
    for (int k = 0; k < S; k++) if ((uint64_t)k < nblk) issue(k, k);
    uint32_t s = TAB == 0 ? base >> 8 : TAB == 2 ? base >> 11 : 0u;
    // swizzle: the 16-byte chunk index is XORed with address bits 7.. (128B: 3 bits, 64B: 2, 32B: 1)
    const uint32_t rowoff = lane * W;
    for (uint64_t bi = 0; bi < nblk; bi++) {
        const int k = (int)(bi % S);
        const uint32_t par = (uint32_t)((bi / S) & 1);
        uint32_t done = 0;
        while (!done)
            asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                         : "=r"(done) : "r"(bars + 8 * k), "r"(par) : "memory");
        uint4 q[W / 16];
        const uint32_t rb = ring + k * 32 * W + rowoff;
#pragma unroll
        for (int j = 0; j < W / 16; j++) {
            uint32_t a = rb + 16 * j;
            if (SW == 128) a ^= ((a >> 7) & 7u) << 4;
            if (SW == 64) a ^= ((a >> 7) & 3u) << 4;
            if (SW == 32) a ^= ((a >> 7) & 1u) << 4;
            asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(q[j].x), "=r"(q[j].y), "=r"(q[j].z), "=r"(q[j].w) : "r"(a));
        }
        __syncwarp();
        if (bi + S < nblk) issue(bi + S, k);
#pragma unroll
        for (int j = 0; j < W / 16; j++) s = step16<TAB>(s, q[j], base);
    }
    out[tid] = s - (TAB == 0 ? base >> 8 : TAB == 2 ? base >> 11 : 0u);
}

static uint64_t rng = 88172645463325252ull;
static uint32_t nxt() { rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17; return (uint32_t)rng; }

template <int W, int S, int SW, int TAB>
int run_g4(const char *name, int threads, uint32_t pad, const uint8_t *dimg, uint32_t bytes, uint8_t *din, uint64_t n, int sms,
           uint32_t *dout, const std::vector<uint8_t> &hin, const std::vector<uint8_t> &delta, const std::vector<uint16_t> &d9) {
    const int grid = sms;
    const uint64_t per = (n / ((uint64_t)grid * threads)) & ~(uint64_t)(W - 1);
    const size_t smem = 2048 + bytes + pad + 1024 + (size_t)(threads / 32) * S * 32 * W + (threads / 32) * S * 8 + 64;
    if (smem > 232448) { printf("{\"g4\": \"%s\", \"W\": %d, \"S\": %d, \"threads\": %d, \"pad\": %u, \"skip\": \"smem %zu\"}\n", name, W, S, threads, pad, smem); return 0; }
    CUtensorMap tm;
    const cuuint64_t dims[2] = {(cuuint64_t)W, (cuuint64_t)((n - W) / 32 + 1)};
    const cuuint64_t strides[1] = {32};
    const cuuint32_t box[2] = {(cuuint32_t)W, 1}, estr[2] = {1, 1};
    CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, din, dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                                         SW == 128 ? CU_TENSOR_MAP_SWIZZLE_128B : SW == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : SW == 32 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) { printf("{\"g4\": \"%s\", \"error\": \"encode %d\"}\n", name, (int)cr); return 0; }
    CK(cudaFuncSetAttribute(gather_g4<W, S, SW, TAB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
    gather_g4<W, S, SW, TAB><<<grid, threads, smem>>>(tm, dimg, bytes, pad, per, dout);
    CK(cudaDeviceSynchronize());
    std::vector<uint32_t> got((size_t)grid * threads);
    CK(cudaMemcpy(got.data(), dout, got.size() * 4, cudaMemcpyDeviceToHost));
    int bad = 0;
    for (uint32_t t : {0u, 777u, (uint32_t)(grid * threads - 1)}) {
        uint32_t hs = 0;
        for (uint64_t i = 0; i < per; i++) hs = TAB != 1 ? delta[hs * 256 + hin[t * per + i]] : d9[hs * 256 + hin[t * per + i]];
        bad += got[t] != hs;
    }
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    for (int r = 0; r < 20; r++) gather_g4<W, S, SW, TAB><<<grid, threads, smem>>>(tm, dimg, bytes, pad, per, dout);
    cudaEventRecord(b);
    CK(cudaEventSynchronize(b));
    float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
    const double bd = (double)per * grid * threads;
    printf("{\"g4\": \"%s\", \"W\": %d, \"S\": %d, \"swizzle\": %d, \"threads\": %d, \"pad\": %u, \"ms\": %.4f, \"GBps\": %.1f, \"check\": \"%s\"}\n",
           name, W, S, SW, threads, pad, ms, bd / ms / 1e6, bad ? "FAIL" : "ok");
    return 0;
}

int main(int argc, char **argv) {
    const uint64_t n = (uint64_t)(argc > 1 ? atoi(argv[1]) : 1024) << 20;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    std::vector<uint8_t> hin(n);
    for (uint64_t i = 0; i < n; i += 4) { uint32_t v = nxt(); memcpy(&hin[i], &v, 4); }
    uint8_t *din; uint32_t *dout;
    CK(cudaMalloc(&din, n + 4096));
    CK(cudaMemcpy(din, hin.data(), n, cudaMemcpyHostToDevice));
    CK(cudaMalloc(&dout, 4u << 20));
    const int nq = 64;
    std::vector<uint8_t> delta(nq * 256);
    for (auto &d : delta) d = nxt() % nq;
    const uint32_t bytes = nq * 256;
    uint8_t *dimg; CK(cudaMalloc(&dimg, bytes));
    CK(cudaMemcpy(dimg, delta.data(), bytes, cudaMemcpyHostToDevice));
    // packed9: 512 states, rows of 87 words
    std::vector<uint16_t> d9(512 * 256);
    for (auto &d : d9) d = nxt() % 512;
    std::vector<uint32_t> img9(512 * 87, 0);
    for (int st = 0; st < 512; st++) for (int c = 0; c < 256; c++) img9[st * 87 + c / 3] |= (uint32_t)d9[st * 256 + c] << (9 * (c % 3));
    const uint32_t bytes9 = 512 * 87 * 4;
    uint8_t *dimg9; CK(cudaMalloc(&dimg9, bytes9));
    CK(cudaMemcpy(dimg9, img9.data(), bytes9, cudaMemcpyHostToDevice));
    for (int threads : {640, 704}) {
        const int grid = sms;
        const uint64_t per = (n / ((uint64_t)grid * threads)) & ~31ull;
        CK(cudaFuncSetAttribute(gather_ldg<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
        const size_t smem = 256 + bytes9 + 64;
        gather_ldg<1><<<grid, threads, smem>>>(dimg9, bytes9, 0, din, per, dout);
        CK(cudaDeviceSynchronize());
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int r = 0; r < 20; r++) gather_ldg<1><<<grid, threads, smem>>>(dimg9, bytes9, 0, din, per, dout);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
        printf("{\"ldg32\": 1, \"table\": \"packed9\", \"threads\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", threads, ms, (double)per * grid * threads / ms / 1e6);
    }
#define RUN9(W, S, SW, T) if (run_g4<W, S, SW, 1>("packed9", T, 0, dimg9, bytes9, din, n, sms, dout, hin, delta, d9)) return 1;
    RUN9(32, 2, 32, 640) RUN9(32, 2, 32, 704) RUN9(32, 3, 32, 512) RUN9(64, 2, 64, 384)
    // rep8_u8 (Random's layout): 64 states x 2 KB
    {
        const uint32_t bytes8 = nq * 2048;
        std::vector<uint8_t> img8(bytes8, 0);
        for (int g = 0; g < 8; g++) for (int st = 0; st < nq; st++) for (int b = 0; b < 256; b++)
            img8[(st << 11) | (((b >> 5) & 7) << 8) | (((b >> 4) & 1) << 7) | (g << 4) | (b & 15)] = delta[st * 256 + b];
        uint8_t *dimg8; CK(cudaMalloc(&dimg8, bytes8));
        CK(cudaMemcpy(dimg8, img8.data(), bytes8, cudaMemcpyHostToDevice));
        for (int threads : {640, 1024}) {
            const int grid = sms;
            const uint64_t per = (n / ((uint64_t)grid * threads)) & ~31ull;
            CK(cudaFuncSetAttribute(gather_ldg<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
            const size_t smem = 2048 + bytes8 + 64;
            gather_ldg<2><<<grid, threads, smem>>>(dimg8, bytes8, 0, din, per, dout);
            CK(cudaDeviceSynchronize());
            cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
            cudaEventRecord(a);
            for (int r = 0; r < 20; r++) gather_ldg<2><<<grid, threads, smem>>>(dimg8, bytes8, 0, din, per, dout);
            cudaEventRecord(b);
            CK(cudaEventSynchronize(b));
            float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
            printf("{\"ldg32\": 1, \"table\": \"rep8_u8\", \"threads\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", threads, ms, (double)per * grid * threads / ms / 1e6);
        }
#define RUN8(W, S, SW, T) if (run_g4<W, S, SW, 2>("rep8_u8", T, 0, dimg8, bytes8, din, n, sms, dout, hin, delta, d9)) return 1;
        RUN8(64, 2, 64, 640) RUN8(32, 2, 32, 640) RUN8(32, 4, 32, 640) RUN8(32, 2, 32, 1024)
    }
    for (int threads : {1024, 640}) {
        const int grid = sms;
        const uint64_t per = (n / ((uint64_t)grid * threads)) & ~31ull;
        CK(cudaFuncSetAttribute(gather_ldg<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448));
        const size_t smem = 256 + bytes + 64;
        gather_ldg<0><<<grid, threads, smem>>>(dimg, bytes, 0, din, per, dout);
        CK(cudaDeviceSynchronize());
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        cudaEventRecord(a);
        for (int r = 0; r < 20; r++) gather_ldg<0><<<grid, threads, smem>>>(dimg, bytes, 0, din, per, dout);
        cudaEventRecord(b);
        CK(cudaEventSynchronize(b));
        float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
        printf("{\"ldg32\": 1, \"threads\": %d, \"ms\": %.4f, \"GBps\": %.1f}\n", threads, ms, (double)per * grid * threads / ms / 1e6);
    }
#define RUN(W, S, SW, T, PAD) if (run_g4<W, S, SW, 0>("ident_u8", T, PAD, dimg, bytes, din, n, sms, dout, hin, delta, d9)) return 1;
    RUN(32, 2, 32, 1024, 0) RUN(32, 4, 32, 1024, 0) RUN(32, 4, 0, 1024, 0)
    RUN(64, 2, 64, 1024, 0) RUN(64, 3, 64, 1024, 0) RUN(64, 2, 0, 1024, 0)
    RUN(128, 2, 128, 640, 0) RUN(64, 2, 64, 640, 0) RUN(64, 4, 64, 640, 0) RUN(32, 2, 32, 640, 0) RUN(32, 4, 32, 640, 0)
    return 0;
}
