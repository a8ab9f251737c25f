// Probe of cp.async.bulk.tensor.2d ... tile::gather4 (sm_100a) for per-lane input staging:
// which tensor-map shapes the driver accepts (overlapping rows: row pitch < row length; box
// height 1 -- height 4 is an illegal instruction --; swizzle modes) and where the four gathered rows land in shared memory.
// Prints one JSON line per variant.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap tmap, uint32_t *out, int c, int r0, int r1, int r2, int r3,
                      uint32_t bytes) {
    extern __shared__ __align__(1024) uint8_t buf[];
    __shared__ uint64_t bar;
    const uint32_t bs = (uint32_t)__cvta_generic_to_shared(buf), ms = (uint32_t)__cvta_generic_to_shared(&bar);
    for (uint32_t i = threadIdx.x; i < 2048 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(buf)[i] = 0xEEEEEEEEu;
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"(ms));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(ms), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
                     :: "r"(bs), "l"(&tmap), "r"(c), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(ms) : "memory");
    }
    __syncthreads();
    uint32_t done = 0, spins = 0;
    while (!done && spins++ < 2000000)
        asm volatile("{ .reg .pred P; mbarrier.try_wait.parity.shared.b64 P, [%1], %2; selp.u32 %0, 1, 0, P; }"
                     : "=r"(done) : "r"(ms), "r"(0) : "memory");
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < 2048 / 4; i += blockDim.x) out[i] = reinterpret_cast<uint32_t *>(buf)[i];
    if (threadIdx.x == 0) out[512] = done;
}

int main() {
    const size_t n = 1 << 20;
    std::vector<uint8_t> h(n);
    // byte at offset o: a value that identifies the 16-byte block (o / 16) and the position
    for (size_t o = 0; o < n; o++) h[o] = (uint8_t)(((o / 16) * 7 + (o % 16)) & 0xFF);
    uint8_t *d;
    cudaMalloc(&d, n);
    cudaMemcpy(d, h.data(), n, cudaMemcpyHostToDevice);
    uint32_t *dout;
    cudaMalloc(&dout, 4 * 520);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 4096);
    struct V { const char *name; uint32_t W, pitch, boxh; CUtensorMapSwizzle sw; };
    const V vs[] = {
        {"w128_pitch128_box1", 128, 128, 1, CU_TENSOR_MAP_SWIZZLE_NONE},
        {"w128_pitch32_box1_overlap", 128, 32, 1, CU_TENSOR_MAP_SWIZZLE_NONE},
        {"w64_pitch32_box1_overlap", 64, 32, 1, CU_TENSOR_MAP_SWIZZLE_NONE},
        {"w32_pitch32_box1", 32, 32, 1, CU_TENSOR_MAP_SWIZZLE_NONE},
        {"w64_pitch16_box1_overlap", 64, 16, 1, CU_TENSOR_MAP_SWIZZLE_NONE},
        {"w128_pitch32_box1_overlap_sw128", 128, 32, 1, CU_TENSOR_MAP_SWIZZLE_128B},
        {"w64_pitch32_box1_overlap_sw64", 64, 32, 1, CU_TENSOR_MAP_SWIZZLE_64B},
        {"w32_pitch32_box1_sw32", 32, 32, 1, CU_TENSOR_MAP_SWIZZLE_32B},
    };
    for (const V &v : vs) {
        CUtensorMap tm;
        const cuuint64_t dims[2] = {v.W, (cuuint64_t)((n - v.W) / v.pitch)};
        const cuuint64_t strides[1] = {v.pitch};
        const cuuint32_t box[2] = {v.W, v.boxh}, estr[2] = {1, 1};
        CUresult cr = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, d, dims, strides, box, estr,
                                             CU_TENSOR_MAP_INTERLEAVE_NONE, v.sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                                             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (cr != CUDA_SUCCESS) { printf("{\"variant\": \"%s\", \"encode_error\": %d}\n", v.name, (int)cr); continue; }
        const int rows[4] = {5, 1000, 77, 3001};
        probe<<<1, 128, 4096>>>(tm, dout, 0, rows[0], rows[1], rows[2], rows[3], 4 * v.W);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("{\"variant\": \"%s\", \"launch_error\": \"%s\"}\n", v.name, cudaGetErrorString(e)); return 1; }
        std::vector<uint32_t> o(520);
        cudaMemcpy(o.data(), dout, 4 * 520, cudaMemcpyDeviceToHost);
        const uint8_t *ob = reinterpret_cast<const uint8_t *>(o.data());
        // where did each row's 16-byte blocks land?  (block b of row r = source offset r*pitch + 16 b)
        printf("{\"variant\": \"%s\", \"done\": %u, \"landing\": [", v.name, o[512]);
        for (int q = 0; q < 4; q++)
            for (uint32_t b = 0; b < v.W / 16; b++) {
                const size_t src = (size_t)rows[q] * v.pitch + 16 * b;
                int at = -1;
                for (uint32_t s = 0; s + 16 <= 2048; s += 16) {
                    bool eq = true;
                    for (int k = 0; k < 16; k++) eq &= ob[s + k] == h[src + k];
                    if (eq) { at = (int)s; break; }
                }
                printf("%s%d", (q || b) ? ", " : "", at);
            }
        printf("]}\n");
    }
    return 0;
}
