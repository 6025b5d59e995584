// TMA load throughput per SM for different box shapes (L2-resident source):
// each CTA (one per SM) streams `iters` boxes through a 4-deep mbarrier ring.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_rate tma_rate.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t b, uint32_t ph) {
    asm volatile("{\n.reg .pred P1;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n@P1 bra D_%=;\nbra W_%=;\nD_%=:\n}" ::"r"(b), "r"(ph) : "memory");
}

// mode 0: 2D tensor box (bw bytes x rows), mode 1: 1D bulk copy of `bytes`
__global__ void __launch_bounds__(32, 1) tma_probe(const __grid_constant__ CUtensorMap map, const uint8_t* src,
                                                   int mode, int bw, int rows, int nx, int iters, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar[4];
    uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    const uint32_t bytes = (uint32_t)bw * rows;
    if (threadIdx.x == 0) {
        for (int i = 0; i < 4; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;");
        long long t0 = clock64();
        for (int i = 0; i < iters + 4; ++i) {
            const int st = i & 3;
            if (i >= 4) wait(su(&bar[st]), ((i >> 2) - 1) & 1);
            if (i >= iters) continue;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar[st])), "r"(bytes));
            const uint32_t dst = su(base + st * bytes);
            const int x = (blockIdx.x * 7 + i) % nx;  // spread over the (L2-resident) source
            if (mode == 0)
                asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
                             "l"((uint64_t)&map), "r"(x * bw), "r"(0), "r"(su(&bar[st])) : "memory");
            else
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                             "l"(src + (size_t)x * bytes), "r"(bytes), "r"(su(&bar[st])) : "memory");
        }
        out[blockIdx.x] = clock64() - t0;
    }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    Enc enc = (Enc)fp;
    const size_t W = 1 << 20, H = 256;  // 256 rows x 1 MiB: 256 MiB (rows up to 256)
    uint8_t* src;
    cudaMalloc(&src, W * H);
    cudaMemset(src, 1, W * H);
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    struct Cfg { int mode, bw, rows, sw; const char* name; } cfgs[] = {
        {0, 64, 128, 2, "2D 64B x 128 rows sw64"},   {0, 128, 64, 3, "2D 128B x 64 rows sw128"},
        {0, 128, 128, 3, "2D 128B x 128 rows sw128"}, {0, 64, 256, 2, "2D 64B x 256 rows sw64"},
        {1, 64, 128, 0, "1D bulk 8 KB"},              {1, 128, 128, 0, "1D bulk 16 KB"},
        {1, 256, 128, 0, "1D bulk 32 KB"}};
    for (auto& c : cfgs) {
        CUtensorMap m;
        const int nx = c.mode == 0 ? (int)(8 << 20 >> 8) / c.bw : 256;  // x extent ~ 8 MB of source per row range
        const cuuint64_t dims[2] = {W, H};
        const cuuint64_t str[1] = {W};
        const cuuint32_t box[2] = {(cuuint32_t)c.bw, (cuuint32_t)c.rows};
        const cuuint32_t es[2] = {1, 1};
        CUtensorMapSwizzle sw = c.sw == 2 ? CU_TENSOR_MAP_SWIZZLE_64B : c.sw == 3 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE;
        if (c.mode == 0)
            enc(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int bytes = c.bw * c.rows, iters = 4000, smem = 4 * bytes + 1024;
        cudaFuncSetAttribute(tma_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        tma_probe<<<148, 32, smem>>>(m, src, c.mode, c.bw, c.rows, nx, 100, d);
        cudaDeviceSynchronize();
        tma_probe<<<148, 32, smem>>>(m, src, c.mode, c.bw, c.rows, nx, iters, d);
        cudaError_t e = cudaDeviceSynchronize();
        long long h[148];
        cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
        long long mx = 0;
        for (int i = 0; i < 148; ++i) mx = h[i] > mx ? h[i] : mx;
        printf("%-26s: %.1f B/clk/SM (slowest SM), %.0f cycles per box (%s)\n", c.name, (double)bytes * iters / mx,
               (double)mx / iters, cudaGetErrorString(e));
    }
    return 0;
}
