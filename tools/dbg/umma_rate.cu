// tcgen05.mma kind::i8 / kind::f16 issue-rate probe: one CTA per SM issues a long
// run of MMAs on zero-filled shared-memory tiles and times them with clock64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_rate umma_rate.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int N, int SW, int KIND>  // SW: 4 = 64B, 2 = 128B swizzle; KIND 0 = i8, 1 = f16
__global__ void __launch_bounds__(128, 1) probe(long long* out, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    for (int i = threadIdx.x; i < 64 * 1024; i += blockDim.x) base[i] = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if ((threadIdx.x >> 5) == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tmem = slot;
    const int rowb = SW == 4 ? 64 : 128;
    auto desc = [&](uint32_t a) {
        uint64_t d = (a >> 4) & 0x3FFF;
        d |= 1ull << 16;
        d |= (uint64_t)((8 * rowb) >> 4) << 32;
        d |= 1ull << 46;
        d |= (uint64_t)SW << 61;
        return d;
    };
    const uint32_t idesc = KIND == 0 ? ((2u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24))
                                     : ((1u << 4) | (1u << 7) | (1u << 10) | ((N >> 3) << 17) | ((128 >> 4) << 24));
    const uint64_t da = desc(su(base)), db = desc(su(base + 32768));
    long long t0 = 0, t1 = 0;
    if (threadIdx.x == 0) {
        t0 = clock64();
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (KIND == 0)
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                                 "l"(da + 2 * (k & 1)), "l"(db + 2 * (k & 1)), "r"(idesc), "r"(1));
                else
                    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
                                 "l"(da + 2 * (k & 1)), "l"(db + 2 * (k & 1)), "r"(idesc), "r"(1));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su(&bar)));
        asm volatile("{\n.reg .pred P1;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n@P1 bra D;\nbra W;\nD:\n}" ::"r"(su(&bar)));
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if ((threadIdx.x >> 5) == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

template <int N, int SW, int KIND>
void run(const char* name) {
    const int iters = 2000, smem = 64 * 1024 + 2048;
    cudaFuncSetAttribute(probe<N, SW, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    long long* d;
    cudaMalloc(&d, 148 * sizeof(long long));
    probe<N, SW, KIND><<<148, 128, smem>>>(d, 10);
    cudaDeviceSynchronize();
    probe<N, SW, KIND><<<148, 128, smem>>>(d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = (double)h[0] / (iters * 8);
    const int K = KIND == 0 ? 32 : 16;
    double macs = 128.0 * N * K;
    printf("%-28s %s: %.1f cycles/MMA, %.0f MAC/clk/SM (%s)\n", name, KIND == 0 ? "i8 " : "f16", cyc, macs / cyc,
           cudaGetErrorString(e));
    cudaFree(d);
}

int main() {
    run<96, 4, 0>("M128 N96  K32 sw64");
    run<128, 4, 0>("M128 N128 K32 sw64");
    run<256, 4, 0>("M128 N256 K32 sw64");
    run<96, 2, 0>("M128 N96  K32 sw128");
    run<128, 2, 0>("M128 N128 K32 sw128");
    run<256, 2, 0>("M128 N256 K32 sw128");
    run<64, 2, 0>("M128 N64  K32 sw128");
    run<128, 2, 1>("M128 N128 K16 sw128 (f16)");
    run<256, 2, 1>("M128 N256 K16 sw128 (f16)");
    return 0;
}
