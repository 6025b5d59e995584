// Microbenchmark: per-step cost of an all-to-all st.async exchange in a
// thread-block cluster (each CTA pushes `per` 16-byte values to every CTA and
// waits on its mbarrier), optionally with two __syncthreads per step.
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;
__device__ unsigned long long g_cyc[64];
__device__ __forceinline__ unsigned smem_addr(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__global__ void ping(int steps, int per, int syncs) {
    cg::cluster_group cl = cg::this_cluster();
    const unsigned C = cl.num_blocks(), rank = cl.block_rank();
    __shared__ __align__(16) double buf[2][16 * 64 * 2];
    __shared__ __align__(8) unsigned long long mbar[2];
    if (threadIdx.x == 0) {
        for (int b = 0; b < 2; ++b) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&mbar[b])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    cl.sync();
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const unsigned dst = lane % C;
    unsigned rb[2], rbar[2];
    for (int b = 0; b < 2; ++b) {
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb[b]) : "r"(smem_addr(&buf[b][0])), "r"(dst));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rbar[b]) : "r"(smem_addr(&mbar[b])), "r"(dst));
    }
    long long t0 = clock64();
    for (int k = 0; k < steps; ++k) {
        const int b = k & 1;
        if (threadIdx.x == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&mbar[b])), "r"(16u * per * C) : "memory");
        // warp w pushes values w, w+nw, ... (< per) to every dst
        if (lane < C)
            for (int v = warp; v < per; v += nw) {
                const unsigned off = (rank * per + v) * 16;
                asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(rb[b] + off),
                             "l"((long long)k), "l"((long long)v), "r"(rbar[b]) : "memory");
            }
        if (syncs) __syncthreads();
        asm volatile("{\n\t.reg .pred P;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n}" ::"r"(smem_addr(&mbar[b])), "r"((k >> 1) & 1) : "memory");
        if (syncs) __syncthreads();
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) g_cyc[rank] = (t1 - t0) / steps;
    cl.sync();
}
int main() {
    cudaFuncSetAttribute(ping, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int C : {16, 8, 4, 2}) for (int thr : {256, 512}) for (int per : {1, 16, 32}) for (int sy : {0, 1}) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(C); cfg.blockDim = dim3(thr);
        cudaLaunchAttribute at[1]; at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = C; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
        cfg.attrs = at; cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, ping, 2000, per, sy) != cudaSuccess) { printf("launch fail C=%d\n", C); continue; }
        cudaDeviceSynchronize();
        unsigned long long cyc[64]; cudaMemcpyFromSymbol(cyc, g_cyc, sizeof(cyc));
        printf("C=%2d threads=%d per=%2d syncs=%d : %llu cycles/step\n", C, thr, per, sy, cyc[0]);
    }
}
