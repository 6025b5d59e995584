// Debug microbenchmark: cycles of topk.cu's device building blocks in isolation
// (elimination-form Cholesky with inverse, the DMMA apply, the Jacobi sweeps).
#include "../../paper_2107_01384_b200/csrc/topk.cu"
namespace tcb {
std::atomic<u64>& launch_counter() { static std::atomic<u64> c{0}; return c; }
bool prof_enabled() { return false; }
void stream_sync(cudaStream_t s) { cudaStreamSynchronize(s); }
ProfScope::ProfScope(Cat c, cudaStream_t s) : cat(c), st(s) {}
ProfScope::~ProfScope() {}
__global__ void chol_apply_bench(long long* cyc, double* sink, int pp, int n) {
    extern __shared__ double smx[];
    const int ld = ((n + 15) & ~15) + 4;
    double* C = smx; double* E = C + 32 * kS; double* rinv = E + 32 * kS; double* Zt = rinv + 64;
    __shared__ int bad;
    long long tc = 0, ta = 0;
    bool b = false;
    for (int rep = 0; rep < 10; ++rep) {
        for (int e = threadIdx.x; e < 32 * kS; e += blockDim.x) {
            const int i = e / kS, j = e % kS;
            C[e] = (i == j ? 40.0 : 0.0) + 1.0 / (1.0 + i + j);
        }
        for (int e = threadIdx.x; e < 32 * ld; e += blockDim.x) Zt[e] = 1e-3 * (e % 17);
        __syncthreads();
        long long t0 = clock64();
        b |= tk_chol_inv(C, E, rinv, pp, &bad);
        long long t1 = clock64();
        tk_apply_inv(Zt, ld, (n + 7) & ~7, E, rinv);
        __syncthreads();
        long long t2 = clock64();
        tc += t1 - t0; ta += t2 - t1;
    }
    if (threadIdx.x == 0) { cyc[0] = tc / 10; cyc[1] = ta / 10; sink[0] = E[5] + rinv[3] + b + Zt[77]; }
}
__global__ void jac_bench(long long* cyc, double* sink, int reps) {
    __shared__ double H[32 * kS], Hb[32 * kS], Y[32 * kS], red[32];
    long long tot = 0;
    int sw = 0;
    for (int rep = 0; rep < reps; ++rep) {
        for (int e = threadIdx.x; e < 32 * kS; e += blockDim.x) {
            const int i = e / kS, j = e % kS;
            H[e] = i == j ? 100.0 / (1 + i) : 1e-3 / (1.0 + ((i * 7 + j * 7) % 13));
            Y[e] = i == j ? 1.0 : 0.0;
        }
        __syncthreads();
        long long t0 = clock64();
        sw += tk_jacobi(H, Hb, Y, 32, red);
        long long t1 = clock64();
        tot += t1 - t0;
    }
    if (threadIdx.x == 0) { cyc[0] = tot / reps; cyc[1] = sw / reps; sink[0] = H[5] + Y[3]; }
}
}  // namespace tcb
int main() {
    long long* c; double* s; cudaMalloc(&c, 64); cudaMalloc(&s, 64);
    long long h[2];
    const int n = 256, smem = (64 * tcb::kS + 64 + 32 * (n + 20)) * 8;
    cudaFuncSetAttribute(tcb::chol_apply_bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    tcb::chol_apply_bench<<<1, 256, smem>>>(c, s, 32, n); cudaDeviceSynchronize();
    cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    printf("tk_chol_inv %lld cycles, tk_apply_inv (n=%d) %lld cycles (%s)\n", h[0], n, h[1],
           cudaGetErrorString(cudaGetLastError()));
    tcb::jac_bench<<<1, 256>>>(c, s, 10); cudaDeviceSynchronize();
    cudaMemcpy(h, c, 16, cudaMemcpyDeviceToHost);
    printf("tk_jacobi %lld cycles, %lld sweeps\n", h[0], h[1]);
}
