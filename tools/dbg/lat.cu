// Debug microbenchmark: single-warp dependent-chain latencies (cycles) of the
// fp64 ops the latency-bound kernels (topk Cholesky / Jacobi) are built from.
#include <cstdio>
#include <cmath>
__global__ void lat(double* out, long long* cyc, double x0, int iters) {
    double x = x0 + threadIdx.x * 1e-9;
    long long t0, t1;
    __shared__ double sm[64];
    sm[threadIdx.x] = x;
    __syncwarp();
    // DFMA chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, 0.999999, 1e-7);
    t1 = clock64(); cyc[0] = t1 - t0;
    // DADD chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = x + 1e-9;
    t1 = clock64(); cyc[1] = t1 - t0;
    // rsqrt chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = rsqrt(x) + 0.5;
    t1 = clock64(); cyc[2] = t1 - t0;
    // sqrt chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = sqrt(x) + 0.5;
    t1 = clock64(); cyc[3] = t1 - t0;
    // div chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = 1.5 / x + 0.5;
    t1 = clock64(); cyc[4] = t1 - t0;
    // shfl (64-bit) chain
    t0 = clock64();
    for (int i = 0; i < iters; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1e-9;
    t1 = clock64(); cyc[5] = t1 - t0;
    // LDS chain (dependent address)
    int idx = threadIdx.x;
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { double v = sm[idx]; idx = ((int)v & 31) ^ (i & 1); x += v; }
    t1 = clock64(); cyc[6] = t1 - t0;
    // __syncwarp + STS/LDS roundtrip
    t0 = clock64();
    for (int i = 0; i < iters; ++i) { sm[threadIdx.x] = x; __syncwarp(); x = sm[(threadIdx.x + 1) & 31] + 1e-9; }
    t1 = clock64(); cyc[7] = t1 - t0;
    out[threadIdx.x] = x;
}
__global__ void bar_lat(long long* cyc, int iters, double* out) {
    __shared__ double sm[256];
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) { sm[threadIdx.x] = x; __syncthreads(); x = sm[(threadIdx.x + 37) & 255] + 1.0; }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[8] = t1 - t0;
    out[threadIdx.x] = x;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 4096); cudaMalloc(&c, 128);
    const int it = 1000;
    lat<<<1, 32>>>(o, c, 1.3, it); cudaDeviceSynchronize();
    lat<<<1, 32>>>(o, c, 1.3, it);
    bar_lat<<<1, 256>>>(c, it, o);
    long long h[16]; cudaMemcpy(h, c, 9 * 8, cudaMemcpyDeviceToHost);
    const char* nm[9] = {"DFMA", "DADD", "rsqrt(f64)+add", "sqrt(f64)+add", "div(f64)+add", "shfl64+add", "LDS dep chain(+cvt,add)", "STS;syncwarp;LDS;+add", "STS;syncthreads(256);LDS;+add"};
    for (int i = 0; i < 9; ++i) printf("%-32s %.1f cycles/iter\n", nm[i], double(h[i]) / it);
}
