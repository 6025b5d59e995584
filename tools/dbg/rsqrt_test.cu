// Debug: accuracy of rsqrt.approx.ftz.f64 and of one cubic refinement step.
#include <cstdio>
#include <cmath>
__device__ __forceinline__ double rsqrt_approx(double x) {
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
    return y;
}
__device__ __forceinline__ double rsqrt_fast(double x) {
    const double y = rsqrt_approx(x);
    const double e = fma(-x * y, y, 1.0);
    return fma(y * e, fma(0.375, e, 0.5), y);
}
__global__ void k(double* out, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double x = 0.25 + 7.75 * (i + 0.5) / n;
    double r = rsqrt(x), a = rsqrt_approx(x), f = rsqrt_fast(x);
    out[3 * i] = a; out[3 * i + 1] = f; out[3 * i + 2] = r;
}
int main() {
    const int n = 1 << 20;
    double* d; cudaMalloc(&d, 3 * n * 8);
    k<<<n / 256, 256>>>(d, n);
    double* h = new double[3 * n];
    cudaMemcpy(h, d, 3 * n * 8, cudaMemcpyDeviceToHost);
    double ea = 0, ef = 0, er = 0;
    for (int i = 0; i < n; ++i) {
        double x = 0.25 + 7.75 * (i + 0.5) / n;
        long double t = 1.0L / sqrtl((long double)x);
        ea = fmax(ea, (double)fabsl((h[3*i] - t) / t));
        ef = fmax(ef, (double)fabsl((h[3*i+1] - t) / t));
        er = fmax(er, (double)fabsl((h[3*i+2] - t) / t));
    }
    printf("approx rel err %.3e, approx+cubic %.3e, rsqrt() %.3e (ulp %.3e)\n", ea, ef, er, 1.1102230246251565e-16);
}
