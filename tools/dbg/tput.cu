// Debug microbenchmark: single-warp issue throughput of shuffles and broadcast shared loads.
#include <cstdio>
__global__ void tput(long long* cyc, double* out) {
    __shared__ __align__(16) double sm[256];
    const int lane = threadIdx.x;
    for (int i = lane; i < 256; i += 32) sm[i] = i * 0.5;
    __syncwarp();
    double x = lane, acc[8] = {};
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < 100; ++it) {
#pragma unroll
        for (int u = 0; u < 32; ++u) acc[u & 7] += __shfl_sync(0xffffffffu, x, u);
        x += 1.0;
    }
    long long t1 = clock64();
    cyc[0] = t1 - t0;
    t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < 100; ++it) {
#pragma unroll
        for (int u = 0; u < 32; ++u) acc[u & 7] += sm[(u + it) & 255];
    }
    t1 = clock64();
    cyc[1] = t1 - t0;
    t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < 100; ++it) {
#pragma unroll
        for (int u = 0; u < 32; u += 2) {
            const double2 v = *reinterpret_cast<const double2*>(sm + ((2 * it + u) & 254));
            acc[u & 7] += v.x;
            acc[(u + 1) & 7] += v.y;
        }
    }
    t1 = clock64();
    cyc[2] = t1 - t0;
    double s = 0;
    for (int u = 0; u < 8; ++u) s += acc[u];
    out[lane] = s + x;
}
int main() {
    long long* c; double* o; cudaMalloc(&c, 64); cudaMalloc(&o, 4096);
    tput<<<1, 32>>>(c, o); cudaDeviceSynchronize();
    tput<<<1, 32>>>(c, o);
    long long h[3]; cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("shfl64 (32 per iter): %.2f cycles per shfl64\n", h[0] / 3200.0);
    printf("LDS.64 broadcast:     %.2f cycles per load\n", h[1] / 3200.0);
    printf("LDS.128 broadcast:    %.2f cycles per 2 doubles\n", h[2] / 1600.0);
}
