// Debug: pinned H2D of a 256 x 65536 fp64 tensor, contiguous vs 8 column chunks (2D copies).
#include <cstdio>
int main() {
    const size_t rows = 256, cols = 65536, n = rows * cols * 8;
    unsigned char *h, *d;
    cudaMallocHost(&h, n);
    cudaMalloc(&d, n);
    cudaStream_t s; cudaStreamCreate(&s);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int mode = 0; mode < 3; ++mode) {
        float best = 1e9;
        for (int it = 0; it < 5; ++it) {
            cudaEventRecord(a, s);
            if (mode == 0) cudaMemcpyAsync(d, h, n, cudaMemcpyHostToDevice, s);
            else {
                const int C = mode == 1 ? 8 : 32;
                for (int c = 0; c < C; ++c) {
                    const size_t k0 = cols * c / C, k1 = cols * (c + 1) / C;
                    cudaMemcpy2DAsync(d + k0 * 8, cols * 8, h + k0 * 8, cols * 8, (k1 - k0) * 8, rows, cudaMemcpyHostToDevice, s);
                }
            }
            cudaEventRecord(b, s);
            cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        printf("%s: %.3f ms (%.1f GB/s)\n", mode == 0 ? "contiguous" : mode == 1 ? "8 x 2D chunks" : "32 x 2D chunks", best, n / best / 1e6);
    }
}
