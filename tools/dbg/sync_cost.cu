// Debug microbenchmark: host round-trip costs (launch + small D2H + sync), pageable vs pinned,
// with and without stream-ordered pool allocations.
#include <chrono>
#include <cstdio>
#include <vector>
__global__ void tiny(unsigned long long* p) { if (threadIdx.x == 0) p[0] += 1; }
int main() {
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    unsigned long long* d; cudaMalloc(&d, 4096);
    unsigned long long* pin; cudaMallocHost(&pin, 4096);
    std::vector<unsigned long long> pg(512);
    cudaMemPool_t pool; cudaDeviceGetDefaultMemPool(&pool, 0);
    unsigned long long thr = ~0ull; cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    auto now = [] { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    for (int mode = 0; mode < 6; ++mode) {
        double best = 1e9, sum = 0;
        for (int it = 0; it < 200; ++it) {
            const double t0 = now();
            if (mode == 5) {
                void* q[8];
                for (int k = 0; k < 8; ++k) cudaMallocAsync(&q[k], 1 << (12 + k), s);
                tiny<<<1, 32, 0, s>>>((unsigned long long*)q[0]);
                cudaMemcpyAsync(pg.data(), q[0], 64, cudaMemcpyDeviceToHost, s);
                for (int k = 0; k < 8; ++k) cudaFreeAsync(q[k], s);
                cudaStreamSynchronize(s);
            } else if (mode == 4) {
                void* q; cudaMallocAsync(&q, 1 << 16, s);
                tiny<<<1, 32, 0, s>>>((unsigned long long*)q);
                cudaMemcpyAsync(pg.data(), q, 64, cudaMemcpyDeviceToHost, s);
                cudaFreeAsync(q, s);
                cudaStreamSynchronize(s);
            } else {
                tiny<<<1, 32, 0, s>>>(d);
                if (mode == 1) cudaMemcpyAsync(pg.data(), d, 64, cudaMemcpyDeviceToHost, s);
                if (mode == 2) cudaMemcpyAsync(pin, d, 64, cudaMemcpyDeviceToHost, s);
                if (mode == 3) cudaMemcpyAsync(d + 64, pg.data(), 64, cudaMemcpyHostToDevice, s);
                cudaStreamSynchronize(s);
            }
            const double dt = now() - t0;
            if (it >= 20) { best = dt < best ? dt : best; sum += dt; }
        }
        const char* nm[6] = {"launch+sync", "launch+D2H pageable+sync", "launch+D2H pinned+sync", "launch+H2D pageable+sync", "mallocAsync+launch+D2H+free+sync", "8x mallocAsync ... +sync"};
        printf("%-36s best %.1f us, mean %.1f us\n", nm[mode], best, sum / 180);
    }
}
