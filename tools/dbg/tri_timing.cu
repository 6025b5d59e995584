// Debug harness: per-phase clock64 totals of tridiag_dsmem (build with -DTCB_TRIDIAG_TIMING).
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>
#include "../../paper_2107_01384_b200/csrc/kernels.cuh"
namespace tcb {
void tri_phase_read(unsigned long long* out);
#ifndef TCB_TRIDIAG_TIMING
void tri_phase_read(unsigned long long*) {}
#endif
std::atomic<u64>& launch_counter() { static std::atomic<u64> c{0}; return c; }
bool prof_enabled() { return false; }
void stream_sync(cudaStream_t s) { cudaStreamSynchronize(s); }
ProfScope::ProfScope(Cat c, cudaStream_t s) : cat(c), st(s) {}
ProfScope::~ProfScope() {}
}
int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 256;
    std::vector<double> b(n * 4 * n), g(n * n, 0.0);
    std::mt19937_64 rng(1);
    std::normal_distribution<double> nd;
    for (auto& v : b) v = nd(rng);
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) { double s = 0; for (int k = 0; k < 4 * n; ++k) s += b[i * 4 * n + k] * b[j * 4 * n + k]; g[i * n + j] = s; }
    cudaStream_t s; cudaStreamCreate(&s);
    tcb::DevBuf<double> G(n * n, s); G.upload(g.data(), n * n);
    for (int it = 0; it < 3; ++it) { tcb::EigWork w; auto ev = tcb::eig_values(G.p, n, w, s); }
    cudaEvent_t a, c; cudaEventCreate(&a); cudaEventCreate(&c);
    tcb::EigWork w; cudaEventRecord(a, s); auto ev = tcb::eig_values(G.p, n, w, s); cudaEventRecord(c, s); cudaEventSynchronize(c);
    float ms; cudaEventElapsedTime(&ms, a, c);
    {
        double tr = 0, fr = 0, s1 = 0, s2 = 0;
        for (int i = 0; i < n; ++i) tr += g[i * n + i];
        for (double v : g) fr += v * v;
        for (double v : ev) { s1 += v; s2 += v * v; }
        printf("check: trace rel err %.3e  frob rel err %.3e\n", std::fabs(s1 - tr) / tr, std::fabs(s2 - fr) / fr);
    }
#ifndef TCB_TRIDIAG_TIMING
    printf("n=%d eig_values %.3f ms\n", n, ms);
    return 0;
#endif
    unsigned long long ph[160]; tcb::tri_phase_read(ph);
    const char* names[10] = {"loop-top", "alpha/t", "mv-sync", "push", "mbar-wait", "K+globals", "update", "rnext", "syncthreads", "matvec"};
    printf("n=%d eig_values %.3f ms; per-step cycles (CTA 0 / CTA 7):\n", n, ms);
    for (int i = 0; i < 10; ++i) printf("  %-12s %8.0f %8.0f\n", names[i], ph[i] / double(n - 2), ph[70 + i] / double(n - 2));
}
