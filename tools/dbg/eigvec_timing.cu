// Debug harness: eig_values vs eig_vectors(r) wall time for an n x n Gram with a
// c3-like spectrum (a few dozen strong directions over a wide noise floor).
#include <chrono>
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>
#include "../../paper_2107_01384_b200/csrc/kernels.cuh"
namespace tcb {
std::atomic<u64>& launch_counter() { static std::atomic<u64> c{0}; return c; }
bool prof_enabled() { return false; }
void stream_sync(cudaStream_t s) { cudaStreamSynchronize(s); }
ProfScope::ProfScope(Cat c, cudaStream_t s) : cat(c), st(s) {}
ProfScope::~ProfScope() {}
}
int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 500, r = argc > 2 ? atoi(argv[2]) : 480, k = 4 * n;
    std::vector<double> b(static_cast<size_t>(n) * k), g(static_cast<size_t>(n) * n, 0.0);
    std::mt19937_64 rng(1);
    std::normal_distribution<double> nd;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < k; ++j) b[static_cast<size_t>(i) * k + j] = nd(rng) * (j < 32 ? 1.0 : 1e-4);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) {
            double s = 0;
            for (int q = 0; q < k; ++q) s += b[static_cast<size_t>(i) * k + q] * b[static_cast<size_t>(j) * k + q];
            g[static_cast<size_t>(i) * n + j] = g[static_cast<size_t>(j) * n + i] = s;
        }
    cudaStream_t s;
    cudaStreamCreate(&s);
    tcb::DevBuf<double> G(static_cast<size_t>(n) * n, s), U(static_cast<size_t>(n) * r, s);
    G.upload(g.data(), g.size());
    auto now = [] { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    for (int it = 0; it < 3; ++it) {
        tcb::EigWork w;
        const double t0 = now();
        auto ev = tcb::eig_values(G.p, n, w, s);
        cudaStreamSynchronize(s);
        const double t1 = now();
        tcb::eig_vectors(w, r, U.p, s);
        cudaStreamSynchronize(s);
        const double t2 = now();
        printf("n=%d r=%d: eig_values %.2f ms, eig_vectors %.2f ms\n", n, r, t1 - t0, t2 - t1);
    }
}
