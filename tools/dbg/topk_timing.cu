// Debug harness: per-phase clock64 totals of topk.cu's tk_cqr (build with -DTCB_TOPK_TIMING).
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>
#include "../../paper_2107_01384_b200/csrc/kernels.cuh"
namespace tcb {
void topk_phase_read(unsigned long long* out);
std::atomic<u64>& launch_counter() { static std::atomic<u64> c{0}; return c; }
bool prof_enabled() { return false; }
void stream_sync(cudaStream_t s) { cudaStreamSynchronize(s); }
ProfScope::ProfScope(Cat c, cudaStream_t s) : cat(c), st(s) {}
ProfScope::~ProfScope() {}
}
int main(int argc, char** argv) {
    const int n = argc > 1 ? atoi(argv[1]) : 256, k = 14;
    std::vector<double> a(n * k), g(n * n, 0.0);
    std::mt19937_64 rng(1);
    std::normal_distribution<double> nd;
    for (int i = 0; i < n * k; ++i) a[i] = nd(rng) * std::pow(0.3, i % k);
    for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) { double s = (i == j) * 1e-9; for (int q = 0; q < k; ++q) s += a[i * k + q] * a[j * k + q]; g[i * n + j] = s; }
    cudaStream_t s; cudaStreamCreate(&s);
    tcb::DevBuf<double> G(n * n, s), X(n * 32, s); G.upload(g.data(), n * n);
    std::vector<double> th, res; double tr;
    for (int it = 0; it < 2; ++it) tcb::topk_eig(G.p, n, 32, 2, X.p, th, res, tr, s);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0, s); tcb::topk_eig(G.p, n, 32, 2, X.p, th, res, tr, s); cudaEventRecord(e1, s); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long ph[32]; tcb::topk_phase_read(ph);
    printf("topk_eig n=%d: %.3f ms; theta0 %.3e res0 %.1e trace %.3e\n", n, ms, th[0], res[0], tr);
    const char* nm[7] = {"cqr load+fro", "cqr gram", "cqr chol+inv", "cqr apply", "rr load+H", "rr jacobi", "rr X+res"};
    for (int i = 0; i < 7; ++i) printf("  %-10s %llu cycles (all launches, 3 passes each)\n", nm[i], ph[i]);
    if (ph[7]) printf("  jacobi sweeps per rr launch: %.2f\n", double(ph[8]) / double(ph[7]));
    const char* cn[12] = {"cl load", "cl gq", "cl gram", "cl sync", "cl reduce", "cl chol", "cl apply", "cl gather", "cl gsync", "cl rr pre", "cl jacobi", "cl tail"};
    for (int i = 0; i < 12; ++i) if (ph[16 + i]) printf("  %-10s %llu cycles (3 calls)\n", cn[i], ph[16 + i]);
}
