// extern "C" boundary (include/tucomp_b200.h).  Each entry point owns one CUDA
// stream for the call, converts exceptions into status + message, and never
// falls back to host computation.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>

#include "../../include/tucomp_b200.h"
#include "exact.cuh"
#include "codec.cuh"
#include "kernels.cuh"
#include "decode.cuh"
#include "decompress.hpp"
#include "nccl_shim.hpp"
#include "pipeline.hpp"
#include "quant.cuh"

namespace tcb {
std::atomic<u64>& launch_counter() {
    static std::atomic<u64> c{0};
    return c;
}

namespace {
bool g_prof = false;
struct Rec {
    int cat;
    cudaEvent_t a, b;
};
std::vector<Rec> g_recs;
}  // namespace

bool prof_enabled() { return g_prof; }

namespace {
std::mutex g_trace_mu;
std::map<std::string, std::pair<double, u64>> g_trace;
// TCB_TIMELINE=1: every ProfScope records a (stream, start, end) event pair without
// serialising anything; dumped relative to the call's first event (debugging aid)
bool timeline_on() {
    static const bool on = [] {
        const char* e = std::getenv("TCB_TIMELINE");
        return e && *e && *e != '0';
    }();
    return on;
}
struct TlRec {
    int cat;
    cudaStream_t st;
    cudaEvent_t a, b;
};
std::vector<TlRec> g_tl;
std::mutex g_tl_mu;
bool trace_on() {
    static const bool on = [] {
        const char* e = std::getenv("TCB_TRACE");
        return e && *e && *e != '0';
    }();
    return on;
}
long long now_ns() {
    return std::chrono::duration_cast<std::chrono::nanoseconds>(
               std::chrono::steady_clock::now().time_since_epoch())
        .count();
}
}  // namespace

HostTrace::HostTrace(const char* l) : label(l) {
    if (trace_on()) t0 = now_ns();
}
void HostTrace::stop() {
    if (done || !trace_on()) return;
    done = true;
    const double ms = (now_ns() - t0) * 1e-6;
    std::lock_guard<std::mutex> lk(g_trace_mu);
    auto& e = g_trace[label];
    e.first += ms;
    e.second += 1;
}
namespace {
std::atomic<u64> g_syncs{0}, g_sync_ns{0};
}
void stream_sync(cudaStream_t s) {
    if (!trace_on()) {
        TCB_CUDA(cudaStreamSynchronize(s));
        return;
    }
    const long long t0 = now_ns();
    TCB_CUDA(cudaStreamSynchronize(s));
    g_syncs += 1;
    g_sync_ns += static_cast<u64>(now_ns() - t0);
}

// Device-to-host reads of small results go through a per-thread pinned bounce
// buffer: a copy into pageable memory is synchronous inside the driver and
// stalls the other host threads' CUDA calls for its duration (measured: a
// factor-prep worker's pageable reads held the mode loop's launches back by
// ~0.15 ms per mode); a pinned copy + stream sync blocks only this thread.
std::atomic<u64>& pinned_staging_allocs() {
    static std::atomic<u64> n{0};
    return n;
}

void d2h(void* h, const void* d, std::size_t bytes, cudaStream_t s) {
    if (!bytes) return;
    constexpr std::size_t kBounce = std::size_t{1} << 20;
    cudaPointerAttributes at{};
    const bool pinned = cudaPointerGetAttributes(&at, h) == cudaSuccess && at.type == cudaMemoryTypeHost;
    if (pinned || bytes > kBounce) {  // already asynchronous: the caller syncs
        TCB_CUDA(cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, s));
        return;
    }
    // per thread; handed back to a process-wide free list when the thread ends
    // (the per-call std::async threads would otherwise pin a fresh buffer each
    // call) and never freed (exit order vs. the context)
    struct Bounce {
        void* buf = nullptr;
        ~Bounce() {
            if (buf) {
                std::lock_guard<std::mutex> lk(pool_mu());
                pool().push_back(buf);
            }
        }
        static std::mutex& pool_mu() {
            static std::mutex* m = new std::mutex;  // leaked: threads may end after static destruction
            return *m;
        }
        static std::vector<void*>& pool() {
            static auto* v = new std::vector<void*>;
            return *v;
        }
    };
    thread_local Bounce b;
    if (!b.buf) {
        {
            std::lock_guard<std::mutex> lk(Bounce::pool_mu());
            if (!Bounce::pool().empty()) {
                b.buf = Bounce::pool().back();
                Bounce::pool().pop_back();
            }
        }
        if (!b.buf) {
            TCB_CUDA(cudaMallocHost(&b.buf, kBounce));
            ++pinned_staging_allocs();
        }
    }
    TCB_CUDA(cudaMemcpyAsync(b.buf, d, bytes, cudaMemcpyDeviceToHost, s));
    stream_sync(s);
    std::memcpy(h, b.buf, bytes);
}

// Host-to-device uploads of small host arrays go through a per-thread ring of
// pinned slots: a copy from pageable memory waits for everything queued on the
// stream before it starts (so the host could not enqueue the kernels that
// follow until the stream drained); from a pinned slot it is asynchronous.  A
// slot is reused once the copy that last read it has completed (its event).
void h2d(void* d, const void* h, std::size_t bytes, cudaStream_t s) {
    if (!bytes) return;
    constexpr std::size_t kSlot = std::size_t{1} << 19;
    constexpr int kSlots = 8;
    if (bytes > kSlot) {
        TCB_CUDA(cudaMemcpyAsync(d, h, bytes, cudaMemcpyHostToDevice, s));
        return;
    }
    struct Ring {
        void* buf = nullptr;
        cudaEvent_t ev[kSlots] = {};
        bool used[kSlots] = {};
        int next = 0;
    };
    // per thread and device; a thread that ends hands its ring (slots, events and
    // their pending state) to a process-wide free list for the next new thread on
    // that device; never freed (exit order vs. the context)
    struct Held {
        Ring r;
        int dev = -1;
        ~Held() {
            if (r.buf) {
                std::lock_guard<std::mutex> lk(pool_mu());
                pool()[dev].push_back(r);
            }
        }
        static std::mutex& pool_mu() {
            static std::mutex* m = new std::mutex;
            return *m;
        }
        static std::map<int, std::vector<Ring>>& pool() {
            static auto* v = new std::map<int, std::vector<Ring>>;
            return *v;
        }
    };
    thread_local Held held;
    const int dev_now = cur_device();
    if (held.r.buf && held.dev != dev_now) {  // the thread moved to another device: its events belong to the old one
        std::lock_guard<std::mutex> lk(Held::pool_mu());
        Held::pool()[held.dev].push_back(held.r);
        held.r = Ring{};
    }
    Ring& r = held.r;
    if (!r.buf) {
        held.dev = dev_now;
        {
            std::lock_guard<std::mutex> lk(Held::pool_mu());
            auto& free_list = Held::pool()[dev_now];
            if (!free_list.empty()) {
                r = free_list.back();
                free_list.pop_back();
            }
        }
        if (!r.buf) {
            TCB_CUDA(cudaMallocHost(&r.buf, kSlot * kSlots));
            ++pinned_staging_allocs();
            for (auto& e : r.ev) TCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        }
    }
    const int i = r.next;
    r.next = (r.next + 1) % kSlots;
    if (r.used[i]) TCB_CUDA(cudaEventSynchronize(r.ev[i]));
    u8* slot = static_cast<u8*>(r.buf) + static_cast<std::size_t>(i) * kSlot;
    std::memcpy(slot, h, bytes);
    TCB_CUDA(cudaMemcpyAsync(d, slot, bytes, cudaMemcpyHostToDevice, s));
    TCB_CUDA(cudaEventRecord(r.ev[i], s));
    r.used[i] = true;
}

void timeline_dump();
void host_trace_dump() {
    timeline_dump();
    if (!trace_on()) return;
    std::lock_guard<std::mutex> lk(g_trace_mu);
    std::fprintf(stderr, "[tcb trace] host syncs: %llu, waiting %.3f ms (all threads)\n",
                 static_cast<unsigned long long>(g_syncs.exchange(0)), g_sync_ns.exchange(0) * 1e-6);
    for (auto& [k, v] : g_trace) std::fprintf(stderr, "[tcb trace] %-28s %8.3f ms  x%llu\n", k.c_str(), v.first,
                                               static_cast<unsigned long long>(v.second));
    g_trace.clear();
}

ProfScope::ProfScope(Cat c, cudaStream_t s) : cat(c), st(s) {
    if (!g_prof && !timeline_on()) return;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
}
ProfScope::~ProfScope() {
    if (!a) return;
    cudaEventRecord(b, st);
    if (g_prof) {
        g_recs.push_back({cat, a, b});
    } else {
        std::lock_guard<std::mutex> lk(g_tl_mu);
        g_tl.push_back({cat, st, a, b});
    }
}

void timeline_dump() {
    if (!timeline_on()) return;
    const cudaError_t se = cudaDeviceSynchronize();
    std::lock_guard<std::mutex> lk(g_tl_mu);
    if (se != cudaSuccess || g_tl.empty()) {
        std::fprintf(stderr, "[tcb tl] sync: %s, %zu records, first query %s\n", cudaGetErrorString(se), g_tl.size(),
                     g_tl.empty() ? "-" : cudaGetErrorString(cudaEventQuery(g_tl[0].a)));
    }
    if (g_tl.empty()) return;
    static const char* names[] = {"ingest", "permute", "gram", "eig", "ttm", "quant", "stats", "emit", "ac", "factor", "sum", "tc"};
    cudaEvent_t ref = g_tl[0].a;
    std::vector<std::pair<float, std::string>> lines;
    std::map<cudaStream_t, int> sid;
    for (auto& r : g_tl) {
        float t0 = 0, t1 = 0;
        const cudaError_t e0 = cudaEventElapsedTime(&t0, ref, r.a);
        const cudaError_t e1 = cudaEventElapsedTime(&t1, ref, r.b);
        if (e0 != cudaSuccess || e1 != cudaSuccess) {
            std::fprintf(stderr, "[tcb tl] event error %s / %s\n", cudaGetErrorString(e0), cudaGetErrorString(e1));
            cudaGetLastError();
        }
        if (!sid.count(r.st)) {
            const int k = static_cast<int>(sid.size());
            sid[r.st] = k;
        }
        char buf[160];
        std::snprintf(buf, sizeof(buf), "[tcb tl] s%-2d %-8s %8.3f -> %8.3f ms (%6.3f)", sid[r.st], names[r.cat], t0, t1,
                      t1 - t0);
        lines.push_back({t0, buf});
    }
    for (auto& r : g_tl) {
        cudaEventDestroy(r.a);
        cudaEventDestroy(r.b);
    }
    std::sort(lines.begin(), lines.end(), [](auto& x, auto& y) { return x.first < y.first; });
    for (auto& l : lines) std::fprintf(stderr, "%s\n", l.second.c_str());
    g_tl.clear();
}

double peak_dmma_tflops();
}  // namespace tcb

using namespace tcb;

namespace tcb {
cudaMemPool_t device_pool() {
    static PerDevice<cudaMemPool_t> pools;
    return pools.get([] {
        cudaMemPool_t mp = nullptr;
        cudaMemPoolProps pp{};
        pp.allocType = cudaMemAllocationTypePinned;
        pp.handleTypes = cudaMemHandleTypeNone;
        pp.location.type = cudaMemLocationTypeDevice;
        pp.location.id = cur_device();
        if (cudaMemPoolCreate(&mp, &pp) != cudaSuccess) {  // the default pool, as the driver configured it
            cudaGetLastError();
            TCB_CUDA(cudaDeviceGetDefaultMemPool(&mp, cur_device()));
            return mp;
        }
        u64 thr = ~u64{0};  // keep freed memory mapped between calls
        TCB_CUDA(cudaMemPoolSetAttribute(mp, cudaMemPoolAttrReleaseThreshold, &thr));
        // A block freed on another stream is reused only once that free has
        // completed: never by making this stream wait for the other stream's
        // pending kernels (the core's emission stalled behind a factor worker's
        // 15 ms kernels in ~1 call of 5: +30..130 ms).  TCB_POOL_DEPS=1 keeps the
        // driver default for measurements.
        if (!std::getenv("TCB_POOL_DEPS")) {
            int off = 0;
            TCB_CUDA(cudaMemPoolSetAttribute(mp, cudaMemPoolReuseAllowInternalDependencies, &off));
        }
        return mp;
    });
}
}  // namespace tcb
namespace {

thread_local std::string g_err;

struct Stream {
    cudaStream_t s = nullptr;
    Stream() {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
            throw Error("tucomp_b200: no CUDA device (the B200 path has no CPU fallback)");
        // the call's own stream carries the critical path (sthosvd, core plan and
        // finalisation): priority over the factor workers' streams, one level
        // below the highest (kept for short speculative work that must overtake it)
        int lo = 0, hi = 0;
        TCB_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        TCB_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, hi < lo ? hi + 1 : hi));
        (void)device_pool();
    }
    ~Stream() {
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        cudaGetLastError();
        return 1;
    }
}

// Result buffers handed to the caller (released with tcb_free).  Large ones
// (decompressed tensors) come from a pool of pinned host blocks, so the
// device-to-host copy runs at PCIe speed into memory that is already mapped;
// tcb_free returns them to the pool.
constexpr std::size_t kPinnedMin = std::size_t{4} << 20;
std::mutex g_pin_mu;
std::map<void*, std::size_t> g_pin_live;              // handed out: block -> capacity
std::multimap<std::size_t, void*> g_pin_free;         // capacity -> block
void* host_alloc(std::size_t bytes) {
    if (bytes < kPinnedMin) return std::malloc(bytes + 1);
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pin_free.lower_bound(bytes);
    if (it != g_pin_free.end() && it->first <= 2 * bytes) {
        void* p = it->second;
        g_pin_live[p] = it->first;
        g_pin_free.erase(it);
        return p;
    }
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes) != cudaSuccess) {
        cudaGetLastError();
        return std::malloc(bytes + 1);
    }
    g_pin_live[p] = bytes;
    return p;
}
bool host_release(void* p) {
    std::lock_guard<std::mutex> lk(g_pin_mu);
    auto it = g_pin_live.find(p);
    if (it == g_pin_live.end()) return false;
    g_pin_free.emplace(it->second, p);
    g_pin_live.erase(it);
    std::size_t cached = 0;  // keep at most ~1 GiB of idle pinned blocks
    for (auto& kv : g_pin_free) cached += kv.first;
    while (cached > (std::size_t{1} << 30) && !g_pin_free.empty()) {
        auto big = std::prev(g_pin_free.end());
        cached -= big->first;
        cudaFreeHost(big->second);
        g_pin_free.erase(big);
    }
    return true;
}

void host_free_any(void* p) {
    if (p && !host_release(p)) std::free(p);
}
// compress results (container bytes) come from the pinned pool too
const bool g_result_alloc_installed = [] {
    set_result_allocator(host_alloc, host_free_any);
    return true;
}();

template <class T>
T* dup(const std::vector<T>& v) {
    T* p = static_cast<T*>(std::malloc(v.size() * sizeof(T) + 1));
    if (!v.empty()) std::memcpy(p, v.data(), v.size() * sizeof(T));
    return p;
}

Params to_params(const tcb_params* p, int d) {
    Params o;
    if (p->has_target_re) o.target_re = p->target_re;
    if (p->has_target_sse) o.target_sse = p->target_sse;
    o.rtmss = p->rtmss;
    o.threads = p->threads;
    o.method = p->method;
    if (p->has_storage_order) o.storage_order = std::vector<u64>(p->storage_order, p->storage_order + d);
    if (p->has_mode_order) o.mode_order = std::vector<u64>(p->mode_order, p->mode_order + d);
    o.coder = p->coder;
    o.split = p->split_planes != 0;
    o.simple = p->simple_factor_weights != 0;
    o.block = p->block_size;
    o.f32 = p->internal_float32 != 0;
    o.backend = p->svd_backend;
    return o;
}

void fill(Result& r, int d, tcb_result* out) {
    std::memset(out, 0, sizeof(*out));
    out->container_size = r.container.size();
    out->container = r.container.release();  // from host_alloc (installed below): tcb_free releases it
    out->truncation_sse = r.trunc;
    out->core_quantization_sse = r.core_quant;
    for (int i = 0; i < d && i < 8; ++i) {
        out->factor_terms[i] = i < static_cast<int>(r.factor_terms.size()) ? r.factor_terms[i] : 0.0;
        out->ranks[i] = r.ranks[i];
    }
    out->estimate_sse = r.estimate;
    out->norm_sq = r.norm_sq;
    out->target_sse = r.target_sse;
    out->order = d;
    out->times = tcb_times{r.times.sthosvd, r.times.quantize, r.times.core, r.times.factor, r.times.serialize,
                           r.times.total};
    out->peak_alloc_estimate = r.peak_alloc;
    out->original_bytes = r.original_bytes;
    out->ingest_precision_loss = r.precision_loss;
    out->core_last_plane = r.core_last_plane;
    out->core_scale_exponent = r.core_k;
    out->uncertified_decisions = r.uncertified;
    out->kernel_launches = launch_counter().load();
    out->rank_tie_modes = r.rank_tie_modes;
}

std::size_t dtype_bytes(int t) {
    static const std::size_t sz[10] = {1, 1, 2, 2, 4, 4, 8, 8, 4, 8};
    if (t < 0 || t > 9) throw Error("container: unknown dtype");
    return sz[t];
}

}  // namespace

extern "C" {

void tcb_default_params(tcb_params* p) {
    std::memset(p, 0, sizeof(*p));
    p->rtmss = 0.5;
    p->threads = 1;
    p->split_planes = 1;
}

const char* tcb_last_error(void) { return g_err.c_str(); }

void tcb_prof_enable(int on) { g_prof = on != 0; }

int tcb_prof_read(double* ms, uint64_t* counts, int ncat) {
    return guard([&] {
        TCB_CUDA(cudaDeviceSynchronize());
        for (int i = 0; i < ncat; ++i) {
            ms[i] = 0.0;
            counts[i] = 0;
        }
        for (auto& r : g_recs) {
            float t = 0.f;
            cudaEventElapsedTime(&t, r.a, r.b);
            if (r.cat < ncat) {
                ms[r.cat] += t;
                counts[r.cat] += 1;
            }
            cudaEventDestroy(r.a);
            cudaEventDestroy(r.b);
        }
        g_recs.clear();
    });
}

double tcb_peak_dmma_tflops(void) {
    try {
        return peak_dmma_tflops();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1.0;
    }
}
void tcb_free(void* p) {
    if (p && !host_release(p)) std::free(p);
}
uint64_t tcb_kernel_launches(void) { return launch_counter().load(); }
uint64_t tcb_pinned_staging_allocs(void) { return pinned_staging_allocs().load(); }

namespace {
// fp64 from pinned host memory with the identity processing order: the upload
// goes in column chunks of the first mode's unfolding (rows x cols, row-major)
// on a copy stream, and the first Gram's split-K blocks for each chunk start as
// soon as it lands, so the Gram hides under the PCIe transfer.  Bitwise the same
// Gram as gram_f64 (same split plan, same reduction).  false: plain upload.
bool upload_overlapping_gram(const u8* host, u64 nbytes, int dtype, const std::vector<u64>& sh, const Params& prm,
                             u8* dev, DevBuf<double>& g0, DevBuf<double>& ws, cudaStream_t s) {
    if (dtype != 9 || prm.f32 || sh.size() < 2 || nbytes < (u64{32} << 20)) return false;
    if (const char* e = std::getenv("TCB_PLAIN_UPLOAD"); e && *e && *e != '0') return false;
    const std::vector<u64> p = prm.mode_order ? *prm.mode_order : stable_ascending(sh);
    for (std::size_t i = 0; i < p.size(); ++i)
        if (p[i] != i) return false;
    const u64 rows = sh[0], cols = nbytes / 8 / rows;
    if (!(prm.backend == 1 || (prm.backend == 0 && rows <= cols))) return false;
    if (ozaki_gram_ok(rows, cols)) return false;  // the mode loop's Gram is the Ozaki one
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, host) != cudaSuccess || pa.type != cudaMemoryTypeHost) {
        cudaGetLastError();
        return false;  // pageable memory: the copies would not overlap anyway
    }
    const double* B = reinterpret_cast<const double*>(dev);
    const GramPlan gp = gram_plan(B, rows, cols);
    g0 = DevBuf<double>(rows * rows, s);
    ws = DevBuf<double>(gram_ws_doubles(gp), s);
    static PerDevice<cudaStream_t> copy_dev;
    cudaStream_t copy = copy_dev.get([] {
        cudaStream_t c;
        TCB_CUDA(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
        return c;
    });
    cudaEvent_t start;
    TCB_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    TCB_CUDA(cudaEventRecord(start, s));  // the buffers exist on `s`
    TCB_CUDA(cudaStreamWaitEvent(copy, start, 0));
    const u64 chunks = std::min<u64>(8, gp.splits);
    std::vector<cudaEvent_t> ev(chunks);
    for (u64 c = 0; c < chunks; ++c) {
        const u64 sp0 = gp.splits * c / chunks, sp1 = gp.splits * (c + 1) / chunks;
        const u64 k0 = gram_split_col(gp, sp0, cols), k1 = gram_split_col(gp, sp1, cols);
        if (k1 > k0)
            TCB_CUDA(cudaMemcpy2DAsync(dev + k0 * 8, cols * 8, host + k0 * 8, cols * 8, (k1 - k0) * 8, rows,
                                       cudaMemcpyHostToDevice, copy));
        TCB_CUDA(cudaEventCreateWithFlags(&ev[c], cudaEventDisableTiming));
        TCB_CUDA(cudaEventRecord(ev[c], copy));
        TCB_CUDA(cudaStreamWaitEvent(s, ev[c], 0));
        gram_splits(B, rows, cols, gp, sp0, sp1, ws.p, s);
    }
    gram_reduce(gp, ws.p, rows, g0.p, s);
    for (auto e : ev) cudaEventDestroy(e);
    cudaEventDestroy(start);
    return true;
}

// fp32 / fp64 from pinned host memory, identity processing order, a first
// unfolding on the Ozaki route: the upload goes in row slabs of the first
// unfolding (rows x cols, row-major: a slab is contiguous) on a copy stream; as
// each lands, its rows are cast to fp64 (fp32 source), their exponents, sums of
// squares and digits computed, and every Gram product tile whose rows are all
// present runs, so the first Gram hides under the PCIe transfer.  Bitwise the
// mode loop's own Gram (exact integer tile products).  false: not applicable.
bool upload_overlapping_ozaki(const u8* host, u64 nbytes, int dtype, const std::vector<u64>& sh, const Params& prm,
                              u8* dev, DevBuf<double>& g0, DevBuf<double>& cast, cudaStream_t s) {
    if ((dtype != 8 && dtype != 9) || prm.f32 || sh.size() < 2 || nbytes < (u64{32} << 20)) return false;
    if (const char* e = std::getenv("TCB_PLAIN_UPLOAD"); e && *e && *e != '0') return false;
    if (ozaki_lt_forced()) return false;
    const std::vector<u64> p = prm.mode_order ? *prm.mode_order : stable_ascending(sh);
    for (std::size_t i = 0; i < p.size(); ++i)
        if (p[i] != i) return false;
    const u64 es = dtype == 8 ? 4 : 8;
    const u64 rows = sh[0], cols = nbytes / es / rows;
    if (rows * cols * es != nbytes || !ozaki_gram_ok(rows, cols)) return false;
    if (!(prm.backend == 1 || (prm.backend == 0 && rows <= cols))) return false;
    if (dtype == 9 && reinterpret_cast<uintptr_t>(dev) % 16) return false;
    cudaPointerAttributes pa{};
    if (cudaPointerGetAttributes(&pa, host) != cudaSuccess || pa.type != cudaMemoryTypeHost) {
        cudaGetLastError();
        return false;  // pageable memory: the copies would not overlap anyway
    }
    if (dtype == 8) cast = DevBuf<double>(rows * cols, s);
    const double* B = dtype == 8 ? cast.p : reinterpret_cast<const double*>(dev);
    OzGramRows gr(rows, cols, s);
    g0 = DevBuf<double>(rows * rows, s);
    static PerDevice<cudaStream_t> copy_dev;
    cudaStream_t copy = copy_dev.get([] {
        cudaStream_t c;
        TCB_CUDA(cudaStreamCreateWithFlags(&c, cudaStreamNonBlocking));
        return c;
    });
    cudaEvent_t start;
    TCB_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
    TCB_CUDA(cudaEventRecord(start, s));  // the buffers exist on `s`
    TCB_CUDA(cudaStreamWaitEvent(copy, start, 0));
    // slabs of 128 rows (the tensor-core tile's row block), at most 16
    const u64 slab = std::max<u64>(128, (rows + 16 * 128 - 1) / (16 * 128) * 128);
    std::vector<cudaEvent_t> ev;
    for (u64 r0 = 0; r0 < rows; r0 += slab) {
        const u64 r1 = std::min(rows, r0 + slab);
        TCB_CUDA(cudaMemcpyAsync(dev + r0 * cols * es, host + r0 * cols * es, (r1 - r0) * cols * es,
                                 cudaMemcpyHostToDevice, copy));
        cudaEvent_t e;
        TCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        ev.push_back(e);
        TCB_CUDA(cudaEventRecord(e, copy));
        TCB_CUDA(cudaStreamWaitEvent(s, e, 0));
        if (dtype == 8) ingest_cast(dev + r0 * cols * es, 8, (r1 - r0) * cols, cast.p + r0 * cols, s);
        gr.rows_ready(B, r1);
    }
    gr.finish(g0.p);
    for (auto e : ev) cudaEventDestroy(e);
    cudaEventDestroy(start);
    return true;
}
}  // namespace

int tcb_compress(const uint8_t* bytes, uint64_t nbytes, int dtype, const uint64_t* shape, int d, uint64_t skip,
                 const tcb_params* params, tcb_result* out) {
    return guard([&] {
        std::vector<u64> sh(shape, shape + d);
        u64 n = 1;
        for (auto v : sh) n *= v;
        const u64 expect = skip + n * dtype_bytes(dtype);
        if (nbytes != expect)
            throw Error("ingest: buffer holds " + std::to_string(nbytes) + " bytes, expected " + std::to_string(expect));
        Stream st;
        const Params prm = to_params(params, d);
        DevBuf<u8> dev(nbytes - skip + 16, st.s);
        DevBuf<double> g0, ws, cast;
        if (!upload_overlapping_ozaki(bytes + skip, nbytes - skip, dtype, sh, prm, dev.p, g0, cast, st.s) &&
            !upload_overlapping_gram(bytes + skip, nbytes - skip, dtype, sh, prm, dev.p, g0, ws, st.s))
            dev.upload(bytes + skip, nbytes - skip);
        Result r = compress_device(dev.p, nbytes - skip, dtype, sh, prm, st.s, g0.p, nullptr, &cast);
        host_trace_dump();
        fill(r, d, out);
    });
}

int tcb_nccl_unique_id(uint8_t out[128]) {
    return guard([&] { nccl_unique_id(out); });
}

int tcb_nccl_comm_init(const uint8_t id[128], int world, int rank, void** comm) {
    return guard([&] {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
            throw Error("tucomp_b200: no CUDA device (the B200 path has no CPU fallback)");
        *comm = nccl_comm_init(id, world, rank);
    });
}

int tcb_nccl_comm_destroy(void* comm) {
    return guard([&] { nccl_comm_destroy(comm); });
}

int tcb_compress_sharded_device(void* comm, int world, int rank, const void* device_bytes, uint64_t nbytes,
                                int dtype, const uint64_t* shape, int d, uint64_t local_extent,
                                const tcb_params* params, tcb_result* out) {
    return guard([&] {
        std::vector<u64> sh(shape, shape + d);
        Stream st;
        ShardComm sc;
        sc.comm = comm;
        sc.world = world;
        sc.rank = rank;
        sc.local_extent = local_extent;
        Result r = compress_device(device_bytes, nbytes, dtype, sh, to_params(params, d), st.s, nullptr, &sc);
        host_trace_dump();
        fill(r, d, out);
    });
}

int tcb_compress_sharded_host(const tcb_host_collectives* coll, int world, int rank, const void* device_bytes,
                              uint64_t nbytes, int dtype, const uint64_t* shape, int d, uint64_t local_extent,
                              const tcb_params* params, tcb_result* out) {
    return guard([&] {
        if (!coll || !coll->allreduce_sum_f64 || !coll->allgather) throw Error("sharded compress: no collectives");
        std::vector<u64> sh(shape, shape + d);
        Stream st;
        HostCollectives hc{coll->ctx, coll->allreduce_sum_f64, coll->allgather};
        ShardComm sc;
        sc.host = &hc;
        sc.world = world;
        sc.rank = rank;
        sc.local_extent = local_extent;
        Result r = compress_device(device_bytes, nbytes, dtype, sh, to_params(params, d), st.s, nullptr, &sc);
        host_trace_dump();
        fill(r, d, out);
    });
}

int tcb_compress_device(const void* device_bytes, uint64_t nbytes, int dtype, const uint64_t* shape, int d,
                        const tcb_params* params, tcb_result* out) {
    return guard([&] {
        std::vector<u64> sh(shape, shape + d);
        Stream st;
        Result r = compress_device(device_bytes, nbytes, dtype, sh, to_params(params, d), st.s);
        host_trace_dump();
        fill(r, d, out);
    });
}

int tcb_measure_error(const uint8_t* bytes, uint64_t nbytes, int dtype, const uint64_t* shape, int d, uint64_t skip,
                      int internal_float32, const uint8_t* container, uint64_t len, double* sse) {
    return guard([&] {
        std::vector<u64> sh(shape, shape + d);
        u64 n = 1;
        for (auto v : sh) n *= v;
        const u64 expect = skip + n * dtype_bytes(dtype);
        if (nbytes != expect)
            throw Error("ingest: buffer holds " + std::to_string(nbytes) + " bytes, expected " + std::to_string(expect));
        Stream st;
        const auto t = decompress_device(container, len, st.s);
        if (t.shape != sh) throw Error("sse_between: shape mismatch");
        DevBuf<u8> dev(nbytes - skip + 16, st.s);
        dev.upload(bytes + skip, nbytes - skip);
        DevBuf<double> x(std::max<u64>(n, 1), st.s);
        ingest_cast(dev.p, dtype, n, x.p, st.s);
        *sse = n ? sse_between(x.p, t.x.p, n, internal_float32 != 0, st.s) : 0.0;
    });
}

int tcb_decompress(const uint8_t* container, uint64_t len, int threads, tcb_decompress_result* out) {
    (void)threads;  // the device path has no host worker count
    return guard([&] {
        Stream st;
        const auto t = decompress_device(container, len, st.s);
        HostTrace ht("decompress: emit+D2H");
        const u64 nb = emit_size(t);
        out->bytes = static_cast<uint8_t*>(host_alloc(nb));
        emit_bytes(t, out->bytes, st.s);
        ht.stop();
        out->nbytes = nb;
        out->dtype = t.dtype;
        out->d = static_cast<int>(t.shape.size());
        for (std::size_t i = 0; i < t.shape.size() && i < 8; ++i) out->shape[i] = t.shape[i];
        out->total_ms = t.ms;
        host_trace_dump();
    });
}

int tcb_decompress_device(const uint8_t* container, uint64_t len, void* device_out, uint64_t capacity,
                          tcb_decompress_result* out) {
    return guard([&] {
        Stream st;
        const auto t = decompress_device(container, len, st.s);
        const u64 nb = emit_size(t);
        if (nb > capacity)
            throw Error("decompress: output buffer holds " + std::to_string(capacity) + " bytes, needs " +
                        std::to_string(nb));
        const u64 total = [&] {
            u64 v = 1;
            for (auto x : t.shape) v *= x;
            return v;
        }();
        if (total) {
            if (t.dtype == 9)
                TCB_CUDA(cudaMemcpyAsync(device_out, t.x.p, nb, cudaMemcpyDeviceToDevice, st.s));
            else
                emit_dtype(t.x.p, total, t.dtype, device_out, st.s);
        }
        stream_sync(st.s);
        out->bytes = nullptr;
        out->nbytes = nb;
        out->dtype = t.dtype;
        out->d = static_cast<int>(t.shape.size());
        for (std::size_t i = 0; i < t.shape.size() && i < 8; ++i) out->shape[i] = t.shape[i];
        out->total_ms = t.ms;
        host_trace_dump();
    });
}

int tcb_decompress_tensor_f64(const uint8_t* container, uint64_t len, double** out, uint64_t* count,
                              uint64_t* shape, int* d) {
    return guard([&] {
        Stream st;
        const auto t = decompress_device(container, len, st.s);
        u64 total = 1;
        for (auto v : t.shape) total *= v;
        *out = static_cast<double*>(host_alloc(total * sizeof(double)));
        if (total) t.x.download(*out, total);
        stream_sync(st.s);
        *count = total;
        *d = static_cast<int>(t.shape.size());
        for (std::size_t i = 0; i < t.shape.size() && i < 8; ++i) shape[i] = t.shape[i];
    });
}

int tcb_read_container_header(const uint8_t* container, uint64_t len, tcb_container_header* out) {
    return guard([&] {
        const auto h = read_container_header(container, len);
        if (h.n.size() > 8) throw Error("container: order above 8 is not supported by this interface");
        *out = tcb_container_header{};
        out->version = h.version;
        out->source_dtype = h.dtype;
        out->internal_float32 = h.f32;
        out->d = static_cast<int>(h.n.size());
        out->coder = h.coder;
        out->method = h.method;
        out->zero_flag = h.zero;
        out->split_planes = h.split;
        out->simple_weights = h.simple;
        for (std::size_t i = 0; i < h.n.size(); ++i) {
            out->mode_sizes[i] = h.n[i];
            out->ranks[i] = h.rk[i];
            out->processing_order[i] = h.order[i];
            out->storage_order[i] = h.storage[i];
        }
        out->core_scale_exponent = h.k;
        out->block_size = h.block;
        out->rtmss = h.rtmss;
        out->target_sse = h.target_sse;
        out->norm_sq = h.norm_sq;
        out->truncation_sse = h.trunc_sse;
        out->core_quant_sse = h.cq_sse;
        out->estimate_sse = h.est_sse;
    });
}

int tcb_sthosvd_f64(const double* a, const uint64_t* shape, int d, double sse_target, const uint64_t* order,
                    int backend, double* core, uint64_t* core_shape, double** factors, uint64_t* ranks, double* trunc,
                    uint64_t* order_out) {
    return guard([&] {
        std::vector<u64> sh(shape, shape + d);
        u64 n = 1;
        for (auto v : sh) n *= v;
        Stream st;
        DevBuf<double> x(n, st.s);
        x.upload(a, n);
        std::optional<std::vector<u64>> ord;
        if (order) ord = std::vector<u64>(order, order + d);
        Tucker f = sthosvd_device(std::move(x), sh, sse_target, ord, backend, st.s);
        u64 nc = 1;
        for (int i = 0; i < d; ++i) {
            core_shape[i] = f.core_shape[i];
            nc *= f.core_shape[i];
            ranks[i] = f.r[i];
            trunc[i] = f.trunc[i];
            order_out[i] = f.order[i];
            f.factors[i].download(factors[i], f.n[i] * f.r[i]);
        }
        f.core.download(core, nc);
        stream_sync(st.s);
    });
}

int tcb_gram_f64(const double* b, uint64_t rows, uint64_t cols, double* g) {
    return guard([&] {
        Stream st;
        DevBuf<double> B(rows * cols, st.s), G(rows * rows, st.s);
        B.upload(b, rows * cols);
        gram_f64(B.p, rows, cols, G.p, st.s);
        G.download(g, rows * rows);
        stream_sync(st.s);
    });
}

int tcb_ttm_f64(const double* b, uint64_t rows, uint64_t cols, const double* u, uint64_t r, double* next) {
    return guard([&] {
        Stream st;
        DevBuf<double> B(rows * cols, st.s), U(rows * r, st.s), O(cols * r, st.s);
        B.upload(b, rows * cols);
        U.upload(u, rows * r);
        ttm_f64(B.p, rows, cols, U.p, r, O.p, st.s);
        O.download(next, cols * r);
        stream_sync(st.s);
    });
}

int tcb_eig_f64(const double* g, uint64_t n, uint64_t r, double* evals_desc, double* u) {
    return guard([&] {
        Stream st;
        DevBuf<double> G(n * n, st.s);
        G.upload(g, n * n);
        EigWork w;
        const auto ev = eig_values(G.p, n, w, st.s);
        std::memcpy(evals_desc, ev.data(), n * sizeof(double));
        if (r > 0) {
            DevBuf<double> U(n * r, st.s);
            eig_vectors(w, r, U.p, st.s);
            fix_column_signs(U.p, n, r, st.s);
            U.download(u, n * r);
        }
        stream_sync(st.s);
    });
}

int tcb_quantize_f64(const double* core, const uint64_t* shape, int d, uint64_t* mag, uint8_t* neg, int* k, int* zero,
                     double* slice_norms_out) {
    return guard([&] {
        std::vector<u64> sh(shape, shape + d);
        u64 n = 1, se = 0;
        for (auto v : sh) {
            n *= v;
            se += v;
        }
        Stream st;
        DevBuf<double> x(n, st.s);
        x.upload(core, n);
        bool fin = true;
        sum_squares(x.p, n, &fin, st.s);
        if (!fin) throw Error("quantize: non-finite core values");
        const double mx = max_abs(x.p, n, st.s);
        *zero = mx == 0.0;
        *k = *zero ? 0 : 63 - std::ilogb(mx);
        if (*zero) {
            std::memset(slice_norms_out, 0, se * sizeof(double));
            return;
        }
        DevBuf<u64> dm(n, st.s);
        DevBuf<u8> dn(n, st.s);
        quantize_f64(x.p, n, *k, dm.p, dn.p, st.s);
        DevBuf<double> sn(se, st.s);
        slice_norms(dm.p, sh, std::ldexp(1.0, -2 * *k), sn.p, st.s);
        dm.download(mag, n);
        dn.download(neg, n);
        sn.download(slice_norms_out, se);
        stream_sync(st.s);
    });
}

int tcb_encode(const uint64_t* mag, const uint8_t* neg, uint64_t n, double target, int coder, uint64_t block,
               int split, int fixed_plane, uint8_t** stream, uint64_t* stream_len, int* last_plane,
               double* achieved, uint64_t* decoded, int* uncertified) {
    return guard([&] {
        Stream st;
        DevBuf<u64> m(n + 1, st.s), dec(n + 1, st.s);
        DevBuf<u8> ng(n + 1, st.s);
        m.upload(mag, n);
        ng.upload(neg, n);
        EncodeOpts o;
        o.coder = coder;
        o.block = block;
        o.split = split != 0;
        if (fixed_plane >= 0) o.fixed_plane = fixed_plane;
        const PlanResult pl = plan_stream(m.p, n, target, o, dec.p, st.s);
        const auto body = finalize_stream(m.p, ng.p, n, pl, coder, n, st.s);
        const double a = exact_backward_sum(kExDiff, 0, m.p, dec.p, n, st.s);
        if (decoded) dec.download(decoded, n);
        stream_sync(st.s);
        *stream = dup(body);
        *stream_len = body.size();
        *last_plane = pl.last_plane;
        *achieved = a;
        if (uncertified) *uncertified = pl.fallbacks;
    });
}

int tcb_exact_sums(const uint64_t* mag, const uint64_t* dec, uint64_t n, const uint64_t* seg_lo,
                   const uint64_t* seg_hi, const int* seg_backward, const double* seg_s0, const double* seg_need,
                   int nseg, const int* kind_term, const int* kind_plane, int nk, int reference, double* sums,
                   uint64_t* c0, uint64_t* c1, int* crossed) {
    return guard([&] {
        Stream st;
        DevBuf<u64> m(n + 1, st.s), d(n + 1, st.s);
        m.upload(mag, n);
        if (dec) d.upload(dec, n);
        std::vector<ExSeg> segs(nseg);
        for (int g = 0; g < nseg; ++g) {
            if (seg_hi[g] < seg_lo[g] || seg_hi[g] > n) throw Error("exact sums: segment out of range");
            segs[g] = ExSeg{seg_lo[g], seg_hi[g], seg_backward[g], seg_s0[g], seg_need[g]};
        }
        std::vector<ExKind> kinds(nk);
        for (int k = 0; k < nk; ++k) {
            if (kind_term[k] < 0 || kind_term[k] > kExDiff || kind_plane[k] < 0 || kind_plane[k] > 64)
                throw Error("exact sums: bad kind");
            kinds[k] = ExKind{kind_term[k], kind_plane[k]};
        }
        const auto out = reference ? exact_serial_reference(m.p, dec ? d.p : nullptr, segs, kinds, st.s)
                                   : exact_serial(m.p, dec ? d.p : nullptr, segs, kinds, st.s);
        for (std::size_t j = 0; j < out.size(); ++j) {
            sums[j] = out[j].sum;
            c0[j] = out[j].c0;
            c1[j] = out[j].c1;
            crossed[j] = out[j].crossed;
        }
    });
}

int tcb_exact_plane_stats(const uint64_t* mag, uint64_t n, uint64_t block, int p_top, int np, double* sums,
                          uint64_t* c0, uint64_t* c1, int* crossed) {
    return guard([&] {
        if (block == 0) throw Error("exact sums: zero block");
        Stream st;
        DevBuf<u64> m(n + 1, st.s);
        m.upload(mag, n);
        const auto out = exact_plane_stats(m.p, n, block, p_top, np, st.s);
        for (std::size_t j = 0; j < out.size(); ++j) {
            sums[j] = out[j].sum;
            c0[j] = out[j].c0;
            c1[j] = out[j].c1;
            crossed[j] = out[j].crossed;
        }
    });
}

int tcb_encode_symbols(int coder, const uint64_t* syms, uint64_t n, uint8_t** out, uint64_t* len) {
    return guard([&] {
        Stream st;
        const auto b = encode_symbols_device(coder, syms, n, st.s);
        *out = dup(b);
        *len = b.size();
    });
}

int tcb_encode_factor_f64(const double* u, uint64_t n, uint64_t r, const uint8_t* dead, const double* sn, int coder,
                          int simple, int core_step_log2, double cap, uint8_t** stream, uint64_t* len, int* k,
                          uint64_t* count, int8_t* flips, double* term, int* plane) {
    return guard([&] {
        Stream st;
        DevBuf<double> U(n * r + 1, st.s);
        U.upload(u, n * r);
        const auto fe = encode_factor_device(U.p, n, r, std::vector<u8>(dead, dead + r),
                                             std::vector<double>(sn, sn + r), coder, simple != 0, core_step_log2, cap,
                                             false, st.s);
        *stream = dup(fe.stream);
        *len = fe.stream.size();
        *k = fe.k;
        *count = fe.count;
        for (u64 j = 0; j < r; ++j) flips[j] = fe.flips[j];
        *term = fe.term;
        *plane = fe.plane;
    });
}

}  // extern "C"

// ---------------------------------------------------------------- device-pointer building blocks
// Used by the sharded multi-GPU mode loop (paper_2107_01384_b200/shard.py):
// inputs/outputs are device pointers on the current device; each call runs on
// a private stream and returns after it completes.
extern "C" {

int tcb_dev_sumsq(const double* x, uint64_t n, double* out, int* finite) {
    return guard([&] {
        Stream st;
        bool f = true;
        *out = sum_squares(x, n, &f, st.s);
        *finite = f ? 1 : 0;
    });
}

int tcb_dev_permute(const double* src, double* dst, const uint64_t* shape, const uint64_t* perm, int d) {
    return guard([&] {
        Stream st;
        permute_axes(src, dst, std::vector<u64>(shape, shape + d), std::vector<u64>(perm, perm + d), st.s);
        stream_sync(st.s);
    });
}

int tcb_dev_gram(const double* b, uint64_t rows, uint64_t cols, double* g) {
    return guard([&] {
        Stream st;
        if (cols == 0) {
            TCB_CUDA(cudaMemsetAsync(g, 0, rows * rows * sizeof(double), st.s));
        } else {
            gram_f64(b, rows, cols, g, st.s);
        }
        stream_sync(st.s);
    });
}

int tcb_dev_gram_ozaki(const double* b, uint64_t rows, uint64_t cols, double* g) {
    return guard([&] {
        Stream st;
        if (cols == 0) TCB_CUDA(cudaMemsetAsync(g, 0, rows * rows * sizeof(double), st.s));
        else gram_ozaki(b, rows, cols, g, st.s);
        stream_sync(st.s);
    });
}

int tcb_dev_ttm_ozaki(const double* b, uint64_t rows, uint64_t cols, const double* u, uint64_t r, double* next) {
    return guard([&] {
        Stream st;
        if (cols > 0 && r > 0) ttm_ozaki(b, rows, cols, u, r, next, st.s);
        stream_sync(st.s);
    });
}

int tcb_dev_factor_from_gram(const double* g, uint64_t n, double budget, double* u, uint64_t* r, double* discarded) {
    return guard([&] {
        Stream st;
        StepOut o = factor_from_gram(g, n, budget, st.s);
        TCB_CUDA(cudaMemcpyAsync(u, o.U.p, n * o.r * sizeof(double), cudaMemcpyDeviceToDevice, st.s));
        stream_sync(st.s);
        *r = o.r;
        *discarded = o.discarded;
    });
}

int tcb_dev_mode_step(const double* b, uint64_t rows, uint64_t cols, double budget, int backend, double* u,
                      double* next, uint64_t* r, double* discarded) {
    return guard([&] {
        Stream st;
        StepOut o = mode_step(b, rows, cols, budget, backend, st.s);
        TCB_CUDA(cudaMemcpyAsync(u, o.U.p, rows * o.r * sizeof(double), cudaMemcpyDeviceToDevice, st.s));
        TCB_CUDA(cudaMemcpyAsync(next, o.next.p, cols * o.r * sizeof(double), cudaMemcpyDeviceToDevice, st.s));
        stream_sync(st.s);
        *r = o.r;
        *discarded = o.discarded;
    });
}

int tcb_dev_ttm(const double* b, uint64_t rows, uint64_t cols, const double* u, uint64_t r, double* next) {
    return guard([&] {
        Stream st;
        if (cols > 0) ttm_f64(b, rows, cols, u, r, next, st.s);
        stream_sync(st.s);
    });
}

namespace {
int encode_tucker_common(const ShardComm* sc, const double* core, const double* const* factors, const uint64_t* n,
                         const uint64_t* r, const uint64_t* order, const double* trunc, int d, int dtype,
                         double norm_sq, double target_sse, const tcb_params* params, tcb_result* out) {
    return guard([&] {
        Stream st;
        Tucker f;
        f.n.assign(n, n + d);
        f.r.assign(r, r + d);
        f.order.assign(order, order + d);
        f.trunc.assign(trunc, trunc + d);
        f.core_shape.resize(d);
        u64 nc = 1;
        for (int i = 0; i < d; ++i) {
            f.core_shape[i] = r[order[i]];
            nc *= f.core_shape[i];
        }
        f.core = DevBuf<double>(nc, st.s);
        TCB_CUDA(cudaMemcpyAsync(f.core.p, core, nc * sizeof(double), cudaMemcpyDeviceToDevice, st.s));
        f.factors.resize(d);
        for (int i = 0; i < d; ++i) {
            f.factors[i] = DevBuf<double>(n[i] * r[i], st.s);
            TCB_CUDA(cudaMemcpyAsync(f.factors[i].p, factors[i], n[i] * r[i] * sizeof(double),
                                     cudaMemcpyDeviceToDevice, st.s));
        }
        Result res = encode_tucker_device(f, dtype, norm_sq, target_sse, to_params(params, d), st.s, sc);
        fill(res, d, out);
    });
}
}  // namespace

int tcb_dev_encode_tucker(const double* core, const double* const* factors, const uint64_t* n, const uint64_t* r,
                          const uint64_t* order, const double* trunc, int d, int dtype, double norm_sq,
                          double target_sse, const tcb_params* params, tcb_result* out) {
    return encode_tucker_common(nullptr, core, factors, n, r, order, trunc, d, dtype, norm_sq, target_sse, params,
                                out);
}

int tcb_dev_encode_tucker_sharded(void* nccl_comm, const tcb_host_collectives* coll, int world, int rank,
                                  const double* core, const double* const* factors, const uint64_t* n,
                                  const uint64_t* r, const uint64_t* order, const double* trunc, int d, int dtype,
                                  double norm_sq, double target_sse, const tcb_params* params, tcb_result* out) {
    HostCollectives hc{};
    ShardComm sc;
    sc.world = world;
    sc.rank = rank;
    if (coll) {
        hc = HostCollectives{coll->ctx, coll->allreduce_sum_f64, coll->allgather};
        sc.host = &hc;
    } else {
        sc.comm = nccl_comm;
    }
    return encode_tucker_common(&sc, core, factors, n, r, order, trunc, d, dtype, norm_sq, target_sse, params, out);
}

}  // extern "C"
