// Shared device/host plumbing for the B200 compress path (sm_100a only).
#pragma once

#include <atomic>
#include <map>
#include <mutex>

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace tcb {

using u8 = std::uint8_t;
using u16 = std::uint16_t;
using u32 = std::uint32_t;
using u64 = std::uint64_t;
using i64 = std::int64_t;

// Same exception type/messages as the reference's tucomp::Error (tensor.hpp:14-17).
struct Error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define TCB_CUDA(expr)                                                                          \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess)                                                                  \
            throw ::tcb::Error(std::string("cuda: ") + cudaGetErrorString(_e) + " at " + #expr + " (" + \
                               __FILE__ + ":" + std::to_string(__LINE__) + ")");               \
    } while (0)

#define TCB_LAUNCH() TCB_CUDA(cudaGetLastError())

constexpr u64 kFull = ~u64{0};

// Host wait on a stream; counted (and timed under TCB_TRACE) per call site class.
void stream_sync(cudaStream_t s);
// device-to-host read; the caller syncs `s` before using `h` (pageable `h` up
// to 1 MiB: through a pinned bounce buffer, complete on return)
void d2h(void* h, const void* d, std::size_t bytes, cudaStream_t s);
// host-to-device copy of a small host array, asynchronous (through pinned staging)
void h2d(void* d, const void* h, std::size_t bytes, cudaStream_t s);

// The library's own stream-ordered memory pool on the current device (capi.cpp):
// freed blocks stay mapped between calls, and a block freed on another stream is
// reused only once that free has completed.  The device's default pool, which
// the host application may be using, is left as the driver set it up.
cudaMemPool_t device_pool();

// Stream-ordered device buffer (from device_pool(); freed on the same stream).
template <class T>
struct DevBuf {
    T* p = nullptr;
    std::size_t n = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    DevBuf(std::size_t count, cudaStream_t st) : n(count), s(st) {
        if (n) TCB_CUDA(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&p), n * sizeof(T), device_pool(), s));
    }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n), s(o.s) { o.p = nullptr; o.n = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        if (this != &o) {
            release();
            p = o.p; n = o.n; s = o.s;
            o.p = nullptr; o.n = 0;
        }
        return *this;
    }
    ~DevBuf() { release(); }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        n = 0;
    }
    void zero() {
        if (n) TCB_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
    void upload(const T* h, std::size_t cnt) {
        if (cnt) h2d(p, h, cnt * sizeof(T), s);
    }
    void download(T* h, std::size_t cnt) const {
        d2h(h, p, cnt * sizeof(T), s);
    }
    std::vector<T> to_host() const {
        std::vector<T> v(n);
        download(v.data(), n);
        stream_sync(s);
        return v;
    }
};

inline int cur_device() {
    int d = 0;
    cudaGetDevice(&d);
    return d;
}

// Per-device state built on first use on each device (function attributes,
// occupancy results, side streams): the library runs on the calling thread's
// current device, so nothing device-bound may be a plain process-wide static.
template <class T>
class PerDevice {
public:
    template <class Make>
    T& get(Make&& make) {
        const int dev = cur_device();
        std::lock_guard<std::mutex> lk(mu_);
        auto it = m_.find(dev);
        if (it == m_.end()) it = m_.emplace(dev, make()).first;
        return it->second;
    }

private:
    std::mutex mu_;
    std::map<int, T> m_;
};
// run `body` once per device at this call site
#define TCB_ONCE_PER_DEVICE(...)                                                 \
    do {                                                                          \
        static ::tcb::PerDevice<bool> tcb_once_;                                  \
        (void)tcb_once_.get([&] {                                                 \
            __VA_ARGS__;                                                          \
            return true;                                                          \
        });                                                                       \
    } while (0)

inline int sm_count() {
    static PerDevice<int> n;
    return n.get([] {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, cur_device());
        return v > 0 ? v : 148;
    });
}

struct EventHandle {
    cudaEvent_t e = nullptr;
    EventHandle() { TCB_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
    EventHandle(const EventHandle&) = delete;
    EventHandle& operator=(const EventHandle&) = delete;
    ~EventHandle() { cudaEventDestroy(e); }
};

inline unsigned cdiv(u64 a, u64 b) { return static_cast<unsigned>((a + b - 1) / b); }

// Grid for a grid-stride pass over n elements: per_sm CTAs per SM for large n,
// but no more CTAs than there are `per_thread`-element slices (a 3k-element
// core gets a handful of CTAs, not 600, and a 600-entry partial array).
inline int grid_for(u64 n, int threads, int per_thread, int per_sm) {
    const u64 want = (n + static_cast<u64>(threads) * per_thread - 1) / (static_cast<u64>(threads) * per_thread);
    const u64 cap = static_cast<u64>(sm_count()) * per_sm;
    return static_cast<int>(want < 1 ? 1 : (want > cap ? cap : want));
}

// Launch counter for the bench's "gpu_launches" claim.
std::atomic<u64>& launch_counter();
inline void count_launch(u64 k = 1) { launch_counter().fetch_add(k, std::memory_order_relaxed); }
// true while tcb_prof_enable(1): the pipeline then runs its stages sequentially
bool prof_enabled();

// Optional per-stage device timing (CUDA events on the launching stream),
// enabled by tcb_prof_enable(); read back with tcb_prof_read().
// kTc: the tcgen05 digit-product launches alone (also inside kGram / kTtm)
enum Cat : int { kIngest = 0, kPermute, kGram, kEig, kTtm, kQuant, kStats, kEmit, kAc, kFactor, kSum, kTc, kNumCat };

// Opt-in host wall-clock trace (TCB_TRACE=1): per-label totals printed to
// stderr by tcb_compress / tcb_compress_device; a debugging aid only.
struct HostTrace {
    explicit HostTrace(const char* label);
    ~HostTrace() { stop(); }
    void stop();  // record now (idempotent)
    const char* label;
    long long t0 = 0;
    bool done = false;
};
void host_trace_dump();
struct ProfScope {
    ProfScope(Cat c, cudaStream_t s);
    ~ProfScope();
    Cat cat;
    cudaStream_t st;
    cudaEvent_t a = nullptr, b = nullptr;
};

}  // namespace tcb
