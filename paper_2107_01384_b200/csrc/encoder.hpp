// Host driver of the device bit-plane encoder (corecodec::Encoder,
// core_codec.cpp:105-413): certified plan decisions + device emission.
#pragma once

#include <functional>
#include <optional>

#include "codec.cuh"

namespace tcb {
struct ShardComm;  // pipeline.hpp
}

namespace tcb {

struct EncodeOpts {
    int coder = 0;       // entropy::Coder (0 = arithmetic)
    u64 block = 0;       // 0 = max(4096, ceil(n/64))
    bool split = true;
    std::optional<int> fixed_plane;
    // called once the last plane is certified (before the stop placement), so
    // work that depends only on it can start early; may be called again with
    // the same value by the exact-mode rerun
    std::function<void(int)> on_last_plane;
    // called once when the breakpoint plane p is found, before the split probe:
    // planes 63 .. p + 1 are full whatever the stops, so their coding can start
    std::function<void(int)> on_breakpoint;
    // speculative full-plane entropy sizes for the split probe (optional)
    ProbeCache* probe = nullptr;
    // sharded encoding: this rank computes the statistics / crossing scans /
    // probes of its own blocks and the ranks exchange them, so every rank takes
    // the same decisions
    const ShardComm* shard = nullptr;
};

// a rank's contiguous share of the nb blocks
inline BlockRange rank_blocks(u64 nb, int world, int rank) {
    return BlockRange{nb * static_cast<u64>(rank) / static_cast<u64>(world),
                      nb * static_cast<u64>(rank + 1) / static_cast<u64>(world)};
}

struct PlanResult {
    int last_plane = 63;
    int nplanes = 0;
    std::vector<u64> stops;  // 2 per block: leading, trailing
    u64 block = 0;
    bool certified = true;   // false when the serial-replay fallback decided
    int fallbacks = 0;
};

u64 default_block(u64 n);

// plan(): decides last_plane and stops exactly as the reference's serial double
// arithmetic would; `dec` receives the decoder-side magnitudes.
PlanResult plan_stream(const u64* m, u64 n, double target_int, const EncodeOpts& o, u64* dec, cudaStream_t s);

// finalize() in two parts: the section head (count, block, last plane, stops,
// plane count) on the host and the (u32 size || payload) body left on the device.
struct StreamParts {
    std::vector<u8> head;
    DevBuf<u8> body;
    u64 body_size = 0;
};
// `upper` (optional, unsharded): returns planes 63 .. last_plane + 1 already
// emitted and coded with these signs (or nullptr); it is called after the last
// plane has been coded, so whatever produces it overlaps that work.
StreamParts finalize_stream_parts(const u64* m, const u8* neg, u64 n, const PlanResult& pl, int coder, u64 count,
                                  cudaStream_t s, const ShardComm* shard = nullptr,
                                  const std::function<EmitDev*()>& upper = {});
// finalize(): emits planes [last_plane, 63] with the given signs and returns
// the serialized stream section (container.cpp:231-247) for `count` elements.
std::vector<u8> finalize_stream(const u64* m, const u8* neg, u64 n, const PlanResult& pl, int coder, u64 count,
                                cudaStream_t s);

}  // namespace tcb
