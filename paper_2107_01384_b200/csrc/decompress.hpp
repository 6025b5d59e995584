// Device decompress (pipeline::decompress / decompress_tensor, pipeline.cpp:197-236, 266-283).
#pragma once

#include <vector>

#include "common.cuh"

namespace tcb {

struct DecompressOut {
    DevBuf<double> x;          // reconstructed tensor, original axis order, row-major
    std::vector<u64> shape;
    int dtype = 9;             // container::Dtype of the source
    bool f32 = false;          // container written with internal_float32
    double ms = 0.0;
};

// read_container's header (container.hpp Header; container.cpp:338-420), host side
struct ContainerHeader {
    int version = 1, dtype = 9, coder = 0, method = 0;
    bool f32 = false, zero = false, split = true, simple = false;
    std::vector<u64> n, rk, order, storage;  // order/storage 0-based
    int k = 0;                               // core scale exponent
    u64 block = 0;
    double rtmss = 0, target_sse = 0, norm_sq = 0, trunc_sse = 0, cq_sse = 0, est_sse = 0;
};
// header fields only; *end = offset of the first section
ContainerHeader parse_header(const u8* container, u64 len, u64* end);
// header plus a structural walk of every section (read_container's validation)
ContainerHeader read_container_header(const u8* container, u64 len);

// container bytes on the host; the result stays on the device
DecompressOut decompress_device(const u8* container, u64 len, cudaStream_t s);
// emit (container.cpp:98-140): the source dtype's bytes, on the host
std::vector<u8> emit_bytes(const DecompressOut& t, cudaStream_t s);
// the same into caller memory of emit_size(t) bytes
u64 emit_size(const DecompressOut& t);
void emit_bytes(const DecompressOut& t, u8* host, cudaStream_t s);

}  // namespace tcb
