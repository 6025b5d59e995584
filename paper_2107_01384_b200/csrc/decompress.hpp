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

// container bytes on the host; the result stays on the device
DecompressOut decompress_device(const u8* container, u64 len, cudaStream_t s);
// emit (container.cpp:98-140): the source dtype's bytes, on the host
std::vector<u8> emit_bytes(const DecompressOut& t, cudaStream_t s);

}  // namespace tcb
