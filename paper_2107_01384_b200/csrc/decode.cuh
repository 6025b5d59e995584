// Device decode of bit-plane streams (corecodec::decode, core_codec.cpp:421-508)
// and dtype emit (container.cpp:98-140); host-built descriptors.
#pragma once

#include <vector>

#include "common.cuh"

namespace tcb {

// one (stream, plane, block) payload: u32 entropy_len | entropy | raw bits
struct DecSection {
    u64 ent_off = 0;   // byte offset of the entropy section in the device container
    u64 ent_len = 0;   // = elen
    u64 raw_off = 0;   // byte offset of the raw bits
    u64 raw_len = 0;
    u64 sym_off = 0;   // decoded run symbols in the symbol buffer
    u64 scratch_off = 0;  // u32 words of global scratch (large models / rANS tables)
    u32 elen = 0;
    u32 nsym = 0;
    u32 cap = 0;       // model capacity (>= distinct symbols + 1), even
    u32 pad = 0;
};

struct DecStream {
    u64 count = 0, block = 0;
    int last_plane = 63;
    u32 nb = 0, nplanes = 0;
    u64 sec_off = 0;            // first section (plane-major: rel * nb + b)
    u64 out_off = 0;            // offset into the magnitude / sign arrays
    const u64* stops_lead = nullptr;   // device, nb entries
    const u64* stops_trail = nullptr;
};

struct DecBlock {
    u32 stream = 0, b = 0;
    u64 lo = 0, hi = 0;         // coefficient range (relative to the stream)
};

enum DecErr : int {
    kDecErrNone = 0,
    kDecErrEntropy = 1,        // entropy: corrupt / truncated payload
    kDecErrCoder = 2,          // entropy: unknown coder id
    kDecErrModel = 3,          // model capacity (internal)
    kDecErrMissingColumn = 4,  // core decode: missing leading column
    kDecErrRle = 5,            // rle: run lengths do not match column length
    kDecErrBits = 6,           // bit reader: read past end
};

u64 decode_model_words(u32 cap);
void decode_entropy(const u8* cont, const DecSection* sec_dev, const std::vector<DecSection>& sec, u64* syms,
                    u32* scratch, int* err, cudaStream_t s);
void decode_streams(const u8* cont, const DecStream* streams, const DecBlock* blocks, u64 nblocks,
                    const DecSection* sec, const u64* syms, u64* mag, u8* neg, u8* pe, u8* colbits, int* err,
                    cudaStream_t s);
// core value = +-ldexp(mag, -k), scattered to order[v] when a vectorisation map is given
void dequantize(const u64* mag, const u8* neg, u64 n, int k, double* out, cudaStream_t s,
                const u64* order = nullptr);
void emit_dtype(const double* x, u64 n, int dtype, void* out, cudaStream_t s);

}  // namespace tcb
