// The reference encoder's per-coefficient double terms, computed exactly as its
// x86-64 build does (separately rounded multiply and subtract, no FMA):
//   sig2 / insig2        core_codec.cpp:20-35
//   trail / lead gains   core_codec.cpp:131-155 (build_block statistics)
//   recalibration term   error_model.cpp:54-72
// Every term is an integer-valued double (|t| <= 2^128).
#pragma once

#include "common.cuh"

namespace tcb {

__device__ __forceinline__ int top_bit64(u64 m) { return m ? 63 - __clzll(static_cast<long long>(m)) : -1; }

// residual^2 of a significant coefficient with planes >= p known
__device__ __forceinline__ double t_sig2(u64 m, int p) {
    if (p == 0) return 0.0;
    const u64 low = m & ((u64{1} << p) - 1);
    const double r = __dsub_rn(__ull2double_rn(low), __ull2double_rn(u64{1} << (p - 1)));
    return __dmul_rn(r, r);
}
__device__ __forceinline__ double t_insig2(u64 m) {
    const double v = __ull2double_rn(m);
    return __dmul_rn(v, v);
}
__device__ __forceinline__ double t_trail_gain(u64 m, int p) { return __dsub_rn(t_sig2(m, p + 1), t_sig2(m, p)); }
__device__ __forceinline__ double t_lead_gain(u64 m, int p) { return __dsub_rn(t_insig2(m), t_sig2(m, p)); }
__device__ __forceinline__ double t_recal(u64 m, int plane) {
    double r;
    if (plane >= 64 || (m >> plane) == 0) r = __ull2double_rn(m);
    else if (plane == 0) r = 0.0;
    else r = __dsub_rn(__ull2double_rn(m & ((u64{1} << plane) - 1)), __ull2double_rn(u64{1} << (plane - 1)));
    return __dmul_rn(r, r);
}
__device__ __forceinline__ double t_diff2(u64 m, u64 dec) {
    const double r = __dsub_rn(__ull2double_rn(m), __ull2double_rn(dec));
    return __dmul_rn(r, r);
}

}  // namespace tcb
