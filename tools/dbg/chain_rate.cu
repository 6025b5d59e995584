// Latency of one range-coder step (range = norm(floor(range / T) * f)) for
// several formulations: one warp, records in registers, clock64 over 1M steps.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o chain_rate chain_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
typedef uint32_t u32;
typedef uint64_t u64;

template <int V>
__global__ void chain(const u32* T_in, const u32* f_in, int n, u32* out, long long* cyc) {
    // 64 distinct records cycled (T in [2^15, 2^16), f <= T)
    u32 T[8], f[8], th1[8], th2[8];
    u64 M[8];
    double inv[8];
    for (int i = 0; i < 8; ++i) {
        T[i] = T_in[i]; f[i] = f_in[i];
        M[i] = (~0ull / T[i]) + 1;
        th1[i] = ((1u << 24) + f[i] - 1) / f[i];
        th2[i] = ((1u << 16) + f[i] - 1) / f[i];
        inv[i] = __drcp_ru((double)T[i]) ;
    }
    u32 range = 0xFFFFFFFFu;
    long long t0 = clock64();
    for (int it = 0; it < n; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            u32 q;
            if (V == 0) {  // two multiply-highs (current)
                const u32 t = __umulhi(range, (u32)M[i]);
                q = (u32)(((u64)range * (u32)(M[i] >> 32) + t) >> 32);
            } else if (V == 1) {  // 64-bit multiply-high
                q = (u32)__umul64hi((u64)range, M[i]);
            } else if (V == 2) {  // fp64: floor(range * (1/T rounded up)), rz
                q = (u32)__double2uint_rz(__dmul_rz((double)range, inv[i]));
            } else {  // fp32 estimate + one integer correction
                const u32 q0 = __float2uint_rz(__fmul_rz(__uint2float_rz(range), __frcp_rz((float)T[i])));
                const u32 r = range - q0 * T[i];
                q = q0 + (r >= T[i]) + (r >= 2 * T[i]);
            }
            const u32 mul = q <= th2[i] - 1 ? f[i] << 16 : (q < th1[i] ? f[i] << 8 : f[i]);
            range = q * mul;
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { out[0] = range; cyc[0] = t1 - t0; }
}

int main() {
    u32 hT[8], hf[8];
    for (int i = 0; i < 8; ++i) { hT[i] = 40000 + 1234 * i; hf[i] = 1 + 777 * i * i; }
    u32 *dT, *df, *dout; long long* dc;
    cudaMalloc(&dT, 32); cudaMalloc(&df, 32); cudaMalloc(&dout, 4); cudaMalloc(&dc, 8);
    cudaMemcpy(dT, hT, 32, cudaMemcpyHostToDevice); cudaMemcpy(df, hf, 32, cudaMemcpyHostToDevice);
    const int n = 1 << 17;
    u32 ref = 0;
    auto run = [&](auto kern, const char* name) {
        kern<<<1, 32>>>(dT, df, 10, dout, dc); cudaDeviceSynchronize();
        kern<<<1, 32>>>(dT, df, n, dout, dc); cudaDeviceSynchronize();
        long long c; u32 o; cudaMemcpy(&c, dc, 8, cudaMemcpyDeviceToHost); cudaMemcpy(&o, dout, 4, cudaMemcpyDeviceToHost);
        printf("%-34s %.1f cycles/step  (final range %08x%s)\n", name, (double)c / (n * 8.0), o, ref && o != ref ? " MISMATCH" : "");
        if (!ref) ref = o;
    };
    run(chain<0>, "two umulhi (current)");
    run(chain<1>, "umul64hi");
    run(chain<2>, "fp64 rz multiply");
    run(chain<3>, "fp32 estimate + correction");
    return 0;
}
