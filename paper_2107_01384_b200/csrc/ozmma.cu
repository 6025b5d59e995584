// Ozaki-scheme digit products on the B200's 5th-generation tensor cores.
//
// ozaki.cu splits fp64 rows into five exact int8 digit slices; the products of
// slice pairs (s, t) of one level L = s + t all carry the weight 2^-(12 + 7 L),
// and levels L <= 4 are kept.  This kernel computes, per 128 x 96 output tile,
// all five level sums at once:
//
// * warp 0 (one thread) stages, per 64-byte k slab, the five A slices
//   (128 rows x 64 B each) and the five B slices (96 rows) into shared memory
//   with two bulk copies (cp.async.bulk: the operands are stored blocked and
//   pre-swizzled, ozmma.cuh), in a 3-stage mbarrier ring -- 10 tiles feed 15
//   slice-pair products, so each byte fetched from L2 is used three times;
// * warp 1 (one thread) issues tcgen05.mma.kind::i8 (M 128, N 96, K 32) for
//   every pair (s, t), s + t <= 4, into accumulator L = s + t: five int32
//   128 x 96 accumulators side by side in tensor memory (480 of its 512
//   columns); tcgen05.commit releases each stage back to the producer;
// * warps 2-5 (the epilogue, one TMEM lane quarter each) read the five
//   accumulators with tcgen05.ld and combine them exactly,
//   T = sum_L C_L 2^(7 (4 - L)) in int64, then either add T to the Gram
//   accumulator (integer atomics: the sum is exact, so the order of the
//   k-chunks does not matter) or scale it into the TTM's fp64 output.
//
// int32 is exact per accumulation: |digit| <= 64, so a level-L term is at
// most (L + 1) 2^12 per k; the Gram runs k-chunks of 2^15 (5 * 2^27 < 2^31),
// the TTM at most 4096 k per slice.
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"
#include "ozmma.cuh"

namespace tcb {

namespace {

constexpr int kTM = 128, kTN = 96;    // tile (M = TMEM lanes, N = columns per accumulator)
constexpr int kBK = 64;               // bytes of k per slab (the swizzle span)
constexpr int kStages = 3;
constexpr u32 kATile = kTM * kBK;     // 8192 B
constexpr u32 kBTile = kTN * kBK;     // 6144 B
constexpr u32 kStageBytes = kOzSlices * (kATile + kBTile);  // 71680 B
constexpr u64 kGramKC = u64{1} << 15;  // k per Gram work item (int32-exact)
constexpr int kEpiWarps = 8;           // two per TMEM lane quarter, each half of the columns
constexpr int kThreads = 32 * (2 + kEpiWarps);  // producer, MMA, epilogue
constexpr size_t kSmem = static_cast<size_t>(kStages) * kStageBytes + 1024 /* alignment */ + 256 /* barriers */;

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ u32 smem_u32(const void* p) { return static_cast<u32>(__cvta_generic_to_shared(p)); }

__device__ __forceinline__ void mbar_init(u32 bar, u32 count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(u32 bar, u32 bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(u32 bar, u32 parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_load(u32 dst, const void* src, u32 bytes, u32 bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(reinterpret_cast<u64>(src)), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(u32 bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tc_mma_i8(u32 d, u64 a, u64 b, u32 idesc, u32 acc) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(a), "l"(b), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void tc_ld16(u32 taddr, int (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void tc_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// K-major operand tile in shared memory, 64-byte swizzle: rows of 64 B, 8-row
// groups 512 B apart (SBO), version 1 (sm_100), layout type 4 = SWIZZLE_64B
__device__ __forceinline__ u64 smem_desc(u32 saddr) {
    u64 d = static_cast<u64>((saddr >> 4) & 0x3FFFu);
    d |= u64{1} << 16;                 // LBO (unused for a swizzled K-major tile)
    d |= static_cast<u64>(512 >> 4) << 32;  // SBO
    d |= u64{1} << 46;                 // descriptor version
    d |= u64{4} << 61;                 // SWIZZLE_64B
    return d;
}
// kind::i8 instruction descriptor: D s32, A and B signed int8, both K-major, M 128, N 96
constexpr u32 kIdesc = (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<u32>(kTN >> 3) << 17) |
                       (static_cast<u32>(kTM >> 4) << 24);

struct OzParams {
    u32 items;          // work items (the grid strides over them)
    const int8_t* A;    // M operand, 128-row blocks
    const int8_t* B;    // N operand, 96-row blocks
    u64 nslab_all;      // slabs per block row (both operands)
    u32 nslab;          // slabs per work item
    int mode;           // 0: Gram (int64 atomics into acc), 1: TTM (fp64 into out)
    // Gram: item -> (lower-triangle tile, k-chunk), chunk-major
    const int2* tiles;  // (m tile, n tile)
    u32 ntiles;
    long long* acc;
    u64 acc_ld;
    // TTM: item -> (m tile, n tile), n fastest
    u32 ntn;
    u64 m_rows, n_rows;
    const int* exa;
    const int* exb;
    double* out;
    int dbg;  // measurement only (TCB_OZ_DBG): 1 = no loads, 2 = no MMAs, 3 = no epilogue
};

__device__ __forceinline__ void item_coords(const OzParams& P, u32 item, int& mt, int& nt, u64& kbase) {
    if (P.mode == 0) {
        const u32 t = item % P.ntiles, c = item / P.ntiles;
        const int2 tl = P.tiles[t];
        mt = tl.x;
        nt = tl.y;
        kbase = static_cast<u64>(c) * (kGramKC / kBK);  // in slabs
    } else {
        mt = static_cast<int>(item / P.ntn);
        nt = static_cast<int>(item % P.ntn);
        kbase = 0;
    }
}

// Persistent: CTA b takes items b, b + grid, ...  The producer runs ahead into
// the next item's slabs while the last MMAs and the epilogue of the current one
// finish; the MMA issuer waits for the epilogue to drain the accumulators
// (tmem_empty) before it starts the next item.
__global__ void __launch_bounds__(kThreads, 1) oz_mma_kernel(const OzParams P) {
    extern __shared__ u8 oz_smem_raw[];
    u8* smem = reinterpret_cast<u8*>((reinterpret_cast<uintptr_t>(oz_smem_raw) + 1023) & ~uintptr_t{1023});
    u64* bars = reinterpret_cast<u64*>(smem + kStages * kStageBytes);  // full[3], empty[3], tmem_full, tmem_empty
    u32* tmem_slot = reinterpret_cast<u32*>(bars + 2 * kStages + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const u32 bar_tfull = smem_u32(&bars[2 * kStages]), bar_tempty = smem_u32(&bars[2 * kStages + 1]);

    if (threadIdx.x == 0) {
        for (int i = 0; i < kStages; ++i) {
            mbar_init(smem_u32(&bars[i]), 1);
            mbar_init(smem_u32(&bars[kStages + i]), 1);
        }
        mbar_init(bar_tfull, 1);
        mbar_init(bar_tempty, kEpiWarps);  // one arrival per epilogue warp
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {  // the whole warp allocates the 512 TMEM columns (one CTA per SM)
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const u32 tmem = *tmem_slot;
    const u32 sbase = smem_u32(smem);

    if (warp == 0 && lane == 0) {
        // ---------------- producer: two bulk copies per slab
        u32 g = 0;  // slab counter over all of this CTA's items (stage ring position)
        for (u32 item = blockIdx.x; item < P.items; item += gridDim.x) {
            int mt, nt;
            u64 kbase;
            item_coords(P, item, mt, nt, kbase);
            const int8_t* srcA = P.A + (static_cast<u64>(mt) * P.nslab_all + kbase) * (kOzSlices * kATile);
            const int8_t* srcB = P.B + (static_cast<u64>(nt) * P.nslab_all + kbase) * (kOzSlices * kBTile);
            for (u32 q = 0; q < P.nslab; ++q, ++g) {
                const u32 st = g % kStages, ph = (g / kStages) & 1u;
                mbar_wait(smem_u32(&bars[kStages + st]), ph ^ 1u);
                const u32 full = smem_u32(&bars[st]);
                if (P.dbg == 1) {
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(full) : "memory");
                    continue;
                }
                mbar_expect_tx(full, kStageBytes);
                const u32 sa = sbase + st * kStageBytes, sb = sa + kOzSlices * kATile;
                bulk_load(sa, srcA + static_cast<u64>(q) * (kOzSlices * kATile), kOzSlices * kATile, full);
                bulk_load(sb, srcB + static_cast<u64>(q) * (kOzSlices * kBTile), kOzSlices * kBTile, full);
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ---------------- MMA issuer
        u32 g = 0, it = 0;
        for (u32 item = blockIdx.x; item < P.items; item += gridDim.x, ++it) {
            if (it > 0) {  // the epilogue has read the previous item's accumulators
                mbar_wait(bar_tempty, (it - 1) & 1u);
                tc_fence_after();
            }
            for (u32 q = 0; q < P.nslab; ++q, ++g) {
                const u32 st = g % kStages, ph = (g / kStages) & 1u;
                mbar_wait(smem_u32(&bars[st]), ph);
                tc_fence_after();
                const u32 sa = sbase + st * kStageBytes, sb = sa + kOzSlices * kATile;
                if (P.dbg != 2) {
#pragma unroll
                    for (int L = 0; L < kOzSlices; ++L) {
#pragma unroll
                        for (int s = 0; s <= L; ++s) {
                            const u64 da = smem_desc(sa + s * kATile), db = smem_desc(sb + (L - s) * kBTile);
#pragma unroll
                            for (int kk = 0; kk < kBK / 32; ++kk)  // K = 32 bytes per MMA: +32 B = +2 in the address field
                                tc_mma_i8(tmem + L * kTN, da + 2 * kk, db + 2 * kk, kIdesc, (q | s | kk) != 0);
                        }
                    }
                }
                tc_commit(smem_u32(&bars[kStages + st]));  // the stage is free once these MMAs have read it
            }
            tc_commit(bar_tfull);  // this item's accumulators are complete
        }
    } else if (warp >= 2) {
        // ---------------- epilogue: lane quarter (warp % 4) of the tile's rows, half of its columns
        const int quarter = warp & 3, half = (warp - 2) >> 2;
        const u32 trow = tmem + (static_cast<u32>(quarter * 32) << 16);
        u32 it = 0;
        for (u32 item = blockIdx.x; item < P.items; item += gridDim.x, ++it) {
            int mt, nt;
            u64 kbase;
            item_coords(P, item, mt, nt, kbase);
            mbar_wait(bar_tfull, it & 1u);
            tc_fence_after();
            const u64 m = static_cast<u64>(mt) * kTM + quarter * 32 + lane;
            const int ea = P.mode == 1 && m < P.m_rows ? P.exa[m] - 40 : 0;
            constexpr int kHalf = kTN / 2;
#pragma unroll 1
            for (int j0 = half * kHalf; j0 < (half + 1) * kHalf; j0 += 16) {
                long long T[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) T[j] = 0;
#pragma unroll
                for (int L = 0; L < kOzSlices; ++L) {
                    int v[16];
                    tc_ld16(trow + L * kTN + j0, v);
                    tc_wait_ld();
#pragma unroll
                    for (int j = 0; j < 16; ++j) T[j] += static_cast<long long>(v[j]) << (7 * (kOzSlices - 1 - L));
                }
                if (P.dbg == 3 && j0 + 16 < (half + 1) * kHalf) continue;  // measurement: accumulators not drained
                if (j0 + 16 >= (half + 1) * kHalf) {  // this warp's accumulators read: the next item may start
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar_tempty) : "memory");
                }
                const u64 n0 = static_cast<u64>(nt) * kTN + j0;
                if (P.dbg == 3) continue;
                if (P.mode == 0) {
                    unsigned long long* a = reinterpret_cast<unsigned long long*>(P.acc + m * P.acc_ld + n0);
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (T[j]) atomicAdd(a + j, static_cast<unsigned long long>(T[j]));
                    continue;
                }
                if (m >= P.m_rows) continue;
                // TTM: scale by the power of two 2^(exa + exb - 40) (exact: normal results);
                // this thread's 16 consecutive outputs of row m, 16 bytes per store
                double o[16];
#pragma unroll
                for (int j = 0; j < 16; ++j) {
                    const int e = ea + (n0 + j < P.n_rows ? __ldg(P.exb + n0 + j) : 0);
                    const double sc = __longlong_as_double(static_cast<long long>(e + 1023) << 52);
                    const double x = static_cast<double>(T[j]);
                    o[j] = e > -1000 && e < 1000 ? x * sc : scalbn(x, e);
                }
                double* dst = P.out + m * P.n_rows + n0;
                if (n0 + 16 <= P.n_rows && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
                    for (int j = 0; j < 16; j += 2) *reinterpret_cast<double2*>(dst + j) = make_double2(o[j], o[j + 1]);
                } else {
#pragma unroll
                    for (int j = 0; j < 16; ++j)
                        if (n0 + j < P.n_rows) dst[j] = o[j];
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// ------------------------------------------------------------------ host side
int dbg_mode() {
    const char* e = std::getenv("TCB_OZ_DBG");
    return e ? std::atoi(e) : 0;
}

void set_smem_attr() {
    TCB_ONCE_PER_DEVICE(TCB_CUDA(cudaFuncSetAttribute(oz_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                      static_cast<int>(kSmem))));
}

}  // namespace

u64 oz_gram_acc_ld(u64 rows) { return (rows + kTN - 1) / kTN * kTN; }

void oz_gram_tc(const int8_t* DA, const int8_t* DB, u64 rows, u64 nslab, long long* acc, u64 acc_ld, cudaStream_t s) {
    // tiles (a, b) meeting the lower triangle: 96 b <= 128 a + 127
    std::vector<int2> tl;
    const u64 nta = (rows + kTM - 1) / kTM, ntb = (rows + kTN - 1) / kTN;
    for (u64 a = 0; a < nta; ++a)
        for (u64 b = 0; b < ntb; ++b)
            if (b * kTN <= a * kTM + kTM - 1) tl.push_back(make_int2(static_cast<int>(a), static_cast<int>(b)));
    oz_gram_tc_tiles(DA, DB, rows, nslab, tl, acc, acc_ld, s);
}

void oz_gram_tc_tiles(const int8_t* DA, const int8_t* DB, u64 rows, u64 nslab, const std::vector<int2>& tl,
                      long long* acc, u64 acc_ld, cudaStream_t s) {
    if (nslab % (kGramKC / kBK)) throw Error("ozaki: Gram k not a multiple of the chunk");
    if (tl.empty()) return;
    set_smem_attr();
    const u64 ntb = (rows + kTN - 1) / kTN;
    if (acc_ld < ntb * kTN) throw Error("ozaki: Gram accumulator too narrow");
    DevBuf<int2> dtl(tl.size(), s);
    dtl.upload(tl.data(), tl.size());
    OzParams P{};
    P.A = DA;
    P.B = DB;
    P.nslab_all = nslab;
    P.nslab = static_cast<u32>(kGramKC / kBK);
    P.mode = 0;
    P.dbg = dbg_mode();
    P.tiles = dtl.p;
    P.ntiles = static_cast<u32>(tl.size());
    P.acc = acc;
    P.acc_ld = acc_ld;
    const u64 items = tl.size() * (nslab / P.nslab);
    P.items = static_cast<u32>(items);
    ProfScope prof(kTc, s);
    oz_mma_kernel<<<static_cast<unsigned>(std::min<u64>(items, sm_count())), kThreads, kSmem, s>>>(P);
    count_launch();
    TCB_LAUNCH();
}

void oz_ttm_tc(const int8_t* A, u64 m_rows, const int8_t* B, u64 n_rows, u64 nslab, const int* exa, const int* exb,
               double* out, cudaStream_t s) {
    if (nslab == 0 || nslab > 64) throw Error("ozaki: TTM k must be at most 4096");
    set_smem_attr();
    OzParams P{};
    P.A = A;
    P.B = B;
    P.nslab_all = nslab;
    P.nslab = static_cast<u32>(nslab);
    P.mode = 1;
    P.dbg = dbg_mode();
    P.ntn = static_cast<u32>((n_rows + kTN - 1) / kTN);
    P.m_rows = m_rows;
    P.n_rows = n_rows;
    P.exa = exa;
    P.exb = exb;
    P.out = out;
    const u64 items = (m_rows + kTM - 1) / kTM * P.ntn;
    P.items = static_cast<u32>(items);
    ProfScope prof(kTc, s);
    oz_mma_kernel<<<static_cast<unsigned>(std::min<u64>(items, sm_count())), kThreads, kSmem, s>>>(P);
    count_launch();
    TCB_LAUNCH();
}

}  // namespace tcb
