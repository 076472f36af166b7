// Shared FP64 tensor-core (DMMA) tile loop of the batched kernels
// (wavekern.cu: butterfly levels, rootmma.cu: root skeletons).
//
// One CTA of kWarps warps computes a kMT x kNT block of C = A * B:
//   A: kMT output rows x K, read from a column-major matrix P (leading
//      dimension ld) either as A(row, k) = P[row + k ld] (AT = false: the
//      forward products T z, S c) or A(row, k) = P[k + row ld] (AT = true: the
//      transposed products T^T c, S^T u) -- one copy of every matrix serves
//      both directions;
//   B: K x kNT, row k starting at bptr(k, n) (R contiguous doubles of V, or
//      the strided chain rows of u), gathered through the caller's functor.
// Both operands go global -> shared by cp.async in a kStages-deep ring of
// 16-deep K chunks (no register prefetch: the loads of chunk c + kStages - 1
// are in flight while chunk c is multiplied).  Warp w owns rows 16w..16w+15
// (two m8 tiles) x all eight n8 tiles: mma.sync.m8n8k4.f64 with the fragment
// layout A[lane/4][lane%4], B[lane%4][lane/4], D[lane/4][2 (lane%4) + {0,1}].
// Shared strides are padded so every fragment load is bank-conflict free.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace bfb {
namespace dmma {

#ifndef BFB_WAVE_WARPS
#define BFB_WAVE_WARPS 4
#endif
#ifndef BFB_MMA_STAGES
#define BFB_MMA_STAGES 2  // measured at c3: 2 stages 640 pairs/s, 3: 598, 4: 503 (occupancy wins)
#endif
#ifndef BFB_MMA_MINB
#define BFB_MMA_MINB 5  // 4-warp CTAs: <= 102 registers, 5 CTAs per SM (c3: 654 vs 640 pairs/s at 4)
#endif
constexpr int kWarps = BFB_WAVE_WARPS;  // default CTA size (warps); NW below per kernel
constexpr int kNT = 64;           // right-hand-side columns per item (NT: 64, or 32 for <= 8 functions)
#ifndef BFB_MMA_KC
#define BFB_MMA_KC 16
#endif
constexpr int kKC = BFB_MMA_KC;   // K chunk
constexpr int kAR = kKC + 4;      // A tile, row-major (AT = true): [row][k]
constexpr int kStages = BFB_MMA_STAGES;
constexpr int kMinBlocks = BFB_MMA_MINB;  // CTAs per SM the register budget is cut for

template <int NW, int NT = kNT, int TPW = 2>
struct Tile {
    static constexpr int kThreads = 32 * NW;
    static constexpr int kMT = 8 * TPW * NW;  // output rows per block (TPW m8 tiles per warp)
    static constexpr int kAK = kMT + 4;   // A tile, k-major (AT = false): [k][row]
    static constexpr int kAStage = (kKC * kAK > kMT * kAR) ? kKC * kAK : kMT * kAR;
    static constexpr int kBS = NT + 4;    // B tile row stride (doubles): conflict-free fragment loads
    static constexpr int kBStage = kKC * kBS;
    static constexpr int kStageD = kAStage + kBStage;  // doubles per ring stage
    static constexpr int kSmemDoubles = kStages * kStageD;
};
constexpr int kThreads = Tile<kWarps>::kThreads;
constexpr int kMT = Tile<kWarps>::kMT;
constexpr int kSmemDoubles = Tile<kWarps>::kSmemDoubles;  // NT = 64 (the larger)

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

// Accumulator start values: zero, or init(row, n) (a double2 for columns n,
// n + 1 of output row `row`) -- the forward's z[sel] term, or the old value of
// a '+=' output.  Loading them into the accumulators before the K loop hides
// their latency behind the operand staging (as an epilogue add they were the
// level kernels' largest stall).
struct ZeroInit {
    __device__ double2 operator()(int, int) const { return make_double2(0.0, 0.0); }
};

// acc = init + A[m0 .. m0 + kMT) x [0, K) * B[0, K) x [n0, n0 + kNT) for this
// warp's 16 rows; rows >= M and columns >= R are zero.  `sm` holds
// kSmemDoubles.  Ends with a barrier, so the caller may reuse `sm` right away.
template <bool AT, int NW = kWarps, int NT = kNT, int TPW = 2, class BP, class IN = ZeroInit>
__device__ __forceinline__ void mma_block(double (&acc)[TPW][NT / 8][2], int M, int K, int m0, int n0, int R,
                                          const double* __restrict__ P, long long ld, BP bptr, double* sm,
                                          IN init = IN{}) {
    using TL = Tile<NW, NT, TPW>;
    constexpr int kThreads = TL::kThreads, kMT = TL::kMT, kAK = TL::kAK, kAStage = TL::kAStage,
                  kStageD = TL::kStageD, kBS = TL::kBS, kNT = NT, NJ = NT / 8;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#pragma unroll
    for (int t = 0; t < TPW; ++t) {
        const int row = m0 + 8 * TPW * warp + 8 * t + (lane >> 2);
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
            const int n = n0 + 8 * j + 2 * (lane & 3);
            double2 v = make_double2(0.0, 0.0);
            if (row < M && n < R) v = init(row, n);
            acc[t][j][0] = v.x;
            acc[t][j][1] = v.y;
        }
    }
    const int tb = m0 + 8 * TPW * warp;
    const int nt = tb >= M ? 0 : min(TPW, (M - tb + 7) / 8);  // this warp's live m8 tiles
    const int nk = (K + kKC - 1) / kKC;
    auto stage = [&](int c) {
        double* As = sm + (c % kStages) * kStageD;
        double* Bs = As + kAStage;
        const int kc = c * kKC;
        for (int e = tid; e < kKC * kMT; e += kThreads) {
            int r, k;
            if (AT) {
                r = e / kKC;
                k = e - r * kKC;
            } else {
                k = e / kMT;
                r = e - k * kMT;
            }
            const int row = m0 + r, kk = kc + k;
            double* d = AT ? As + r * kAR + k : As + k * kAK + r;
            if (row < M && kk < K)
                cp_async8(d, AT ? P + kk + static_cast<long long>(row) * ld : P + row + static_cast<long long>(kk) * ld);
            else
                *d = 0.0;
        }
        for (int e = tid; e < kKC * (kNT / 2); e += kThreads) {
            const int k = e / (kNT / 2), h = e - k * (kNT / 2);
            const int n = n0 + 2 * h, kk = kc + k;
            double* d = Bs + k * kBS + 2 * h;
            if (kk < K && n < R) {
                cp_async16(d, bptr(kk, n));
            } else {
                d[0] = 0.0;
                d[1] = 0.0;
            }
        }
    };
#pragma unroll
    for (int s = 0; s < kStages - 1; ++s) {
        if (s < nk) stage(s);
        cp_async_commit();
    }
    const int ka = lane & 3, ra = 8 * TPW * warp + (lane >> 2);
    for (int c = 0; c < nk; ++c) {
        cp_async_wait<kStages - 2>();  // this thread's copies of chunk c landed
        __syncthreads();               // everyone's; and chunk c - 1 is done (its slot is restaged next)
        if (c + kStages - 1 < nk) stage(c + kStages - 1);
        cp_async_commit();
        const double* As = sm + (c % kStages) * kStageD;
        const double* b = As + kAStage + ka * kBS + (lane >> 2);
        if (nt > 0) {
#pragma unroll
            for (int s = 0; s < kKC / 4; ++s) {
                const int k = 4 * s + ka;
                double bv[NJ];
#pragma unroll
                for (int j = 0; j < NJ; ++j) bv[j] = b[4 * s * kBS + 8 * j];
#pragma unroll
                for (int t = 0; t < TPW; ++t) {
                    if (t < nt) {
                        const double at = AT ? As[(ra + 8 * t) * kAR + k] : As[k * kAK + ra + 8 * t];
#pragma unroll
                        for (int j = 0; j < NJ; ++j) dmma(acc[t][j], at, bv[j]);
                    }
                }
            }
        }
    }
    cp_async_wait<0>();
    __syncthreads();
}

}  // namespace dmma
}  // namespace bfb
