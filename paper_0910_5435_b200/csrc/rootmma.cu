// Batched root stage of the split SHT programs on the FP64 tensor cores.
//
// The root stage of every butterfly plan (reference src/butterfly.cpp:430-440
// forward, :452-460 transpose) multiplies each root stripe's dense skeleton S
// (rows x rank, the "leaf-level dense Legendre block" of the north_star) with
// that stripe's coefficient vector.  With a batch of B functions there are
// R = 4B right-hand sides (+-m x re/im per function) and the product becomes a
// real dense contraction:
//   forward:   Y[stripe rows][R] = S   * C[stripe cells][R]
//   transpose: C[stripe cells][R] = S^T * U[stripe rows][R]
// so each skeleton word is read from HBM once per launch for all R right-hand
// sides instead of once per function (rootmv.cu), and the work is FP64 DMMA
// (mma.sync.m8n8k4.f64) rather than HBM streaming.
//
// CTA = 8 warps, one work item = (stripe, 128-row block of the output) x a
// 64-column chunk of the right-hand sides.  Warp w owns output rows
// 16w..16w+15 of the block (two m8 tiles) x all 8 n8 tiles: 32 accumulators
// per lane.  A fragments (the skeleton, read exactly once per item) come
// straight from global memory one K chunk ahead; B (the coefficient / row
// vectors, shared by the 8 warps) is staged per 16-deep K chunk in a
// double-buffered shared-memory tile with cp.async, rows padded to 68 doubles
// so the fragment loads are bank-conflict free.
//
// Layouts (cell-major, so a stripe's operand is one dense row-major matrix):
//   C     [c_cells][batch][4]   written by the event program (ShtIO::cell_major)
//   ypart [y_rows][batch][4]    summed over root groups by combine_kernel
//   u     [plan][batch][l][4]   (transpose input, the engine's usual staging)
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "rootmv.hpp"

namespace bfb {

namespace {

constexpr int kWarps = 8;
constexpr int kThreads = 32 * kWarps;
constexpr int kMT = 16 * kWarps;  // output rows per item
constexpr int kNT = 64;           // right-hand-side columns per item
constexpr int kKC = 16;           // K chunk staged in shared memory
constexpr int kBS = kNT + 4;      // padded row stride of the B tile (doubles)
constexpr int kKS = kKC / 4;      // k4 steps per chunk

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait0() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
// D(8x8) += A(8x4) * B(4x8); lane holds A[lane/4][lane%4], B[lane%4][lane/4],
// D[lane/4][2*(lane%4) + {0,1}].
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

template <bool BWD>
__global__ void __launch_bounds__(kThreads, 2) root_mma_kernel(RootMmaArgs a) {
    __shared__ __align__(16) double bs[2][kKC * kBS];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint2 it = reinterpret_cast<const uint2*>(a.items)[blockIdx.x];
    const RootStripeDesc d = a.stripes[it.x];
    const int m0 = static_cast<int>(it.y);
    const int R = 4 * a.batch;
    const int n0 = kNT * static_cast<int>(blockIdx.y);
    const int M = BWD ? static_cast<int>(d.rank) : static_cast<int>(d.rows);
    const int K = BWD ? static_cast<int>(d.rows) : static_cast<int>(d.rank);
    const double* S = a.data + d.s_off;
    const long long lds = d.lds;

    // ---- B tile staging: chunk kc of K, 64 columns from n0 -------------------
    auto stage = [&](int buf, int kc) {
        double* dst = bs[buf];
        for (int e = tid; e < kKC * (kNT / 2); e += kThreads) {
            const int k = e / (kNT / 2), h = e - k * (kNT / 2);
            const int n = n0 + 2 * h;
            double* p = dst + k * kBS + 2 * h;
            const int kk = kc + k;
            if (kk < K && n < R) {
                const double* src;
                if (!BWD) {
                    src = a.C + (static_cast<long long>(d.coff) + kk) * R + n;
                } else {
                    const int b = n >> 2, c = n & 3;
                    src = a.u + ((static_cast<long long>(d.plan) * a.batch + b) * a.l + d.yin + kk) * 4 + c;
                }
                cp_async16(p, src);
            } else {
                p[0] = 0.0;
                p[1] = 0.0;
            }
        }
    };
    // ---- A fragments of one K chunk (two m8 tiles x kKS k-steps) ------------
    const int ra = m0 + 16 * warp + (lane >> 2);  // output row of tile 0 (tile 1: +8)
    const int tb = m0 + 16 * warp, nt = tb >= M ? 0 : (tb + 8 >= M ? 1 : 2);  // this warp's live m8 tiles
    const int ka = lane & 3;
    auto load_a = [&](double (&av)[2][kKS], int kc) {
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int s = 0; s < kKS; ++s) {
                const int row = ra + 8 * t, k = kc + 4 * s + ka;
                const bool ok = row < M && k < K;
                // forward A = S[row][k]; transpose A = S^T[row][k] = S[k][row]
                const long long off = BWD ? static_cast<long long>(row) * lds + k : static_cast<long long>(k) * lds + row;
                av[t][s] = ok ? __ldcs(S + off) : 0.0;
            }
    };

    double acc[2][8][2];
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[t][j][0] = acc[t][j][1] = 0.0;

    const int nk = (K + kKC - 1) / kKC;
    double av[2][kKS], an[2][kKS];
    if (nk > 0) {
        stage(0, 0);
        cp_async_commit();
        load_a(av, 0);
    }
    for (int c = 0; c < nk; ++c) {
        const int buf = c & 1;
        if (c + 1 < nk) {
            stage(buf ^ 1, (c + 1) * kKC);
            cp_async_commit();
            load_a(an, (c + 1) * kKC);
            cp_async_wait1();
        } else {
            cp_async_wait0();
        }
        __syncthreads();
        const double* b = bs[buf] + ka * kBS + (lane >> 2);
        // m8 tiles past M would multiply zeros: skipped (warp-uniform), which
        // matters for the many nodes / stripes whose rank is below 128
        if (nt == 2) {
#pragma unroll
            for (int s = 0; s < kKS; ++s) {
                double bv[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) bv[j] = b[4 * s * kBS + 8 * j];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    dmma(acc[0][j], av[0][s], bv[j]);
                    dmma(acc[1][j], av[1][s], bv[j]);
                }
            }
        } else if (nt == 1) {
#pragma unroll
            for (int s = 0; s < kKS; ++s) {
                double bv[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) bv[j] = b[4 * s * kBS + 8 * j];
#pragma unroll
                for (int j = 0; j < 8; ++j) dmma(acc[0][j], av[0][s], bv[j]);
            }
        }
        __syncthreads();  // the buffer is restaged two chunks later
        if (c + 1 < nk) {
#pragma unroll
            for (int t = 0; t < 2; ++t)
#pragma unroll
                for (int s = 0; s < kKS; ++s) av[t][s] = an[t][s];
        }
    }

    // ---- epilogue ---------------------------------------------------------------
    // transpose: '=' into the stripe's coefficient cells; forward: '=' into its
    // partial rows, or straight into the chain rows u (a.to_u; '+=' for root
    // groups after the first, which run as later launches)
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int row = ra + 8 * t;
        if (row >= M) continue;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int n = n0 + 8 * j + 2 * (lane & 3);
            if (n >= R) continue;
            double2 v = make_double2(acc[t][j][0], acc[t][j][1]);
            double* p;
            if (BWD)
                p = a.C + (static_cast<long long>(d.coff) + row) * R + n;
            else if (!a.to_u)
                p = a.ypart + (static_cast<long long>(d.yout) + row) * R + n;
            else
                p = a.u_out + ((static_cast<long long>(d.plan) * a.batch + (n >> 2)) * a.l + d.yin + row) * 4 + (n & 3);
            if (!BWD && a.accumulate) {
                const double2 o = *reinterpret_cast<const double2*>(p);
                v.x += o.x;
                v.y += o.y;
            }
            *reinterpret_cast<double2*>(p) = v;
        }
    }
}

}  // namespace

cudaError_t launch_roots_mma(const RootMmaArgs& args, bool transpose, cudaStream_t st, int item0, int n_items) {
    if (n_items < 0) n_items = (transpose ? args.n_bwd : args.n_fwd) - item0;
    if (n_items <= 0 || args.batch == 0) return cudaSuccess;
    RootMmaArgs a = args;
    a.items = (transpose ? args.bwd_items : args.fwd_items) + 2 * item0;
    const dim3 grid(static_cast<unsigned>(n_items), static_cast<unsigned>((4 * args.batch + kNT - 1) / kNT));
    if (transpose)
        root_mma_kernel<true><<<grid, kThreads, 0, st>>>(a);
    else
        root_mma_kernel<false><<<grid, kThreads, 0, st>>>(a);
    return cudaGetLastError();
}

// Work items of the tensor-core root kernels: (stripe, first output row) per
// 128-row block of S (forward) or of S^T (transpose), largest stripes first
// (the stripes are already sorted by size).
// fwd_group[g] = first forward item of root group g (stripes sorted by group).
void root_mma_items(const std::vector<RootStripeDesc>& stripes, std::vector<std::uint32_t>& fwd,
                    std::vector<std::uint32_t>& bwd, std::vector<int>* fwd_group) {
    fwd.clear();
    bwd.clear();
    for (std::uint32_t s = 0; s < stripes.size(); ++s) {
        if (fwd_group)
            while (static_cast<int>(fwd_group->size()) <= static_cast<int>(stripes[s].pad[0]))
                fwd_group->push_back(static_cast<int>(fwd.size() / 2));
        for (std::uint32_t m = 0; m < stripes[s].rows; m += kMT) {
            fwd.push_back(s);
            fwd.push_back(m);
        }
        for (std::uint32_t m = 0; m < stripes[s].rank; m += kMT) {
            bwd.push_back(s);
            bwd.push_back(m);
        }
    }
}

}  // namespace bfb
