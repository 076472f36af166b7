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
// A work item = (stripe, kMT-row block of the output) x a 64-column chunk of
// the right-hand sides; the tile loop (both operands through a cp.async ring,
// DMMA m8n8k4) is dmma_tile.cuh.  S is stored once, column-major, and read as
// S (forward) or S^T (transpose).
//
// Layouts (cell-major, so a stripe's operand is one dense row-major matrix):
//   C     [c_cells][batch][4]   written by the event program (ShtIO::cell_major)
//   ypart [y_rows][batch][4]    summed over root groups by combine_kernel
//   u     [plan][batch][l][4]   (transpose input, the engine's usual staging)
#include <cuda_runtime.h>

#include <algorithm>
#include <type_traits>
#include <mutex>
#include <vector>

#include "dmma_tile.cuh"
#include "rootmv.hpp"

namespace bfb {

namespace {

using namespace dmma;

// CTA size of the transpose (S^T blocks); the forward uses the default.

#ifndef BFB_ROOT_BWD_WARPS
#define BFB_ROOT_BWD_WARPS 4  // 8 measured 3.82 vs 3.10 ms at c3
#endif
constexpr int kBwdWarps = BFB_ROOT_BWD_WARPS;
template <bool BWD>
constexpr int root_warps() { return BWD ? kBwdWarps : kWarps; }

template <bool BWD, int NT>
__global__ void __launch_bounds__(32 * root_warps<BWD>(), 16 / root_warps<BWD>()) root_mma_kernel(RootMmaArgs a) {
    constexpr int NW = root_warps<BWD>();
    extern __shared__ __align__(16) double ring[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint2 it = reinterpret_cast<const uint2*>(a.items)[blockIdx.x];
    const RootStripeDesc d = a.stripes[it.x];
    const int m0 = static_cast<int>(it.y);
    const int R = 4 * a.batch;
    const int n0 = NT * static_cast<int>(blockIdx.y);
    const int M = BWD ? static_cast<int>(d.rank) : static_cast<int>(d.rows);
    const int K = BWD ? static_cast<int>(d.rows) : static_cast<int>(d.rank);
    const double* S = a.data + d.s_off;
    double acc[2][NT / 8][2];
    if (!BWD) {
        const double* C = a.C + static_cast<long long>(d.coff) * R;
        auto bp = [&](int k, int n) { return C + static_cast<long long>(k) * R + n; };
        if (a.accumulate && a.to_u)  // later root groups add onto the chain rows
            mma_block<false, NW, NT>(acc, M, K, m0, n0, R, S, d.lds, bp, ring, [&](int row, int n) {
                return *reinterpret_cast<const double2*>(
                    a.u_out + ((static_cast<long long>(d.plan) * a.batch + (n >> 2)) * a.l + d.yin + row) * 4 + (n & 3));
            });
        else
            mma_block<false, NW, NT>(acc, M, K, m0, n0, R, S, d.lds, bp, ring);
    } else if (a.rows_cm) {  // plan-set apply: stacked rows, R contiguous doubles per row
        const double* Wr = a.rows_cm + static_cast<long long>(d.pad[1]) * R;
        mma_block<true, NW, NT>(acc, M, K, m0, n0, R, S, d.lds,
                                [&](int k, int n) { return Wr + static_cast<long long>(k) * R + n; }, ring);
    } else {
        const double* U = a.u + (static_cast<long long>(d.plan) * a.batch * a.l + d.yin) * 4;
        const long long bs = static_cast<long long>(a.l) * 4;  // between members
        mma_block<true, NW, NT>(acc, M, K, m0, n0, R, S, d.lds,
                        [&](int k, int n) { return U + (n >> 2) * bs + static_cast<long long>(k) * 4 + (n & 3); }, ring);
    }

    // ---- epilogue ---------------------------------------------------------------
    // transpose: '=' into the stripe's coefficient cells; forward: '=' into its
    // partial rows, or straight into the chain rows u (a.to_u; '+=' for root
    // groups after the first, which run as later launches)
#pragma unroll
    for (int t = 0; t < 2; ++t) {
        const int row = m0 + 16 * warp + 8 * t + (lane >> 2);
        if (row >= M) continue;
#pragma unroll
        for (int j = 0; j < NT / 8; ++j) {
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
            if (!BWD && a.accumulate && !a.to_u) {
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
    // column tiles as narrow as the right-hand sides allow (8 / 16 / 32 / 64)
    const int R = 4 * args.batch;
    const int nt = R <= 8 ? 8 : R <= 16 ? 16 : R <= 32 ? 32 : kNT;
    const dim3 grid(static_cast<unsigned>(n_items), static_cast<unsigned>((R + nt - 1) / nt));
    auto go = [&](auto kern, int threads, std::size_t smem) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        kern<<<grid, threads, smem, st>>>(a);
    };
    constexpr int WB = root_warps<true>(), WF = root_warps<false>();
    auto run = [&](auto ntc) {
        constexpr int NT = decltype(ntc)::value;
        if (transpose)
            go(root_mma_kernel<true, NT>, 32 * WB, Tile<WB, NT>::kSmemDoubles * sizeof(double));
        else
            go(root_mma_kernel<false, NT>, 32 * WF, Tile<WF, NT>::kSmemDoubles * sizeof(double));
    };
    switch (nt) {
    case 8: run(std::integral_constant<int, 8>{}); break;
    case 16: run(std::integral_constant<int, 16>{}); break;
    case 32: run(std::integral_constant<int, 32>{}); break;
    default: run(std::integral_constant<int, 64>{}); break;
    }
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
        for (std::uint32_t m = 0; m < stripes[s].rank; m += Tile<kBwdWarps>::kMT) {
            bwd.push_back(s);
            bwd.push_back(m);
        }
    }
}

}  // namespace bfb
