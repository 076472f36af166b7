// Device side of the level-synchronous wave programs (waves.hpp): one launch
// per butterfly level applies every StripeId of every plan to all R = 4B
// right-hand sides on the FP64 tensor cores (mma.sync.m8n8k4.f64 -> DMMA).
//
// CTA = 8 warps; a work item is one node (forward) or one pair of nodes that
// share an input vector (transpose) x a 64-column chunk of the right-hand
// sides (blockIdx.y).  The output rows are walked in 128-row blocks: warp w
// owns rows 16w..16w+15 (two m8 tiles) x eight n8 tiles.  A (the
// interpolation matrix, read exactly once per item) is loaded from global
// memory one K chunk ahead; B (rows of V gathered through the node's index
// list, shared by the 8 warps) is staged per 16-deep K chunk in a
// double-buffered shared-memory tile with cp.async (rows padded to 68 doubles:
// conflict-free fragment loads).
//
//   forward   c[i]        = z[sel[i]] + sum_q T[i, q] z[others[q]]          (src/butterfly.cpp:51-63)
//   transpose z[others[q]] (=|+=) sum_i T[i, q] c[i];  z[sel[i]] (=|+=) c[i]  (:67-79)
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>

#include "waves_dev.hpp"

namespace bfb {

namespace {

#ifndef BFB_WAVE_WARPS
#define BFB_WAVE_WARPS 4
#endif
// 4 warps (64-row blocks): most nodes have rank <= 64 (leaves: <= the block
// width), so small CTAs keep every warp on DMMA work and 4 CTAs share an SM
constexpr int kWarps = BFB_WAVE_WARPS;
constexpr int kThreads = 32 * kWarps;
constexpr int kMT = 16 * kWarps;  // output rows per block
constexpr int kMinBlocks = 16 / kWarps;
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
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

using Tile = double[2][kKC * kBS];

// acc (this warp's 16 rows x 64 columns of the block at m0) = A[m0.., 0..K) *
// B[0..K, n0..n0+64).  aval(row, k) reads A (row < M, k < K); brow(k) is the
// start of B row k (R contiguous doubles), the columns n0.. of it are staged.
template <class AV, class BR>
__device__ __forceinline__ void mma_block(double (&acc)[2][8][2], int M, int K, int m0, int n0, int R, AV aval,
                                          BR brow, Tile& bs) {
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
#pragma unroll
    for (int t = 0; t < 2; ++t)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[t][j][0] = acc[t][j][1] = 0.0;
    auto stage = [&](int buf, int kc) {
        double* dst = bs[buf];
        for (int e = tid; e < kKC * (kNT / 2); e += kThreads) {
            const int k = e / (kNT / 2), h = e - k * (kNT / 2);
            const int n = n0 + 2 * h;
            double* p = dst + k * kBS + 2 * h;
            if (kc + k < K && n < R) {
                cp_async16(p, brow(kc + k) + n);
            } else {
                p[0] = 0.0;
                p[1] = 0.0;
            }
        }
    };
    const int ra = m0 + 16 * warp + (lane >> 2), ka = lane & 3;
    const int tb = m0 + 16 * warp, nt = tb >= M ? 0 : (tb + 8 >= M ? 1 : 2);  // this warp's live m8 tiles
    auto load_a = [&](double (&av)[2][kKS], int kc) {
#pragma unroll
        for (int t = 0; t < 2; ++t)
#pragma unroll
            for (int s = 0; s < kKS; ++s) {
                const int row = ra + 8 * t, k = kc + 4 * s + ka;
                av[t][s] = (row < M && k < K) ? aval(row, k) : 0.0;
            }
    };
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
}

// The node's index list (sel then others) in shared memory when it fits: the
// B staging gathers through it every K chunk.
constexpr int kIdxMax = 1024;
__device__ __forceinline__ const std::uint32_t* node_index(const WaveArgs& a, const WaveNode& nd, std::uint32_t* sidx) {
    const int n = static_cast<int>(nd.rank + nd.nothers);
    const std::uint32_t* g = a.idx + nd.idx;
    if (n > kIdxMax) return g;
    for (int e = threadIdx.x; e < n; e += kThreads) sidx[e] = __ldg(g + e);
    __syncthreads();
    return sidx;
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) wave_fwd_kernel(WaveArgs a, int item0) {
    __shared__ __align__(16) Tile bs;
    __shared__ std::uint32_t sidx[kIdxMax];
    const WaveNode nd = a.nodes[a.fwd[item0 + blockIdx.x]];
    const int R = 4 * a.batch, n0 = kNT * static_cast<int>(blockIdx.y);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double* T = a.T + nd.t_off;
    const std::uint32_t* sel = node_index(a, nd, sidx);
    const std::uint32_t* oth = sel + nd.rank;
    const int M = static_cast<int>(nd.rank), K = static_cast<int>(nd.nothers);
    double* V = a.V;
    for (int m0 = 0; m0 < M; m0 += kMT) {
        double acc[2][8][2];
        mma_block(
            acc, M, K, m0, n0, R, [&](int i, int q) { return __ldcs(T + i + static_cast<long long>(q) * M); },
            [&](int q) { return V + static_cast<long long>(oth[q]) * R; }, bs);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int i = m0 + 16 * warp + 8 * t + (lane >> 2);
            if (i >= M) continue;
            const double* zs = V + static_cast<long long>(sel[i]) * R;
            double* out = V + (static_cast<long long>(nd.cA) + i) * R;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int n = n0 + 8 * j + 2 * (lane & 3);
                if (n < R) {
                    const double2 z = *reinterpret_cast<const double2*>(zs + n);
                    *reinterpret_cast<double2*>(out + n) = make_double2(z.x + acc[t][j][0], z.y + acc[t][j][1]);
                }
            }
        }
    }
}

__global__ void __launch_bounds__(kThreads, kMinBlocks) wave_bwd_kernel(WaveArgs a, int item0) {
    __shared__ __align__(16) Tile bs;
    __shared__ std::uint32_t sidx[kIdxMax];
    const int R = 4 * a.batch, n0 = kNT * static_cast<int>(blockIdx.y);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint2 pr = reinterpret_cast<const uint2*>(a.pairs)[item0 + blockIdx.x];
    double* V = a.V;
    for (int t2 = 0; t2 < 2; ++t2) {
        const std::uint32_t ni = t2 == 0 ? pr.x : pr.y;
        if (ni == ~0u) break;
        const bool first = t2 == 0;
        const WaveNode nd = a.nodes[ni];
        const double* T = a.T + nd.t_off;
        const std::uint32_t* sel = node_index(a, nd, sidx);
        const std::uint32_t* oth = sel + nd.rank;
        const int M = static_cast<int>(nd.nothers), K = static_cast<int>(nd.rank);
        const double* c = V + static_cast<long long>(nd.cA) * R;
        for (int m0 = 0; m0 < M; m0 += kMT) {
            double acc[2][8][2];
            mma_block(
                acc, M, K, m0, n0, R, [&](int q, int i) { return __ldcs(T + i + static_cast<long long>(q) * K); },
                [&](int i) { return c + static_cast<long long>(i) * R; }, bs);
#pragma unroll
            for (int t = 0; t < 2; ++t) {
                const int q = m0 + 16 * warp + 8 * t + (lane >> 2);
                if (q >= M) continue;
                double* z = V + static_cast<long long>(oth[q]) * R;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int n = n0 + 8 * j + 2 * (lane & 3);
                    if (n < R) {
                        double2 v = make_double2(acc[t][j][0], acc[t][j][1]);
                        if (!first) {
                            const double2 o = *reinterpret_cast<const double2*>(z + n);
                            v.x += o.x;
                            v.y += o.y;
                        }
                        *reinterpret_cast<double2*>(z + n) = v;
                    }
                }
            }
        }
        // z[sel[i]] (=|+=) c[i] over this item's columns
        const int nn = min(kNT, R - n0) / 2;
        for (int e = threadIdx.x; e < K * nn; e += kThreads) {
            const int i = e / nn, n = n0 + 2 * (e - i * nn);
            double2 v = *reinterpret_cast<const double2*>(c + static_cast<long long>(i) * R + n);
            double2* z = reinterpret_cast<double2*>(V + static_cast<long long>(sel[i]) * R + n);
            if (!first) {
                const double2 o = *z;
                v.x += o.x;
                v.y += o.y;
            }
            *z = v;
        }
        __syncthreads();  // the second node of the pair adds into the same z cells
    }
}

__device__ __forceinline__ long long coeff_index(int l, int mu, int sign, int col, int parity) {
    const long long L = l;
    const long long base = mu == 0 ? 0 : 2 * L + static_cast<long long>(mu - 1) * (4 * L - mu);
    return base + sign * (2 * L - mu) + 2LL * col + parity;
}

// Chain coefficients <-> the plans' input cells: V[plan_in + j][b][4] =
// (re, im of beta^{+mu}_{mu + 2j + p}, re, im of beta^{-mu}_{...}) of member b.
template <bool SCATTER>
__global__ void __launch_bounds__(256) wave_io_kernel(WaveArgs a, const double* beta_in, double* beta_out) {
    const int plan = blockIdx.x;
    const int mu = static_cast<int>(a.plan_mu[plan]), par = static_cast<int>(a.plan_parity[plan]);
    const int n = static_cast<int>(a.plan_cols[plan]) * a.batch;
    const long long in0 = a.plan_in[plan];
    const int R = 4 * a.batch;
    for (int e = threadIdx.x; e < n; e += blockDim.x) {
        const int j = e / a.batch, b = e - j * a.batch;
        double2* v = reinterpret_cast<double2*>(a.V + (in0 + j) * R + 4 * b);
        if (a.real_members > 0) {
            // real fields, half layout (m >= 0 only): the cell's two halves are
            // fields 2b and 2b + 1 (beta^{-m} = (-1)^m conj(beta^m) is implied)
            const long long mu_l = mu, L = a.l;
            const long long k = 2 * (mu_l * 2 * L - mu_l * (mu_l - 1) / 2 + 2LL * j + par);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int m = 2 * b + h;
                const long long off = k + m * a.beta_stride;
                if (!SCATTER)
                    v[h] = m < a.real_members ? *reinterpret_cast<const double2*>(beta_in + off) : make_double2(0.0, 0.0);
                else if (m < a.real_members)
                    *reinterpret_cast<double2*>(beta_out + off) = v[h];
            }
            continue;
        }
        const long long ip = 2 * coeff_index(a.l, mu, 0, j, par) + b * a.beta_stride;
        const long long im = 2 * coeff_index(a.l, mu, 1, j, par) + b * a.beta_stride;
        if (!SCATTER) {
            v[0] = *reinterpret_cast<const double2*>(beta_in + ip);
            v[1] = mu == 0 ? make_double2(0.0, 0.0) : *reinterpret_cast<const double2*>(beta_in + im);
        } else {
            *reinterpret_cast<double2*>(beta_out + ip) = v[0];
            if (mu != 0) *reinterpret_cast<double2*>(beta_out + im) = v[1];
        }
    }
}

template <class T>
T* upload(const std::vector<T>& v) {
    T* d = nullptr;
    if (v.empty()) return nullptr;
    if (cudaMalloc(&d, v.size() * sizeof(T)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed (waves)");
    if (cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy failed (waves)");
    return d;
}

}  // namespace

DeviceWaveSet upload_waves(const WaveSet& w) {
    DeviceWaveSet d;
    d.T = upload(w.T);
    d.idx = upload(w.idx);
    d.nodes = upload(w.nodes);
    d.fwd = upload(w.fwd);
    d.pairs = upload(w.pairs);
    d.plan_in = upload(w.plan_in);
    d.plan_mu = upload(w.plan_mu);
    d.plan_parity = upload(w.plan_parity);
    d.plan_cols = upload(w.plan_cols);
    d.n_T = w.T.size();
    d.n_idx = w.idx.size();
    d.n_nodes = w.nodes.size();
    d.n_fwd = w.fwd.size();
    d.n_pairs = w.pairs.size();
    d.fwd_begin = w.fwd_begin;
    d.bwd_begin = w.bwd_begin;
    d.levels = w.levels;
    d.n_plans = static_cast<int>(w.plan_in.size());
    d.v_cells = w.v_cells;
    d.roots = upload_roots(w.roots, true);
    d.event_words = w.event_words;
    d.root_words = w.root_words;
    return d;
}

void free_waves(DeviceWaveSet& d) {
    cudaFree(d.T);
    cudaFree(d.idx);
    cudaFree(d.nodes);
    cudaFree(d.fwd);
    cudaFree(d.pairs);
    cudaFree(d.plan_in);
    cudaFree(d.plan_mu);
    cudaFree(d.plan_parity);
    cudaFree(d.plan_cols);
    free_roots(d.roots);
    d = DeviceWaveSet{};
}

WaveArgs wave_args(const DeviceWaveSet& d, double* V, int l, int batch, long long beta_stride) {
    WaveArgs a;
    a.T = d.T;
    a.idx = d.idx;
    a.nodes = d.nodes;
    a.fwd = d.fwd;
    a.pairs = d.pairs;
    a.plan_in = d.plan_in;
    a.plan_mu = d.plan_mu;
    a.plan_parity = d.plan_parity;
    a.plan_cols = d.plan_cols;
    a.V = V;
    a.l = l;
    a.batch = batch;
    a.beta_stride = beta_stride;
    return a;
}

cudaError_t launch_wave_gather(const DeviceWaveSet& d, const WaveArgs& a, const double* beta, cudaStream_t st) {
    if (d.n_plans == 0) return cudaSuccess;
    wave_io_kernel<false><<<d.n_plans, 256, 0, st>>>(a, beta, nullptr);
    return cudaGetLastError();
}

cudaError_t launch_wave_scatter(const DeviceWaveSet& d, const WaveArgs& a, double* beta, cudaStream_t st) {
    if (d.n_plans == 0) return cudaSuccess;
    wave_io_kernel<true><<<d.n_plans, 256, 0, st>>>(a, nullptr, beta);
    return cudaGetLastError();
}

cudaError_t launch_wave_level(const DeviceWaveSet& d, const WaveArgs& a, int level, bool transpose, cudaStream_t st) {
    const std::vector<std::uint32_t>& beg = transpose ? d.bwd_begin : d.fwd_begin;
    const int i0 = static_cast<int>(beg[level - 1]), n = static_cast<int>(beg[level]) - i0;
    if (n == 0) return cudaSuccess;
    const dim3 grid(static_cast<unsigned>(n), static_cast<unsigned>((4 * a.batch + kNT - 1) / kNT));
    if (transpose)
        wave_bwd_kernel<<<grid, kThreads, 0, st>>>(a, i0);
    else
        wave_fwd_kernel<<<grid, kThreads, 0, st>>>(a, i0);
    return cudaGetLastError();
}

}  // namespace bfb
