// Device side of the wave programs (waves.hpp): upload, and the kernels that
// move vectors between the caller's layouts and the cell-major V / row buffers.
// The butterfly levels and roots themselves run in the graph kernel (wgraph.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <type_traits>

#include "waves_dev.hpp"

namespace bfb {

namespace {

// Chain coefficients <-> the plans' input cells, one block per order mu (both
// degree parities, so consecutive threads touch consecutive coefficients):
// V[plan_in + j][b][4] = (re, im of beta^{+mu}_{mu + 2j + p}, re, im of
// beta^{-mu}_{...}) of member b, p the plan's parity.
template <bool SCATTER>
__global__ void __launch_bounds__(256) wave_io_kernel(WaveArgs a, const double* beta_in, double* beta_out) {
    // Tiled through shared memory so both sides stay coalesced: 32 degrees x 16
    // members at a time; the coefficient side runs along the degrees (16-byte
    // pieces of the +m / -m blocks, or of the two real fields of a slot), the V
    // side along whole 512-byte rows.
    constexpr int TT = 32, G = 16, TS = 4 * G + 2;  // row stride (doubles), padded
    __shared__ __align__(16) double tile[TT * TS];
    const int o = blockIdx.x, mu = a.mu0 + o, L = a.l;
    const std::uint32_t pe = a.order_plan[2 * o], po = a.order_plan[2 * o + 1];
    const long long ie = a.plan_in[pe], io = po == ~0u ? 0 : a.plan_in[po];
    const int nk = 2 * L - mu;  // degrees mu .. 2l - 1
    const int R = 4 * a.batch;
    const bool real = a.real_members > 0;
    const long long base = real ? static_cast<long long>(mu) * 2 * L - static_cast<long long>(mu) * (mu - 1) / 2
                                : (mu == 0 ? 0 : 2LL * L + static_cast<long long>(mu - 1) * (4LL * L - mu));
    for (int g0 = 0; g0 < a.batch; g0 += G) {
        const int gn = min(G, a.batch - g0);
        for (int t0 = 0; t0 < nk; t0 += TT) {
            const int tn = min(TT, nk - t0);
            // coefficient side: piece (member m, half h) of degree t0 + t
            auto coef = [&](int m, int h, int t, bool& ok) -> long long {
                const int b = g0 + m;
                if (real) {
                    const int f = 2 * b + h;
                    ok = f < a.real_members;
                    return 2 * (base + t0 + t) + static_cast<long long>(f) * a.beta_stride;
                }
                ok = !(h == 1 && mu == 0);
                return 2 * (base + t0 + t) + static_cast<long long>(b) * a.beta_stride + h * 2LL * (2 * L - mu);
            };
            if (!SCATTER) {
                for (int e = threadIdx.x; e < gn * 2 * TT; e += blockDim.x) {
                    const int t = e % TT, mh = e / TT, m = mh >> 1, h = mh & 1;
                    if (t >= tn) continue;
                    bool ok;
                    const long long off = coef(m, h, t, ok);
                    *reinterpret_cast<double2*>(tile + t * TS + 4 * m + 2 * h) =
                        ok ? *reinterpret_cast<const double2*>(beta_in + off) : make_double2(0.0, 0.0);
                }
                __syncthreads();
                for (int e = threadIdx.x; e < tn * 2 * gn; e += blockDim.x) {
                    const int t = e / (2 * gn), q = e - t * (2 * gn);
                    const long long cell = ((t0 + t) & 1 ? io : ie) + ((t0 + t) >> 1);
                    *reinterpret_cast<double2*>(a.V + cell * R + 4 * g0 + 2 * q) =
                        *reinterpret_cast<const double2*>(tile + t * TS + 2 * q);
                }
            } else {
                for (int e = threadIdx.x; e < tn * 2 * gn; e += blockDim.x) {
                    const int t = e / (2 * gn), q = e - t * (2 * gn);
                    const long long cell = ((t0 + t) & 1 ? io : ie) + ((t0 + t) >> 1);
                    *reinterpret_cast<double2*>(tile + t * TS + 2 * q) =
                        *reinterpret_cast<const double2*>(a.V + cell * R + 4 * g0 + 2 * q);
                }
                __syncthreads();
                for (int e = threadIdx.x; e < gn * 2 * TT; e += blockDim.x) {
                    const int t = e % TT, mh = e / TT, m = mh >> 1, h = mh & 1;
                    if (t >= tn) continue;
                    bool ok;
                    const long long off = coef(m, h, t, ok);
                    if (ok)
                        *reinterpret_cast<double2*>(beta_out + off) =
                            *reinterpret_cast<const double2*>(tile + t * TS + 4 * m + 2 * h);
                }
            }
            __syncthreads();
        }
    }
}

// Plan-set apply (bfly_dev_apply with many right-hand sides): the stacked
// column-major vectors of the reference layout (plan p, rhs r, entry k at
// prefix[p] * nrhs + r * n(p) + k) <-> cell-major V / row buffers (R = 4 * batch
// doubles per cell, columns >= nrhs zero).  One block per plan.
template <bool TO_CELLS>
__global__ void __launch_bounds__(256) plan_io_kernel(const double* __restrict__ src, double* __restrict__ dst,
                                                     const std::uint64_t* __restrict__ prefix,
                                                     const std::uint32_t* __restrict__ cell0, int nrhs, int R,
                                                     int r0, int nrhs_total) {
    // columns r0 .. r0 + nrhs of the stacked layout with nrhs_total columns
    const int p = blockIdx.x;
    const int n = static_cast<int>(prefix[p + 1] - prefix[p]);
    const long long base = static_cast<long long>(prefix[p]) * nrhs_total + static_cast<long long>(r0) * n;
    const long long c0 = cell0 ? cell0[p] : static_cast<long long>(prefix[p]);
    for (int e = threadIdx.x; e < n * R; e += blockDim.x) {
        const int k = e / R, r = e - k * R;  // cell-major side contiguous
        if (TO_CELLS)
            dst[(c0 + k) * R + r] = r < nrhs ? src[base + static_cast<long long>(r) * n + k] : 0.0;
        else if (r < nrhs)
            dst[base + static_cast<long long>(r) * n + k] = src[(c0 + k) * R + r];
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

cudaError_t launch_plan_cells_in(const double* src, double* V, const std::uint64_t* prefix, const std::uint32_t* cell0,
                                 int n_plans, int nrhs, int R, cudaStream_t st, int r0, int nrhs_total) {
    if (n_plans == 0) return cudaSuccess;
    plan_io_kernel<true><<<n_plans, 256, 0, st>>>(src, V, prefix, cell0, nrhs, R, r0, nrhs_total > 0 ? nrhs_total : nrhs);
    return cudaGetLastError();
}
cudaError_t launch_plan_cells_out(const double* V, double* dst, const std::uint64_t* prefix, const std::uint32_t* cell0,
                                  int n_plans, int nrhs, int R, cudaStream_t st, int r0, int nrhs_total) {
    if (n_plans == 0) return cudaSuccess;
    plan_io_kernel<false><<<n_plans, 256, 0, st>>>(V, dst, prefix, cell0, nrhs, R, r0, nrhs_total > 0 ? nrhs_total : nrhs);
    return cudaGetLastError();
}
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
    // per order: its even / odd plan (plans are sorted by order, even first)
    std::vector<std::uint32_t> op;
    const int mu0 = w.plan_mu.empty() ? 0 : static_cast<int>(w.plan_mu[0]);
    for (std::size_t i = 0; i < w.plan_mu.size(); ++i) {
        const std::size_t o = w.plan_mu[i] - mu0;
        if (op.size() < 2 * (o + 1)) op.resize(2 * (o + 1), ~0u);
        op[2 * o + w.plan_parity[i]] = static_cast<std::uint32_t>(i);
    }
    d.order_plan = upload(op);
    d.n_orders = static_cast<int>(op.size() / 2);
    d.mu0 = mu0;
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
    // root stripes: tiled S (packer.hpp) and the descriptors, as built
    d.roots.data = upload(w.roots.data);
    d.roots.stripes = upload(w.roots.stripes);
    d.roots.n_stripes = w.roots.stripes.size();
    d.roots.bytes = w.roots.data.size() * sizeof(double);
    d.roots.stored_words = w.roots.stored_words;
    {
        std::uint32_t groups = 0;
        for (const RootStripeDesc& r : w.roots.stripes) groups = std::max(groups, r.pad[0] + 1);
        d.root_groups = static_cast<int>(groups);
    }
    d.plan_row0 = upload(w.plan_row0);
    d.event_words = w.event_words;
    d.root_words = w.root_words;
    d.node_src = w.node_src;
    d.plan_node_begin = w.plan_node_begin;
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
    cudaFree(d.order_plan);
    cudaFree(d.plan_row0);
    cudaFree(d.roots.data);
    cudaFree(d.roots.stripes);
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
    a.order_plan = d.order_plan;
    a.mu0 = d.mu0;
    a.V = V;
    a.l = l;
    a.batch = batch;
    a.beta_stride = beta_stride;
    return a;
}

cudaError_t launch_wave_gather(const DeviceWaveSet& d, const WaveArgs& a, const double* beta, cudaStream_t st) {
    if (d.n_plans == 0) return cudaSuccess;
    wave_io_kernel<false><<<d.n_orders, 256, 0, st>>>(a, beta, nullptr);
    return cudaGetLastError();
}

cudaError_t launch_wave_scatter(const DeviceWaveSet& d, const WaveArgs& a, double* beta, cudaStream_t st) {
    if (d.n_plans == 0) return cudaSuccess;
    wave_io_kernel<true><<<d.n_orders, 256, 0, st>>>(a, nullptr, beta);
    return cudaGetLastError();
}

}  // namespace bfb
