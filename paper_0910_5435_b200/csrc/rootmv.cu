// Root-stage kernels of the split SHT programs.
//
// The root stage of every butterfly plan (reference src/butterfly.cpp:432-440,
// forward; :452-460, transpose) is a dense skeleton product per root stripe,
// independent across stripes.  Once the event program has left each stripe's
// coefficient vector in C, the whole stage is a batched matrix-vector product
// over ~80 % of the plan bytes with no dependency chain, so it runs as a flat
// grid of warps streaming the skeletons with coalesced, read-once loads:
//   forward:   ypart[stripe rows] = S   * c      (lane = output row)
//   transpose: C[stripe]          = S^T * u[rows] (lane = output column; reads
//              the transposed copy so the loads stay coalesced)
// Each warp owns one 32-output block of one stripe for one batch member; the
// right-hand sides (4 per function: +-m x re/im) are broadcast loads.
#include <cuda_runtime.h>

#include <algorithm>
#include <mutex>

#include "rootmv.hpp"

namespace bfb {

namespace {

constexpr int kWarpsPerCta = 8;
constexpr int kUnroll = 8;

__device__ __forceinline__ double4 ld_vec4(const double* p) {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p));
    const double2 b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    return make_double4(a.x, a.y, b.x, b.y);
}

// Two adjacent outputs per lane: out[t][4] = sum_k A[k * lda + t] * V[k][0..3]
// (t = 0, 1; A column stride lda, V rows of 4 doubles), kUnroll independent
// 16-byte loads in flight.
__device__ __forceinline__ void dot4x2(const double* A, long long lda, const double* V, int n, bool ok,
                                       double (&acc)[2][4]) {
    int k = 0;
    for (; k + kUnroll <= n; k += kUnroll) {
        double2 a[kUnroll];
        double4 v[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            a[u] = ok ? __ldcs(reinterpret_cast<const double2*>(A + (k + u) * lda)) : make_double2(0.0, 0.0);
            v[u] = ld_vec4(V + 4 * (k + u));
        }
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            acc[0][0] = fma(a[u].x, v[u].x, acc[0][0]);
            acc[0][1] = fma(a[u].x, v[u].y, acc[0][1]);
            acc[0][2] = fma(a[u].x, v[u].z, acc[0][2]);
            acc[0][3] = fma(a[u].x, v[u].w, acc[0][3]);
            acc[1][0] = fma(a[u].y, v[u].x, acc[1][0]);
            acc[1][1] = fma(a[u].y, v[u].y, acc[1][1]);
            acc[1][2] = fma(a[u].y, v[u].z, acc[1][2]);
            acc[1][3] = fma(a[u].y, v[u].w, acc[1][3]);
        }
    }
    for (; k < n; ++k) {
        const double2 a = ok ? __ldcs(reinterpret_cast<const double2*>(A + k * lda)) : make_double2(0.0, 0.0);
        const double4 v = ld_vec4(V + 4 * k);
        acc[0][0] = fma(a.x, v.x, acc[0][0]);
        acc[0][1] = fma(a.x, v.y, acc[0][1]);
        acc[0][2] = fma(a.x, v.z, acc[0][2]);
        acc[0][3] = fma(a.x, v.w, acc[0][3]);
        acc[1][0] = fma(a.y, v.x, acc[1][0]);
        acc[1][1] = fma(a.y, v.y, acc[1][1]);
        acc[1][2] = fma(a.y, v.z, acc[1][2]);
        acc[1][3] = fma(a.y, v.w, acc[1][3]);
    }
}

template <bool BWD>
__global__ void __launch_bounds__(32 * kWarpsPerCta) root_kernel(RootArgs a) {
    const int lane = threadIdx.x & 31;
    const long long warps = static_cast<long long>(gridDim.x) * kWarpsPerCta;
    const long long n_tasks = static_cast<long long>(a.n_items) * a.batch;
    for (long long task = static_cast<long long>(blockIdx.x) * kWarpsPerCta + (threadIdx.x >> 5); task < n_tasks;
         task += warps) {
        const std::uint32_t item = a.items[task / a.batch];
        const int b = static_cast<int>(task % a.batch);
        const RootStripeDesc d = a.stripes[item >> 8];
        const int o = 64 * static_cast<int>(item & 255u) + 2 * lane;  // first of two outputs
        const int n_out = BWD ? static_cast<int>(d.rank) : static_cast<int>(d.rows);
        const bool ok = o < n_out;  // o + 1 may be padding (zeros)
        double acc[2][4] = {{0.0, 0.0, 0.0, 0.0}, {0.0, 0.0, 0.0, 0.0}};
        double* out;
        if (!BWD) {
            const double* A = a.data + d.s_off + (ok ? o : 0);
            const double* V = a.C + (static_cast<long long>(b) * a.c_cells + d.coff) * 4;
            dot4x2(A, d.lds, V, static_cast<int>(d.rank), ok, acc);
            out = a.ypart + (static_cast<long long>(b) * a.y_rows + d.yout + o) * 4;
        } else {
            const double* A = a.data + d.st_off + (ok ? o : 0);
            const double* V = a.u + ((static_cast<long long>(d.plan) * a.batch + b) * a.l + d.yin) * 4;
            dot4x2(A, d.ldt, V, static_cast<int>(d.rows), ok, acc);
            out = a.C + (static_cast<long long>(b) * a.c_cells + d.coff + o) * 4;
        }
        if (ok) {
            double2* y = reinterpret_cast<double2*>(out);
            y[0] = make_double2(acc[0][0], acc[0][1]);
            y[1] = make_double2(acc[0][2], acc[0][3]);
            if (o + 1 < n_out) {
                y[2] = make_double2(acc[1][0], acc[1][1]);
                y[3] = make_double2(acc[1][2], acc[1][3]);
            }
        }
    }
}

struct GridCache {
    std::mutex mu;
    int device = -1;
    int grid[2] = {0, 0};
};

template <bool BWD>
int grid_for() {
    static GridCache cache;
    std::lock_guard<std::mutex> lk(cache.mu);
    int dev = 0;
    cudaGetDevice(&dev);
    if (cache.device != dev || cache.grid[BWD] == 0) {
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, root_kernel<BWD>, 32 * kWarpsPerCta, 0);
        cache.device = dev;
        cache.grid[BWD] = std::max(1, sms * std::max(1, per_sm));
    }
    return cache.grid[BWD];
}

}  // namespace

cudaError_t launch_roots(const RootArgs& args, bool transpose, cudaStream_t st) {
    if (args.n_items == 0 || args.batch == 0) return cudaSuccess;
    const long long tasks = static_cast<long long>(args.n_items) * args.batch;
    if (transpose) {
        const int grid = static_cast<int>(std::min<long long>(grid_for<true>(), (tasks + kWarpsPerCta - 1) / kWarpsPerCta));
        root_kernel<true><<<grid, 32 * kWarpsPerCta, 0, st>>>(args);
    } else {
        const int grid = static_cast<int>(std::min<long long>(grid_for<false>(), (tasks + kWarpsPerCta - 1) / kWarpsPerCta));
        root_kernel<false><<<grid, 32 * kWarpsPerCta, 0, st>>>(args);
    }
    return cudaGetLastError();
}

DeviceRootSet upload_roots(const RootSet& r, bool mma) {
    DeviceRootSet d;
    auto up = [](const void* src, std::size_t bytes, void** dst) {
        if (bytes == 0) return;
        if (cudaMalloc(dst, bytes) != cudaSuccess) throw std::runtime_error("cudaMalloc failed (root set)");
        if (cudaMemcpy(*dst, src, bytes, cudaMemcpyHostToDevice) != cudaSuccess)
            throw std::runtime_error("cudaMemcpy failed (root set)");
    };
    if (mma) {
        // S only, stripes back to back (32-byte aligned)
        std::vector<RootStripeDesc> st = r.stripes;
        std::size_t words = 0;
        for (const RootStripeDesc& s : st) words += (static_cast<std::size_t>(s.lds) * s.rank + 3) & ~std::size_t{3};
        std::vector<double> data(words, 0.0);
        std::size_t off = 0;
        for (RootStripeDesc& s : st) {
            const std::size_t n = static_cast<std::size_t>(s.lds) * s.rank;
            std::copy(r.data.begin() + static_cast<std::ptrdiff_t>(s.s_off),
                      r.data.begin() + static_cast<std::ptrdiff_t>(s.s_off + n), data.begin() + static_cast<std::ptrdiff_t>(off));
            s.s_off = off;  // st_off is kept (the wave programs' producer record)
            off += (n + 3) & ~std::size_t{3};
        }
        std::vector<std::uint32_t> fi, bi;
        root_mma_items(st, fi, bi, &d.mma_fwd_group);
        d.mma_fwd_group.push_back(static_cast<int>(fi.size() / 2));
        up(data.data(), data.size() * sizeof(double), reinterpret_cast<void**>(&d.data));
        up(st.data(), st.size() * sizeof(RootStripeDesc), reinterpret_cast<void**>(&d.stripes));
        up(fi.data(), fi.size() * sizeof(std::uint32_t), reinterpret_cast<void**>(&d.mma_fwd));
        up(bi.data(), bi.size() * sizeof(std::uint32_t), reinterpret_cast<void**>(&d.mma_bwd));
        d.n_mma_fwd = static_cast<int>(fi.size() / 2);
        d.n_mma_bwd = static_cast<int>(bi.size() / 2);
        d.mma = true;
        d.n_stripes = st.size();
        d.stored_words = r.stored_words;
        d.bytes = data.size() * sizeof(double);
        return d;
    }
    up(r.data.data(), r.data.size() * sizeof(double), reinterpret_cast<void**>(&d.data));
    up(r.stripes.data(), r.stripes.size() * sizeof(RootStripeDesc), reinterpret_cast<void**>(&d.stripes));
    up(r.fwd_items.data(), r.fwd_items.size() * sizeof(std::uint32_t), reinterpret_cast<void**>(&d.fwd_items));
    up(r.bwd_items.data(), r.bwd_items.size() * sizeof(std::uint32_t), reinterpret_cast<void**>(&d.bwd_items));
    d.n_fwd = static_cast<int>(r.fwd_items.size());
    d.n_bwd = static_cast<int>(r.bwd_items.size());
    d.stored_words = r.stored_words;
    d.bytes = r.data.size() * sizeof(double);
    return d;
}

void free_roots(DeviceRootSet& d) {
    cudaFree(d.data);
    cudaFree(d.stripes);
    cudaFree(d.fwd_items);
    cudaFree(d.bwd_items);
    cudaFree(d.mma_fwd);
    cudaFree(d.mma_bwd);
    d = DeviceRootSet{};
}

}  // namespace bfb
