// The butterfly engine: one persistent, warp-specialised kernel per direction
// that applies every butterfly plan of a plan set (reference bfly::apply /
// bfly::apply_transpose, src/butterfly.cpp:384-513) for many right-hand sides.
//
// CTA = 4 consumer warps + 1 producer warp.  The producer claims jobs from a
// global work counter and streams each job's stages (engine_format.hpp) into
// a 4-slot shared-memory ring with cp.async.bulk + mbarrier complete_tx; it
// runs ahead across job boundaries, so HBM stays busy while consumers finish
// a job.  Consumers replay the job's records (forward: in order; transpose:
// stages and records reversed) against coefficient vectors that never leave
// shared memory.  FP64 throughout; every matrix word is read from HBM once per
// apply and reused for all RC right-hand sides of the job.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <stdexcept>
#include <string>

#include "engine.hpp"

namespace bfb {

namespace {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kNT = kConsumerThreads;

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* b, std::uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* b, std::uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(std::uint64_t* b, std::uint32_t parity) {
    std::uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Waits for the phase with the given parity.  A wait that exceeds ~2^35
// cycles (well over ten seconds) traps instead of hanging the device.
__device__ __forceinline__ void mbar_wait(std::uint64_t* b, std::uint32_t parity) {
    if (mbar_try_wait(b, parity)) return;
    const long long t0 = clock64();
    while (!mbar_try_wait(b, parity)) {
        if (clock64() - t0 > (1LL << 35)) __trap();
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, std::uint32_t bytes, std::uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// Barrier over the 128 consumer threads only (the producer never joins).
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Index of the first element >= 0 of the arithmetic slice owned by thread t
// when element e is owned by thread (base + e) mod kNT.
__device__ __forceinline__ int first_of(std::uint32_t base, int t) {
    return (t - static_cast<int>(base & (kNT - 1))) & (kNT - 1);
}

struct JobCtx {
    int task, chunk;
    int n_plans, mu;
    std::uint32_t plan[2], yA[2], n_cols[2], n_rows;
};

template <int RC>
struct Cells {
    double* a;
    __device__ __forceinline__ void load(std::uint32_t c, double (&v)[RC]) const {
        const double2* p = reinterpret_cast<const double2*>(a + static_cast<std::size_t>(c) * RC);
#pragma unroll
        for (int r = 0; r < RC / 2; ++r) {
            const double2 x = p[r];
            v[2 * r] = x.x;
            v[2 * r + 1] = x.y;
        }
    }
    __device__ __forceinline__ void store(std::uint32_t c, const double (&v)[RC]) const {
        double2* p = reinterpret_cast<double2*>(a + static_cast<std::size_t>(c) * RC);
#pragma unroll
        for (int r = 0; r < RC / 2; ++r) p[r] = make_double2(v[2 * r], v[2 * r + 1]);
    }
    __device__ __forceinline__ void put(std::uint32_t c, const double (&v)[RC], bool assign) const {
        if (assign) {
            store(c, v);
        } else {
            double o[RC];
            load(c, o);
#pragma unroll
            for (int r = 0; r < RC; ++r) o[r] += v[r];
            store(c, o);
        }
    }
};

__device__ __forceinline__ std::uint32_t zcell(const Rec& r, std::uint32_t k) {
    return k < r.kl ? r.zA + k : r.zB + (k - r.kl);
}

// ---- I/O policies -----------------------------------------------------------

struct GenericPolicy {
    GenericIO io;

    template <int RC>
    __device__ void load_rows(const JobCtx& j, int ps, std::uint32_t row0, int n, std::uint32_t zA, double* arena,
                              int t) const {
        const std::uint64_t base = io.in_prefix[j.plan[ps]] * static_cast<std::uint64_t>(io.nrhs);
        const std::uint32_t ld = j.n_cols[ps];
        for (int idx = t; idx < n * RC; idx += kNT) {
            const int r = idx / n, k = idx - r * n;
            const int rhs = j.chunk * RC + r;
            const double v = rhs < io.nrhs ? io.in[base + static_cast<std::uint64_t>(rhs) * ld + row0 + k] : 0.0;
            arena[static_cast<std::size_t>(zA + k) * RC + r] = v;
        }
    }
    template <int RC>
    __device__ void store_rows(const JobCtx& j, int ps, std::uint32_t row0, int n, std::uint32_t zA,
                               const double* arena, int t) const {
        const std::uint64_t base = io.out_prefix[j.plan[ps]] * static_cast<std::uint64_t>(io.nrhs);
        const std::uint32_t ld = j.n_cols[ps];
        for (int idx = t; idx < n * RC; idx += kNT) {
            const int r = idx / n, k = idx - r * n;
            const int rhs = j.chunk * RC + r;
            if (rhs < io.nrhs)
                io.out[base + static_cast<std::uint64_t>(rhs) * ld + row0 + k] =
                    arena[static_cast<std::size_t>(zA + k) * RC + r];
        }
    }
    template <int RC>
    __device__ void epilogue(const JobCtx& j, const double* arena, int t) const {
        const int n = static_cast<int>(j.n_rows);
        for (int ps = 0; ps < j.n_plans; ++ps) {
            const std::uint64_t base = io.out_prefix[j.plan[ps]] * static_cast<std::uint64_t>(io.nrhs);
            for (int idx = t; idx < n * RC; idx += kNT) {
                const int r = idx / n, i = idx - r * n;
                const int rhs = j.chunk * RC + r;
                if (rhs < io.nrhs)
                    io.out[base + static_cast<std::uint64_t>(rhs) * n + i] =
                        arena[static_cast<std::size_t>(j.yA[ps] + i) * RC + r];
            }
        }
    }
    template <int RC>
    __device__ void prologue(const JobCtx& j, double* arena, int t) const {
        const int n = static_cast<int>(j.n_rows);
        for (int ps = 0; ps < j.n_plans; ++ps) {
            const std::uint64_t base = io.in_prefix[j.plan[ps]] * static_cast<std::uint64_t>(io.nrhs);
            for (int idx = t; idx < n * RC; idx += kNT) {
                const int r = idx / n, i = idx - r * n;
                const int rhs = j.chunk * RC + r;
                arena[static_cast<std::size_t>(j.yA[ps] + i) * RC + r] =
                    rhs < io.nrhs ? io.in[base + static_cast<std::uint64_t>(rhs) * n + i] : 0.0;
            }
        }
    }
};

// SHT: chunk = batch member b, RC = 4 right-hand sides r = 2*sign + reim,
// sign 0 -> m = +mu, sign 1 -> m = -mu (absent for mu = 0).
struct ShtPolicy {
    ShtIO io;

    __device__ __forceinline__ long long coeff_index(int mu, int sign, int col, int parity) const {
        const long long l = io.l;
        const long long base = mu == 0 ? 0 : 2 * l + static_cast<long long>(mu - 1) * (4 * l - mu);
        return base + sign * (2 * l - mu) + 2LL * col + parity;
    }

    template <int RC>
    __device__ void load_rows(const JobCtx& j, int ps, std::uint32_t row0, int n, std::uint32_t zA, double* arena,
                              int t) const {
        static_assert(RC == 4, "SHT jobs carry (sign, re/im) x 1 function");
        const double* src = io.beta_in + static_cast<long long>(j.chunk) * io.beta_stride;
        for (int idx = t; idx < n * 4; idx += kNT) {
            const int k = idx >> 2, r = idx & 3, sign = r >> 1, reim = r & 1;
            double v = 0.0;
            if (!(j.mu == 0 && sign)) v = src[2 * coeff_index(j.mu, sign, static_cast<int>(row0) + k, ps) + reim];
            arena[static_cast<std::size_t>(zA + k) * 4 + r] = v;
        }
    }
    template <int RC>
    __device__ void store_rows(const JobCtx& j, int ps, std::uint32_t row0, int n, std::uint32_t zA,
                               const double* arena, int t) const {
        double* dst = io.beta_out + static_cast<long long>(j.chunk) * io.beta_stride;
        for (int idx = t; idx < n * 4; idx += kNT) {
            const int k = idx >> 2, r = idx & 3, sign = r >> 1, reim = r & 1;
            if (!(j.mu == 0 && sign))
                dst[2 * coeff_index(j.mu, sign, static_cast<int>(row0) + k, ps) + reim] =
                    arena[static_cast<std::size_t>(zA + k) * 4 + r];
        }
    }
    // g_m(+-x_i) = (u_even +- u_odd) / sqrt(rho_i) into DFT bin m mod N of
    // latitude rows t = l + i (x > 0) and l - 1 - i (x < 0).
    template <int RC>
    __device__ void epilogue(const JobCtx& j, const double* arena, int t) const {
        const int l = io.l, N = io.N;
        double* dst = io.grid_out + static_cast<long long>(j.chunk) * io.grid_stride;
        for (int idx = t; idx < l * 4; idx += kNT) {
            const int i = idx >> 2, r = idx & 3, sign = r >> 1, reim = r & 1;
            if (j.mu == 0 && sign) continue;
            const double ue = arena[static_cast<std::size_t>(j.yA[0] + i) * 4 + r];
            const double uo = j.n_plans > 1 ? arena[static_cast<std::size_t>(j.yA[1] + i) * 4 + r] : 0.0;
            const double s = io.isr[i];
            const int bin = sign ? N - j.mu : j.mu;
            dst[(static_cast<long long>(l + i) * N + bin) * 2 + reim] = (ue + uo) * s;
            dst[(static_cast<long long>(l - 1 - i) * N + bin) * 2 + reim] = (ue - uo) * s;
        }
    }
    // u_even,i = sqrt(rho_i)/2 (g(+x_i) + g(-x_i)) / N, u_odd with '-'.
    template <int RC>
    __device__ void prologue(const JobCtx& j, double* arena, int t) const {
        const int l = io.l, N = io.N;
        const double* src = io.grid_in + static_cast<long long>(j.chunk) * io.grid_stride;
        for (int idx = t; idx < l * 4; idx += kNT) {
            const int i = idx >> 2, r = idx & 3, sign = r >> 1, reim = r & 1;
            double ye = 0.0, yo = 0.0;
            if (!(j.mu == 0 && sign)) {
                const int bin = sign ? N - j.mu : j.mu;
                const double gp = src[(static_cast<long long>(l + i) * N + bin) * 2 + reim];
                const double gm = src[(static_cast<long long>(l - 1 - i) * N + bin) * 2 + reim];
                const double s = io.hsr[i];
                ye = (gp + gm) * s;
                yo = (gp - gm) * s;
            }
            arena[static_cast<std::size_t>(j.yA[0] + i) * 4 + r] = ye;
            if (j.n_plans > 1) arena[static_cast<std::size_t>(j.yA[1] + i) * 4 + r] = yo;
        }
    }
};

// ---- record execution -------------------------------------------------------

template <int RC, bool BWD, class Policy>
__device__ __forceinline__ void run_record(const Rec& r, const unsigned char* stage, double* arena, int t,
                                           const JobCtx& j, const Policy& pol) {
    const Cells<RC> cells{arena};
    switch (r.op) {
    case OP_LOADZ:
        if (!BWD)
            pol.template load_rows<RC>(j, r.pslot, r.zB, r.nr, r.zA, arena, t);
        else
            pol.template store_rows<RC>(j, r.pslot, r.zB, r.nr, r.zA, arena, t);
        break;
    case OP_SEL: {
        const std::uint16_t* sel = reinterpret_cast<const std::uint16_t*>(stage + r.data);
        if (!BWD) {
            for (int i = first_of(r.cA, t); i < r.nr; i += kNT) {
                double v[RC];
                cells.load(zcell(r, sel[i]), v);
                cells.store(r.cA + i, v);
            }
        } else {
            const bool assign = r.flags & F_ASSIGN_BWD;
            for (int i = t; i < r.nr; i += kNT) {
                double v[RC];
                cells.load(r.cA + i, v);
                cells.put(zcell(r, sel[i]), v, assign);
            }
        }
        break;
    }
    case OP_TPANEL: {
        const std::uint16_t* idx = reinterpret_cast<const std::uint16_t*>(stage + r.data);
        const double* T = reinterpret_cast<const double*>(stage + r.data + ((2u * r.nc + 15u) & ~15u));
        if (!BWD) {
            for (int i = first_of(r.cA, t); i < r.nr; i += kNT) {
                double acc[RC];
#pragma unroll
                for (int q = 0; q < RC; ++q) acc[q] = 0.0;
#pragma unroll 4
                for (int q = 0; q < r.nc; ++q) {
                    const double a = T[i + q * r.ld];
                    double z[RC];
                    cells.load(zcell(r, idx[q]), z);
#pragma unroll
                    for (int c = 0; c < RC; ++c) acc[c] = fma(a, z[c], acc[c]);
                }
                cells.put(r.cA + i, acc, false);
            }
        } else {
            const bool assign = r.flags & F_ASSIGN_BWD;
            for (int q = first_of(r.q0, t); q < r.nc; q += kNT) {
                const double* col = T + q * r.ld;
                double acc[RC];
#pragma unroll
                for (int c = 0; c < RC; ++c) acc[c] = 0.0;
#pragma unroll 4
                for (int i = 0; i < r.nr; ++i) {
                    const double a = col[i];
                    double v[RC];
                    cells.load(r.cA + i, v);
#pragma unroll
                    for (int c = 0; c < RC; ++c) acc[c] = fma(a, v[c], acc[c]);
                }
                cells.put(zcell(r, idx[q]), acc, assign);
            }
        }
        break;
    }
    case OP_SPANEL: {
        const double* S = reinterpret_cast<const double*>(stage + r.data);
        if (!BWD) {
            const bool assign = r.flags & F_ASSIGN_FWD;
            for (int i = first_of(r.zA, t); i < r.nr; i += kNT) {
                double acc[RC];
#pragma unroll
                for (int c = 0; c < RC; ++c) acc[c] = 0.0;
#pragma unroll 4
                for (int q = 0; q < r.nc; ++q) {
                    const double a = S[i + q * r.ld];
                    double v[RC];
                    cells.load(r.cA + q, v);
#pragma unroll
                    for (int c = 0; c < RC; ++c) acc[c] = fma(a, v[c], acc[c]);
                }
                cells.put(r.zA + i, acc, assign);
            }
        } else {
            const bool assign = r.flags & F_ASSIGN_BWD;
            for (int q = first_of(r.cA, t); q < r.nc; q += kNT) {
                const double* col = S + q * r.ld;
                double acc[RC];
#pragma unroll
                for (int c = 0; c < RC; ++c) acc[c] = 0.0;
#pragma unroll 4
                for (int i = 0; i < r.nr; ++i) {
                    const double a = col[i];
                    double v[RC];
                    cells.load(r.zA + i, v);
#pragma unroll
                    for (int c = 0; c < RC; ++c) acc[c] = fma(a, v[c], acc[c]);
                }
                cells.put(r.cA + q, acc, assign);
            }
        }
        break;
    }
    default:
        break;
    }
}

template <int RC, class Policy, bool BWD>
__global__ void __launch_bounds__(kEngineThreads, 2)
    engine_kernel(const std::uint8_t* __restrict__ stream, const std::uint64_t* __restrict__ stage_off,
                  const std::uint32_t* __restrict__ stage_bytes, const Job* __restrict__ jobs,
                  unsigned* __restrict__ counters, int n_tasks, int n_chunks, Policy pol) {
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned char* ring = smem;
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kRingStages * kStageBytes);
    std::uint64_t* empty = full + kRingStages;
    int4* info = reinterpret_cast<int4*>(empty + kRingStages);
    double* arena = reinterpret_cast<double*>(info + kRingStages);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kRingStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kNT / 32);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == kNT / 32) {
        // ------------------------------ producer ------------------------------
        std::uint32_t g = 0;
        for (;;) {
            int task = 0;
            if (lane == 0) task = static_cast<int>(atomicAdd(&counters[0], 1u));
            task = __shfl_sync(kFull, task, 0);
            if (task >= n_tasks) {
                const std::uint32_t slot = g % kRingStages, use = g / kRingStages;
                if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);
                if (lane == 0) {
                    info[slot] = make_int4(-1, 0, 0, 0);
                    mbar_arrive(&full[slot]);
                    __threadfence();
                    if (atomicAdd(&counters[1], 1u) == gridDim.x - 1) {
                        counters[0] = 0;
                        counters[1] = 0;
                    }
                }
                return;
            }
            const int job = task / n_chunks;
            const std::uint64_t s0 = jobs[job].stage0;
            const int ns = static_cast<int>(jobs[job].n_stages);
            for (int base = 0; base < ns; base += 32) {
                const int k = base + lane;
                std::uint64_t off = 0;
                std::uint32_t bytes = 0;
                if (k < ns) {
                    const std::uint64_t st = BWD ? s0 + static_cast<std::uint64_t>(ns - 1 - k) : s0 + k;
                    off = stage_off[st];
                    bytes = stage_bytes[st];
                }
                const int cnt = min(32, ns - base);
                for (int kk = 0; kk < cnt; ++kk) {
                    const std::uint64_t o = __shfl_sync(kFull, off, kk);
                    const std::uint32_t b = __shfl_sync(kFull, bytes, kk);
                    const std::uint32_t slot = g % kRingStages, use = g / kRingStages;
                    if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);
                    if (lane == 0) {
                        info[slot] = make_int4(task, base + kk, ns, 0);
                        mbar_expect_tx(&full[slot], b);
                        bulk_g2s(ring + slot * kStageBytes, stream + o, b, &full[slot]);
                    }
                    __syncwarp();
                    ++g;
                }
            }
        }
    }

    // ------------------------------ consumers --------------------------------
    const int t = tid;
    JobCtx j{};
    std::uint32_t g = 0;
    for (;;) {
        const std::uint32_t slot = g % kRingStages;
        mbar_wait(&full[slot], (g / kRingStages) & 1);
        const int4 inf = info[slot];
        if (inf.x < 0) break;
        const unsigned char* stage = ring + slot * kStageBytes;
        if (inf.y == 0) {
            j.task = inf.x;
            const int job = inf.x / n_chunks;
            j.chunk = inf.x - job * n_chunks;
            const Job& J = jobs[job];
            j.n_plans = J.n_plans;
            j.mu = J.mu;
            j.plan[0] = J.plan[0];
            j.plan[1] = J.plan[1];
            j.yA[0] = J.yA[0];
            j.yA[1] = J.yA[1];
            j.n_cols[0] = J.n_cols[0];
            j.n_cols[1] = J.n_cols[1];
            j.n_rows = J.n_rows;
            if (BWD) pol.template prologue<RC>(j, arena, t);
            consumer_sync();
        }
        const StageHeader* h = reinterpret_cast<const StageHeader*>(stage);
        const Rec* recs = reinterpret_cast<const Rec*>(stage + sizeof(StageHeader));
        const int n = static_cast<int>(h->n_rec);
        for (int q = 0; q < n; ++q) {
            const Rec r = recs[BWD ? n - 1 - q : q];
            if (r.flags & (BWD ? F_SYNC_BWD : F_SYNC_FWD)) consumer_sync();
            run_record<RC, BWD>(r, stage, arena, t, j, pol);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (inf.y == inf.z - 1) {
            consumer_sync();
            if (!BWD) pol.template epilogue<RC>(j, arena, t);
            consumer_sync();
        }
        ++g;
    }
}

template <class Policy, bool BWD>
cudaError_t launch(const DeviceProgram& prog, const Policy& pol, int n_chunks, cudaStream_t st) {
    if (prog.n_jobs == 0 || n_chunks == 0) return cudaSuccess;
    auto kern = engine_kernel<kRC, Policy, BWD>;
    const std::size_t smem = engine_smem_bytes(prog);
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    if (e != cudaSuccess) return e;
    int dev = 0, sms = 0, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kEngineThreads, smem);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaErrorInvalidConfiguration;
    const long long tasks = static_cast<long long>(prog.n_jobs) * n_chunks;
    const int grid = static_cast<int>(std::min<long long>(tasks, static_cast<long long>(sms) * per_sm));
    kern<<<grid, kEngineThreads, smem, st>>>(prog.stream, prog.stage_off, prog.stage_bytes, prog.jobs, prog.counters,
                                             static_cast<int>(tasks), n_chunks, pol);
    return cudaGetLastError();
}

template <class T>
T* upload(const std::vector<T>& v) {
    T* d = nullptr;
    if (v.empty()) return nullptr;
    if (cudaMalloc(&d, v.size() * sizeof(T)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
    if (cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy failed");
    return d;
}

}  // namespace

std::size_t engine_smem_bytes(const DeviceProgram& prog) {
    return static_cast<std::size_t>(kRingStages) * kStageBytes + 2 * kRingStages * sizeof(std::uint64_t) +
           kRingStages * sizeof(int4) + static_cast<std::size_t>(prog.arena_cells) * kRC * sizeof(double);
}

DeviceProgram upload_program(const PackedProgram& p, int device) {
    if (cudaSetDevice(device) != cudaSuccess) throw std::runtime_error("cudaSetDevice failed");
    DeviceProgram d;
    d.device = device;
    d.stream = upload(p.stream);
    d.stage_off = upload(p.stage_off);
    d.stage_bytes = upload(p.stage_bytes);
    d.jobs = upload(p.jobs);
    if (cudaMalloc(&d.counters, 2 * sizeof(unsigned)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
    cudaMemset(d.counters, 0, 2 * sizeof(unsigned));
    d.n_jobs = static_cast<int>(p.jobs.size());
    d.arena_cells = p.arena_cells;
    d.stream_bytes = p.stream.size();
    d.fetched_bytes = p.fetched_bytes;
    d.stored_words = p.stored_words;
    const std::size_t smem = engine_smem_bytes(d);
    int optin = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
    if (static_cast<long long>(smem) > optin) {
        free_program(d);
        throw std::runtime_error("engine: job arena needs " + std::to_string(smem) +
                                 " bytes of shared memory, device allows " + std::to_string(optin));
    }
    return d;
}

void free_program(DeviceProgram& d) {
    cudaFree(d.stream);
    cudaFree(d.stage_off);
    cudaFree(d.stage_bytes);
    cudaFree(d.jobs);
    cudaFree(d.counters);
    d = DeviceProgram{};
}

cudaError_t launch_generic(const DeviceProgram& prog, bool transpose, const GenericIO& io, cudaStream_t st) {
    const int chunks = (io.nrhs + kRC - 1) / kRC;
    GenericPolicy pol{io};
    return transpose ? launch<GenericPolicy, true>(prog, pol, chunks, st)
                     : launch<GenericPolicy, false>(prog, pol, chunks, st);
}

cudaError_t launch_sht(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st) {
    ShtPolicy pol{io};
    return transpose ? launch<ShtPolicy, true>(prog, pol, batch, st) : launch<ShtPolicy, false>(prog, pol, batch, st);
}

}  // namespace bfb
