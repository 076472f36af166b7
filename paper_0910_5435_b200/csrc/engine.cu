// The butterfly engine: one persistent, warp-specialised kernel per direction
// that applies every butterfly plan of a plan set (reference bfly::apply /
// bfly::apply_transpose, src/butterfly.cpp:384-513) for a few right-hand sides
// (RC = 4: the +-m x re/im columns of one function).  Batches of functions run
// on the graph program instead (waves.cpp, wgraph.cu).
//
// CTA = kConsumerWarps (4; 8 in engine_wide.cu) consumer warps + 1 producer
// warp.  The producer claims jobs (one (mu, parity) chain x one function) from
// a global work counter and streams each job's stages (engine_format.hpp) into
// a kRingStages-slot (2) shared-memory ring with cp.async.bulk + mbarrier
// complete_tx.  Consumers replay the records against coefficient vectors that
// never leave shared memory:
//   * matrix panels are contracted with FP64 FMAs on the CUDA cores: forward,
//     32-row items (lane = output row, whole K per lane); transpose, 16-column
//     items (lane = output column, half-warps split the rows, one shuffle).
//     At RC = 4 the DMMA m8n8k4 tile would be half padding; dmma() below is
//     kept only for the measured alternative;
//   * leaf inputs are prefetched one event ahead with cp.async;
//   * the SHT prologue / epilogue fold the +-x parity combine and the
//     sqrt(rho) scaling into the chain-value buffers read by the phi kernels.
// FP64 throughout.  Every matrix word is read from HBM once per apply.
#include <cuda_runtime.h>
#include <cstdlib>

#include <algorithm>
#include <cstdio>
#include <mutex>
#include <stdexcept>
#include <string>

#include "engine.hpp"

namespace bfb {

namespace {

#ifndef BFB_ENGINE_WIDE
#define BFB_ENGINE_WIDE 0  // engine_wide.cu: the same engine with 8 consumer warps, 1 CTA per SM
#endif
#ifndef BFB_MIN_BLOCKS
#define BFB_MIN_BLOCKS 3
#endif

constexpr unsigned kFull = 0xffffffffu;
constexpr int kNT = kConsumerThreads;
constexpr int kNW = kConsumerWarps;

// ---- PTX wrappers ------------------------------------------------------------

__device__ __forceinline__ std::uint32_t smem_u32(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* b, std::uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* b, std::uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(std::uint64_t* b, std::uint32_t parity) {
    std::uint32_t ok;
    asm volatile(
        "{\n"
        ".reg .pred P1;\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\n"
        "selp.u32 %0, 1, 0, P1;\n"
        "}\n"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity), "r"(1000000u)  // suspend up to 1 ms instead of spinning
        : "memory");
    return ok != 0;
}
// Waits for the phase with the given parity; a wait beyond ~2^35 cycles
// (well over ten seconds) traps instead of hanging the device.
__device__ __forceinline__ void mbar_wait(std::uint64_t* b, std::uint32_t parity) {
    if (mbar_try_wait(b, parity)) return;
    long long t0 = 0;
    for (std::uint32_t it = 1; !mbar_try_wait(b, parity); ++it) {
        if ((it & 1023u) == 0) {  // look at the clock only now and then
            const long long now = clock64();
            if (t0 == 0) t0 = now;
            else if (now - t0 > (1LL << 35)) __trap();
        }
    }
}
// The plan stream is read once per apply: evict-first in L2 so it does not
// push out the vectors (u, coefficients) the neighbouring kernels reuse.
__device__ __forceinline__ std::uint64_t l2_evict_first_policy() {
    std::uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, std::uint32_t bytes, std::uint64_t* bar,
                                         std::uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async16_l2(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }
// Barrier over the consumer warps only (the producer never joins).
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kNT) : "memory"); }
// D(8x8) += A(8x4) * B(4x8), FP64 tensor core.
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

struct JobCtx {
    int chunk, n_plans, mu, parity, kind;
    std::uint32_t plan[2], yA[2], n_cols[2], n_rows, yin, yout;
};

__device__ __forceinline__ std::uint32_t zcell(const Rec& r, std::uint32_t k) {
    return k < r.kl ? r.zA + k : r.zB + (k - r.kl);
}

// ---- I/O policies -------------------------------------------------------------

struct GenericPolicy {
    GenericIO io;

    template <int RC>
    __device__ void c_xchg(const JobCtx&, bool, std::uint32_t, std::uint32_t, int, double*, int) const {}
    template <bool BWD>
    __device__ void job_wait(const JobCtx&) const {}
    template <bool BWD>
    __device__ void job_signal(const JobCtx&) const {}

    // Input rows row0..row0+n of plan slot ps -> cells (cp.async, 8 B each).
    template <int RC>
    __device__ void load_rows(const JobCtx& j, int ps, std::uint32_t row0, int n, std::uint32_t cells, double* arena,
                              int t) const {
        const std::uint64_t base = io.in_prefix[j.plan[ps]] * static_cast<std::uint64_t>(io.nrhs);
        const std::uint32_t ld = j.n_cols[ps];
        for (int idx = t; idx < n * RC; idx += kNT) {
            const int r = idx / n, k = idx - r * n;
            const int rhs = j.chunk * RC + r;
            double* dst = arena + static_cast<std::size_t>(cells + k) * RC + r;
            if (rhs < io.nrhs)
                cp_async8(dst, io.in + base + static_cast<std::uint64_t>(rhs) * ld + row0 + k);
            else
                *dst = 0.0;
        }
    }
    template <int RC>
    __device__ void store_rows(const JobCtx& j, int ps, std::uint32_t row0, int n, std::uint32_t cells,
                               const double* arena, int t) const {
        const std::uint64_t base = io.out_prefix[j.plan[ps]] * static_cast<std::uint64_t>(io.nrhs);
        const std::uint32_t ld = j.n_cols[ps];
        for (int idx = t; idx < n * RC; idx += kNT) {
            const int r = idx / n, k = idx - r * n;
            const int rhs = j.chunk * RC + r;
            if (rhs < io.nrhs)
                io.out[base + static_cast<std::uint64_t>(rhs) * ld + row0 + k] =
                    arena[static_cast<std::size_t>(cells + k) * RC + r];
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
                double* dst = arena + static_cast<std::size_t>(j.yA[ps] + i) * RC + r;
                if (rhs < io.nrhs)
                    cp_async8(dst, io.in + base + static_cast<std::uint64_t>(rhs) * n + i);
                else
                    *dst = 0.0;
            }
        }
        cp_async_wait_all();
    }
};

// SHT: one job = one degree chain (mu, parity) for one batch member b = chunk;
// RC = 4 right-hand sides r = 2*sign + reim, sign 0 -> m = +mu, sign 1 ->
// m = -mu (absent for mu = 0).  The job's rows go to / come from the staging
// buffer u[plan][b][i][4] (weighted node values sqrt(rho_i) * chain sum); the
// +-x parity combine and the phi-stage layout are handled by combine_kernel /
// split_kernel below.
template <int MODE>  // 0: whole chains (u staging), 1: event program, 2: root program, 3: merged
struct ShtPolicyT {
    ShtIO io;

    // Merged programs: a job waits for the jobs it depends on, and publishes
    // its own completion (thread 0; the caller brackets with barriers).
    __device__ __forceinline__ unsigned long long* dep_word(const JobCtx& j) const {
        return io.dep + static_cast<long long>(j.plan[0]) * io.batch + j.chunk;
    }
    template <bool BWD>
    __device__ void job_wait(const JobCtx& j) const {
        if (MODE != 3) return;
        const bool waits = BWD ? j.kind == 0 : j.kind == 1;
        if (!waits) return;
        const unsigned long long target = BWD ? io.epoch * io.plan_roots[j.plan[0]] : io.epoch;
        const unsigned long long* w = dep_word(j);
        const long long t0 = clock64();
        for (;;) {
            unsigned long long v;
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(w) : "memory");
            if (v >= target) break;
            __nanosleep(200);
            if (clock64() - t0 > (1LL << 35)) __trap();
        }
    }
    template <bool BWD>
    __device__ void job_signal(const JobCtx& j) const {
        if (MODE != 3) return;
        const bool signals = BWD ? j.kind == 1 : j.kind == 0;
        if (!signals) return;
        __threadfence();
        if (BWD)
            atomicAdd(dep_word(j), 1ull);
        else
            asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(dep_word(j)), "l"(io.epoch) : "memory");
    }

    // Real fields (RC = 2): coefficients of m >= 0 only, order blocks of 2l - mu
    // degrees back to back (beta^{-m} = conj(beta^m) is implied).
    __device__ __forceinline__ long long coeff_index_half(int mu, int col, int parity) const {
        const long long l = io.l;
        return static_cast<long long>(mu) * 2 * l - static_cast<long long>(mu) * (mu - 1) / 2 + 2LL * col + parity;
    }
    __device__ __forceinline__ long long coeff_index(int mu, int sign, int col, int parity) const {
        const long long l = io.l;
        const long long base = mu == 0 ? 0 : 2 * l + static_cast<long long>(mu - 1) * (4 * l - mu);
        return base + sign * (2 * l - mu) + 2LL * col + parity;
    }
    template <int RC>
    __device__ __forceinline__ double* urow(const JobCtx& j) const {  // u[chain][b][i][RC]
        return io.u + (static_cast<long long>(j.plan[0]) * io.batch + j.chunk) * io.l * RC;
    }

    // cells <-> C[b][off .. off + n]
    template <int RC>
    __device__ void c_xchg(const JobCtx& j, bool load, std::uint32_t cells, std::uint32_t off, int n, double* arena,
                           int t) const {
        double* ca = arena + static_cast<std::size_t>(cells) * 4;
        if (io.cell_major) {  // C[cell][b][4]
            for (int idx = t; idx < n * 2; idx += kNT) {
                double* cg = io.c + ((static_cast<long long>(off) + (idx >> 1)) * io.batch + j.chunk) * 4 + 2 * (idx & 1);
                if (load)
                    cp_async16_l2(ca + 2 * idx, cg);
                else
                    *reinterpret_cast<double2*>(cg) = *reinterpret_cast<const double2*>(ca + 2 * idx);
            }
            return;
        }
        double* cg = io.c + (static_cast<long long>(j.chunk) * io.c_cells + off) * 4;
        for (int idx = t; idx < n * 2; idx += kNT) {
            if (load)
                cp_async16_l2(ca + 2 * idx, cg + 2 * idx);  // written by another SM: bypass L1
            else
                *reinterpret_cast<double2*>(cg + 2 * idx) = *reinterpret_cast<const double2*>(ca + 2 * idx);
        }
    }

    template <int RC>
    __device__ void load_rows(const JobCtx& j, int, std::uint32_t row0, int n, std::uint32_t cells, double* arena,
                              int t) const {
        static_assert(RC == 4 || RC == 2, "SHT jobs carry (+-m, re/im) or, for real fields, (re/im) of +m");
        const double* src = io.beta_in + static_cast<long long>(j.chunk) * io.beta_stride;
        if (RC == 2) {
            for (int idx = t; idx < n; idx += kNT)
                cp_async16(arena + static_cast<std::size_t>(cells + idx) * 2,
                           src + 2 * coeff_index_half(j.mu, static_cast<int>(row0) + idx, j.parity));
            return;
        }
        if (io.real_per_task == 2) {  // two real fields per task: cell = (field 2c, field 2c + 1)
            for (int idx = t; idx < n * 2; idx += kNT) {
                const int k = idx >> 1, h = idx & 1, m = 2 * j.chunk + h;
                double* dst = arena + static_cast<std::size_t>(cells + k) * 4 + 2 * h;
                if (m < io.real_members) {
                    cp_async16(dst, io.beta_in + static_cast<long long>(m) * io.beta_stride +
                                        2 * coeff_index_half(j.mu, static_cast<int>(row0) + k, j.parity));
                } else {
                    dst[0] = 0.0;
                    dst[1] = 0.0;
                }
            }
            return;
        }
        for (int idx = t; idx < n * 2; idx += kNT) {
            const int k = idx >> 1, sign = idx & 1;
            double* dst = arena + static_cast<std::size_t>(cells + k) * 4 + 2 * sign;
            if (j.mu == 0 && sign) {
                dst[0] = 0.0;
                dst[1] = 0.0;
            } else {
                cp_async16(dst, src + 2 * coeff_index(j.mu, sign, static_cast<int>(row0) + k, j.parity));
            }
        }
    }
    template <int RC>
    __device__ void store_rows(const JobCtx& j, int, std::uint32_t row0, int n, std::uint32_t cells,
                               const double* arena, int t) const {
        if (io.real_per_task == 2) {
            for (int idx = t; idx < n * 2; idx += kNT) {
                const int k = idx >> 1, h = idx & 1, m = 2 * j.chunk + h;
                if (m >= io.real_members) continue;
                *reinterpret_cast<double2*>(io.beta_out + static_cast<long long>(m) * io.beta_stride +
                                            2 * coeff_index_half(j.mu, static_cast<int>(row0) + k, j.parity)) =
                    *reinterpret_cast<const double2*>(arena + static_cast<std::size_t>(cells + k) * 4 + 2 * h);
            }
            return;
        }
        double* dst = io.beta_out + static_cast<long long>(j.chunk) * io.beta_stride;
        if (RC == 2) {
            for (int idx = t; idx < n; idx += kNT)
                *reinterpret_cast<double2*>(dst + 2 * coeff_index_half(j.mu, static_cast<int>(row0) + idx, j.parity)) =
                    *reinterpret_cast<const double2*>(arena + static_cast<std::size_t>(cells + idx) * 2);
            return;
        }
        for (int idx = t; idx < n * 2; idx += kNT) {
            const int k = idx >> 1, sign = idx & 1;
            if (j.mu == 0 && sign) continue;
            const double2 v =
                *reinterpret_cast<const double2*>(arena + static_cast<std::size_t>(cells + k) * 4 + 2 * sign);
            *reinterpret_cast<double2*>(dst + 2 * coeff_index(j.mu, sign, static_cast<int>(row0) + k, j.parity)) = v;
        }
    }
    // forward end of job: whole chains -> u; root jobs -> their group partial rows
    template <int RC>
    __device__ void epilogue(const JobCtx& j, const double* arena, int t) const {
        if (MODE == 1 || (MODE == 3 && j.kind == 0)) return;
        double2* dst = MODE == 0 ? reinterpret_cast<double2*>(urow<RC>(j))
                                 : reinterpret_cast<double2*>(io.ypart + (static_cast<long long>(j.chunk) * io.y_rows + j.yout) * 4);
        const double2* src = reinterpret_cast<const double2*>(arena + static_cast<std::size_t>(j.yA[0]) * RC);
        for (int idx = t; idx < static_cast<int>(j.n_rows) * (RC / 2); idx += kNT) dst[idx] = src[idx];
    }
    // transpose start of job: u rows (whole chain, or the root stripe's rows)
    template <int RC>
    __device__ void prologue(const JobCtx& j, double* arena, int t) const {
        if (MODE == 1 || (MODE == 3 && j.kind == 0)) return;
        const double* src = urow<RC>(j) + (MODE >= 2 ? static_cast<long long>(j.yin) * RC : 0);
        double* dst = arena + static_cast<std::size_t>(j.yA[0]) * RC;
        for (int idx = t; idx < static_cast<int>(j.n_rows) * (RC / 2); idx += kNT)
            cp_async16(dst + 2 * idx, src + 2 * idx);
        cp_async_wait_all();
    }
};
using ShtPolicy = ShtPolicyT<0>;
using ShtEventPolicy = ShtPolicyT<1>;
using ShtRootPolicy = ShtPolicyT<2>;
using ShtMergedPolicy = ShtPolicyT<3>;

// Plan index of chain (mu, p) in the SHT plan order (mu ascending, even then
// odd; the odd chain of mu = 2l - 1 is empty).
__device__ __forceinline__ int plan_index(int mu, int p) { return 2 * mu + p; }

#if !BFB_ENGINE_WIDE
// Synthesis phi-prep: g_m(+-x_i) = (u_even +- u_odd) / sqrt(rho_i) into the
// [bin][b][t] buffer (bins mu and N - mu).  One block per (mu, b).
__global__ void __launch_bounds__(256) combine_kernel(ShtIO io) {
    const int mu = io.mu0 + blockIdx.x, b = blockIdx.y, l = io.l, N = io.N;
    const bool odd = mu < 2 * l - 1;
    const int p0 = plan_index(mu, 0) - plan_index(io.mu0, 0);
    const double* ue = io.u + (static_cast<long long>(p0) * io.batch + b) * l * 4;
    const double* uo = odd ? io.u + (static_cast<long long>(p0 + 1) * io.batch + b) * l * 4 : nullptr;
    // split programs: u = sum of the plan's root-group partials
    const double* pe = nullptr;
    const double* po = nullptr;
    int ge = 0, go = 0;
    // partial row r of member b: member-major [b][y_rows][4] or cell-major [y_rows][b][4]
    long long rstride = 4, bstride = static_cast<long long>(io.y_rows) * 4;
    if (io.cell_major) {
        rstride = 4LL * io.batch;
        bstride = 4;
    }
    if (io.ypart) {
        pe = io.ypart + b * bstride + io.plan_yoff[p0] * rstride;
        ge = static_cast<int>(io.plan_groups[p0]);
        if (odd) {
            po = io.ypart + b * bstride + io.plan_yoff[p0 + 1] * rstride;
            go = static_cast<int>(io.plan_groups[p0 + 1]);
        }
    }
    double2* g = reinterpret_cast<double2*>(io.g_out);
    const long long rp = (static_cast<long long>(mu) * io.batch + b) * 2 * l;
    const long long rm = (static_cast<long long>(N - mu) * io.batch + b) * 2 * l;
    for (int i = threadIdx.x; i < l; i += blockDim.x) {
        const double s = io.isr[i];
        double4 e, o = make_double4(0.0, 0.0, 0.0, 0.0);
        if (pe) {
            e = *reinterpret_cast<const double4*>(pe + rstride * i);
            for (int k = 1; k < ge; ++k) {
                const double4 v = *reinterpret_cast<const double4*>(pe + rstride * (static_cast<long long>(k) * l + i));
                e.x += v.x;
                e.y += v.y;
                e.z += v.z;
                e.w += v.w;
            }
            if (odd) {
                o = *reinterpret_cast<const double4*>(po + rstride * i);
                for (int k = 1; k < go; ++k) {
                    const double4 v = *reinterpret_cast<const double4*>(po + rstride * (static_cast<long long>(k) * l + i));
                    o.x += v.x;
                    o.y += v.y;
                    o.z += v.z;
                    o.w += v.w;
                }
            }
        } else {
            e = *reinterpret_cast<const double4*>(ue + 4 * i);
            if (odd) o = *reinterpret_cast<const double4*>(uo + 4 * i);
        }
        g[rp + l + i] = make_double2((e.x + o.x) * s, (e.y + o.y) * s);
        g[rp + l - 1 - i] = make_double2((e.x - o.x) * s, (e.y - o.y) * s);
        if (mu > 0) {
            g[rm + l + i] = make_double2((e.z + o.z) * s, (e.w + o.w) * s);
            g[rm + l - 1 - i] = make_double2((e.z - o.z) * s, (e.w - o.w) * s);
        }
    }
}

// Analysis phi-prep: u_even,i = sqrt(rho_i)/(2N) (G(+x_i) + G(-x_i)), u_odd
// with '-', from the unnormalised forward DFT rows G (bins mu and N - mu).
__global__ void __launch_bounds__(256) split_kernel(ShtIO io) {
    const int mu = io.mu0 + blockIdx.x, b = blockIdx.y, l = io.l, N = io.N;
    const bool odd = mu < 2 * l - 1;
    const int p0 = plan_index(mu, 0) - plan_index(io.mu0, 0);
    double* ue = io.u + (static_cast<long long>(p0) * io.batch + b) * l * 4;
    double* uo = odd ? io.u + (static_cast<long long>(p0 + 1) * io.batch + b) * l * 4 : nullptr;
    const double2* g = reinterpret_cast<const double2*>(io.g_in);
    const long long rp = (static_cast<long long>(mu) * io.batch + b) * 2 * l;
    const long long rm = (static_cast<long long>(N - mu) * io.batch + b) * 2 * l;
    for (int i = threadIdx.x; i < l; i += blockDim.x) {
        const double s = io.hsr[i];
        const double2 pp = g[rp + l + i], pm = g[rp + l - 1 - i];
        double2 mp = make_double2(0.0, 0.0), mm = make_double2(0.0, 0.0);
        if (mu > 0) {
            mp = g[rm + l + i];
            mm = g[rm + l - 1 - i];
        }
        *reinterpret_cast<double4*>(ue + 4 * i) =
            make_double4((pp.x + pm.x) * s, (pp.y + pm.y) * s, (mp.x + mm.x) * s, (mp.y + mm.y) * s);
        if (odd)
            *reinterpret_cast<double4*>(uo + 4 * i) =
                make_double4((pp.x - pm.x) * s, (pp.y - pm.y) * s, (mp.x - mm.x) * s, (mp.y - mm.y) * s);
    }
}

#endif  // !BFB_ENGINE_WIDE

// ---- panel contraction (FP64 FMA, warp-granular work items) -----------------
//
// Work items are 16 outputs wide and owned by one warp: lane = (output o =
// lane & 15, half h = lane >> 4); the two half-warps split the reduction
// dimension (even / odd columns forward, even / odd rows transpose) and are
// combined with one shuffle.  Forward: the outputs are a unit's rows, the
// item lives across all of the unit's panels.  Transpose: the outputs are a
// panel's columns (the odd leading dimension keeps the lanes' strided reads
// bank-conflict free).  Items are dealt round-robin to the consumer warps
// from a running counter, so warps overlap across consecutive units and
// panels without barriers.

// Work items: forward = kItemWF rows of a unit (lane = row, kKSplitF lane
// groups split the columns), transpose = kItemWB columns of a panel (lane =
// column, kKSplitB groups split the rows).  Measured at l=256: whole-row
// lanes (32-row items, no split) are fastest forward, 16-column items with a
// two-way row split fastest in the transpose.
#ifndef BFB_ITEM_WF
#define BFB_ITEM_WF 32
#endif
#ifndef BFB_ITEM_WB
#define BFB_ITEM_WB 16
#endif
constexpr int kItemWF = BFB_ITEM_WF, kKSplitF = 32 / kItemWF;
constexpr int kItemWB = BFB_ITEM_WB, kKSplitB = 32 / kItemWB;
static_assert((kItemWF == 8 || kItemWF == 16 || kItemWF == 32) && (kItemWB == 8 || kItemWB == 16 || kItemWB == 32),
              "item width");

// Sum over the lane groups (lanes l, l + W, l + 2W, ...) of width W.
template <int W>
__device__ __forceinline__ double ksplit_sum(double v) {
#pragma unroll
    for (int off = W; off < 32; off <<= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
    return v;
}

// First k >= 0 with (item + k) mod kNW == w: items are dealt round-robin.
__device__ __forceinline__ int rr_first(int item, int w) {
    const int m = (w - item) % kNW;
    return m < 0 ? m + kNW : m;
}

// Row blocks a warp may own in one unit (kChunkRows / kItemW items dealt over
// kNW warps).
constexpr int kMaxOwn = (kChunkRows / kItemWF + kNW - 1) / kNW;

template <int RC>
struct FwdItem {
    double acc[kMaxOwn][RC];
    int row[kMaxOwn];  // unit row of this lane's output per owned block (>= nr if none)
    int n_own;         // row blocks owned by this warp in the current unit
};

#ifndef BFB_KU
#define BFB_KU 8
#endif
constexpr int kU = BFB_KU;  // columns (forward) / rows (transpose) per batched step

// Forward panel: acc[k][c] += sum_q P[row_k, q] * B(q)[c] over this half-warp's
// contiguous half of the panel's columns, B(q) = z(others[q]) (TPANEL) or
// cell(cA + q) (SPANEL).  kU columns per step: all operand loads of a step are
// issued before its FMAs, and the B operand is shared by the warp's row blocks.
template <int RC, bool TP>
__device__ __forceinline__ void fwd_panel(const Rec& r, const unsigned char* stage, const double* arena,
                                          FwdItem<RC>& it, int ks) {
    const std::uint16_t* oth = reinterpret_cast<const std::uint16_t*>(stage + r.data);
    const double* P = reinterpret_cast<const double*>(stage + r.data + r.moff);
    const int nc = r.nc, ld = r.ld;
    const int qs = (nc + kKSplitF - 1) / kKSplitF;
    const int q_begin = min(nc, ks * qs), q_end = min(nc, q_begin + qs);
    bool ok[kMaxOwn];
    const double* pr[kMaxOwn];
    double acc[kMaxOwn][RC];
#pragma unroll
    for (int k = 0; k < kMaxOwn; ++k) {
        ok[k] = k < it.n_own && it.row[k] < r.nr;
        pr[k] = P + (ok[k] ? it.row[k] : 0);
#pragma unroll
        for (int c = 0; c < RC; ++c) acc[k][c] = it.acc[k][c];
    }
    auto bcell = [&](int q) -> const double2* {
        const std::uint32_t cell = TP ? zcell(r, oth[q]) : r.cA + q;
        return reinterpret_cast<const double2*>(arena + static_cast<std::size_t>(cell) * RC);
    };
    int q = q_begin;
    for (; q + kU <= q_end; q += kU) {
        double2 b[kU][RC / 2];
        double a[kMaxOwn][kU];
#pragma unroll
        for (int u = 0; u < kU; ++u) {
            const double2* bp = bcell(q + u);
#pragma unroll
            for (int c2 = 0; c2 < RC / 2; ++c2) b[u][c2] = bp[c2];
        }
#pragma unroll
        for (int k = 0; k < kMaxOwn; ++k)
#pragma unroll
            for (int u = 0; u < kU; ++u) a[k][u] = ok[k] ? pr[k][(q + u) * ld] : 0.0;
#pragma unroll
        for (int u = 0; u < kU; ++u)
#pragma unroll
            for (int k = 0; k < kMaxOwn; ++k)
#pragma unroll
                for (int c2 = 0; c2 < RC / 2; ++c2) {
                    acc[k][2 * c2] = fma(a[k][u], b[u][c2].x, acc[k][2 * c2]);
                    acc[k][2 * c2 + 1] = fma(a[k][u], b[u][c2].y, acc[k][2 * c2 + 1]);
                }
    }
    for (; q < q_end; ++q) {
        const double2* bp = bcell(q);
#pragma unroll
        for (int k = 0; k < kMaxOwn; ++k) {
            const double a = ok[k] ? pr[k][q * ld] : 0.0;
#pragma unroll
            for (int c2 = 0; c2 < RC / 2; ++c2) {
                const double2 v = bp[c2];
                acc[k][2 * c2] = fma(a, v.x, acc[k][2 * c2]);
                acc[k][2 * c2 + 1] = fma(a, v.y, acc[k][2 * c2 + 1]);
            }
        }
    }
#pragma unroll
    for (int k = 0; k < kMaxOwn; ++k)
#pragma unroll
        for (int c = 0; c < RC; ++c) it.acc[k][c] = acc[k][c];
}

// Transpose panel: out(col)[c] = sum_i P[i, col] * V(i)[c] for this warp's
// 16-column blocks (half-warps take contiguous halves of the rows, combined
// with one shuffle), V = cell(cA + i) (TPANEL) or cell(zA + i) (SPANEL); the
// result goes to z(others[col]) or cell(cA + col), '=' or '+='.
template <int RC, bool TP>
__device__ __forceinline__ void bwd_panel(const Rec& r, const unsigned char* stage, double* arena, int& item, int w,
                                          int lane) {
    const std::uint16_t* oth = reinterpret_cast<const std::uint16_t*>(stage + r.data);
    const double* P = reinterpret_cast<const double*>(stage + r.data + r.moff);
    const int nc = r.nc, nr = r.nr, ld = r.ld;
    const int nblk = (nc + kItemWB - 1) / kItemWB;
    const bool assign = r.flags & F_ASSIGN_BWD;
    const int o = lane & (kItemWB - 1), ks = lane / kItemWB;
    const int is = (nr + kKSplitB - 1) / kKSplitB;
    const int i_begin = min(nr, ks * is), i_end = min(nr, i_begin + is);
    const double2* vb = reinterpret_cast<const double2*>(arena + static_cast<std::size_t>(TP ? r.cA : r.zA) * RC);
    for (int blk = rr_first(item, w); blk < nblk; blk += kNW) {
        const int col = kItemWB * blk + o;
        const bool ok = col < nc;
        const double* pc = P + static_cast<std::size_t>(ok ? col : 0) * ld;
        double acc[RC];
#pragma unroll
        for (int c = 0; c < RC; ++c) acc[c] = 0.0;
        int i = i_begin;
        for (; i + kU <= i_end; i += kU) {
            double a[kU];
            double2 b[kU][RC / 2];
#pragma unroll
            for (int u = 0; u < kU; ++u) {
                a[u] = ok ? pc[i + u] : 0.0;
#pragma unroll
                for (int c2 = 0; c2 < RC / 2; ++c2) b[u][c2] = vb[(i + u) * (RC / 2) + c2];
            }
#pragma unroll
            for (int u = 0; u < kU; ++u)
#pragma unroll
                for (int c2 = 0; c2 < RC / 2; ++c2) {
                    acc[2 * c2] = fma(a[u], b[u][c2].x, acc[2 * c2]);
                    acc[2 * c2 + 1] = fma(a[u], b[u][c2].y, acc[2 * c2 + 1]);
                }
        }
        for (; i < i_end; ++i) {
            const double a = ok ? pc[i] : 0.0;
#pragma unroll
            for (int c2 = 0; c2 < RC / 2; ++c2) {
                const double2 v = vb[i * (RC / 2) + c2];
                acc[2 * c2] = fma(a, v.x, acc[2 * c2]);
                acc[2 * c2 + 1] = fma(a, v.y, acc[2 * c2 + 1]);
            }
        }
#pragma unroll
        for (int c = 0; c < RC; ++c) acc[c] = ksplit_sum<kItemWB>(acc[c]);
        if (ok && ks == 0) {
            const std::uint32_t cell = TP ? zcell(r, oth[col]) : r.cA + col;
            double2* p = reinterpret_cast<double2*>(arena + static_cast<std::size_t>(cell) * RC);
#pragma unroll
            for (int c2 = 0; c2 < RC / 2; ++c2) {
                double2 v = make_double2(acc[2 * c2], acc[2 * c2 + 1]);
                if (!assign) {
                    const double2 q2 = p[c2];
                    v.x += q2.x;
                    v.y += q2.y;
                }
                p[c2] = v;
            }
        }
    }
    item += nblk;
}

template <int RC, class Policy, bool BWD>
__global__ void __launch_bounds__(kEngineThreads, BFB_MIN_BLOCKS)
    engine_kernel(const std::uint8_t* __restrict__ stream, const std::uint64_t* __restrict__ stage_off,
                  const std::uint32_t* __restrict__ stage_bytes, const Job* __restrict__ jobs,
                  unsigned* __restrict__ counters, unsigned claim_base, int n_tasks, int n_chunks,
                  std::uint32_t zo_cells,
                  unsigned long long* __restrict__ trace, int debug, std::uint32_t stage_cap,
                  const std::uint32_t* __restrict__ order, Policy pol) {
    extern __shared__ __align__(128) unsigned char smem[];
    // Programmatic dependent launch: the next kernel on the stream may be
    // scheduled as soon as SM resources free up; it waits for this grid's
    // completion itself (griddepcontrol.wait) before reading our outputs.
    asm volatile("griddepcontrol.launch_dependents;");
    unsigned char* ring = smem;
    std::uint64_t* full = reinterpret_cast<std::uint64_t*>(smem + kRingStages * stage_cap);
    std::uint64_t* empty = full + kRingStages;
    int4* info = reinterpret_cast<int4*>(empty + kRingStages);
    double* arena = reinterpret_cast<double*>(info + kRingStages);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (int s = 0; s < kRingStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], kNW);
        }
        mbar_fence_init();
    }
    __syncthreads();

    if (warp == kNW) {
        // ------------------------------ producer ------------------------------
        const std::uint64_t policy = l2_evict_first_policy();
        std::uint32_t g = 0;
        // First task: the CTA's own index (no atomic round trip before the first
        // bulk copy); later tasks come from the counter, offset by the grid.
        int task = static_cast<int>(blockIdx.x);
        bool waited = false;
        for (;;) {
            if (task >= n_tasks) {
                const std::uint32_t slot = g % kRingStages, use = g / kRingStages;
                if (use > 0) mbar_wait(&empty[slot], (use - 1) & 1);
                if (lane == 0) {
                    info[slot] = make_int4(-1, 0, 0, 0);
                    mbar_arrive(&full[slot]);
                }
                return;
            }
            // The next task is claimed once this one's last stage is issued: the
            // ring still holds up to kRingStages stages, which hides the atomic,
            // and a CTA never reserves a task it cannot start soon (claiming at
            // the start of a long job let early CTAs hoard first-wave tasks and
            // left a tail of one late job per hoarding CTA).
            const int job = order ? static_cast<int>(order[task / n_chunks]) : task / n_chunks;
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
                        bulk_g2s(ring + slot * stage_cap, stream + o, b, &full[slot], policy);
                    }
                    __syncwarp();
                    ++g;
                }
            }
            int nxt = 0;
            // The counter is never reset: every launch takes exactly n_tasks
            // increments (n_tasks - grid claims plus one failing claim per CTA),
            // so the host passes the running total as claim_base.  Under
            // programmatic dependent launch the preceding grid on the stream
            // may be an engine launch of the same program whose CTAs are still
            // claiming from this counter: wait for it to complete before the
            // first claim (the first task, blockIdx.x, needs no claim, so its
            // plan stages still stream while the predecessor drains).
            if (!waited) {
                asm volatile("griddepcontrol.wait;" ::: "memory");
                waited = true;
            }
            if (lane == 0) nxt = static_cast<int>(gridDim.x + (atomicAdd(&counters[0], 1u) - claim_base));
            task = __shfl_sync(kFull, nxt, 0);
        }
    }

    // ------------------------------ consumers --------------------------------
    // When launched as a programmatic dependent (e.g. after the fused phi
    // analysis), the producer already streams plan stages (read-only) while
    // the consumers wait here for the predecessor's outputs.  No-op otherwise.
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int t = tid;
    const bool prof = (debug & 2) && trace;  // debug bit 1: per-category cycle counts into trace
    long long tcat[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long ncat[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    const long long t_begin = prof ? clock64() : 0;
#define BFB_T0 long long _t0 = prof ? clock64() : 0
#define BFB_T1(cat) if (prof) { tcat[cat] += clock64() - _t0; ncat[cat] += 1; }
    JobCtx j{};
    FwdItem<RC> fi{};
    int item = 0;  // running work-item counter (forward: row blocks, transpose: column blocks)
    std::uint32_t g = 0;
    for (;;) {
        const std::uint32_t slot = g % kRingStages;
        {
            BFB_T0;
            mbar_wait(&full[slot], (g / kRingStages) & 1);
            BFB_T1(0);
        }
        const int4 inf = info[slot];
        if (inf.x < 0) {
            if (prof && lane == 0) {
                tcat[7] = clock64() - t_begin;
                for (int c = 0; c < 8; ++c) {
                    atomicAdd(reinterpret_cast<unsigned long long*>(trace) + c, static_cast<unsigned long long>(tcat[c]));
                    atomicAdd(reinterpret_cast<unsigned long long*>(trace) + 8 + c, static_cast<unsigned long long>(ncat[c]));
                }
            }
            break;
        }
        const unsigned char* stage = ring + slot * stage_cap;
        if (inf.y == 0) {
            const int jt = inf.x / n_chunks;
            const int job = order ? static_cast<int>(order[jt]) : jt;
            j.chunk = inf.x - jt * n_chunks;
            const Job& J = jobs[job];
            j.n_plans = J.n_plans;
            j.mu = J.mu;
            j.parity = static_cast<int>(J.parity);
            j.yin = J.yin;
            j.yout = J.yout;
            j.kind = static_cast<int>(J.kind);
            j.plan[0] = J.plan[0];
            j.plan[1] = J.plan[1];
            j.yA[0] = J.yA[0];
            j.yA[1] = J.yA[1];
            j.n_cols[0] = J.n_cols[0];
            j.n_cols[1] = J.n_cols[1];
            j.n_rows = J.n_rows;
            if (trace && !prof && t == 0) {
                unsigned long long now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                unsigned smid;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
                trace[4 * inf.x + 0] = now;
                trace[4 * inf.x + 2] = smid;
                trace[4 * inf.x + 3] = static_cast<unsigned long long>(inf.z);
            }
            BFB_T0;
            if (t == 0) pol.template job_wait<BWD>(j);
            consumer_sync();
            if (BWD) pol.template prologue<RC>(j, arena, t);
            consumer_sync();
            BFB_T1(6);
        }
        const StageHeader* h = reinterpret_cast<const StageHeader*>(stage);
        const Rec* recs = reinterpret_cast<const Rec*>(stage + sizeof(StageHeader));
        const int n = (debug & 1) ? 0 : static_cast<int>(h->n_rec);  // debug bit 0: stream only
        const bool no_math = debug & 4;  // debug bit 2: records and barriers, no panel arithmetic
        for (int q = 0; q < n; ++q) {
            const Rec r = recs[BWD ? n - 1 - q : q];
            if (r.flags & (BWD ? F_SYNC_BWD : F_SYNC_FWD)) {
                BFB_T0;
                cp_async_wait_all();
                consumer_sync();
                BFB_T1(1);
            }
            BFB_T0;
            switch (r.op) {
            case OP_LOADZ:
                if (!BWD)
                    pol.template load_rows<RC>(j, r.pslot, r.zB, r.nr, r.zA, arena, t);
                else
                    pol.template store_rows<RC>(j, r.pslot, r.zB, r.nr, r.zA, arena, t);
                break;
            case OP_CXCH:
                pol.template c_xchg<RC>(j, ((r.flags & F_CLOAD_FWD) != 0) != BWD, r.zA, r.zB, r.nr, arena, t);
                break;
            case OP_SEL: {
                const std::uint16_t* sel = reinterpret_cast<const std::uint16_t*>(stage + r.data);
                for (int idx = t; idx < r.nr * RC; idx += kNT) {
                    const int i = idx / RC, c = idx - i * RC;
                    const std::size_t zc = static_cast<std::size_t>(zcell(r, sel[i])) * RC + c;
                    const std::size_t cc = static_cast<std::size_t>(r.cA + i) * RC + c;
                    if (!BWD)
                        arena[cc] = arena[zc];
                    else
                        arena[zc] = (r.flags & F_ASSIGN_BWD) ? arena[cc] : arena[zc] + arena[cc];
                }
                break;
            }
            case OP_TPANEL:
            case OP_SPANEL: {
                const bool tp = r.op == OP_TPANEL;
                if (!BWD) {
                    if (r.flags & F_BEGIN) {
                        // deal this unit's 16-row blocks round-robin; lane owns a row of
                        // each of its blocks, half-warps split K
                        const int nrb = (r.nr + kItemWF - 1) / kItemWF;
                        const std::uint16_t* sel =
                            reinterpret_cast<const std::uint16_t*>(stage + r.data + ((2u * r.nc + 7u) & ~7u));
                        fi.n_own = 0;
#pragma unroll
                        for (int k = 0; k < kMaxOwn; ++k) {
                            const int blk = rr_first(item, warp) + k * kNW;
                            const int row = kItemWF * blk + (lane & (kItemWF - 1));
                            const bool own = blk < nrb;
                            fi.n_own += own ? 1 : 0;
                            fi.row[k] = own ? row : 0x7fffffff;
                            const bool init = tp && own && row < r.nr && lane < kItemWF;
                            const double* zp = arena + static_cast<std::size_t>(init ? zcell(r, sel[row]) : 0) * RC;
#pragma unroll
                            for (int c = 0; c < RC; ++c) fi.acc[k][c] = init ? zp[c] : 0.0;
                        }
                        item += nrb;
                    }
                    if (fi.n_own > 0 && !no_math) {
                        if (tp)
                            fwd_panel<RC, true>(r, stage, arena, fi, lane / kItemWF);
                        else
                            fwd_panel<RC, false>(r, stage, arena, fi, lane / kItemWF);
                        if (r.flags & F_END) {
                            const bool assign = tp || (r.flags & F_ASSIGN_FWD);
#pragma unroll
                            for (int k = 0; k < kMaxOwn; ++k) {
#pragma unroll
                                for (int c = 0; c < RC; ++c)
                                    fi.acc[k][c] = ksplit_sum<kItemWF>(fi.acc[k][c]);
                                if (fi.row[k] < r.nr && lane < kItemWF) {
                                    double2* p = reinterpret_cast<double2*>(
                                        arena + static_cast<std::size_t>((tp ? r.cA : r.zA) + fi.row[k]) * RC);
#pragma unroll
                                    for (int c2 = 0; c2 < RC / 2; ++c2) {
                                        double2 v = make_double2(fi.acc[k][2 * c2], fi.acc[k][2 * c2 + 1]);
                                        if (!assign) {
                                            const double2 o = p[c2];
                                            v.x += o.x;
                                            v.y += o.y;
                                        }
                                        p[c2] = v;
                                    }
                                }
                            }
                        }
                    }
                } else if (!no_math) {
                    if (tp)
                        bwd_panel<RC, true>(r, stage, arena, item, warp, lane);
                    else
                        bwd_panel<RC, false>(r, stage, arena, item, warp, lane);
                    if (tp && (r.flags & F_BEGIN)) {
                        // z(sel[i]) (=|+=) c[i] for the chunk rows (disjoint from z(others)).
                        const std::uint16_t* sel =
                            reinterpret_cast<const std::uint16_t*>(stage + r.data + ((2u * r.nc + 7u) & ~7u));
                        const bool asg = r.flags & F_ASSIGN_SEL_BWD;
                        for (int idx = t; idx < r.nr * RC; idx += kNT) {
                            const int i = idx / RC, c = idx - i * RC;
                            const std::size_t zc = static_cast<std::size_t>(zcell(r, sel[i])) * RC + c;
                            const double v = arena[static_cast<std::size_t>(r.cA + i) * RC + c];
                            arena[zc] = asg ? v : arena[zc] + v;
                        }
                    }
                }
                break;
            }
            default:
                break;
            }
            BFB_T1(r.op < 4 ? 2 + r.op : 6);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[slot]);
        if (inf.y == inf.z - 1) {
            BFB_T0;
            if (!BWD) cp_async_wait_all();
            consumer_sync();
            if (!BWD) pol.template epilogue<RC>(j, arena, t);
            cp_async_wait_all();
            consumer_sync();
            if (t == 0) pol.template job_signal<BWD>(j);
            BFB_T1(6);
            if (trace && !prof && t == 0) {
                unsigned long long now;
                asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(now));
                trace[4 * inf.x + 1] = now;
            }
        }
        ++g;
    }
}

// Per-instantiation launch configuration, computed once per (device, smem).
struct LaunchCache {
    std::mutex mu;
    int device = -1;
    std::size_t smem_set = 0;
    std::size_t smem_occ = 0;
    int sms = 0, per_sm = 0;
};

template <class Policy, bool BWD, int RC = kRC>
cudaError_t launch(const DeviceProgram& prog, const Policy& pol, int n_chunks, cudaStream_t st,
                   const std::uint32_t* order = nullptr, bool pdl = false) {
    if (prog.n_jobs == 0 || n_chunks == 0) return cudaSuccess;
    auto kern = engine_kernel<RC, Policy, BWD>;
    static LaunchCache cache;
    const std::size_t smem = engine_smem_bytes(prog, RC);
    int grid_cap = 0;
    {
        std::lock_guard<std::mutex> lk(cache.mu);
        int dev = 0;
        cudaError_t e = cudaGetDevice(&dev);
        if (e != cudaSuccess) return e;
        if (dev != cache.device) {
            cache.device = dev;
            cache.smem_set = cache.smem_occ = 0;
            cache.per_sm = 0;
            e = cudaDeviceGetAttribute(&cache.sms, cudaDevAttrMultiProcessorCount, dev);
            if (e != cudaSuccess) return e;
        }
        if (smem > cache.smem_set) {
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
            if (e != cudaSuccess) return e;
            e = cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     cudaSharedmemCarveoutMaxShared);
            if (e != cudaSuccess) return e;
            cache.smem_set = smem;
        }
        if (smem != cache.smem_occ) {
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&cache.per_sm, kern, kEngineThreads, smem);
            if (e != cudaSuccess) return e;
            cache.smem_occ = smem;
        }
        if (cache.per_sm < 1) return cudaErrorInvalidConfiguration;
        grid_cap = cache.sms * cache.per_sm;
    }
    const long long tasks = static_cast<long long>(prog.n_jobs) * n_chunks;
    const int grid = static_cast<int>(std::min<long long>(tasks, grid_cap));
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(kEngineThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    static const bool no_pdl = std::getenv("BFLY_NO_PDL") != nullptr;  // diagnostics
    cfg.numAttrs = (pdl && !no_pdl) ? 1 : 0;
    // The claim base advances only when the grid was actually launched (a failed
    // launch takes no increments).  One handle = one stream: the counter and the
    // scratch buffers are not guarded against concurrent launches on two streams.
    const unsigned base = prog.claimed;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, kern, prog.stream, prog.stage_off, prog.stage_bytes, prog.jobs,
                                             prog.counters, base, static_cast<int>(tasks), n_chunks, prog.zo_cells,
                                             prog.trace, prog.debug, prog.stage_capacity, order, pol);
    if (e == cudaSuccess) prog.claimed += static_cast<unsigned>(tasks);
    return e;
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

#if BFB_ENGINE_WIDE
namespace wide {
#else
namespace narrow {
#endif
cudaError_t launch_generic(const DeviceProgram& prog, bool transpose, const GenericIO& io, cudaStream_t st) {
    const int chunks = (io.nrhs + kRC - 1) / kRC;
    GenericPolicy pol{io};
    return transpose ? launch<GenericPolicy, true>(prog, pol, chunks, st)
                     : launch<GenericPolicy, false>(prog, pol, chunks, st);
}

cudaError_t launch_sht(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st,
                       bool pdl, bool real_field) {
    ShtPolicy pol{io};
    pol.io.batch = batch;
    if (real_field)
        return transpose ? launch<ShtPolicy, true, 2>(prog, pol, batch, st, nullptr, pdl)
                         : launch<ShtPolicy, false, 2>(prog, pol, batch, st, nullptr, pdl);
    return transpose ? launch<ShtPolicy, true>(prog, pol, batch, st, nullptr, pdl)
                     : launch<ShtPolicy, false>(prog, pol, batch, st, nullptr, pdl);
}

cudaError_t launch_sht_events(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st) {
    ShtEventPolicy pol{io};
    pol.io.batch = batch;
    return transpose ? launch<ShtEventPolicy, true>(prog, pol, batch, st)
                     : launch<ShtEventPolicy, false>(prog, pol, batch, st);
}

cudaError_t launch_sht_roots(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st) {
    ShtRootPolicy pol{io};
    pol.io.batch = batch;
    return transpose ? launch<ShtRootPolicy, true>(prog, pol, batch, st)
                     : launch<ShtRootPolicy, false>(prog, pol, batch, st);
}

cudaError_t launch_sht_merged(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st) {
    ShtMergedPolicy pol{io};
    pol.io.batch = batch;
    return transpose ? launch<ShtMergedPolicy, true>(prog, pol, batch, st, prog.order[1])
                     : launch<ShtMergedPolicy, false>(prog, pol, batch, st, prog.order[0]);
}

}  // namespace wide / narrow

#if !BFB_ENGINE_WIDE
std::size_t engine_smem_bytes(const DeviceProgram& prog, int rc) {
    return static_cast<std::size_t>(kRingStages) * prog.stage_capacity + 2 * kRingStages * sizeof(std::uint64_t) +
           kRingStages * sizeof(int4) +
           static_cast<std::size_t>(prog.arena_cells) * rc * sizeof(double);
}

DeviceProgram upload_program(const PackedProgram& p, int device) {
    if (cudaSetDevice(device) != cudaSuccess) throw std::runtime_error("cudaSetDevice failed");
    DeviceProgram d;
    d.device = device;
    d.stream = upload(p.stream);
    d.stage_off = upload(p.stage_off);
    d.stage_bytes = upload(p.stage_bytes);
    d.jobs = upload(p.jobs);
    d.order[0] = upload(p.order_fwd);
    d.order[1] = upload(p.order_bwd);
    d.plan_roots = upload(p.plan_roots);
    if (cudaMalloc(&d.counters, 2 * sizeof(unsigned)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed");
    cudaMemset(d.counters, 0, 2 * sizeof(unsigned));
    d.n_jobs = static_cast<int>(p.jobs.size());
    d.n_stages = p.stage_off.size();
    d.arena_cells = p.arena_cells;
    d.zo_cells = p.zo_cells;
    d.stage_capacity = p.stage_capacity;
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
    cudaFree(d.order[0]);
    cudaFree(d.order[1]);
    cudaFree(d.plan_roots);
    cudaFree(d.counters);
    d = DeviceProgram{};
}

// Programs whose arena leaves room for only one CTA per SM (large l) run the
// wide build (engine_wide.cu: 8 consumer warps per CTA; +12 % at c3, where 4
// warps per SM cannot hide the shared-memory latency); BFLY_ENGINE_WIDE=0/1
// forces either (diagnostics).
namespace wide {
cudaError_t launch_generic(const DeviceProgram& prog, bool transpose, const GenericIO& io, cudaStream_t st);
cudaError_t launch_sht(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st,
                       bool pdl, bool real_field);
cudaError_t launch_sht_events(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st);
cudaError_t launch_sht_roots(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st);
cudaError_t launch_sht_merged(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st);
}  // namespace wide

bool use_wide(const DeviceProgram& prog, int rc) {
    static const int force = [] {
        const char* e = std::getenv("BFLY_ENGINE_WIDE");
        return e ? static_cast<int>(std::strtol(e, nullptr, 10)) : -1;
    }();
    if (force >= 0) return force != 0;
    constexpr std::size_t kSmemPerSm = 228u * 1024u, kReserved = 1024u;
    return 2 * (engine_smem_bytes(prog, rc) + kReserved) > kSmemPerSm;
}

cudaError_t launch_generic(const DeviceProgram& prog, bool transpose, const GenericIO& io, cudaStream_t st) {
    return use_wide(prog, kRC) ? wide::launch_generic(prog, transpose, io, st)
                               : narrow::launch_generic(prog, transpose, io, st);
}
cudaError_t launch_sht(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st,
                       bool pdl, bool real_field) {
    return use_wide(prog, real_field ? 2 : kRC) ? wide::launch_sht(prog, transpose, io, batch, st, pdl, real_field)
                                                : narrow::launch_sht(prog, transpose, io, batch, st, pdl, real_field);
}
cudaError_t launch_sht_events(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st) {
    return use_wide(prog, kRC) ? wide::launch_sht_events(prog, transpose, io, batch, st)
                               : narrow::launch_sht_events(prog, transpose, io, batch, st);
}
cudaError_t launch_sht_roots(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st) {
    return use_wide(prog, kRC) ? wide::launch_sht_roots(prog, transpose, io, batch, st)
                               : narrow::launch_sht_roots(prog, transpose, io, batch, st);
}
cudaError_t launch_sht_merged(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st) {
    return use_wide(prog, kRC) ? wide::launch_sht_merged(prog, transpose, io, batch, st)
                               : narrow::launch_sht_merged(prog, transpose, io, batch, st);
}

cudaError_t launch_sht_combine(const ShtIO& io, int mu_begin, int mu_end, cudaStream_t st) {
    if (mu_end <= mu_begin) return cudaSuccess;
    ShtIO a = io;
    a.mu0 = mu_begin;
    dim3 grid(static_cast<unsigned>(mu_end - mu_begin), static_cast<unsigned>(io.batch));
    combine_kernel<<<grid, std::min(256, std::max(32, (io.l + 31) / 32 * 32)), 0, st>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_sht_split(const ShtIO& io, int mu_begin, int mu_end, cudaStream_t st) {
    if (mu_end <= mu_begin) return cudaSuccess;
    ShtIO a = io;
    a.mu0 = mu_begin;
    dim3 grid(static_cast<unsigned>(mu_end - mu_begin), static_cast<unsigned>(io.batch));
    split_kernel<<<grid, std::min(256, std::max(32, (io.l + 31) / 32 * 32)), 0, st>>>(a);
    return cudaGetLastError();
}

#endif  // !BFB_ENGINE_WIDE

}  // namespace bfb
