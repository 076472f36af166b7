// Fused phi stage: parity combine / split + the length-N DFT over the orders,
// one CTA per (colatitude pair, batch member), entirely in shared memory.
//
// Synthesis f(theta_t, phi_n) = sum_m g_m(theta_t) e^{+2 pi i m n / N} and
// analysis G_m(theta_t) = sum_n f(theta_t, phi_n) e^{-2 pi i m n / N}, N = 4l - 1
// (SURVEY.md §8 row a10).  The engine leaves (synthesis) or expects (analysis)
// the weighted chain values u[plan][b][i][4]; one CTA owns node i of member b,
// i.e. the two grid rows t = l + i (+x_i) and t = l - 1 - i (-x_i), so the
// +-x parity combine/split happens next to the DFT and no [bin][b][t]
// intermediate exists: each grid row is read or written once, coalesced.  The
// two rows are transformed concurrently by the two halves of the CTA.
//
// DFT: mixed-radix Stockham autosort over the odd prime factors of N (N is
// always odd), ping-ponging between two row buffers.  A butterfly of radix R
// loads v_r (pre-twiddled), forms s_r = v_r + v_{R-r}, d_r = v_r - v_{R-r}
// (r = 1..h, h = (R-1)/2) and writes V_0 = v_0 + sum s_r and the pairs
//   V_k, V_{R-k} = v_0 + sum_r s_r cos(2 pi rk/R) +- i S sum_r d_r sin(2 pi rk/R),
// i.e. 4h^2 real FMAs instead of R^2 complex multiply-adds.  For the radices in
// kRegRadix the butterfly is one thread with everything in registers and the
// cos/sin factors as compile-time-indexed constant-bank operands; other odd
// radices (up to kPhiMaxRadix) take a generic two-phase path through a scratch
// row.  Twiddles come from one table W[k] = e^{+2 pi i k/N}.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <string>
#include <vector>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "phi.hpp"

namespace bfb {

namespace {

#ifndef BFB_PHI_THREADS
#define BFB_PHI_THREADS 128
#endif
#ifndef BFB_PHI_MIN_BLOCKS
#define BFB_PHI_MIN_BLOCKS 3
#endif
constexpr int kPhiThreads = BFB_PHI_THREADS;  // two halves: one grid row each
constexpr int kHalf = kPhiThreads / 2;

// cos / sin (2 pi e / R) for the register-blocked radices, e = 0..R-1, at
// offset kTrigOff(R); filled from the host in long double.
constexpr int kRegRadix[] = {3, 5, 7, 11, 13, 31};
constexpr int kTrigOff(int R) {
    int off = 0;
    for (int q : kRegRadix) {
        if (q == R) return off;
        off += q;
    }
    return -1;
}
constexpr int kTrigTotal = 3 + 5 + 7 + 11 + 13 + 31;
__constant__ double c_cos[kTrigTotal];
__constant__ double c_sin[kTrigTotal];

struct PhiConst {
    int N, n_pass, dbg;  // dbg (BFLY_PHI_DEBUG, diagnostics only): 1 = skip the DFT
    int stage_w;         // 1: copy the twiddle table into shared memory (after the 4 rows)
    int tma;             // small synthesis kernel: chain gather by TMA (else cp.async)
    int radix[kPhiMaxPasses];
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}

template <int S>
__device__ __forceinline__ double2 twiddle(const double2* __restrict__ W, int k) {
    const double2 w = W[k];  // shared-memory copy of the table when it fits
    return S > 0 ? w : make_double2(w.x, -w.y);
}

// One Stockham pass of compile-time radix R: in -> out, butterflies dealt to
// the T threads of this half.
// PW (power twiddles): load w = W[t] and w^R = W[t R] only and form w^r,
// w^{R-r} = w^R conj(w^r) by complex multiplication -- for the large-row
// kernels, whose twiddle table does not fit shared memory next to the rows
// (two table reads per butterfly instead of R - 1 from L2).
template <int R, int S, bool PW = false>
__device__ void reg_pass(const double2* __restrict__ in, double2* __restrict__ out, int N, int Ns,
                         const double2* __restrict__ W, int tid, int T) {
    constexpr int h = (R - 1) / 2;
    constexpr int off = kTrigOff(R);
    const int NR = N / R, tws = NR / Ns;
    for (int j = tid; j < NR; j += T) {
        const int jq = j / Ns, jr = j - jq * Ns;
        const int t = jr * tws;
        const double2 v0 = in[j];
        double2* o = out + jq * Ns * R + jr;
        // h <= 6: s and d stay in registers; larger radices park d_r in the
        // butterfly's own output slot R - r right away (read back below).
        constexpr int hd = h <= 6 ? h : 1;
        double2 s[h], d[hd];
        double2 w1 = make_double2(1.0, 0.0), wR = w1, wr = w1;
        if (PW && t != 0) {
            w1 = twiddle<S>(W, t);
            wR = twiddle<S>(W, t * R);
            wr = w1;
        }
#pragma unroll
        for (int r = 1; r <= h; ++r) {
            double2 a = in[j + r * NR], b = in[j + (R - r) * NR];
            if (t != 0) {
                if (PW) {
                    a = cmul(a, wr);
                    b = cmul(b, cmul(wR, make_double2(wr.x, -wr.y)));
                    wr = cmul(wr, w1);
                } else {
                    a = cmul(a, twiddle<S>(W, t * r));
                    b = cmul(b, twiddle<S>(W, t * (R - r)));
                }
            }
            s[r - 1] = make_double2(a.x + b.x, a.y + b.y);
            const double2 dr = make_double2(a.x - b.x, a.y - b.y);
            if constexpr (h <= 6)
                d[r - 1] = dr;
            else
                o[(R - r) * Ns] = dr;
        }
        double2 acc = v0;
#pragma unroll
        for (int r = 0; r < h; ++r) {
            acc.x += s[r].x;
            acc.y += s[r].y;
        }
        o[0] = acc;
        if constexpr (h <= 6) {
#pragma unroll
            for (int k = 1; k <= h; ++k) {
                double2 ar = v0, bv = make_double2(0.0, 0.0);
#pragma unroll
                for (int r = 1; r <= h; ++r) {
                    const double c = c_cos[off + (r * k) % R], sn = c_sin[off + (r * k) % R];
                    ar.x = fma(s[r - 1].x, c, ar.x);
                    ar.y = fma(s[r - 1].y, c, ar.y);
                    bv.x = fma(d[r - 1].x, sn, bv.x);
                    bv.y = fma(d[r - 1].y, sn, bv.y);
                }
                o[k * Ns] = make_double2(ar.x - S * bv.y, ar.y + S * bv.x);
                o[(R - k) * Ns] = make_double2(ar.x + S * bv.y, ar.y - S * bv.x);
            }
        } else {
            // Large radix: keep only s or d live.  The butterfly's own output
            // slots park d_r (slots R - r) and the cosine halves ar_k (slots k)
            // between the two sweeps; no other thread touches them.
#pragma unroll
            for (int k = 1; k <= h; ++k) {
                double2 ar = v0;
#pragma unroll
                for (int r = 1; r <= h; ++r) {
                    const double c = c_cos[off + (r * k) % R];
                    ar.x = fma(s[r - 1].x, c, ar.x);
                    ar.y = fma(s[r - 1].y, c, ar.y);
                }
                o[k * Ns] = ar;
            }
            double2 dd[h];
#pragma unroll
            for (int r = 1; r <= h; ++r) dd[r - 1] = o[(R - r) * Ns];
#pragma unroll
            for (int k = 1; k <= h; ++k) {
                double2 bv = make_double2(0.0, 0.0);
#pragma unroll
                for (int r = 1; r <= h; ++r) {
                    const double sn = c_sin[off + (r * k) % R];
                    bv.x = fma(dd[r - 1].x, sn, bv.x);
                    bv.y = fma(dd[r - 1].y, sn, bv.y);
                }
                const double2 ar = o[k * Ns];
                o[k * Ns] = make_double2(ar.x - S * bv.y, ar.y + S * bv.x);
                o[(R - k) * Ns] = make_double2(ar.x + S * bv.y, ar.y - S * bv.x);
            }
        }
    }
}

// Generic odd radix: phase 1 writes v_0, s_r, d_r of every butterfly to
// `scratch`, phase 2 combines them into `in` (the pass is in place).  The
// caller's barrier separates the phases of all threads (both halves).
template <int S>
__device__ void generic_pass_phase1(const double2* in, double2* scratch, int N, int R, int Ns,
                                    const double2* __restrict__ W, int tid, int T) {
    const int h = (R - 1) >> 1, NR = N / R, H = h + 1, tws = NR / Ns;
    for (int idx = tid; idx < NR * H; idx += T) {
        const int j = idx / H, r = idx - j * H;
        if (r == 0) {
            scratch[j * R] = in[j];
        } else {
            const int t = (j % Ns) * tws;
            const double2 a = cmul(in[j + r * NR], twiddle<S>(W, t * r));
            const double2 b = cmul(in[j + (R - r) * NR], twiddle<S>(W, t * (R - r)));
            scratch[j * R + r] = make_double2(a.x + b.x, a.y + b.y);
            scratch[j * R + h + r] = make_double2(a.x - b.x, a.y - b.y);
        }
    }
}

template <int S>
__device__ void generic_pass_phase2(double2* in, const double2* scratch, int N, int R, int Ns,
                                    const double2* __restrict__ W, int tid, int T) {
    const int h = (R - 1) >> 1, NR = N / R, H = h + 1;
    for (int idx = tid; idx < NR * H; idx += T) {
        const int j = idx / H, k = idx - j * H;
        const int base = (j / Ns) * Ns * R + j % Ns;
        const double2* sj = scratch + j * R;
        const double2 v0 = sj[0];
        if (k == 0) {
            double2 acc = v0;
            for (int r = 1; r <= h; ++r) {
                acc.x += sj[r].x;
                acc.y += sj[r].y;
            }
            in[base] = acc;
        } else {
            double2 ar = v0, bv = make_double2(0.0, 0.0);
            int e = k;
            for (int r = 1; r <= h; ++r) {
                const double2 c = W[e * NR];  // (cos, sin)(2 pi rk / R)
                ar.x = fma(sj[r].x, c.x, ar.x);
                ar.y = fma(sj[r].y, c.x, ar.y);
                bv.x = fma(sj[h + r].x, c.y, bv.x);
                bv.y = fma(sj[h + r].y, c.y, bv.y);
                e += k;
                if (e >= R) e -= R;
            }
            in[base + k * Ns] = make_double2(ar.x - S * bv.y, ar.y + S * bv.x);
            in[base + (R - k) * Ns] = make_double2(ar.x + S * bv.y, ar.y - S * bv.x);
        }
    }
}

// Length-N DFT of this half's row: data in X, scratch Y; returns the buffer
// holding the result.  Called by all threads of the CTA (barriers inside).
#ifndef BFB_PHI_SMALL_MAXREG
#define BFB_PHI_SMALL_MAXREG 31
#endif
template <int S, int kMaxReg = BFB_PHI_SMALL_MAXREG, bool PW = false>  // register passes for radices <= kMaxReg, two-phase passes otherwise
__device__ double2* row_dft(double2* X, double2* Y, const PhiConst& pc, const double2* __restrict__ W, int tid,
                            int T = kHalf) {
    const int N = pc.N;
    int Ns = 1;
    for (int p = 0; p < pc.n_pass; ++p) {
        const int R = pc.radix[p];
        bool reg = false;  // a register pass ran (result in Y: swap)
        switch (R) {
#define BFB_REG_PASS(RR)                                 \
    case RR:                                             \
        if constexpr (RR <= kMaxReg) {                   \
            reg_pass<RR, S, PW>(X, Y, N, Ns, W, tid, T); \
            reg = true;                                  \
        }                                                \
        break;
            BFB_REG_PASS(3)
            BFB_REG_PASS(5)
            BFB_REG_PASS(7)
            BFB_REG_PASS(11)
            BFB_REG_PASS(13)
            BFB_REG_PASS(31)
#undef BFB_REG_PASS
            default:
                break;
        }
        if (!reg) {
            generic_pass_phase1<S>(X, Y, N, R, Ns, W, tid, T);
            __syncthreads();
            generic_pass_phase2<S>(X, Y, N, R, Ns, W, tid, T);
        }
        const bool swapped = reg;
        __syncthreads();
        if (swapped) {
            double2* tmp = X;
            X = Y;
            Y = tmp;
        }
        Ns *= R;
    }
    return X;
}

__device__ __forceinline__ double* urow(const ShtIO& io, int plan, int b) {
    return io.u + (static_cast<long long>(plan) * io.batch + b) * io.l * 4;
}

__device__ __forceinline__ std::uint32_t smem_addr(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// Chain-value gather by TMA: the tensor map views u[chain][b][i][4] as a 4-D
// tensor (4 doubles, node i, member b, chain c), so one box of 256 chains x 32 B
// for fixed (i, b) is one cp.async.bulk.tensor: 16 instructions per CTA at
// l = 1024 instead of 16K 16-byte cp.async, landing chain-ordered in shared
// memory (OOB chains are zero-filled).
constexpr int kTmaBox = 256;
constexpr std::size_t kBigStage = 65536;  // 128-byte aligned offset of the staging / B / C region

__device__ __forceinline__ void mbar_init1(std::uint64_t* b) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(b)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_wait0(std::uint64_t* b) {
    std::uint32_t ok = 0;
    while (!ok)
        asm volatile(
            "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], 0, 1000000;\nselp.u32 %0, 1, 0, P1;\n}\n"
            : "=r"(ok)
            : "r"(smem_addr(b))
            : "memory");
}
__device__ __forceinline__ void tma_gather_chains(const CUtensorMap* tm, void* dst, std::uint64_t* bar, int i, int b,
                                                  int n_chains) {
    const int nbox = (n_chains + kTmaBox - 1) / kTmaBox;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
                 "r"(static_cast<std::uint32_t>(nbox * kTmaBox * 32))
                 : "memory");
    for (int k = 0; k < nbox; ++k)
        asm volatile(
            "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(
                smem_addr(static_cast<char*>(dst) + static_cast<std::size_t>(k) * kTmaBox * 32)),
            "l"(reinterpret_cast<std::uint64_t>(tm)), "r"(0), "r"(i), "r"(b), "r"(k * kTmaBox), "r"(smem_addr(bar))
            : "memory");
}
// One contiguous grid row (N complex) global -> shared by the bulk-copy engine.
__device__ __forceinline__ void bulk_row(void* dst, const void* src, std::uint32_t bytes, std::uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void tma_prefetch_chains(const CUtensorMap* tm, int i, int b, int n_chains) {
    for (int k = 0; k * kTmaBox < n_chains; ++k)
        asm volatile("cp.async.bulk.prefetch.tensor.4d.L2.global.tile [%0, {%1, %2, %3, %4}];" ::"l"(
                         reinterpret_cast<std::uint64_t>(tm)),
                     "r"(0), "r"(i), "r"(b), "r"(k * kTmaBox)
                     : "memory");
}

// Shared memory (128-byte aligned): [Y(+x) Y(-x)][X(+x) X(-x)][W]; the Y rows
// (at least 2 N complex, rounded up to whole TMA boxes) first receive all 4l - 1
// chain values of the node by TMA (chain-ordered, 32 B each), then serve as the
// DFT scratch rows.
__host__ __device__ constexpr std::size_t small_stage_bytes(int N) {
    return ((2 * static_cast<std::size_t>(N) * 16 > static_cast<std::size_t>((N + kTmaBox - 1) / kTmaBox) * kTmaBox * 32
                 ? 2 * static_cast<std::size_t>(N) * 16
                 : static_cast<std::size_t>((N + kTmaBox - 1) / kTmaBox) * kTmaBox * 32) +
            127) &
           ~std::size_t{127};
}

__global__ void __launch_bounds__(kPhiThreads, BFB_PHI_MIN_BLOCKS)
    phi_synth_kernel(ShtIO io, PhiConst pc, const double2* __restrict__ W, double2* __restrict__ grid,
                     const __grid_constant__ CUtensorMap umap) {
    extern __shared__ __align__(16) double2 sm_raw[];
    __shared__ std::uint64_t bar;
    asm volatile("griddepcontrol.wait;" ::: "memory");  // launched as a dependent of the engine
    asm volatile("griddepcontrol.launch_dependents;");  // a following analysis may get scheduled
    const int N = pc.N, l = io.l, i = blockIdx.x, b = blockIdx.y;
    const int half = threadIdx.x / kHalf, tid = threadIdx.x % kHalf;
    double2* sm = reinterpret_cast<double2*>(reinterpret_cast<char*>(sm_raw) + ((128u - (smem_addr(sm_raw) & 127u)) & 127u));
    double2* Y = sm;
    double2* Xp = reinterpret_cast<double2*>(reinterpret_cast<char*>(sm) + small_stage_bytes(N));
    double2* Xm = Xp + N;
    if (pc.tma) {
        if (threadIdx.x == 0) {
            mbar_init1(&bar);
            tma_gather_chains(&umap, Y, &bar, i, b, 4 * l - 1);
        }
    } else {  // 16-byte cp.async per half chain value (BFLY_PHI_TMA=0)
        for (int c = threadIdx.x; c < 4 * l - 1; c += blockDim.x) {
            const double* src = urow(io, c, b) + 4 * i;
            double* dst = reinterpret_cast<double*>(Y) + 4 * c;
            cp_async16(dst, src);
            cp_async16(dst + 2, src + 2);
        }
    }
    if (pc.stage_w) {
        for (int n = threadIdx.x; n < N; n += blockDim.x) cp_async16(Xp + 2 * N + n, W + n);
        W = Xp + 2 * N;
    }
    cp_async_wait_all();
    __syncthreads();  // also: the barrier is initialised
    if (pc.tma) mbar_wait0(&bar);
    const double4* Ys = reinterpret_cast<const double4*>(Y);
    const double s = io.isr[i];
    for (int mu = threadIdx.x; mu < 2 * l; mu += blockDim.x) {  // staging (Y) -> bins (X)
        const double4 ue = Ys[2 * mu];
        double4 uo = make_double4(0.0, 0.0, 0.0, 0.0);
        if (mu < 2 * l - 1) uo = Ys[2 * mu + 1];
        Xp[mu] = make_double2((ue.x + uo.x) * s, (ue.y + uo.y) * s);
        Xm[mu] = make_double2((ue.x - uo.x) * s, (ue.y - uo.y) * s);
        if (mu > 0) {
            Xp[N - mu] = make_double2((ue.z + uo.z) * s, (ue.w + uo.w) * s);
            Xm[N - mu] = make_double2((ue.z - uo.z) * s, (ue.w - uo.w) * s);
        }
    }
    __syncthreads();
    double2* X = Xp + half * N;
    const double2* res = pc.dbg & 1 ? X : row_dft<1>(X, Y + half * N, pc, W, tid);
    const int t = half ? l - 1 - i : l + i;  // half 0: +x_i, half 1: -x_i
    double2* out = grid + (static_cast<long long>(b) * 2 * l + t) * N;
    for (int n = tid; n < N; n += kHalf) __stcs(out + n, res[n]);
}

__global__ void __launch_bounds__(kPhiThreads, BFB_PHI_MIN_BLOCKS)
    phi_anal_kernel(ShtIO io, PhiConst pc, const double2* __restrict__ W, const double2* __restrict__ grid) {
    extern __shared__ __align__(16) double2 sm[];
    asm volatile("griddepcontrol.wait;" ::: "memory");  // as a dependent: the grid rows are ready
    asm volatile("griddepcontrol.launch_dependents;");  // the engine's producers may start streaming
    const int N = pc.N, l = io.l, i = blockIdx.x, b = blockIdx.y;
    const int half = threadIdx.x / kHalf, tid = threadIdx.x % kHalf;
    __shared__ std::uint64_t bar;
    double2* X = sm + half * N;
    if (threadIdx.x == 0) {  // both rows of the pair by the bulk-copy engine
        mbar_init1(&bar);
        const std::uint32_t bytes = static_cast<std::uint32_t>(N) * 16u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar)), "r"(2 * bytes)
                     : "memory");
        bulk_row(sm, grid + (static_cast<long long>(b) * 2 * l + l + i) * N, bytes, &bar);
        bulk_row(sm + N, grid + (static_cast<long long>(b) * 2 * l + l - 1 - i) * N, bytes, &bar);
    }
    if (pc.stage_w) {
        for (int n = threadIdx.x; n < N; n += blockDim.x) cp_async16(sm + 4 * N + n, W + n);
        W = sm + 4 * N;
    }
    cp_async_wait_all();
    __syncthreads();  // also: the barrier is initialised
    mbar_wait0(&bar);
    const double2* res = pc.dbg & 1 ? X : row_dft<-1>(X, X + 2 * N, pc, W, tid);
    // both halves run the same pass sequence: both results are in X or both in Y
    const double2* Gp = res == X ? sm : sm + 2 * N;
    const double2* Gm = Gp + N;
    const double s = io.hsr[i];
    for (int mu = threadIdx.x; mu < 2 * l; mu += blockDim.x) {
        const double2 pp = Gp[mu], pm = Gm[mu];
        double2 mp = make_double2(0.0, 0.0), mm = make_double2(0.0, 0.0);
        if (mu > 0) {
            mp = Gp[N - mu];
            mm = Gm[N - mu];
        }
        *reinterpret_cast<double4*>(urow(io, 2 * mu, b) + 4 * i) =
            make_double4((pp.x + pm.x) * s, (pp.y + pm.y) * s, (mp.x + mm.x) * s, (mp.y + mm.y) * s);
        if (mu < 2 * l - 1)
            *reinterpret_cast<double4*>(urow(io, 2 * mu + 1, b) + 4 * i) =
                make_double4((pp.x - pm.x) * s, (pp.y - pm.y) * s, (mp.x - mm.x) * s, (mp.y - mm.y) * s);
    }
}

// ---- large rows (4 N complex do not fit shared memory, 3 N do) --------------
// The colatitude pair's two rows are transformed one after the other by the
// whole CTA (kBigThreads) in three N-complex buffers A, B, C: c3 (l = 1024,
// N = 4095) at 196 KB per CTA instead of the stage-wise cuFFT route.
#ifndef BFB_PHI_BIG_THREADS
#define BFB_PHI_BIG_THREADS 512
#endif
constexpr int kBigThreads = BFB_PHI_BIG_THREADS;
constexpr int kBigPer = 2560 / kBigThreads;  // orders per thread: 2l <= 2560 (l <= 1280)
#ifndef BFB_PHI_BIG_MAXREG
#define BFB_PHI_BIG_MAXREG 13
#endif
#ifndef BFB_PHI_BIG_PW
#define BFB_PHI_BIG_PW 1
#endif
constexpr bool kBigPW = BFB_PHI_BIG_PW != 0;  // power twiddles in the large-row kernels
constexpr int kBigMaxReg = BFB_PHI_BIG_MAXREG;  // register passes up to radix 13 (N = 4095 = 3^2 5 7 13) keep 128 registers

__global__ void __launch_bounds__(kBigThreads, 1)
    phi_synth_big_kernel(ShtIO io, PhiConst pc, const double2* __restrict__ W, double2* __restrict__ grid,
                         const __grid_constant__ CUtensorMap umap) {
    extern __shared__ __align__(16) double2 sm_raw[];
    __shared__ std::uint64_t bar;
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    const int N = pc.N, l = io.l, i = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
    // TMA writes 128-byte aligned shared memory: align the dynamic base (the
    // allocation carries 128 bytes of slack)
    double2* sm = reinterpret_cast<double2*>(reinterpret_cast<char*>(sm_raw) + ((128u - (smem_addr(sm_raw) & 127u)) & 127u));
    double2* A = sm;
    double2* B = reinterpret_cast<double2*>(reinterpret_cast<char*>(sm) + kBigStage);
    double2* C = B + N;
    // chain values staged chain-ordered from B on: (4l - 1) x 32 B (+ the last box's tail)
    const double4* Ys = reinterpret_cast<const double4*>(B);
    if (tid == 0) {
        mbar_init1(&bar);
        tma_gather_chains(&umap, B, &bar, i, b, 4 * l - 1);
        // warm L2 for the CTA one wave later (one CTA per SM is resident, so
        // this gather is exposed latency; that CTA runs on some SM meanwhile)
        unsigned nsm;
        asm("mov.u32 %0, %%nsmid;" : "=r"(nsm));
        const long long lin = static_cast<long long>(b) * gridDim.x + i + nsm;
        if (lin < static_cast<long long>(gridDim.x) * gridDim.y)
            tma_prefetch_chains(&umap, static_cast<int>(lin % gridDim.x), static_cast<int>(lin / gridDim.x), 4 * l - 1);
    }
    __syncthreads();  // the barrier is initialised
    mbar_wait0(&bar);
    const double s = io.isr[i];
    double2 mp[kBigPer], mm[kBigPer];  // the -x row's bins wait in registers until the staging is consumed
#pragma unroll
    for (int k = 0; k < kBigPer; ++k) {
        const int mu = tid + k * kBigThreads;
        if (mu >= 2 * l) break;
        const double4 ue = Ys[2 * mu];
        double4 uo = make_double4(0.0, 0.0, 0.0, 0.0);
        if (mu < 2 * l - 1) uo = Ys[2 * mu + 1];
        A[mu] = make_double2((ue.x + uo.x) * s, (ue.y + uo.y) * s);
        if (mu > 0) A[N - mu] = make_double2((ue.z + uo.z) * s, (ue.w + uo.w) * s);
        mp[k] = make_double2((ue.x - uo.x) * s, (ue.y - uo.y) * s);
        mm[k] = make_double2((ue.z - uo.z) * s, (ue.w - uo.w) * s);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kBigPer; ++k) {
        const int mu = tid + k * kBigThreads;
        if (mu >= 2 * l) break;
        B[mu] = mp[k];
        if (mu > 0) B[N - mu] = mm[k];
    }
    __syncthreads();
    const double2* res = pc.dbg & 1 ? A : row_dft<1, kBigMaxReg, kBigPW>(A, C, pc, W, tid, kBigThreads);
    double2* out = grid + (static_cast<long long>(b) * 2 * l + l + i) * N;  // +x_i
    for (int n = tid; n < N; n += kBigThreads) __stcs(out + n, res[n]);
    __syncthreads();
    res = pc.dbg & 1 ? B : row_dft<1, kBigMaxReg, kBigPW>(B, C, pc, W, tid, kBigThreads);
    out = grid + (static_cast<long long>(b) * 2 * l + l - 1 - i) * N;  // -x_i
    for (int n = tid; n < N; n += kBigThreads) __stcs(out + n, res[n]);
}

__global__ void __launch_bounds__(kBigThreads, 1)
    phi_anal_big_kernel(ShtIO io, PhiConst pc, const double2* __restrict__ W, const double2* __restrict__ grid) {
    extern __shared__ __align__(16) double2 sm[];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    const int N = pc.N, l = io.l, i = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
    double2* A = sm;
    double2* B = sm + N;
    double2* C = sm + 2 * N;
    const double2* rp = grid + (static_cast<long long>(b) * 2 * l + l + i) * N;
    const double2* rm = grid + (static_cast<long long>(b) * 2 * l + l - 1 - i) * N;
    __shared__ std::uint64_t bar;
    if (tid == 0) {  // both rows by the bulk-copy engine
        mbar_init1(&bar);
        const std::uint32_t bytes = static_cast<std::uint32_t>(N) * 16u;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(&bar)), "r"(2 * bytes)
                     : "memory");
        bulk_row(A, rp, bytes, &bar);
        bulk_row(B, rm, bytes, &bar);
    }
    if (tid == 0) {  // warm L2 with the rows of the CTA one wave later (see phi_synth_big_kernel)
        unsigned nsm;
        asm("mov.u32 %0, %%nsmid;" : "=r"(nsm));
        const long long lin = static_cast<long long>(b) * gridDim.x + i + nsm;
        if (lin < static_cast<long long>(gridDim.x) * gridDim.y) {
            const int bn = static_cast<int>(lin / gridDim.x), in = static_cast<int>(lin % gridDim.x);
            const std::uint32_t bytes = static_cast<std::uint32_t>(N) * 16u & ~15u;
            const double2* np = grid + (static_cast<long long>(bn) * 2 * l + l + in) * N;
            const double2* nm = grid + (static_cast<long long>(bn) * 2 * l + l - 1 - in) * N;
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(np), "r"(bytes) : "memory");
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(nm), "r"(bytes) : "memory");
        }
    }
    __syncthreads();  // the barrier is initialised
    mbar_wait0(&bar);
    const double2* Gp = pc.dbg & 1 ? A : row_dft<-1, kBigMaxReg, kBigPW>(A, C, pc, W, tid, kBigThreads);
    const double2* Gm = pc.dbg & 1 ? B : row_dft<-1, kBigMaxReg, kBigPW>(B, Gp == A ? C : A, pc, W, tid, kBigThreads);
    const double s = io.hsr[i];
    for (int mu = tid; mu < 2 * l; mu += kBigThreads) {
        const double2 pp = Gp[mu], pm = Gm[mu];
        double2 mp = make_double2(0.0, 0.0), mm = make_double2(0.0, 0.0);
        if (mu > 0) {
            mp = Gp[N - mu];
            mm = Gm[N - mu];
        }
        *reinterpret_cast<double4*>(urow(io, 2 * mu, b) + 4 * i) =
            make_double4((pp.x + pm.x) * s, (pp.y + pm.y) * s, (mp.x + mm.x) * s, (mp.y + mm.y) * s);
        if (mu < 2 * l - 1)
            *reinterpret_cast<double4*>(urow(io, 2 * mu + 1, b) + 4 * i) =
                make_double4((pp.x - pm.x) * s, (pp.y - pm.y) * s, (mp.x - mm.x) * s, (mp.y - mm.y) * s);
    }
}

// ---- real fields (beta^{-m} = conj(beta^m), Im beta^0 = 0) -----------------
// g_{-m} = conj(g_m), so each colatitude row is real.  The two rows of a node
// go through ONE complex DFT: z = f(+x) + i f(-x) has spectrum
// Z_m = G+_m + i G-_m, with G-+_{-m} = conj(G-+_m).  u[chain][b][i][2] holds the
// +m chain values only (re, im).
__global__ void __launch_bounds__(kHalf) phi_synth_real_kernel(ShtIO io, PhiConst pc, const double2* __restrict__ W,
                                                              double* __restrict__ grid) {
    extern __shared__ __align__(16) double2 sm[];
    asm volatile("griddepcontrol.wait;" ::: "memory");  // launched as a dependent of the engine
    const int N = pc.N, l = io.l, i = blockIdx.x, b = blockIdx.y;
    double2* X = sm;
    double2* S = sm + 2 * N;  // chain values of the node: S[c] = u[c][b][i]
    // u[chain][task][i][2 * per]: field b is task b / per, half b % per
    const int per = io.real_per_task, n_task = (io.batch + per - 1) / per, q = b / per, h = b % per;
    for (int c = threadIdx.x; c < 4 * l - 1; c += blockDim.x)
        cp_async16(S + c, io.u + ((static_cast<long long>(c) * n_task + q) * l + i) * 2 * per + 2 * h);
    cp_async_wait_all();
    __syncthreads();
    const double s = io.isr[i];
    for (int mu = threadIdx.x; mu < 2 * l; mu += blockDim.x) {
        const double2 ue = S[2 * mu];
        const double2 uo = mu < 2 * l - 1 ? S[2 * mu + 1] : make_double2(0.0, 0.0);
        double2 gp = make_double2((ue.x + uo.x) * s, (ue.y + uo.y) * s);
        double2 gm = make_double2((ue.x - uo.x) * s, (ue.y - uo.y) * s);
        if (mu == 0) gp.y = gm.y = 0.0;                        // g_0 is real for a real field
        X[mu] = make_double2(gp.x - gm.y, gp.y + gm.x);        // Z_m = G+ + i G-
        if (mu > 0) X[N - mu] = make_double2(gp.x + gm.y, gm.x - gp.y);  // conj(G+) + i conj(G-)
    }
    __syncthreads();
    const double2* z = row_dft<1>(X, sm + N, pc, W, threadIdx.x);
    double* rp = grid + (static_cast<long long>(b) * 2 * l + l + i) * N;
    double* rm = grid + (static_cast<long long>(b) * 2 * l + l - 1 - i) * N;
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
        const double2 v = z[n];
        __stcs(rp + n, v.x);
        __stcs(rm + n, v.y);
    }
}

__global__ void __launch_bounds__(kHalf) phi_anal_real_kernel(ShtIO io, PhiConst pc, const double2* __restrict__ W,
                                                             const double* __restrict__ grid) {
    extern __shared__ __align__(16) double2 sm[];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    const int N = pc.N, l = io.l, i = blockIdx.x, b = blockIdx.y;
    double2* X = sm;
    const double* rp = grid + (static_cast<long long>(b) * 2 * l + l + i) * N;
    const double* rm = grid + (static_cast<long long>(b) * 2 * l + l - 1 - i) * N;
    for (int n = threadIdx.x; n < N; n += blockDim.x) X[n] = make_double2(__ldcs(rp + n), __ldcs(rm + n));
    __syncthreads();
    const double2* Z = row_dft<-1>(X, sm + N, pc, W, threadIdx.x);
    const double s = io.hsr[i];
    const int per = io.real_per_task, n_task = (io.batch + per - 1) / per, q = b / per, h = b % per;
    auto uat = [&](int chain) {
        return reinterpret_cast<double2*>(io.u + ((static_cast<long long>(chain) * n_task + q) * l + i) * 2 * per + 2 * h);
    };
    for (int mu = threadIdx.x; mu < 2 * l; mu += blockDim.x) {
        const double2 zm = Z[mu], zc = Z[mu == 0 ? 0 : N - mu];
        // G+ = (Z_m + conj Z_{-m}) / 2, G- = (Z_m - conj Z_{-m}) / (2i)
        const double2 gp = make_double2(0.5 * (zm.x + zc.x), 0.5 * (zm.y - zc.y));
        const double2 gm = make_double2(0.5 * (zm.y + zc.y), -0.5 * (zm.x - zc.x));
        *uat(2 * mu) = make_double2((gp.x + gm.x) * s, (gp.y + gm.y) * s);
        if (mu < 2 * l - 1) *uat(2 * mu + 1) = make_double2((gp.x - gm.x) * s, (gp.y - gm.y) * s);
    }
}

// ---- order-sharded transform (one process per GPU) --------------------------
// Exchange buffers of rank r (orders [mu0, mu_end), local bins: +mu then -mu)
// with rank j (latitude slab of T_j rows): [local bin][member][slab row],
// complex, blocks back to back by peer.  row_base[t] / row_T[t] locate grid row
// t in this rank's order-side buffer (synthesis send / analysis receive);
// bin_off[bin] locates a bin in the slab-side buffer (synthesis receive /
// analysis send), member stride = this rank's slab rows.
__device__ __forceinline__ int local_bin(const ShtIO& io, int mu, int minus) {
    const int n_plus = io.mu_end - io.mu0;
    return minus ? n_plus + mu - max(io.mu0, 1) : mu - io.mu0;
}

__global__ void __launch_bounds__(256) shard_pack_kernel(ShtIO io, double2* __restrict__ send,
                                                        const long long* __restrict__ row_base,
                                                        const int* __restrict__ row_T) {
    const int mu = io.mu0 + blockIdx.x, b = blockIdx.y, l = io.l;
    const bool odd = mu < 2 * l - 1;
    const int p0 = 2 * (mu - io.mu0);
    const double* ue = io.u + (static_cast<long long>(p0) * io.batch + b) * l * 4;
    const double* uo = odd ? io.u + (static_cast<long long>(p0 + 1) * io.batch + b) * l * 4 : nullptr;
    const int ip = local_bin(io, mu, 0), im = mu > 0 ? local_bin(io, mu, 1) : 0;
    for (int i = threadIdx.x; i < l; i += blockDim.x) {
        const double s = io.isr[i];
        const double4 e = *reinterpret_cast<const double4*>(ue + 4 * i);
        const double4 o = odd ? *reinterpret_cast<const double4*>(uo + 4 * i) : make_double4(0.0, 0.0, 0.0, 0.0);
        const int tp = l + i, tm = l - 1 - i;
        const long long sp = static_cast<long long>(row_T[tp]), sm_ = static_cast<long long>(row_T[tm]);
        send[row_base[tp] + (static_cast<long long>(ip) * io.batch + b) * sp] =
            make_double2((e.x + o.x) * s, (e.y + o.y) * s);
        send[row_base[tm] + (static_cast<long long>(ip) * io.batch + b) * sm_] =
            make_double2((e.x - o.x) * s, (e.y - o.y) * s);
        if (mu > 0) {
            send[row_base[tp] + (static_cast<long long>(im) * io.batch + b) * sp] =
                make_double2((e.z + o.z) * s, (e.w + o.w) * s);
            send[row_base[tm] + (static_cast<long long>(im) * io.batch + b) * sm_] =
                make_double2((e.z - o.z) * s, (e.w - o.w) * s);
        }
    }
}

__global__ void __launch_bounds__(256) shard_unpack_kernel(ShtIO io, const double2* __restrict__ recv,
                                                          const long long* __restrict__ row_base,
                                                          const int* __restrict__ row_T) {
    const int mu = io.mu0 + blockIdx.x, b = blockIdx.y, l = io.l;
    const bool odd = mu < 2 * l - 1;
    const int p0 = 2 * (mu - io.mu0);
    double* ue = io.u + (static_cast<long long>(p0) * io.batch + b) * l * 4;
    double* uo = odd ? io.u + (static_cast<long long>(p0 + 1) * io.batch + b) * l * 4 : nullptr;
    const int ip = local_bin(io, mu, 0), im = mu > 0 ? local_bin(io, mu, 1) : 0;
    for (int i = threadIdx.x; i < l; i += blockDim.x) {
        const double s = io.hsr[i];
        const int tp = l + i, tm = l - 1 - i;
        const long long sp = static_cast<long long>(row_T[tp]), sm_ = static_cast<long long>(row_T[tm]);
        const double2 pp = recv[row_base[tp] + (static_cast<long long>(ip) * io.batch + b) * sp];
        const double2 pm = recv[row_base[tm] + (static_cast<long long>(ip) * io.batch + b) * sm_];
        double2 mp = make_double2(0.0, 0.0), mm = make_double2(0.0, 0.0);
        if (mu > 0) {
            mp = recv[row_base[tp] + (static_cast<long long>(im) * io.batch + b) * sp];
            mm = recv[row_base[tm] + (static_cast<long long>(im) * io.batch + b) * sm_];
        }
        *reinterpret_cast<double4*>(ue + 4 * i) =
            make_double4((pp.x + pm.x) * s, (pp.y + pm.y) * s, (mp.x + mm.x) * s, (mp.y + mm.y) * s);
        if (odd)
            *reinterpret_cast<double4*>(uo + 4 * i) =
                make_double4((pp.x - pm.x) * s, (pp.y - pm.y) * s, (mp.x - mm.x) * s, (mp.y - mm.y) * s);
    }
}

// Slab rows: one CTA per (slab row, member); T threads (kHalf, or kBigThreads
// for long rows, where 2 N complex leave room for one CTA per SM only).
template <int S, int T = kHalf>
__global__ void __launch_bounds__(T) shard_phi_kernel(PhiConst pc, const double2* __restrict__ W,
                                                     const double2* __restrict__ src, double2* __restrict__ dst,
                                                     const long long* __restrict__ bin_off, int n_rows) {
    extern __shared__ __align__(16) double2 sm[];
    const int N = pc.N, t = blockIdx.x, b = blockIdx.y;
    double2* X = sm;
    const long long o = static_cast<long long>(b) * n_rows + t;
    if (S > 0) {  // synthesis: gather the bins of this row from every rank's block
        for (int bin = threadIdx.x; bin < N; bin += blockDim.x) X[bin] = src[bin_off[bin] + o];
    } else {      // analysis: the grid row
        for (int n = threadIdx.x; n < N; n += blockDim.x) X[n] = src[o * N + n];
    }
    __syncthreads();
    const double2* res = T == kHalf ? row_dft<S>(X, sm + N, pc, W, threadIdx.x)
                                    : row_dft<S, kBigMaxReg, kBigPW>(X, sm + N, pc, W, threadIdx.x, T);
    if (S > 0) {
        for (int n = threadIdx.x; n < N; n += blockDim.x) __stcs(dst + o * N + n, res[n]);
    } else {
        for (int bin = threadIdx.x; bin < N; bin += blockDim.x) dst[bin_off[bin] + o] = res[bin];
    }
}

// Bins <-> contiguous slab rows (the cuFFT slab path), tiled through shared
// memory: 32 bins x 32 (member, row) pairs per block so both sides stay coalesced.
template <bool TO_ROWS>
__global__ void __launch_bounds__(256) shard_bins_rows_kernel(const double2* __restrict__ src, double2* __restrict__ dst,
                                                             const long long* __restrict__ bin_off, int N,
                                                             long long n_pairs) {
    __shared__ double2 tile[32][33];
    const int bin0 = blockIdx.x * 32;
    const long long p0 = static_cast<long long>(blockIdx.y) * 32;
    const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;  // 8 rows of 32
    if (TO_ROWS) {
        for (int r = ty; r < 32; r += 8) {  // r: bin, tx: pair
            const int bin = bin0 + r;
            const long long p = p0 + tx;
            if (bin < N && p < n_pairs) tile[r][tx] = src[bin_off[bin] + p];
        }
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {  // r: pair, tx: bin
            const int bin = bin0 + tx;
            const long long p = p0 + r;
            if (bin < N && p < n_pairs) dst[p * N + bin] = tile[tx][r];
        }
    } else {
        for (int r = ty; r < 32; r += 8) {  // r: pair, tx: bin
            const int bin = bin0 + tx;
            const long long p = p0 + r;
            if (bin < N && p < n_pairs) tile[tx][r] = src[p * N + bin];
        }
        __syncthreads();
        for (int r = ty; r < 32; r += 8) {  // r: bin, tx: pair
            const int bin = bin0 + r;
            const long long p = p0 + tx;
            if (bin < N && p < n_pairs) dst[bin_off[bin] + p] = tile[r][tx];
        }
    }
}

PhiConst phi_const(const PhiPlan& p) {
    PhiConst c{};
    c.N = p.N;
    c.n_pass = p.n_pass;
    c.dbg = p.dbg;
    c.stage_w = p.stage_w ? 1 : 0;
    c.tma = p.tma ? 1 : 0;
    for (int k = 0; k < p.n_pass; ++k) c.radix[k] = p.radix[k];
    return c;
}

constexpr long double kTwoPi = 6.283185307179586476925286766559005768L;

void upload_trig() {
    std::vector<double> c(kTrigTotal), s(kTrigTotal);
    for (int R : kRegRadix) {
        const int off = kTrigOff(R);
        for (int e = 0; e < R; ++e) {
            const long double a = kTwoPi * e / R;
            c[static_cast<std::size_t>(off + e)] = static_cast<double>(std::cos(a));
            s[static_cast<std::size_t>(off + e)] = static_cast<double>(std::sin(a));
        }
    }
    if (cudaMemcpyToSymbol(c_cos, c.data(), sizeof(double) * kTrigTotal) != cudaSuccess ||
        cudaMemcpyToSymbol(c_sin, s.data(), sizeof(double) * kTrigTotal) != cudaSuccess)
        throw std::runtime_error("cudaMemcpyToSymbol failed (phi trig tables)");
}

}  // namespace

PhiPlan make_phi_plan(int N) {
    PhiPlan p;
    p.N = N;
    if (N < 1 || N % 2 == 0) return p;
    {
        const char* e = std::getenv("BFLY_PHI_RADER");  // 1: Rader kernels for any prime N >= 5 (tests)
        const bool force = e && std::strtol(e, nullptr, 10) != 0;
        bool prime = N >= 5;
        for (int f = 2; prime && f * f <= N; ++f) prime = N % f != 0;
        if (prime && (N > kPhiMaxRadix || force) && make_rader_plan(p)) return p;
    }
    int n = N;
    for (int f = 3; n > 1 && f <= kPhiMaxRadix; f += 2)
        while (n % f == 0) {
            if (p.n_pass == kPhiMaxPasses) return p;
            p.radix[p.n_pass++] = f;
            n /= f;
        }
    if (n != 1) return p;  // a prime factor above kPhiMaxRadix
    p.smem_synth = 4 * static_cast<std::size_t>(N) * sizeof(double2);
    int dev = 0, max_smem = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    const char* fb = std::getenv("BFLY_PHI_BIG");  // BFLY_PHI_BIG=1: large-row kernels at any N (tests)
    const bool force_big = fb && std::strtol(fb, nullptr, 10) != 0;
    if (p.smem_synth > static_cast<std::size_t>(max_smem) || force_big) {
        // large rows: the pair's two rows one after the other in 3 N complex
        p.smem_synth = 3 * static_cast<std::size_t>(N) * sizeof(double2);
        if (p.smem_synth > static_cast<std::size_t>(max_smem) || (N + 1) / 2 > kBigPer * kBigThreads) return p;
        p.big = true;
        // synthesis: A, then the 128-byte aligned TMA staging (= B, C) at kBigStage
        p.smem_big_synth = std::max(kBigStage, static_cast<std::size_t>(N) * sizeof(double2)) +
                           std::max(2 * static_cast<std::size_t>(N) * sizeof(double2),
                                    static_cast<std::size_t>((N + kTmaBox - 1) / kTmaBox) * kTmaBox * 32) +
                           128;  // alignment slack
        if (static_cast<std::size_t>(N) * sizeof(double2) > kBigStage ||
            p.smem_big_synth > static_cast<std::size_t>(max_smem))
            return p;
    }
    if (!p.big &&
        p.smem_synth + static_cast<std::size_t>(N) * sizeof(double2) <= static_cast<std::size_t>(max_smem) / 2) {
        p.stage_w = true;  // still two CTAs per SM with the twiddles in shared memory
        p.smem_synth += static_cast<std::size_t>(N) * sizeof(double2);
    }
    p.smem_anal = p.smem_synth;
    if (!p.big)  // synthesis: TMA staging rows first (see phi_synth_kernel)
        p.smem_synth = small_stage_bytes(N) + (p.stage_w ? 3 : 2) * static_cast<std::size_t>(N) * sizeof(double2) + 128;
    std::vector<double> w(2 * static_cast<std::size_t>(N));
    for (int k = 0; k < N; ++k) {
        const long double a = kTwoPi * static_cast<long double>(k) / N;
        w[2 * static_cast<std::size_t>(k)] = static_cast<double>(std::cos(a));
        w[2 * static_cast<std::size_t>(k) + 1] = static_cast<double>(std::sin(a));
    }
    upload_trig();
    if (cudaMalloc(&p.W, w.size() * sizeof(double)) != cudaSuccess)
        throw std::runtime_error("cudaMalloc failed (phi twiddles)");
    if (cudaMemcpy(p.W, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy failed (phi twiddles)");
    p.smem_real_synth = 3 * static_cast<std::size_t>(N) * sizeof(double2);
    p.smem_real_anal = 2 * static_cast<std::size_t>(N) * sizeof(double2);
    cudaFuncSetAttribute(phi_synth_real_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(p.smem_real_synth));
    cudaFuncSetAttribute(phi_anal_real_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(p.smem_real_anal));
    cudaFuncSetAttribute(shard_phi_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(2 * static_cast<std::size_t>(N) * sizeof(double2)));
    cudaFuncSetAttribute(shard_phi_kernel<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(2 * static_cast<std::size_t>(N) * sizeof(double2)));
    cudaFuncSetAttribute(shard_phi_kernel<1, kBigThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(2 * static_cast<std::size_t>(N) * sizeof(double2)));
    cudaFuncSetAttribute(shard_phi_kernel<-1, kBigThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(2 * static_cast<std::size_t>(N) * sizeof(double2)));
    if (p.big)
        cudaFuncSetAttribute(phi_synth_big_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(p.smem_big_synth));
    else
        cudaFuncSetAttribute(phi_synth_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             static_cast<int>(p.smem_synth));
    cudaFuncSetAttribute(p.big ? phi_anal_big_kernel : phi_anal_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(p.smem_anal));
    // same L1/shared split as the engine: no reconfiguration between the launches
    cudaFuncSetAttribute(phi_synth_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    cudaFuncSetAttribute(phi_anal_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, cudaSharedmemCarveoutMaxShared);
    if (const char* e = std::getenv("BFLY_PHI_DEBUG")) p.dbg = static_cast<int>(std::strtol(e, nullptr, 10));
    if (const char* e = std::getenv("BFLY_PHI_TMA")) p.tma = std::strtol(e, nullptr, 10) != 0;
    p.ok = true;
    return p;
}

void free_phi_plan(PhiPlan& p) {
    free_rader_plan(p);
    cudaFree(p.W);
    p = PhiPlan{};
}

// Tensor map of u[chain][b][i][4] for the TMA chain gather (cached per buffer
// and shape: the engine's staging buffer only moves when the batch grows).
const CUtensorMap& u_tensor_map(const PhiPlan& p, const ShtIO& io) {
    const int chains = 4 * io.l - 1;
    if (p.umap_u == io.u && p.umap_batch == io.batch && p.umap_l == io.l) return p.umap;
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess || !fn)
            throw std::runtime_error("phi: cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    const cuuint64_t dims[4] = {4, static_cast<cuuint64_t>(io.l), static_cast<cuuint64_t>(io.batch),
                                static_cast<cuuint64_t>(chains)};
    const cuuint64_t strides[3] = {32, 32ull * io.l, 32ull * io.l * io.batch};
    const cuuint32_t box[4] = {4, 1, 1, kTmaBox};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode(&p.umap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, io.u, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw std::runtime_error("phi: cuTensorMapEncodeTiled failed (" + std::to_string(r) + ")");
    p.umap_u = io.u;
    p.umap_batch = io.batch;
    p.umap_l = io.l;
    return p.umap;
}

cudaError_t launch_phi_synth_fused(const PhiPlan& p, const ShtIO& io, double* grid, cudaStream_t st) {
    if (p.rader) return launch_phi_synth_rader(p, io, grid, st);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(io.l), static_cast<unsigned>(io.batch));
    cfg.blockDim = dim3(p.big ? kBigThreads : kPhiThreads);
    cfg.dynamicSmemBytes = p.big ? p.smem_big_synth : p.smem_synth;
    cfg.stream = st;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;  // overlap the engine's tail
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    static const bool no_pdl = std::getenv("BFLY_NO_PDL") != nullptr;  // diagnostics
    cfg.numAttrs = no_pdl ? 0 : 1;
    if (p.big)
        return cudaLaunchKernelEx(&cfg, phi_synth_big_kernel, io, phi_const(p), reinterpret_cast<const double2*>(p.W),
                                  reinterpret_cast<double2*>(grid), u_tensor_map(p, io));
    return cudaLaunchKernelEx(&cfg, phi_synth_kernel, io, phi_const(p), reinterpret_cast<const double2*>(p.W),
                              reinterpret_cast<double2*>(grid), u_tensor_map(p, io));
}

cudaError_t launch_phi_anal_fused(const PhiPlan& p, const ShtIO& io, const double* grid, cudaStream_t st) {
    if (p.rader) return launch_phi_anal_rader(p, io, grid, st);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(io.l), static_cast<unsigned>(io.batch));
    cfg.blockDim = dim3(p.big ? kBigThreads : kPhiThreads);
    cfg.dynamicSmemBytes = p.smem_anal;
    cfg.stream = st;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;  // waits before reading the grid
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    static const bool no_pdl = std::getenv("BFLY_NO_PDL") != nullptr;  // diagnostics
    cfg.numAttrs = no_pdl ? 0 : 1;
    return cudaLaunchKernelEx(&cfg, p.big ? phi_anal_big_kernel : phi_anal_kernel, io, phi_const(p), reinterpret_cast<const double2*>(p.W),
                              reinterpret_cast<const double2*>(grid));
}

cudaError_t launch_phi_synth_real(const PhiPlan& p, const ShtIO& io, double* grid, cudaStream_t st) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(io.l), static_cast<unsigned>(io.batch));
    cfg.blockDim = dim3(kHalf);
    cfg.dynamicSmemBytes = p.smem_real_synth;
    cfg.stream = st;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, phi_synth_real_kernel, io, phi_const(p), reinterpret_cast<const double2*>(p.W), grid);
}

cudaError_t launch_phi_anal_real(const PhiPlan& p, const ShtIO& io, const double* grid, cudaStream_t st) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(io.l), static_cast<unsigned>(io.batch));
    cfg.blockDim = dim3(kHalf);
    cfg.dynamicSmemBytes = p.smem_real_anal;
    cfg.stream = st;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, phi_anal_real_kernel, io, phi_const(p), reinterpret_cast<const double2*>(p.W), grid);
}

cudaError_t launch_shard_pack(const ShtIO& io, double* send, const long long* row_base, const int* row_T, int mu_begin,
                              int mu_end, cudaStream_t st) {
    ShtIO a = io;
    a.mu0 = mu_begin;
    a.mu_end = mu_end;
    dim3 g(static_cast<unsigned>(mu_end - mu_begin), static_cast<unsigned>(io.batch));
    shard_pack_kernel<<<g, 256, 0, st>>>(a, reinterpret_cast<double2*>(send), row_base, row_T);
    return cudaGetLastError();
}

cudaError_t launch_shard_unpack(const ShtIO& io, const double* recv, const long long* row_base, const int* row_T,
                                int mu_begin, int mu_end, cudaStream_t st) {
    ShtIO a = io;
    a.mu0 = mu_begin;
    a.mu_end = mu_end;
    dim3 g(static_cast<unsigned>(mu_end - mu_begin), static_cast<unsigned>(io.batch));
    shard_unpack_kernel<<<g, 256, 0, st>>>(a, reinterpret_cast<const double2*>(recv), row_base, row_T);
    return cudaGetLastError();
}

cudaError_t launch_shard_phi(const PhiPlan& p, bool synthesis, const double* src, double* dst,
                             const long long* bin_off, int n_rows, int batch, cudaStream_t st) {
    if (n_rows == 0) return cudaSuccess;
    dim3 g(static_cast<unsigned>(n_rows), static_cast<unsigned>(batch));
    const std::size_t smem = 2 * static_cast<std::size_t>(p.N) * sizeof(double2);
    const auto W = reinterpret_cast<const double2*>(p.W);
    const auto in = reinterpret_cast<const double2*>(src);
    const auto out = reinterpret_cast<double2*>(dst);
    if (p.big) {  // c3: N = 4095, 64 threads per SM took 2x the single-GPU transform
        if (synthesis)
            shard_phi_kernel<1, kBigThreads><<<g, kBigThreads, smem, st>>>(phi_const(p), W, in, out, bin_off, n_rows);
        else
            shard_phi_kernel<-1, kBigThreads><<<g, kBigThreads, smem, st>>>(phi_const(p), W, in, out, bin_off, n_rows);
    } else if (synthesis) {
        shard_phi_kernel<1><<<g, kHalf, smem, st>>>(phi_const(p), W, in, out, bin_off, n_rows);
    } else {
        shard_phi_kernel<-1><<<g, kHalf, smem, st>>>(phi_const(p), W, in, out, bin_off, n_rows);
    }
    return cudaGetLastError();
}

cudaError_t launch_shard_bins_rows(bool to_rows, const double* src, double* dst, const long long* bin_off, int N,
                                   int n_rows, int batch, cudaStream_t st) {
    const long long pairs = static_cast<long long>(batch) * n_rows;
    if (pairs == 0 || N == 0) return cudaSuccess;
    const dim3 grid(static_cast<unsigned>((N + 31) / 32), static_cast<unsigned>((pairs + 31) / 32));
    if (to_rows)
        shard_bins_rows_kernel<true><<<grid, 256, 0, st>>>(reinterpret_cast<const double2*>(src),
                                                            reinterpret_cast<double2*>(dst), bin_off, N, pairs);
    else
        shard_bins_rows_kernel<false><<<grid, 256, 0, st>>>(reinterpret_cast<const double2*>(src),
                                                             reinterpret_cast<double2*>(dst), bin_off, N, pairs);
    return cudaGetLastError();
}

}  // namespace bfb
