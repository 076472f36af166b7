// Fused phi stage for PRIME row lengths N = 4l - 1 (e.g. c4: l = 2048,
// N = 8191) by Rader's algorithm, one CTA per (colatitude pair, member),
// entirely in shared memory.
//
// For prime N with a primitive root g, every nonzero index is a power of g,
// and the length-N DFT X_n = sum_m x_m w^{mn} (w = e^{+-2 pi i / N}) becomes
//   X_0          = sum_m x_m
//   X_{g^{-q}}   = x_0 + (a (*) b)_q,   a_p = x_{g^p},  b_t = w^{g^{-t}},
// a cyclic convolution of length M = N - 1 (8190 = 2 3^2 5 7 13: all small
// radices).  The convolution runs as
//   forward mixed-radix DIF FFT in place (natural order in, digit-reversed
//   order out), pointwise product with the precomputed, digit-reversed,
//   1/M-scaled spectrum of b, inverse DIT FFT in place (digit-reversed in,
//   natural out)
// so no permutation pass is needed inside the FFTs, and one M-complex buffer
// (131 KB at N = 8191) holds the whole row: the Stockham kernels of phi.cu need
// two (plus staging) and do not fit shared memory at this length.  The Rader
// permutations are folded into the gather (row values scattered to their
// position p = log_g m) and the write-out (X_n read from position -log_g n).
//
// Synthesis CTA: gathers the node's chain values u[chain][b][i][4], forms
// g_m(+x_i) into the buffer and keeps g_m(-x_i) in registers, transforms and
// writes row +x_i, then row -x_i.  Analysis CTA: row +x_i is transformed and
// the values each thread will need for the parity split stay in registers;
// row -x_i is transformed and both are combined into u (sqrt(rho)/(2N)).
// Math: arXiv 0910.5435 eqs. (thetas), (phis), (alternate_expansion)
// (PAPER.md:158-177); the reference has no phi stage.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <stdexcept>
#include <vector>

#include "phi.hpp"

namespace bfb {

namespace {

constexpr int kRThreads = 512;
constexpr int kRPer = 8;           // orders per thread: 2l <= kRPer * kRThreads (l <= 2048)
constexpr int kTwLo = 128;         // twiddle w^e = Tlo[e % 128] * Thi[e / 128]
// cos / sin (2 pi e / R), e < R: the odd prime radices' butterflies and the
// twiddles inside the composite radices 9 = 3 x 3, 10 = 2 x 5
constexpr int kTrig[] = {3, 5, 7, 11, 13, 9, 10};
constexpr int kTrigOff(int R) {
    int off = 0;
    for (int q : kTrig) {
        if (q == R) return off;
        off += q;
    }
    return -1;
}
constexpr int kTrigTotal = 3 + 5 + 7 + 11 + 13 + 9 + 10;
__constant__ double r_cos[kTrigTotal];
__constant__ double r_sin[kTrigTotal];

struct RaderConst {
    int N, M, n_stage, n_hi;
    int radix[kRaderMaxStages];
    int L[kRaderMaxStages];  // block stride after stage s (L_s = L_{s-1} / R_s, L_0 = M)
    int P[kRaderMaxStages];  // M / L_{s-1}: twiddle exponent step
};

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

// w^e, e in [0, M): the table holds e^{-2 pi i e / M}; S = +1 conjugates
template <int S>
__device__ __forceinline__ double2 tw(const double2* Tlo, const double2* Thi, int e) {
    const double2 w = cmul(Tlo[e & (kTwLo - 1)], Thi[e >> 7]);
    return S > 0 ? make_double2(w.x, -w.y) : w;
}

// In-register DFT of length R with kernel e^{S 2 pi i r k / R} (S = -1: forward).
template <int R, int S>
__device__ __forceinline__ void small_dft(double2 (&x)[R]) {
    if constexpr (R == 2) {
        const double2 a = x[0], b = x[1];
        x[0] = cadd(a, b);
        x[1] = csub(a, b);
    } else if constexpr (R == 4) {
        const double2 a = cadd(x[0], x[2]), b = csub(x[0], x[2]);
        const double2 c = cadd(x[1], x[3]), d = csub(x[1], x[3]);
        // d * (S i)
        const double2 di = S > 0 ? make_double2(-d.y, d.x) : make_double2(d.y, -d.x);
        x[0] = cadd(a, c);
        x[2] = csub(a, c);
        x[1] = cadd(b, di);
        x[3] = csub(b, di);
    } else {
        constexpr int h = (R - 1) / 2;
        constexpr int off = kTrigOff(R);
        double2 s[h], d[h];
        const double2 v0 = x[0];
#pragma unroll
        for (int r = 1; r <= h; ++r) {
            s[r - 1] = cadd(x[r], x[R - r]);
            d[r - 1] = csub(x[r], x[R - r]);
        }
        double2 acc = v0;
#pragma unroll
        for (int r = 0; r < h; ++r) acc = cadd(acc, s[r]);
        x[0] = acc;
#pragma unroll
        for (int k = 1; k <= h; ++k) {
            double2 ar = v0, bv = make_double2(0.0, 0.0);
#pragma unroll
            for (int r = 1; r <= h; ++r) {
                const double c = r_cos[off + (r * k) % R], sn = r_sin[off + (r * k) % R];
                ar.x = fma(s[r - 1].x, c, ar.x);
                ar.y = fma(s[r - 1].y, c, ar.y);
                bv.x = fma(d[r - 1].x, sn, bv.x);
                bv.y = fma(d[r - 1].y, sn, bv.y);
            }
            x[k] = make_double2(ar.x - S * bv.y, ar.y + S * bv.x);
            x[R - k] = make_double2(ar.x + S * bv.y, ar.y - S * bv.x);
        }
    }
}

// Composite radix R = R1 x R2 entirely in registers (natural order in and
// out): R2 DFTs of length R1 over x[R2 n1 + n2], twiddles e^{S 2 pi i n2 k1 / R},
// then R1 DFTs of length R2 -> X[k1 + R1 k2].  One shared-memory pass instead of
// two (8190 = 13 7 9 10: four passes instead of six).
template <int R>
struct Composite {
    static constexpr int R1 = R == 9 ? 3 : R == 10 ? 2 : 0;
    static constexpr int R2 = R1 ? R / R1 : 0;
};
template <int R, int S>
__device__ __forceinline__ void dft(double2 (&x)[R]) {
    if constexpr (Composite<R>::R1 == 0) {
        small_dft<R, S>(x);
    } else {
        constexpr int R1 = Composite<R>::R1, R2 = Composite<R>::R2, off = kTrigOff(R);
        double2 y[R];
#pragma unroll
        for (int n2 = 0; n2 < R2; ++n2) {
            double2 t[R1];
#pragma unroll
            for (int n1 = 0; n1 < R1; ++n1) t[n1] = x[R2 * n1 + n2];
            small_dft<R1, S>(t);
#pragma unroll
            for (int k1 = 0; k1 < R1; ++k1) {
                double2 v = t[k1];
                if ((n2 * k1) % R != 0) {
                    const int e = (n2 * k1) % R;
                    v = cmul(v, make_double2(r_cos[off + e], S * r_sin[off + e]));
                }
                y[n2 * R1 + k1] = v;
            }
        }
#pragma unroll
        for (int k1 = 0; k1 < R1; ++k1) {
            double2 t[R2];
#pragma unroll
            for (int n2 = 0; n2 < R2; ++n2) t[n2] = y[n2 * R1 + k1];
            small_dft<R2, S>(t);
#pragma unroll
            for (int k2 = 0; k2 < R2; ++k2) x[k1 + R1 * k2] = t[k2];
        }
    }
}

// One in-place stage over the whole buffer.  DIF (forward, S = -1): butterfly
// then twiddle w^{j k P}; DIT (inverse, S = +1): conjugate twiddle w^{-j r P}
// then butterfly.  Butterfly bf: block bf / L (stride Lp = R L), offset j = bf % L,
// elements j + r L of the block.
template <int R, int S, bool DIF>
__device__ void stage(double2* A, int M, int L, int P, const double2* Tlo, const double2* Thi) {
    // U butterflies per thread and iteration: their loads are issued together
    // (the compiler cannot move one butterfly's loads above another's stores)
    constexpr int U = 1;
    const int nb = M / R, Lp = R * L;
    for (int bf0 = threadIdx.x; bf0 < nb; bf0 += U * kRThreads) {
        double2 x[U][R];
        double2* base[U];
        int e1[U];
        bool ok[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int bf = bf0 + u * kRThreads;
            ok[u] = bf < nb;
            const int blk = ok[u] ? bf / L : 0, j = ok[u] ? bf - blk * L : 0;
            base[u] = A + blk * Lp + j;
            e1[u] = j * P;
            if (ok[u]) {
#pragma unroll
                for (int r = 0; r < R; ++r) x[u][r] = base[u][r * L];
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!ok[u]) continue;
            // power twiddles: one table read (w = w^e1) per butterfly, w^r by
            // repeated multiplication (error ~ r ulp, r < 13)
            const double2 w1 = e1[u] != 0 ? tw<S>(Tlo, Thi, e1[u]) : make_double2(1.0, 0.0);
            if (!DIF && e1[u] != 0) {
                double2 wk = w1;
#pragma unroll
                for (int r = 1; r < R; ++r) {
                    x[u][r] = cmul(x[u][r], wk);
                    if (r + 1 < R) wk = cmul(wk, w1);
                }
            }
            dft<R, S>(x[u]);
            if (DIF && e1[u] != 0) {
                double2 wk = w1;
#pragma unroll
                for (int k = 1; k < R; ++k) {
                    x[u][k] = cmul(x[u][k], wk);
                    if (k + 1 < R) wk = cmul(wk, w1);
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (!ok[u]) continue;
#pragma unroll
            for (int r = 0; r < R; ++r) base[u][r * L] = x[u][r];
        }
    }
}

template <int S, bool DIF>
__device__ void run_stage(double2* A, const RaderConst& rc, int s, const double2* Tlo, const double2* Thi) {
    const int L = rc.L[s], P = rc.P[s];
    switch (rc.radix[s]) {
    case 2: stage<2, S, DIF>(A, rc.M, L, P, Tlo, Thi); break;
    case 3: stage<3, S, DIF>(A, rc.M, L, P, Tlo, Thi); break;
    case 4: stage<4, S, DIF>(A, rc.M, L, P, Tlo, Thi); break;
    case 5: stage<5, S, DIF>(A, rc.M, L, P, Tlo, Thi); break;
    case 7: stage<7, S, DIF>(A, rc.M, L, P, Tlo, Thi); break;
    case 11: stage<11, S, DIF>(A, rc.M, L, P, Tlo, Thi); break;
    case 13: stage<13, S, DIF>(A, rc.M, L, P, Tlo, Thi); break;
    case 9: stage<9, S, DIF>(A, rc.M, L, P, Tlo, Thi); break;
    case 10: stage<10, S, DIF>(A, rc.M, L, P, Tlo, Thi); break;
    default: break;
    }
    __syncthreads();
}

// The last forward stage, the pointwise product with the spectrum of b and the
// first inverse stage act on the same R consecutive elements (stride L = 1, no
// twiddles): one shared-memory pass instead of three.
template <int R>
__device__ void middle(double2* A, int M, const double2* __restrict__ Bhat) {
    for (int bf = threadIdx.x; bf < M / R; bf += kRThreads) {
        double2* base = A + bf * R;
        double2 b[R], x[R];
#pragma unroll
        for (int r = 0; r < R; ++r) b[r] = __ldg(Bhat + bf * R + r);  // issued first: L2 latency
#pragma unroll
        for (int r = 0; r < R; ++r) x[r] = base[r];
        dft<R, -1>(x);
#pragma unroll
        for (int r = 0; r < R; ++r) x[r] = cmul(x[r], b[r]);
        dft<R, 1>(x);
#pragma unroll
        for (int r = 0; r < R; ++r) base[r] = x[r];
    }
    __syncthreads();
}

// The cyclic convolution of A (Rader order, natural) with b: A <- a (*) b.
__device__ void rader_convolve(double2* A, const RaderConst& rc, const double2* __restrict__ Bhat,
                               const double2* Tlo, const double2* Thi) {
    const int last = rc.n_stage - 1;
    for (int s = 0; s < last; ++s) run_stage<-1, true>(A, rc, s, Tlo, Thi);
    switch (rc.radix[last]) {
    case 2: middle<2>(A, rc.M, Bhat); break;
    case 3: middle<3>(A, rc.M, Bhat); break;
    case 4: middle<4>(A, rc.M, Bhat); break;
    case 5: middle<5>(A, rc.M, Bhat); break;
    case 7: middle<7>(A, rc.M, Bhat); break;
    case 9: middle<9>(A, rc.M, Bhat); break;
    case 10: middle<10>(A, rc.M, Bhat); break;
    case 11: middle<11>(A, rc.M, Bhat); break;
    case 13: middle<13>(A, rc.M, Bhat); break;
    default: break;
    }
    for (int s = last - 1; s >= 0; --s) run_stage<1, false>(A, rc, s, Tlo, Thi);
}

// Block sum of one complex value per thread (all threads call; result to all).
__device__ double2 block_sum(double2 v, double2* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        v.x += __shfl_xor_sync(0xffffffffu, v.x, o);
        v.y += __shfl_xor_sync(0xffffffffu, v.y, o);
    }
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double2 t = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < kRThreads / 32; ++k) t = cadd(t, red[k]);
    __syncthreads();
    return t;
}

struct RaderTabs {
    const double2* Tlo;       // e^{-2 pi i e / M}, e < 128
    const double2* Thi;       // e^{-2 pi i 128 e / M}
    const double2* Bhat;      // digit-reversed spectrum of b, / M (direction-specific)
    const std::uint32_t* pos; // pos[m] = log_g m (m = 1..N-1; pos[0] unused)
};

__device__ __forceinline__ void load_twiddles(const RaderTabs& t, const RaderConst& rc, double2* sTlo, double2* sThi) {
    for (int e = threadIdx.x; e < kTwLo; e += kRThreads) sTlo[e] = t.Tlo[e];
    for (int e = threadIdx.x; e < rc.n_hi; e += kRThreads) sThi[e] = t.Thi[e];
}

// Row output: X_0 = total, X_n = x0 + A[(M - pos[n]) mod M].
__device__ __forceinline__ void write_row(double2* __restrict__ out, const double2* A, const RaderConst& rc,
                                          const std::uint32_t* __restrict__ pos, double2 x0, double2 total) {
    for (int n = threadIdx.x; n < rc.N; n += kRThreads) {
        double2 v = total;
        if (n > 0) {
            int q = rc.M - static_cast<int>(__ldg(pos + n));
            if (q == rc.M) q = 0;
            v = cadd(x0, A[q]);
        }
        __stcs(out + n, v);
    }
}

__device__ __forceinline__ double2 read_bin(const double2* A, const RaderConst& rc, const std::uint32_t* __restrict__ pos,
                                            int m, double2 x0, double2 total) {
    if (m == 0) return total;
    int q = rc.M - static_cast<int>(__ldg(pos + m));
    if (q == rc.M) q = 0;
    return cadd(x0, A[q]);
}

__global__ void __launch_bounds__(kRThreads, 1)
    phi_synth_rader_kernel(ShtIO io, RaderConst rc, RaderTabs tb, double2* __restrict__ grid) {
    extern __shared__ __align__(16) double2 sm[];
    __shared__ double2 red[kRThreads / 32];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    const int N = rc.N, l = io.l, i = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
    double2* A = sm;
    double2* sTlo = A + rc.M;
    double2* sThi = sTlo + kTwLo;
    load_twiddles(tb, rc, sTlo, sThi);
    const double s = io.isr[i];
    // gather the node's chain values: g(+x) into A (Rader order), g(-x) kept
    double2 mp[kRPer], mm[kRPer];
    double2 sum = make_double2(0.0, 0.0), x0p = make_double2(0.0, 0.0), x0m = x0p;
#pragma unroll
    for (int k = 0; k < kRPer; ++k) {
        const int mu = tid + k * kRThreads;
        mp[k] = mm[k] = make_double2(0.0, 0.0);
        if (mu >= 2 * l) continue;
        const double4 ue = reinterpret_cast<const double4*>(io.u + (static_cast<long long>(2 * mu) * io.batch + b) * l * 4)[i];
        double4 uo = make_double4(0.0, 0.0, 0.0, 0.0);
        if (mu < 2 * l - 1)
            uo = reinterpret_cast<const double4*>(io.u + (static_cast<long long>(2 * mu + 1) * io.batch + b) * l * 4)[i];
        const double2 pp = make_double2((ue.x + uo.x) * s, (ue.y + uo.y) * s);  // g_{+mu}(+x)
        mp[k] = make_double2((ue.x - uo.x) * s, (ue.y - uo.y) * s);          // g_{+mu}(-x)
        sum = cadd(sum, pp);
        if (mu == 0) {
            x0p = pp;
            x0m = mp[k];
        } else {
            A[__ldg(tb.pos + mu)] = pp;
            const double2 pm = make_double2((ue.z + uo.z) * s, (ue.w + uo.w) * s);  // g_{-mu}(+x)
            mm[k] = make_double2((ue.z - uo.z) * s, (ue.w - uo.w) * s);          // g_{-mu}(-x)
            sum = cadd(sum, pm);
            A[__ldg(tb.pos + N - mu)] = pm;
        }
    }
    x0p = block_sum(x0p, red);  // only thread 0 contributed
    x0m = block_sum(x0m, red);
    double2 total = block_sum(sum, red);  // also: A and the twiddles are complete
    rader_convolve(A, rc, tb.Bhat, sTlo, sThi);
    write_row(grid + (static_cast<long long>(b) * 2 * l + l + i) * N, A, rc, tb.pos, x0p, total);
    __syncthreads();
    sum = make_double2(0.0, 0.0);
#pragma unroll
    for (int k = 0; k < kRPer; ++k) {
        const int mu = tid + k * kRThreads;
        if (mu >= 2 * l) continue;
        sum = cadd(sum, mp[k]);
        if (mu > 0) {
            A[__ldg(tb.pos + mu)] = mp[k];
            A[__ldg(tb.pos + N - mu)] = mm[k];
            sum = cadd(sum, mm[k]);
        }
    }
    total = block_sum(sum, red);
    rader_convolve(A, rc, tb.Bhat, sTlo, sThi);
    write_row(grid + (static_cast<long long>(b) * 2 * l + l - 1 - i) * N, A, rc, tb.pos, x0m, total);
}

__global__ void __launch_bounds__(kRThreads, 1)
    phi_anal_rader_kernel(ShtIO io, RaderConst rc, RaderTabs tb, const double2* __restrict__ grid) {
    extern __shared__ __align__(16) double2 sm[];
    __shared__ double2 red[kRThreads / 32];
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    const int N = rc.N, l = io.l, i = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
    double2* A = sm;
    double2* sTlo = A + rc.M;
    double2* sThi = sTlo + kTwLo;
    load_twiddles(tb, rc, sTlo, sThi);
    double2 gp[kRPer], gm[kRPer];  // row +x_i: G_{+mu}, G_{-mu} of this thread's orders
    for (int row = 0; row < 2; ++row) {
        const double2* f = grid + (static_cast<long long>(b) * 2 * l + (row == 0 ? l + i : l - 1 - i)) * N;
        double2 sum = make_double2(0.0, 0.0), x0 = sum;
        for (int n = tid; n < N; n += kRThreads) {
            const double2 v = __ldcs(f + n);
            sum = cadd(sum, v);
            if (n == 0)
                x0 = v;
            else
                A[__ldg(tb.pos + n)] = v;
        }
        x0 = block_sum(x0, red);
        const double2 total = block_sum(sum, red);
        rader_convolve(A, rc, tb.Bhat, sTlo, sThi);
        if (row == 0) {
#pragma unroll
            for (int k = 0; k < kRPer; ++k) {
                const int mu = tid + k * kRThreads;
                gp[k] = gm[k] = make_double2(0.0, 0.0);
                if (mu >= 2 * l) continue;
                gp[k] = read_bin(A, rc, tb.pos, mu, x0, total);
                if (mu > 0) gm[k] = read_bin(A, rc, tb.pos, N - mu, x0, total);
            }
            __syncthreads();  // A is overwritten by row -x
        } else {
            const double s = io.hsr[i];
#pragma unroll
            for (int k = 0; k < kRPer; ++k) {
                const int mu = tid + k * kRThreads;
                if (mu >= 2 * l) continue;
                const double2 pp = gp[k], pm = read_bin(A, rc, tb.pos, mu, x0, total);
                double2 mp = make_double2(0.0, 0.0), mm = mp;
                if (mu > 0) {
                    mp = gm[k];
                    mm = read_bin(A, rc, tb.pos, N - mu, x0, total);
                }
                *reinterpret_cast<double4*>(io.u + (static_cast<long long>(2 * mu) * io.batch + b) * l * 4 + 4 * i) =
                    make_double4((pp.x + pm.x) * s, (pp.y + pm.y) * s, (mp.x + mm.x) * s, (mp.y + mm.y) * s);
                if (mu < 2 * l - 1)
                    *reinterpret_cast<double4*>(io.u + (static_cast<long long>(2 * mu + 1) * io.batch + b) * l * 4 +
                                                4 * i) =
                        make_double4((pp.x - pm.x) * s, (pp.y - pm.y) * s, (mp.x - mm.x) * s, (mp.y - mm.y) * s);
            }
        }
    }
}

constexpr long double kTwoPi = 6.283185307179586476925286766559005768L;

bool is_prime(int n) {
    if (n < 2) return false;
    for (int f = 2; static_cast<long long>(f) * f <= n; ++f)
        if (n % f == 0) return false;
    return true;
}

long long powmod(long long a, long long e, long long m) {
    long long r = 1;
    a %= m;
    while (e > 0) {
        if (e & 1) r = r * a % m;
        a = a * a % m;
        e >>= 1;
    }
    return r;
}

int primitive_root(int N) {
    const int M = N - 1;
    std::vector<int> fs;
    int n = M;
    for (int f = 2; f * f <= n; ++f)
        if (n % f == 0) {
            fs.push_back(f);
            while (n % f == 0) n /= f;
        }
    if (n > 1) fs.push_back(n);
    for (int g = 2; g < N; ++g) {
        bool ok = true;
        for (int f : fs)
            if (powmod(g, M / f, N) == 1) {
                ok = false;
                break;
            }
        if (ok) return g;
    }
    return -1;
}

template <class T>
T* upload_vec(const std::vector<T>& v) {
    T* d = nullptr;
    if (cudaMalloc(&d, v.size() * sizeof(T)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed (rader)");
    if (cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy failed (rader)");
    return d;
}

RaderConst rader_const(const PhiPlan& p) {
    RaderConst c{};
    c.N = p.N;
    c.M = p.N - 1;
    c.n_stage = p.r_stages;
    c.n_hi = (c.M + kTwLo - 1) / kTwLo;
    int L = c.M;
    for (int s = 0; s < p.r_stages; ++s) {
        c.radix[s] = p.r_radix[s];
        c.P[s] = c.M / L;
        L /= p.r_radix[s];
        c.L[s] = L;
    }
    return c;
}

}  // namespace

bool make_rader_plan(PhiPlan& p) {
    const int N = p.N;
    if (!is_prime(N) || N < 5) return false;
    const int M = N - 1;
    // radices of M: 4 before 2, largest first
    std::vector<int> rad;
    int n = M;
    for (int f : {13, 11, 7, 5, 3}) {
        while (n % f == 0) {
            rad.push_back(f);
            n /= f;
        }
    }
    while (n % 4 == 0) {
        rad.push_back(4);
        n /= 4;
    }
    while (n % 2 == 0) {
        rad.push_back(2);
        n /= 2;
    }
    if (n != 1) return false;
    // composite register radices: 3 x 3 -> 9, 5 x 2 -> 10 (fewer shared-memory passes)
    if (!std::getenv("BFLY_RADER_PRIME_RADICES")) {
        auto take = [&](int f) {
            auto it = std::find(rad.begin(), rad.end(), f);
            if (it == rad.end()) return false;
            rad.erase(it);
            return true;
        };
        std::vector<int> comp;
        while (std::count(rad.begin(), rad.end(), 3) >= 2) {
            take(3);
            take(3);
            comp.push_back(9);
        }
        while (std::count(rad.begin(), rad.end(), 5) >= 1 && std::count(rad.begin(), rad.end(), 2) >= 1) {
            take(5);
            take(2);
            comp.push_back(10);
        }
        rad.insert(rad.end(), comp.begin(), comp.end());
        std::stable_sort(rad.begin(), rad.end(), [](int a, int b) { return a > b; });
    }
    if (static_cast<int>(rad.size()) > kRaderMaxStages) return false;
    const std::size_t smem = static_cast<std::size_t>(M) * 16 + 16 * (kTwLo + (M + kTwLo - 1) / kTwLo);
    int dev = 0, max_smem = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    if (smem + 1024 > static_cast<std::size_t>(max_smem) || (N + 1) / 2 > kRPer * kRThreads) return false;
    p.r_stages = static_cast<int>(rad.size());
    for (int s = 0; s < p.r_stages; ++s) p.r_radix[s] = rad[static_cast<std::size_t>(s)];
    const int g = primitive_root(N);
    // pos[m] = log_g m
    std::vector<std::uint32_t> pos(static_cast<std::size_t>(N), 0);
    std::vector<int> gpow(static_cast<std::size_t>(M));  // g^t mod N
    long long v = 1;
    for (int t = 0; t < M; ++t) {
        gpow[static_cast<std::size_t>(t)] = static_cast<int>(v);
        pos[static_cast<std::size_t>(v)] = static_cast<std::uint32_t>(t);
        v = v * g % N;
    }
    // twiddle tables e^{-2 pi i e / M}
    const int nhi = (M + kTwLo - 1) / kTwLo;
    std::vector<double2> tlo(kTwLo), thi(static_cast<std::size_t>(nhi));
    for (int e = 0; e < kTwLo; ++e) {
        const long double a = -kTwoPi * e / M;
        tlo[static_cast<std::size_t>(e)] = make_double2(static_cast<double>(std::cos(a)), static_cast<double>(std::sin(a)));
    }
    for (int e = 0; e < nhi; ++e) {
        const long double a = -kTwoPi * static_cast<long double>(e) * kTwLo / M;
        thi[static_cast<std::size_t>(e)] = make_double2(static_cast<double>(std::cos(a)), static_cast<double>(std::sin(a)));
    }
    // digit-reversed output position of spectrum index k after the DIF stages
    std::vector<int> kpos(static_cast<std::size_t>(M));
    {
        const RaderConst rc = rader_const(p);
        for (int k = 0; k < M; ++k) {
            int rem = k, ps = 0;
            for (int s = 0; s < rc.n_stage; ++s) {
                ps += (rem % rc.radix[s]) * rc.L[s];
                rem /= rc.radix[s];
            }
            kpos[static_cast<std::size_t>(k)] = ps;
        }
    }
    // b_t = w^{g^{-t}}, w = e^{S 2 pi i / N}; Bhat_k = sum_t b_t e^{-2 pi i t k / M} / M
    std::vector<long double> cM(static_cast<std::size_t>(M)), sM(static_cast<std::size_t>(M));
    for (int e = 0; e < M; ++e) {
        cM[static_cast<std::size_t>(e)] = std::cos(kTwoPi * e / M);
        sM[static_cast<std::size_t>(e)] = std::sin(kTwoPi * e / M);
    }
    for (int dir = 0; dir < 2; ++dir) {
        const long double S = dir == 0 ? 1.0L : -1.0L;  // synthesis e^{+}, analysis e^{-}
        std::vector<long double> br(static_cast<std::size_t>(M)), bi(static_cast<std::size_t>(M));
        for (int t = 0; t < M; ++t) {
            const int ginv = gpow[static_cast<std::size_t>((M - t) % M)];
            const long double a = S * kTwoPi * ginv / N;
            br[static_cast<std::size_t>(t)] = std::cos(a);
            bi[static_cast<std::size_t>(t)] = std::sin(a);
        }
        std::vector<double2> bh(static_cast<std::size_t>(M));
        for (int k = 0; k < M; ++k) {
            long double re = 0, im = 0;
            long long e = 0;
            for (int t = 0; t < M; ++t) {  // e = t k mod M; factor e^{-i 2 pi e / M}
                const long double c = cM[static_cast<std::size_t>(e)], s = sM[static_cast<std::size_t>(e)];
                re += br[static_cast<std::size_t>(t)] * c + bi[static_cast<std::size_t>(t)] * s;
                im += bi[static_cast<std::size_t>(t)] * c - br[static_cast<std::size_t>(t)] * s;
                e += k;
                if (e >= M) e -= M;
            }
            bh[static_cast<std::size_t>(kpos[static_cast<std::size_t>(k)])] =
                make_double2(static_cast<double>(re / M), static_cast<double>(im / M));
        }
        (dir == 0 ? p.r_bsyn : p.r_banal) = reinterpret_cast<double*>(upload_vec(bh));
    }
    p.r_tlo = reinterpret_cast<double*>(upload_vec(tlo));
    p.r_thi = reinterpret_cast<double*>(upload_vec(thi));
    p.r_pos = upload_vec(pos);
    std::vector<double> c(kTrigTotal), s(kTrigTotal);
    for (int R : kTrig) {
        const int off = kTrigOff(R);
        for (int e = 0; e < R; ++e) {
            c[static_cast<std::size_t>(off + e)] = static_cast<double>(std::cos(kTwoPi * e / R));
            s[static_cast<std::size_t>(off + e)] = static_cast<double>(std::sin(kTwoPi * e / R));
        }
    }
    if (cudaMemcpyToSymbol(r_cos, c.data(), sizeof(double) * kTrigTotal) != cudaSuccess ||
        cudaMemcpyToSymbol(r_sin, s.data(), sizeof(double) * kTrigTotal) != cudaSuccess)
        throw std::runtime_error("cudaMemcpyToSymbol failed (rader trig tables)");
    p.smem_rader = smem;
    cudaFuncSetAttribute(phi_synth_rader_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaFuncSetAttribute(phi_anal_rader_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    p.rader = true;
    return true;
}

void free_rader_plan(PhiPlan& p) {
    cudaFree(p.r_bsyn);
    cudaFree(p.r_banal);
    cudaFree(p.r_tlo);
    cudaFree(p.r_thi);
    cudaFree(p.r_pos);
    p.r_bsyn = p.r_banal = p.r_tlo = p.r_thi = nullptr;
    p.r_pos = nullptr;
    p.rader = false;
}

static cudaError_t launch_rader(const PhiPlan& p, const ShtIO& io, bool synthesis, double* grid_out,
                                const double* grid_in, cudaStream_t st) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(io.l), static_cast<unsigned>(io.batch));
    cfg.blockDim = dim3(kRThreads);
    cfg.dynamicSmemBytes = p.smem_rader;
    cfg.stream = st;
    cudaLaunchAttribute attr{};
    attr.id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr.val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = &attr;
    static const bool no_pdl = std::getenv("BFLY_NO_PDL") != nullptr;
    cfg.numAttrs = no_pdl ? 0 : 1;
    RaderTabs t;
    t.Tlo = reinterpret_cast<const double2*>(p.r_tlo);
    t.Thi = reinterpret_cast<const double2*>(p.r_thi);
    t.pos = p.r_pos;
    if (synthesis) {
        t.Bhat = reinterpret_cast<const double2*>(p.r_bsyn);
        return cudaLaunchKernelEx(&cfg, phi_synth_rader_kernel, io, rader_const(p), t,
                                  reinterpret_cast<double2*>(grid_out));
    }
    t.Bhat = reinterpret_cast<const double2*>(p.r_banal);
    return cudaLaunchKernelEx(&cfg, phi_anal_rader_kernel, io, rader_const(p), t,
                              reinterpret_cast<const double2*>(grid_in));
}

cudaError_t launch_phi_synth_rader(const PhiPlan& p, const ShtIO& io, double* grid, cudaStream_t st) {
    return launch_rader(p, io, true, grid, nullptr, st);
}

cudaError_t launch_phi_anal_rader(const PhiPlan& p, const ShtIO& io, const double* grid, cudaStream_t st) {
    return launch_rader(p, io, false, nullptr, grid, st);
}

}  // namespace bfb
