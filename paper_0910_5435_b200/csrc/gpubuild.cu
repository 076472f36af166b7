// GPU plan construction (see gpubuild.hpp for the design and the reference
// semantics it reproduces).
#include "gpubuild.hpp"

#include "hostpar.hpp"

#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <stdexcept>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>

namespace cg = cooperative_groups;

namespace bfb {

namespace {

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("gpu plan builder: ") + what + ": " + cudaGetErrorString(e));
}

// ---------------------------------------------------------------------------
// Legendre matrices.  One thread per (order, node): the normalised three-term
// recurrence in the degree (the same restatement as LegendreColumns,
// builder.cpp) with a per-node binary exponent, emitting degree mu + d into
// column d / 2 of chain d % 2, scaled by sqrt(rho_i).  Columns are stored
// column-major with leading dimension l, so the writes of a warp (consecutive
// nodes) are contiguous.

struct ColTarget {
    double* even;  // l x n_even (nullptr when empty)
    double* odd;   // l x n_odd
    int mu;
};

__global__ void __launch_bounds__(128) gb_columns_kernel(const double* __restrict__ x, const double* __restrict__ srho,
                                                          int l, const ColTarget* __restrict__ tg) {
    extern __shared__ double coef[];  // a[d], ia[d] for d = 0 .. 2l - mu - 1
    const ColTarget t = tg[blockIdx.y];
    const int mu = t.mu, nd = 2 * l - mu;
    double* a = coef;
    double* ia = coef + nd;
    for (int d = threadIdx.x; d < nd; d += blockDim.x) {
        const double k = mu + d, m2 = static_cast<double>(mu) * mu, k1 = k + 1.0;
        a[d] = d == 0 ? 0.0 : sqrt((k * k - m2) / (4.0 * k * k - 1.0));
        ia[d] = sqrt((4.0 * k1 * k1 - 1.0) / (k1 * k1 - m2));
    }
    __syncthreads();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= l) return;
    const double xi = x[i], s = srho[i];
    // seed: Pbar^mu_mu(x) = (1/sqrt 2) prod_{k<=mu} sqrt((2k+1)/(2k)) (1 - x^2)^{mu/2}, kept as m * 2^e
    double m = 0.70710678118654752440;
    long long e = 0;
    auto norm = [&]() {
        int ee;
        m = frexp(m, &ee);
        e += ee;
    };
    for (int k = 1; k <= mu; ++k) {
        m *= sqrt((2.0 * k + 1.0) / (2.0 * k));
        if ((k & 15) == 0) norm();
    }
    norm();
    {
        const double s2 = (1.0 - xi) * (1.0 + xi);
        int es;
        double bm = frexp(s2, &es);
        long long be = es;
        int p = mu / 2;
        while (p > 0) {  // binary powering, renormalised every product
            if (p & 1) {
                m *= bm;
                e += be;
                norm();
            }
            bm *= bm;
            be *= 2;
            int eb;
            bm = frexp(bm, &eb);
            be += eb;
            p >>= 1;
        }
        if (mu & 1) {
            m *= sqrt(s2);
            norm();
        }
    }
    double prev = 0.0, cur = m;
    const double big = 0x1p+256, small = 0x1p-256;
    for (int d = 0; d < nd; ++d) {
        const double v = e < -1200 ? 0.0 : ldexp(cur, static_cast<int>(max(e, -1200LL)));
        double* col = (d & 1) ? t.odd : t.even;
        col[static_cast<long long>(d >> 1) * l + i] = s * v;
        const double nxt = (xi * cur - a[d] * prev) * ia[d];
        prev = cur;
        cur = nxt;
        const double mag = fmax(fabs(cur), fabs(prev));
        if (mag > big) {
            prev *= small;
            cur *= small;
            e += 256;
        } else if (mag < small && mag != 0.0) {
            prev *= big;
            cur *= big;
            e -= 256;
        }
    }
}

// Full-column norms (over all l rows): the col_norm every skeleton column
// carries into the adaptive epsilon of later merges.  One warp per column.
__global__ void gb_colnorm_kernel(const double* __restrict__ A, int l, long long ncols, double* __restrict__ out) {
    const long long c = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (c >= ncols) return;
    const double* p = A + c * l;
    double s = 0.0;
    for (int i = lane; i < l; i += 32) s = fma(p[i], p[i], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) out[c] = sqrt(s);
}

// ---------------------------------------------------------------------------
// Batched interpolative decompositions, one cluster of C CTAs per request.

struct IdTask {
    const double* A;      // the plan's matrix (column-major, leading dimension lda)
    long long ws;         // R workspace offset (doubles), ldr = min(m, n)
    int lda, row0, m, n;  // block = A[row0 : row0 + m, cols[c0 : c0 + n]]
    int c0;               // column list offset (also the perm output offset)
    int fixed;            // 0: pivoted, adaptive rank; > 0: exactly `fixed` unpivoted steps
    double eps, nn;       // nn < 0: eps as given (leaf); else min(0.5, max(eps, eps nn / ||block||_F))
};

constexpr int kIdThreads = 256;
constexpr int kIdSmemDoubles = 27000;  // per CTA: row slice + exchange + replicated vectors (216 KB)

__host__ __device__ inline int id_ld(int m, int C) { return ((m + C - 1) / C) | 1; }
__host__ __device__ inline long long id_smem_doubles(int m, int n, int C) {
    return static_cast<long long>(id_ld(m, C)) * n + 8LL * n + 8;
}

template <int C>
__global__ void __launch_bounds__(kIdThreads) gb_id_kernel(const IdTask* __restrict__ tasks,
                                                           const std::uint32_t* __restrict__ cols,
                                                           double* __restrict__ Rws, int* __restrict__ perm_out,
                                                           int* __restrict__ rank_out) {
    cg::cluster_group cl = cg::this_cluster();
    const int cr = static_cast<int>(cl.block_rank());
    const IdTask tk = tasks[blockIdx.x / C];
    const int m = tk.m, n = tk.n, tid = threadIdx.x;
    const int rl = (m + C - 1) / C, r0 = cr * rl, rc = max(0, min(m - r0, rl)), ld = id_ld(m, C);
    extern __shared__ __align__(16) double sm[];
    double* W = sm;                                   // ld x n: this CTA's rows of the working block
    double* X = W + static_cast<long long>(ld) * n;   // 2 exchange buffers of 2n
    double* nrm = X + 4 * n;                          // trailing column norms^2 (replicated), then
    double* rowj = nrm + n;                           //   the pivot row j of the working block
    double* wv = rowj + n;                            // reflector products w_q
    int* pm = reinterpret_cast<int*>(wv + n);         // column permutation (pivot order)
    __shared__ int s_piv;
    __shared__ unsigned long long s_max;

    if (tid == 0) s_max = 0ull;
    __syncthreads();
    double mx = 0.0;
    for (long long e = tid; e < static_cast<long long>(rc) * n; e += kIdThreads) {
        const int q = static_cast<int>(e / rc), i = static_cast<int>(e - static_cast<long long>(q) * rc);
        const double v = __ldg(tk.A + static_cast<long long>(cols[tk.c0 + q]) * tk.lda + tk.row0 + r0 + i);
        W[q * ld + i] = v;
        mx = fmax(mx, fabs(v));
    }
    for (int q = tid; q < n; q += kIdThreads) pm[q] = q;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) atomicMax(&s_max, static_cast<unsigned long long>(__double_as_longlong(mx)));
    __syncthreads();  // (also: the block is loaded element-wise, the norms below read whole columns)
    // Scale the block by a power of two so its largest entry is ~1: the ID is invariant, and the
    // squared norms of blocks next to the poles (entries below 1e-154 at high orders) neither
    // underflow nor turn the reflector scale into inf / NaN.
    if (tid == 0) X[0] = __longlong_as_double(static_cast<long long>(s_max));
    cl.sync();
    double gmax = 0.0;
#pragma unroll
    for (int c = 0; c < C; ++c) gmax = fmax(gmax, cl.map_shared_rank(X, c)[0]);
    cl.sync();  // X is free again
    double scale = 1.0;
    if (gmax > 0.0 && gmax < 0x1p-64) {
        int ex;
        frexp(gmax, &ex);
        scale = ldexp(1.0, min(-ex, 1000));
        for (long long e = tid; e < static_cast<long long>(rc) * n; e += kIdThreads) {
            const int q = static_cast<int>(e / rc), i = static_cast<int>(e - static_cast<long long>(q) * rc);
            W[q * ld + i] *= scale;
        }
        __syncthreads();
    }

    int buf = 0;
    // Sum the cluster's partials X[buf][lo, hi) and X[buf][n + lo, n + hi) (when two) into dst, in
    // CTA order (bit-identical sums in every CTA, so every decision below is the cluster's).
    auto reduce = [&](int lo, int hi, bool two, double* dst) {
        cl.sync();
        const double* mine = X + buf * 2 * n;
        const int len = hi - lo;
        for (int e = tid; e < (two ? 2 * len : len); e += kIdThreads) {
            const int off = e < len ? lo + e : n + lo + (e - len);
            double s = 0.0;
#pragma unroll
            for (int c = 0; c < C; ++c) s += cl.map_shared_rank(const_cast<double*>(mine), c)[off];
            dst[off] = s;
        }
        buf ^= 1;
        __syncthreads();
    };
    // partial trailing norms^2 over rows >= j of columns [j, n), and row j (its owner)
    auto post_norms = [&](int j) {
        double* P = X + buf * 2 * n;
        const int lo = max(0, j - r0);
        const bool own = j >= r0 && j < r0 + rc;
        for (int q = j + tid; q < n; q += kIdThreads) {
            const double* c = W + q * ld;
            double s = 0.0;
            for (int i = lo; i < rc; ++i) s = fma(c[i], c[i], s);
            P[q] = s;
            P[n + q] = own ? c[j - r0] : 0.0;
        }
    };

    post_norms(0);
    reduce(0, n, true, nrm);
    double fro2 = 0.0;
    for (int q = 0; q < n; ++q) fro2 += nrm[q];
    const int kcap = min(m, n);
    int k = 0;
    if (fro2 == 0.0) {
        k = 1;  // zero block: one zero skeleton column, T = 0 (reference id.cpp zero-norm branch)
        if (r0 == 0 && rc > 0)
            for (int q = tid; q < n; q += kIdThreads) W[q * ld] = 0.0;
    } else {
        const double fro = sqrt(fro2);
        const double eps = tk.nn < 0.0 ? tk.eps : fmin(0.5, fmax(tk.eps, tk.eps * (tk.nn * scale) / fro));
        const double thr = eps * fro / sqrt(static_cast<double>(n));
        const int steps = tk.fixed > 0 ? min(tk.fixed, kcap) : kcap;
        for (int j = 0; j < steps; ++j) {
            int piv = j;
            if (tk.fixed == 0) {
                if (tid < 32) {
                    double bv = -1.0;
                    int bi = INT_MAX;  // (no candidate / NaN norms: falls back to j below)
                    for (int q = j + tid; q < n; q += 32)
                        if (nrm[q] > bv) {
                            bv = nrm[q];
                            bi = q;
                        }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) {
                        const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
                        if (ov > bv || (ov == bv && oi < bi)) {
                            bv = ov;
                            bi = oi;
                        }
                    }
                    if (tid == 0) s_piv = bi < n ? bi : j;
                }
                __syncthreads();
                piv = s_piv;
                if (j > 0 && sqrt(nrm[piv]) <= thr) break;  // every CTA holds the same nrm: uniform
            }
            if (piv != j) {
                for (int i = tid; i < rc; i += kIdThreads) {
                    const double t = W[j * ld + i];
                    W[j * ld + i] = W[piv * ld + i];
                    W[piv * ld + i] = t;
                }
                __syncthreads();
                if (tid == 0) {
                    double t = nrm[j];
                    nrm[j] = nrm[piv];
                    nrm[piv] = t;
                    t = rowj[j];
                    rowj[j] = rowj[piv];
                    rowj[piv] = t;
                    const int p = pm[j];
                    pm[j] = pm[piv];
                    pm[piv] = p;
                }
                __syncthreads();
            }
            // Householder reflector of column j (rows >= j): alpha = -sign(x0) sigma
            const double sigma2 = nrm[j], sigma = sqrt(sigma2), x0 = rowj[j];
            const double alpha = x0 >= 0.0 ? -sigma : sigma, v0 = x0 - alpha;
            const double vn2 = v0 * v0 + (sigma2 - x0 * x0);
            const double beta = vn2 > 0x1p-1000 ? 2.0 / vn2 : 0.0;
            const int lo = max(0, j - r0), jj = j - r0;
            const bool own = j >= r0 && j < r0 + rc;
            const double* vj = W + j * ld;
            // G lanes share a trailing column (its rows dealt round robin, partial sums by shuffles): as
            // many as keep the CTA's threads busy with the n - j - 1 columns left
            const int rem = n - j - 1;
            const int G = rem <= 32 ? 8 : rem <= 64 ? 4 : rem <= 128 ? 2 : 1;
            const int sub = tid & (G - 1), colt = tid / G, cstep = kIdThreads / G;
            const unsigned gmask = ((G == 32 ? 0u : (1u << G)) - 1u) << ((tid & 31) & ~(G - 1));
            {
                double* P = X + buf * 2 * n;
                for (int q = j + 1 + colt; q < n; q += cstep) {
                    const double* c = W + q * ld;
                    double s = 0.0;
                    for (int i = lo + sub; i < rc; i += G) s = fma(own && i == jj ? v0 : vj[i], c[i], s);
                    for (int o = G >> 1; o > 0; o >>= 1) s += __shfl_xor_sync(gmask, s, o);
                    if (sub == 0) P[q] = s;
                }
            }
            reduce(j + 1, n, false, wv);
            {
                double* P = X + buf * 2 * n;
                const int lo1 = max(0, j + 1 - r0);
                const bool own1 = j + 1 >= r0 && j + 1 < r0 + rc;
                const int i1 = j + 1 - r0;
                for (int q = j + 1 + colt; q < n; q += cstep) {
                    double* c = W + q * ld;
                    const double wq = beta * wv[q];
                    double s = 0.0, rv = 0.0;
                    for (int i = lo + sub; i < rc; i += G) {
                        const double v = c[i] - wq * (own && i == jj ? v0 : vj[i]);
                        c[i] = v;
                        if (i >= lo1) s = fma(v, v, s);
                        if (own1 && i == i1) rv = v;
                    }
                    for (int o = G >> 1; o > 0; o >>= 1) {
                        s += __shfl_xor_sync(gmask, s, o);
                        rv += __shfl_xor_sync(gmask, rv, o);
                    }
                    if (sub == 0) {
                        P[q] = s;
                        P[n + q] = rv;
                    }
                }
            }
            __syncthreads();
            for (int i = lo + tid; i < rc; i += kIdThreads) W[j * ld + i] = (own && i == jj) ? alpha : 0.0;
            k = j + 1;
            if (j + 1 < n) reduce(j + 1, n, true, nrm);
        }
    }
    // R = rows [0, k) of the working block, column-major, leading dimension min(m, n)
    __syncthreads();
    const int ldr = kcap;
    double* R = Rws + tk.ws;
    for (long long e = tid; e < static_cast<long long>(rc) * n; e += kIdThreads) {
        const int q = static_cast<int>(e / rc), i = static_cast<int>(e - static_cast<long long>(q) * rc);
        const int g = r0 + i;
        if (g < k) R[static_cast<long long>(q) * ldr + g] = W[q * ld + i];
    }
    if (cr == 0) {
        for (int q = tid; q < n; q += kIdThreads) perm_out[tk.c0 + q] = pm[q];
        if (tid == 0) rank_out[blockIdx.x / C] = k;
    }
    cl.sync();  // no CTA leaves while a peer may still read its exchange buffer
}

// T = R11^-1 R12 for a chunk of <= 32 columns of T: column-oriented back
// substitution (zero pivots give zero rows, reference solve semantics).
struct SolveChunk {
    long long ws, t_off;  // R workspace offset; T output offset (k x (n - k), column-major)
    int ldr, k, n, c0;
};

__global__ void __launch_bounds__(256) gb_solve_kernel(const SolveChunk* __restrict__ chunks,
                                                       const double* __restrict__ Rws, double* __restrict__ Tout) {
    extern __shared__ double B[];  // k x 32
    const SolveChunk ch = chunks[blockIdx.x];
    const int k = ch.k, nt = min(32, ch.n - k - ch.c0);
    const double* R = Rws + ch.ws;
    const int c = threadIdx.x & 31, g = threadIdx.x >> 5;
    for (int e = threadIdx.x; e < k * 32; e += 256) {
        const int q = e >> 5, cc = e & 31;
        B[e] = cc < nt ? R[static_cast<long long>(k + ch.c0 + cc) * ch.ldr + q] : 0.0;
    }
    __syncthreads();
    for (int i = k - 1; i >= 0; --i) {
        const double d = R[static_cast<long long>(i) * ch.ldr + i];
        const double ti = d == 0.0 ? 0.0 : B[i * 32 + c] / d;
        __syncthreads();
        if (g == 0) B[i * 32 + c] = ti;
        for (int q = g; q < i; q += 8) B[q * 32 + c] -= R[static_cast<long long>(i) * ch.ldr + q] * ti;
        __syncthreads();
    }
    for (int e = threadIdx.x; e < k * 32; e += 256) {
        const int q = e >> 5, cc = e & 31;
        if (cc < nt) Tout[ch.t_off + static_cast<long long>(ch.c0 + cc) * k + q] = B[e];
    }
}

// Root skeletons: source columns restricted to the stripe rows, packed.
struct GatherCol {
    const double* src;  // first element (row_begin of the source column)
    long long dst;
    int rows;
};
__global__ void gb_gather_kernel(const GatherCol* __restrict__ g, long long n, double* __restrict__ out) {
    const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    if (w >= n) return;
    const GatherCol c = g[w];
    for (int i = threadIdx.x & 31; i < c.rows; i += 32) out[c.dst + i] = c.src[i];
}

// ---------------------------------------------------------------------------
// Device buffers that grow.
template <class T>
struct DevBuf {
    T* p = nullptr;
    std::size_t cap = 0;
    void need(std::size_t n) {
        if (n <= cap) return;
        if (p) cudaFree(p);
        p = nullptr;
        cap = std::max<std::size_t>(n, cap + cap / 2);
        ck(cudaMalloc(&p, cap * sizeof(T)), "cudaMalloc");
    }
    void put(const std::vector<T>& v, cudaStream_t st) {
        need(std::max<std::size_t>(1, v.size()));
        if (!v.empty()) ck(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st), "H2D");
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

int cluster_size(int m, int n) {
    for (int C : {1, 2, 4, 8, 16})
        if (id_smem_doubles(m, n, C) <= kIdSmemDoubles) return C;
    throw std::runtime_error("gpu plan builder: block " + std::to_string(m) + " x " + std::to_string(n) +
                             " exceeds a 16-CTA cluster");
}

// ---------------------------------------------------------------------------
// Host side: resumable depth-first builds and the round loop.

struct Span {
    int begin, count;
};

// A stripe of a pending block: its rows and the source columns of its
// skeleton (pivot order); the skeleton itself is A[rows, src].
struct SrcStripe {
    int row0, rows;
    std::vector<std::uint32_t> src;
};
struct Block {
    int level;
    std::vector<SrcStripe> st;
};

struct PlanBuild;

// One interpolative decomposition, possibly over several rounds (|T| refinement).
struct IdJob {
    PlanBuild* owner;
    int slot;                          // index in the owner's current attempt
    int row0, m;
    std::vector<std::uint32_t> cols;   // input columns (source indices), input order
    double eps, nn;
    // state
    std::vector<int> perm;             // pivot order (input positions)
    int k = 0, passes = 0;
    bool fixed = false, done = false;
    IdResult out;
};

struct PlanBuild {
    int mu, parity, l;
    std::int64_t n;
    double* A = nullptr;               // device, l x n
    std::vector<double> colnorm;       // full-column norms
    double eps;
    std::int64_t width;
    ButterflyPlan plan;
    std::vector<Block> stack;
    std::vector<std::vector<Span>> parts;
    int ceiling = INT_MAX;
    std::int64_t next_leaf = 0, n_leaves = 0;
    std::vector<IdResult> leaves;
    int phase = 0;                     // 0 leaves, 1 tail, 2 closed
    bool blocked = false;
    // the attempt in flight
    bool waiting = false, promote = false;
    std::vector<IdJob*> att;
    std::vector<std::vector<std::uint32_t>> att_cat;  // per input stripe: concatenated source columns
    std::vector<int> att_left;                        // per input stripe: left rank

    const std::vector<Span>& rows_at(int level) {
        if (parts.empty()) {
            parts.push_back({});
            parts.push_back({Span{0, l}});
        }
        while (static_cast<int>(parts.size()) <= level) {
            std::vector<Span> nxt;
            for (const Span& s : parts.back()) {
                const int top = (s.count + 1) / 2;
                nxt.push_back(Span{s.begin, top});
                nxt.push_back(Span{s.begin + top, s.count - top});
            }
            parts.push_back(std::move(nxt));
        }
        return parts[static_cast<std::size_t>(level)];
    }
};

class Scheduler {
public:
    Scheduler(int l, double eps, std::int64_t width, GpuBuildStats& stats) : l_(l), eps_(eps), width_(width), stats_(stats) {
        ck(cudaStreamCreateWithFlags(&st_, cudaStreamNonBlocking), "stream");
    }
    ~Scheduler() {
        for (IdJob* j : jobs_) delete j;
        cudaStreamDestroy(st_);
    }

    void run(std::vector<PlanBuild>& plans) {
        // round 0: every leaf of every plan
        for (PlanBuild& b : plans) {
            b.n_leaves = (b.n + b.width - 1) / b.width;
            b.leaves.resize(static_cast<std::size_t>(b.n_leaves));
            for (std::int64_t c = 0; c < b.n_leaves; ++c) {
                IdJob* j = new IdJob{};
                j->owner = &b;
                j->slot = static_cast<int>(c);
                j->row0 = 0;
                j->m = l_;
                const std::int64_t c0 = c * b.width, nc = std::min(b.width, b.n - c0);
                for (std::int64_t q = 0; q < nc; ++q) j->cols.push_back(static_cast<std::uint32_t>(c0 + q));
                j->eps = eps_;
                j->nn = -1.0;
                queue_.push_back(j);
            }
        }
        rounds(plans, true);
        for (PlanBuild& b : plans) advance(b);
        while (!queue_.empty()) rounds(plans, false);
        for (PlanBuild& b : plans)
            if (b.phase != 2) throw std::runtime_error("gpu plan builder: a plan did not finish");
        gather_roots(plans);
    }

private:
    // Run queued jobs until none is left unfinished among them (refinements
    // re-queue), then hand results to their plans.
    void rounds(std::vector<PlanBuild>& plans, bool leaves) {
        (void)plans;
        std::vector<IdJob*> finished;
        while (!queue_.empty()) {
            std::vector<IdJob*> batch;
            batch.swap(queue_);
            execute(batch);
            for (IdJob* j : batch) (j->done ? finished : queue_).push_back(j);
            ++stats_.rounds;
            if (!leaves) break;  // merge rounds: refinements wait for the next round with the new attempts
        }
        const auto h0 = std::chrono::steady_clock::now();
        for (IdJob* j : finished) {
            PlanBuild& b = *j->owner;
            if (leaves) {
                b.leaves[static_cast<std::size_t>(j->slot)] = std::move(j->out);
                delete j;
            } else {
                jobs_done_[&b] += 1;
            }
        }
        if (!leaves) {
            // plans whose whole attempt is done resolve it and post the next one
            std::vector<PlanBuild*> ready;
            for (auto& [b, cnt] : jobs_done_)
                if (cnt == static_cast<int>(b->att.size())) ready.push_back(b);
            for (PlanBuild* b : ready) {
                jobs_done_.erase(b);
                resolve(*b);
                advance(*b);
            }
        }
        stats_.host_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - h0).count();
    }

    // ---- the depth-first policy, resumable -----------------------------------
    void push_leaf(PlanBuild& b) {
        const std::int64_t c = b.next_leaf++;
        const std::int64_t c0 = c * b.width, nc = std::min(b.width, b.n - c0);
        IdResult& r = b.leaves[static_cast<std::size_t>(c)];
        Block blk{1, {}};
        SrcStripe s{0, l_, {}};
        for (auto q : r.selected) s.src.push_back(static_cast<std::uint32_t>(c0 + static_cast<std::int64_t>(q)));
        blk.st.push_back(std::move(s));
        PlanEvent ev;
        ev.kind = EventKind::leaf;
        ev.col_begin = static_cast<std::uint64_t>(c0);
        ev.col_count = static_cast<std::uint64_t>(nc);
        ev.ids.push_back(StripeId{std::move(r.selected), std::move(r.t)});
        b.plan.events.push_back(std::move(ev));
        b.stack.push_back(std::move(blk));
    }

    // Post the IDs of a merge (or promote) of the top block(s); false when the
    // level ceiling or the thinnest-stripe rule refuses it without any ID.
    bool post(PlanBuild& b, bool promote) {
        const Block& top = b.stack.back();
        const int lv = top.level + 1;
        if (lv > b.ceiling) return false;
        const std::vector<Span>& part = b.rows_at(lv);
        int thinnest = l_;
        for (const Span& s : part) thinnest = std::min(thinnest, s.count);
        if (thinnest < b.width) {
            b.ceiling = top.level;
            return false;
        }
        const Block& a = promote ? top : b.stack[b.stack.size() - 2];
        const Block* c = promote ? nullptr : &top;
        b.promote = promote;
        b.att.clear();
        b.att_cat.clear();
        b.att_left.clear();
        for (std::size_t s = 0; s < a.st.size(); ++s) {
            std::vector<std::uint32_t> cat = a.st[s].src;
            b.att_left.push_back(static_cast<int>(cat.size()));
            if (c) cat.insert(cat.end(), c->st[s].src.begin(), c->st[s].src.end());
            double nn = 0.0;
            for (auto q : cat) nn += b.colnorm[q] * b.colnorm[q];
            nn = std::sqrt(nn);
            for (int h = 0; h < 2; ++h) {
                const Span& sp = part[2 * s + static_cast<std::size_t>(h)];
                IdJob* j = new IdJob{};
                j->owner = &b;
                j->slot = static_cast<int>(b.att.size());
                j->row0 = sp.begin;
                j->m = sp.count;
                j->cols = cat;
                j->eps = eps_;
                j->nn = nn;
                b.att.push_back(j);
                queue_.push_back(j);
            }
            b.att_cat.push_back(std::move(cat));
        }
        b.waiting = true;
        return true;
    }

    // The attempt's IDs are back: accept (replace the input blocks) or refuse
    // (freeze the level).
    void resolve(PlanBuild& b) {
        b.waiting = false;
        const Block& top = b.stack.back();
        const int lv = top.level + 1;
        const Block& a = b.promote ? top : b.stack[b.stack.size() - 2];
        const Block* c = b.promote ? nullptr : &top;
        std::uint64_t skel = 0, interp = 0, freed = 0;
        bool ok = true;
        for (IdJob* j : b.att) {
            const std::int64_t k = static_cast<std::int64_t>(j->out.selected.size());
            if (10 * k > 9 * static_cast<std::int64_t>(j->m)) ok = false;
            skel += static_cast<std::uint64_t>(j->m) * static_cast<std::uint64_t>(k);
            interp += j->out.t.words();
        }
        for (const auto& s : a.st) freed += static_cast<std::uint64_t>(s.rows) * s.src.size();
        if (c)
            for (const auto& s : c->st) freed += static_cast<std::uint64_t>(s.rows) * s.src.size();
        if (!ok || 10 * (skel + interp) > 17 * freed) {
            b.ceiling = top.level;
            b.blocked = true;
        } else {
            PlanEvent ev;
            ev.kind = b.promote ? EventKind::promote : EventKind::merge;
            Block nb{lv, {}};
            for (std::size_t s = 0; s < b.att_cat.size(); ++s) {
                if (!b.promote) ev.left_ranks.push_back(static_cast<std::uint64_t>(b.att_left[s]));
                for (int h = 0; h < 2; ++h) {
                    IdJob* j = b.att[2 * s + static_cast<std::size_t>(h)];
                    SrcStripe ns{j->row0, j->m, {}};
                    for (auto q : j->out.selected) ns.src.push_back(b.att_cat[s][static_cast<std::size_t>(q)]);
                    nb.st.push_back(std::move(ns));
                    ev.ids.push_back(StripeId{std::move(j->out.selected), std::move(j->out.t)});
                }
            }
            b.stack.pop_back();
            if (!b.promote) b.stack.pop_back();
            b.plan.events.push_back(std::move(ev));
            b.stack.push_back(std::move(nb));
            b.blocked = false;
        }
        for (IdJob* j : b.att) delete j;
        b.att.clear();
    }

    // Advance a plan until it posts an attempt or closes.
    void advance(PlanBuild& b) {
        for (;;) {
            if (b.waiting || b.phase == 2) return;
            const bool can = b.stack.size() >= 2;
            if (b.phase == 0) {
                if (!b.blocked && can && b.stack[b.stack.size() - 2].level == b.stack.back().level) {
                    if (post(b, false)) return;
                    b.blocked = true;
                    continue;
                }
                b.blocked = false;
                if (b.next_leaf < b.n_leaves) {
                    push_leaf(b);
                    continue;
                }
                b.phase = 1;
                continue;
            }
            if (!b.blocked && can) {
                const bool aligned = b.stack[b.stack.size() - 2].level == b.stack.back().level;
                if (post(b, !aligned)) return;
            }
            close(b);
            return;
        }
    }

    void close(PlanBuild& b) {
        b.plan.levels = 0;
        for (Block& blk : b.stack) {
            b.plan.levels = std::max<std::uint64_t>(b.plan.levels, static_cast<std::uint64_t>(blk.level));
            std::vector<RootStripe> group;
            for (SrcStripe& s : blk.st) {
                RootStripe rs;
                rs.row_begin = static_cast<std::uint64_t>(s.row0);
                rs.row_count = static_cast<std::uint64_t>(s.rows);
                rs.skeleton.rows = s.rows;  // storage: gather_roots (allocated by its workers)
                rs.skeleton.cols = static_cast<std::int64_t>(s.src.size());
                roots_.push_back(RootRef{&b, b.plan.root_groups.size(), group.size(), std::move(s.src)});
                group.push_back(std::move(rs));
            }
            b.plan.root_groups.push_back(std::move(group));
        }
        b.stack.clear();
        b.phase = 2;
    }

    // ---- device execution of a batch of IDs -------------------------------------
    void execute(std::vector<IdJob*>& batch) {
        const auto t0 = std::chrono::steady_clock::now();
        // tasks by cluster size
        std::vector<IdTask> tasks(batch.size());
        std::vector<std::uint32_t> cols;
        std::vector<int> csize(batch.size());
        long long ws = 0;
        std::vector<long long> wsoff(batch.size());
        for (std::size_t t = 0; t < batch.size(); ++t) {
            IdJob& j = *batch[t];
            IdTask& k = tasks[t];
            const int n = static_cast<int>(j.cols.size());
            k.A = j.owner->A;
            k.lda = l_;
            k.row0 = j.row0;
            k.m = j.m;
            k.n = n;
            k.c0 = static_cast<int>(cols.size());
            k.fixed = j.fixed ? j.k : 0;
            k.eps = j.eps;
            k.nn = j.nn;
            k.ws = ws;
            wsoff[t] = ws;
            ws += static_cast<long long>(std::min(j.m, n)) * n;
            if (j.fixed) {
                for (int q = 0; q < n; ++q) cols.push_back(j.cols[static_cast<std::size_t>(j.perm[static_cast<std::size_t>(q)])]);
            } else {
                cols.insert(cols.end(), j.cols.begin(), j.cols.end());
            }
            csize[t] = cluster_size(j.m, n);
        }
        // order tasks by cluster size (one launch per size)
        std::vector<std::size_t> order(batch.size());
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) { return csize[a] < csize[b]; });
        std::vector<IdTask> sorted(batch.size());
        for (std::size_t i = 0; i < order.size(); ++i) sorted[i] = tasks[order[i]];
        d_tasks_.put(sorted, st_);
        d_cols_.put(cols, st_);
        d_R_.need(static_cast<std::size_t>(std::max(1LL, ws)));
        d_perm_.need(std::max<std::size_t>(1, cols.size()));
        d_rank_.need(std::max<std::size_t>(1, batch.size()));
        std::size_t i0 = 0;
        while (i0 < order.size()) {
            const int C = csize[order[i0]];
            std::size_t i1 = i0;
            long long maxsm = 0;
            while (i1 < order.size() && csize[order[i1]] == C) {
                const IdTask& k = sorted[i1];
                maxsm = std::max(maxsm, id_smem_doubles(k.m, k.n, C));
                ++i1;
            }
            launch_ids(C, d_tasks_.p + i0, static_cast<int>(i1 - i0), static_cast<std::size_t>(maxsm) * sizeof(double),
                       d_rank_.p + i0);
            i0 = i1;
        }
        // ranks and permutations back
        std::vector<int>&rk = h_rk_, &pm = h_pm_;  // (members: pages stay mapped across rounds)
        if (rk.size() < batch.size()) rk.resize(batch.size());
        if (pm.size() < cols.size()) pm.resize(cols.size());
        ck(cudaMemcpyAsync(rk.data(), d_rank_.p, batch.size() * sizeof(int), cudaMemcpyDeviceToHost, st_), "D2H ranks");
        if (!cols.empty())
            ck(cudaMemcpyAsync(pm.data(), d_perm_.p, cols.size() * sizeof(int), cudaMemcpyDeviceToHost, st_), "D2H perms");
        ck(cudaStreamSynchronize(st_), "id kernels");
        // T = R11^-1 R12, compact
        std::vector<SolveChunk> chunks;
        std::vector<long long> toff(batch.size());
        long long tsz = 0;
        for (std::size_t i = 0; i < order.size(); ++i) {
            const std::size_t t = order[i];
            const IdTask& k = sorted[i];
            const int kk = rk[i], nt = k.n - kk;
            toff[t] = tsz;
            for (int c0 = 0; c0 < nt; c0 += 32) chunks.push_back(SolveChunk{wsoff[t], tsz, std::min(k.m, k.n), kk, k.n, c0});
            tsz += static_cast<long long>(kk) * nt;
        }
        std::vector<double>& T = h_T_;
        if (T.size() < static_cast<std::size_t>(tsz)) T.resize(static_cast<std::size_t>(tsz));
        if (!chunks.empty()) {
            d_chunks_.put(chunks, st_);
            d_T_.need(static_cast<std::size_t>(tsz));
            int maxk = 0;
            for (const auto& c : chunks) maxk = std::max(maxk, c.k);
            const std::size_t sm = static_cast<std::size_t>(std::max(1, maxk)) * 32 * sizeof(double);
            ck(cudaFuncSetAttribute(gb_solve_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm)),
               "solve smem");
            gb_solve_kernel<<<static_cast<unsigned>(chunks.size()), 256, sm, st_>>>(d_chunks_.p, d_R_.p, d_T_.p);
            ck(cudaGetLastError(), "solve launch");
            ck(cudaMemcpyAsync(T.data(), d_T_.p, static_cast<std::size_t>(tsz) * sizeof(double), cudaMemcpyDeviceToHost, st_),
               "D2H T");
            ck(cudaStreamSynchronize(st_), "solve");
        }
        if (std::getenv("BFLY_GPU_BUILD_CHECK")) {
            // debugging aid: (1) T against a host back substitution of the same R; (2) the ID launches run
            // a second time must reproduce R bit for bit
            std::vector<double> Rh(static_cast<std::size_t>(ws));
            ck(cudaMemcpy(Rh.data(), d_R_.p, Rh.size() * sizeof(double), cudaMemcpyDeviceToHost), "check D2H R");
            int bad = 0;
            for (std::size_t i = 0; i < order.size(); ++i) {
                const std::size_t t = order[i];
                const IdTask& k = sorted[i];
                const int kk = rk[i], nt = k.n - kk, ldr = std::min(k.m, k.n);
                const double* R = Rh.data() + wsoff[t];
                double worst = 0.0;
                for (int c = 0; c < nt; ++c) {
                    std::vector<double> x(static_cast<std::size_t>(kk));
                    for (int q = 0; q < kk; ++q) x[static_cast<std::size_t>(q)] = R[static_cast<std::size_t>(kk + c) * ldr + q];
                    for (int r = kk - 1; r >= 0; --r) {
                        const double d = R[static_cast<std::size_t>(r) * ldr + r];
                        const double v = d == 0.0 ? 0.0 : x[static_cast<std::size_t>(r)] / d;
                        x[static_cast<std::size_t>(r)] = v;
                        for (int q = 0; q < r; ++q) x[static_cast<std::size_t>(q)] -= R[static_cast<std::size_t>(r) * ldr + q] * v;
                    }
                    for (int q = 0; q < kk; ++q)
                        worst = std::max(worst, std::fabs(x[static_cast<std::size_t>(q)] -
                                                          T[static_cast<std::size_t>(toff[t]) + static_cast<std::size_t>(c) * kk + q]));
                }
                if (worst > 1e-9 && bad++ < 8)
                    std::fprintf(stderr, "  CHECK solve: task %zu (row0 %d m %d n %d k %d fixed %d): |T_dev - T_host| max %.3e\n", t,
                                 k.row0, k.m, k.n, kk, k.fixed, worst);
            }
            std::size_t j0 = 0;
            while (j0 < order.size()) {
                const int C = csize[order[j0]];
                std::size_t j1 = j0;
                long long maxsm = 0;
                while (j1 < order.size() && csize[order[j1]] == C) {
                    maxsm = std::max(maxsm, id_smem_doubles(sorted[j1].m, sorted[j1].n, C));
                    ++j1;
                }
                launch_ids(C, d_tasks_.p + j0, static_cast<int>(j1 - j0), static_cast<std::size_t>(maxsm) * sizeof(double),
                           d_rank_.p + j0);
                j0 = j1;
            }
            std::vector<double> R2(static_cast<std::size_t>(ws));
            ck(cudaStreamSynchronize(st_), "check rerun");
            ck(cudaMemcpy(R2.data(), d_R_.p, R2.size() * sizeof(double), cudaMemcpyDeviceToHost), "check D2H R2");
            int diff = 0;
            for (std::size_t i = 0; i < order.size(); ++i) {
                const std::size_t t = order[i];
                const IdTask& k = sorted[i];
                const int kk = rk[i], ldr = std::min(k.m, k.n);
                double worst = 0.0;
                for (int q = 0; q < k.n; ++q)
                    for (int g = 0; g < kk; ++g) {
                        const std::size_t at = static_cast<std::size_t>(wsoff[t]) + static_cast<std::size_t>(q) * ldr + g;
                        worst = std::max(worst, std::fabs(Rh[at] - R2[at]));
                    }
                if (worst != 0.0 && diff++ < 8)
                    std::fprintf(stderr, "  CHECK rerun: task %zu (row0 %d m %d n %d k %d fixed %d C %d): R differs by %.3e\n", t,
                                 k.row0, k.m, k.n, kk, k.fixed, csize[t], worst);
            }
            std::fprintf(stderr, "  CHECK batch of %zu: %d solve mismatches, %d rerun differences\n", batch.size(), bad, diff);
        }
        stats_.ids_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        stats_.id_tasks += static_cast<long long>(batch.size());
        // finish or refine each job
        std::atomic<long long> refined{0};
        parallel_for(order.size(), [&](std::size_t i) {
            const std::size_t t = order[i];
            IdJob& j = *batch[t];
            const IdTask& k = sorted[i];
            const int n = k.n, kk = rk[i], nt = n - kk;
            if (kk < 1 || kk > std::min(k.m, n)) throw std::runtime_error("gpu plan builder: an ID returned an impossible rank");
            if (!j.fixed) {
                j.perm.assign(pm.begin() + k.c0, pm.begin() + k.c0 + n);
                std::vector<char> seen(static_cast<std::size_t>(n), 0);
                for (int v : j.perm) {
                    if (v < 0 || v >= n || seen[static_cast<std::size_t>(v)])
                        throw std::runtime_error("gpu plan builder: an ID returned an invalid column permutation");
                    seen[static_cast<std::size_t>(v)] = 1;
                }
                j.k = kk;
            }
            const double* Tt = T.data() + toff[t];
            // the largest |T| (first in column-major order)
            double worst = -1.0;
            int bi = 0, bj = 0;
            for (int c = 0; c < nt; ++c)
                for (int r = 0; r < kk; ++r) {
                    const double a = std::fabs(Tt[static_cast<std::size_t>(c) * kk + r]);
                    if (a > worst) {
                        worst = a;
                        bi = r;
                        bj = c;
                    }
                }
            if (nt > 0 && worst > 2.0 && j.passes < 64) {
                std::swap(j.perm[static_cast<std::size_t>(bi)], j.perm[static_cast<std::size_t>(kk + bj)]);
                j.fixed = true;
                ++j.passes;
                ++refined;
                return;  // re-factor in the next round
            }
            // result: selected in pivot order; T columns in ascending input order
            IdResult& r = j.out;
            r.selected.assign(j.perm.begin(), j.perm.begin() + kk);
            std::vector<int> ord(static_cast<std::size_t>(nt));
            std::iota(ord.begin(), ord.end(), 0);
            std::sort(ord.begin(), ord.end(), [&](int a, int b2) {
                return j.perm[static_cast<std::size_t>(kk + a)] < j.perm[static_cast<std::size_t>(kk + b2)];
            });
            r.t = Mat(kk, nt);
            for (int c = 0; c < nt; ++c)
                std::copy(Tt + static_cast<std::size_t>(ord[static_cast<std::size_t>(c)]) * kk,
                          Tt + static_cast<std::size_t>(ord[static_cast<std::size_t>(c)]) * kk + kk, r.t.col(c));
            j.done = true;
        });
        stats_.refinements += refined.load();
    }

    template <int C>
    void launch_one(const IdTask* tasks, int n, std::size_t smem, int* rank) {
        auto kern = gb_id_kernel<C>;
        ck(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)), "id smem");
        if (C > 8) ck(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1), "cluster 16");
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(static_cast<unsigned>(n) * C);
        cfg.blockDim = dim3(kIdThreads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st_;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = C;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        ck(cudaLaunchKernelEx(&cfg, kern, tasks, static_cast<const std::uint32_t*>(d_cols_.p), d_R_.p, d_perm_.p, rank),
           "id launch");
    }
    void launch_ids(int C, const IdTask* tasks, int n, std::size_t smem, int* rank) {
        switch (C) {
        case 1: launch_one<1>(tasks, n, smem, rank); break;
        case 2: launch_one<2>(tasks, n, smem, rank); break;
        case 4: launch_one<4>(tasks, n, smem, rank); break;
        case 8: launch_one<8>(tasks, n, smem, rank); break;
        default: launch_one<16>(tasks, n, smem, rank); break;
        }
    }

    struct RootRef {
        PlanBuild* b;
        std::size_t group, stripe;
        std::vector<std::uint32_t> src;
    };

    void gather_roots(std::vector<PlanBuild>& plans) {
        (void)plans;
        if (roots_.empty()) return;
        // chunks of whole stripes, <= kChunk doubles each, through one pinned staging buffer
        constexpr long long kChunk = 1LL << 27;  // 1 GiB
        double* stage = nullptr;
        long long biggest = 0;
        for (const RootRef& r : roots_) {
            const RootStripe& rs = r.b->plan.root_groups[r.group][r.stripe];
            biggest = std::max(biggest, static_cast<long long>(rs.row_count) * static_cast<long long>(r.src.size()));
        }
        const long long cap = std::max(kChunk, biggest);
        ck(cudaMallocHost(&stage, static_cast<std::size_t>(cap) * sizeof(double)), "pinned staging");
        DevBuf<GatherCol> dg;
        DevBuf<double> dout;
        dout.need(static_cast<std::size_t>(cap));
        std::vector<GatherCol> gc;
        std::vector<long long> off;
        std::size_t r0 = 0;
        try {
            while (r0 < roots_.size()) {
                gc.clear();
                off.clear();
                long long total = 0;
                std::size_t r1 = r0;
                while (r1 < roots_.size()) {
                    const RootRef& r = roots_[r1];
                    const RootStripe& rs = r.b->plan.root_groups[r.group][r.stripe];
                    const long long words = static_cast<long long>(rs.row_count) * static_cast<long long>(r.src.size());
                    if (r1 > r0 && total + words > cap) break;
                    off.push_back(total);
                    for (auto q : r.src) {
                        gc.push_back(GatherCol{r.b->A + static_cast<long long>(q) * l_ + static_cast<long long>(rs.row_begin),
                                               total, static_cast<int>(rs.row_count)});
                        total += static_cast<long long>(rs.row_count);
                    }
                    ++r1;
                }
                if (!gc.empty()) {
                    dg.put(gc, st_);
                    const long long threads = static_cast<long long>(gc.size()) * 32;
                    gb_gather_kernel<<<static_cast<unsigned>((threads + 255) / 256), 256, 0, st_>>>(
                        dg.p, static_cast<long long>(gc.size()), dout.p);
                    ck(cudaGetLastError(), "gather launch");
                    ck(cudaMemcpyAsync(stage, dout.p, static_cast<std::size_t>(total) * sizeof(double), cudaMemcpyDeviceToHost, st_),
                       "D2H roots");
                    ck(cudaStreamSynchronize(st_), "gather");
                }
                parallel_for(r1 - r0, [&](std::size_t i) {
                    const RootRef& r = roots_[r0 + i];
                    RootStripe& rs = r.b->plan.root_groups[r.group][r.stripe];
                    const std::size_t words = static_cast<std::size_t>(rs.row_count) * r.src.size();
                    rs.skeleton.a.assign(stage + off[i], stage + off[i] + words);
                });
                r0 = r1;
            }
        } catch (...) {
            cudaFreeHost(stage);
            throw;
        }
        cudaFreeHost(stage);
        roots_.clear();
    }

    int l_;
    double eps_;
    std::int64_t width_;
    GpuBuildStats& stats_;
    cudaStream_t st_ = nullptr;
    std::vector<IdJob*> queue_, jobs_;
    std::unordered_map<PlanBuild*, int> jobs_done_;
    std::vector<RootRef> roots_;
    DevBuf<IdTask> d_tasks_;
    DevBuf<std::uint32_t> d_cols_;
    DevBuf<double> d_R_, d_T_;
    DevBuf<int> d_perm_, d_rank_;
    DevBuf<SolveChunk> d_chunks_;
    std::vector<int> h_rk_, h_pm_;
    std::vector<double> h_T_;
};

}  // namespace

std::vector<ButterflyPlan> build_glrow_planset_gpu(int l, int mu_begin, int mu_end, double eps,
                                                   std::int64_t block_width, std::vector<PlanKey>* keys_out,
                                                   const GlRule* rule_in, GpuBuildStats* stats_out) {
    if (!(eps > 0.0)) throw std::invalid_argument("build_plan: epsilon must be positive");
    if (block_width < 2) throw std::invalid_argument("build_plan: block_width must be >= 2");
    if (l < 1 || mu_begin < 0 || mu_end > 2 * l || mu_begin >= mu_end)
        throw std::invalid_argument("planset: bad (l, mu range)");
    const auto t0 = std::chrono::steady_clock::now();
    if (std::getenv("BFLY_BUILD_VERBOSE")) std::fprintf(stderr, "gpu plan build: start\n");
    GpuBuildStats stats;
    std::vector<PlanKey> keys;
    for (int mu = mu_begin; mu < mu_end; ++mu)
        for (int p = 0; p < 2; ++p)
            if (chain_cols(l, mu, p) > 0) keys.push_back(PlanKey{mu, p});
    const GlRule rule = rule_in ? *rule_in : gauss_legendre_positive(l);
    if (static_cast<int>(rule.nodes.size()) != l || static_cast<int>(rule.rho.size()) != l)
        throw std::invalid_argument("planset: the rule must have l nodes and weights");
    std::vector<double> srho(static_cast<std::size_t>(l));
    for (int i = 0; i < l; ++i) srho[static_cast<std::size_t>(i)] = std::sqrt(rule.rho[static_cast<std::size_t>(i)]);
    DevBuf<double> d_x, d_s;
    cudaStream_t st;
    ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
    d_x.put(rule.nodes, st);
    d_s.put(srho, st);

    // groups of whole orders whose dense matrices fit the workspace
    std::size_t free_b = 0, total_b = 0;
    ck(cudaMemGetInfo(&free_b, &total_b), "meminfo");
    std::size_t budget = static_cast<std::size_t>(static_cast<double>(free_b) * 0.35);
    if (const char* e = std::getenv("BFLY_GPU_BUILD_GB")) budget = static_cast<std::size_t>(std::atof(e) * 1e9);
    budget = std::max<std::size_t>(budget, static_cast<std::size_t>(l) * 2 * l * 8 * 2);

    std::vector<ButterflyPlan> plans(keys.size());
    std::size_t k0 = 0;
    while (k0 < keys.size()) {
        std::size_t k1 = k0, bytes = 0;
        while (k1 < keys.size()) {
            // whole orders only (both chains share one recurrence)
            std::size_t k2 = k1, b2 = 0;
            while (k2 < keys.size() && keys[k2].mu == keys[k1].mu) {
                b2 += static_cast<std::size_t>(l) * static_cast<std::size_t>(chain_cols(l, keys[k2].mu, keys[k2].parity)) * 8;
                ++k2;
            }
            if (k1 > k0 && bytes + b2 > budget) break;
            bytes += b2;
            k1 = k2;
        }
        const auto tc = std::chrono::steady_clock::now();
        DevBuf<double> d_A, d_norm;
        d_A.need(bytes / 8);
        std::vector<PlanBuild> pb(k1 - k0);
        std::vector<ColTarget> tg;
        long long off = 0, ncols = 0;
        for (std::size_t i = k0; i < k1; ++i) {
            PlanBuild& b = pb[i - k0];
            b.mu = keys[i].mu;
            b.parity = keys[i].parity;
            b.l = l;
            b.n = chain_cols(l, b.mu, b.parity);
            b.A = d_A.p + off;
            b.eps = eps;
            b.width = block_width;
            b.plan.n_rows = static_cast<std::uint64_t>(l);
            b.plan.n_cols = static_cast<std::uint64_t>(b.n);
            b.plan.epsilon = eps;
            b.plan.block_width = static_cast<std::uint64_t>(block_width);
            if (b.parity == 0) tg.push_back(ColTarget{b.A, nullptr, b.mu});
            else if (!tg.empty() && tg.back().mu == b.mu) tg.back().odd = b.A;
            else tg.push_back(ColTarget{nullptr, b.A, b.mu});
            off += static_cast<long long>(l) * b.n;
            ncols += b.n;
        }
        // a chain with no plan (odd at mu = 2l - 1) still gets written by the kernel: give it scratch
        DevBuf<double> scratch;
        scratch.need(static_cast<std::size_t>(l) * 2);
        for (auto& t : tg) {
            if (!t.even) t.even = scratch.p;
            if (!t.odd) t.odd = scratch.p;
        }
        DevBuf<ColTarget> d_tg;
        d_tg.put(tg, st);
        int maxnd = 0;
        for (const auto& t : tg) maxnd = std::max(maxnd, 2 * l - t.mu);
        const std::size_t csm = static_cast<std::size_t>(2 * maxnd) * sizeof(double);
        ck(cudaFuncSetAttribute(gb_columns_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(csm)),
           "columns smem");
        gb_columns_kernel<<<dim3(static_cast<unsigned>((l + 127) / 128), static_cast<unsigned>(tg.size())), 128, csm, st>>>(
            d_x.p, d_s.p, l, d_tg.p);
        ck(cudaGetLastError(), "columns launch");
        d_norm.need(static_cast<std::size_t>(ncols));
        gb_colnorm_kernel<<<static_cast<unsigned>((ncols * 32 + 255) / 256), 256, 0, st>>>(d_A.p, l, ncols, d_norm.p);
        ck(cudaGetLastError(), "colnorm launch");
        std::vector<double> norms(static_cast<std::size_t>(ncols));
        ck(cudaMemcpyAsync(norms.data(), d_norm.p, norms.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H norms");
        ck(cudaStreamSynchronize(st), "columns");
        long long co = 0;
        for (PlanBuild& b : pb) {
            b.colnorm.assign(norms.begin() + co, norms.begin() + co + b.n);
            co += b.n;
        }
        stats.columns_s += std::chrono::duration<double>(std::chrono::steady_clock::now() - tc).count();
        {
            Scheduler sch(l, eps, block_width, stats);
            sch.run(pb);
        }
        for (std::size_t i = k0; i < k1; ++i) {
            ButterflyPlan& p = pb[i - k0].plan;
            p.stored_words = p.count_stored_words();
            p.m_max_words = p.stored_words;
            plans[i] = std::move(p);
        }
        ++stats.groups;
        k0 = k1;
    }
    cudaStreamDestroy(st);
    stats.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    for (auto& p : plans) p.t_comp_seconds = stats.seconds / static_cast<double>(std::max<std::size_t>(1, plans.size()));
    if (std::getenv("BFLY_BUILD_VERBOSE"))
        std::fprintf(stderr,
                     "gpu plan build: l=%d mu [%d, %d) %zu plans in %.2f s (columns %.2f, IDs %.2f, host %.2f; %lld IDs, "
                     "%lld rounds, %lld refinements, %lld groups)\n",
                     l, mu_begin, mu_end, plans.size(), stats.seconds, stats.columns_s, stats.ids_s, stats.host_s,
                     stats.id_tasks, stats.rounds, stats.refinements, stats.groups);
    if (stats_out) *stats_out = stats;
    if (keys_out) *keys_out = std::move(keys);
    return plans;
}

std::vector<ButterflyPlan> build_glrow_planset_auto(int l, int mu_begin, int mu_end, double eps,
                                                    std::int64_t block_width, int threads, std::vector<PlanKey>* keys,
                                                    const GlRule* rule) {
    const char* e = std::getenv("BFLY_BUILDER");
    int ndev = 0;
    const bool gpu = !(e && std::string(e) == "host") && cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0;
    if (!gpu) {
        cudaGetLastError();
        return build_glrow_planset(l, mu_begin, mu_end, eps, block_width, threads, keys, rule);
    }
    return build_glrow_planset_gpu(l, mu_begin, mu_end, eps, block_width, keys, rule);
}

}  // namespace bfb
