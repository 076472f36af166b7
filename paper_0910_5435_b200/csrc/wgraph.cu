// Persistent graph kernel of the wave programs (wgraph.hpp): one launch runs
// a whole direction of the batched butterfly apply on the FP64 tensor cores.
//
// Every CTA (forward: 4 warps, four per SM; transpose: 8 warps, three per SM)
// loops: take the next (item, column block) -- claimed from an atomic counter
// one item ahead, its 64-byte record prefetched into shared memory while the
// current item runs; items start in queue order and the queue is topological,
// which makes the dependency spin deadlock-free (every item an item waits for
// was claimed earlier by a running CTA and waits only on even earlier ones) --
// wait until the items it depends on have published (per-(item, column block)
// flags = this launch's epoch, polled by a few lanes while the other threads
// fetch the descriptors), stage the node's index lists (a root block: its chunk
// table) in shared memory, and run its passes: up to 64 output rows x NT (<= 64)
// columns, K-chunks of 16 through a 2- / 3-stage cp.async ring in which every
// thread gathers its fixed 16-byte pieces (the matrix tiles -- 16 x 16 swizzled
// tiles of T / S, packer.hpp -- and the vector rows named by the index list),
// DMMA m8n8k4 with each warp running exactly its live m8 tiles, accumulators
// starting from the forward's z[sel] term / the transpose's old z, epilogue
// straight to V / u, then a gpu-scope release of the item's flag.
//
// Why this shape (measured at c3, l = 1024, 16 functions, and on l = 2048
// order ranges): a warp-specialised version (producer warps
// feeding one consumer group per SM by TMA bulk copies) was bound by the TMA
// unit's rate for small copies (~100 cycles per 512-byte vector row per SM);
// with cp.async gathers spread over all threads and several items in flight per
// SM, the gathers issue in parallel and one CTA's item latency (dependency,
// descriptors, index lists, pipeline fill) hides behind the others' MMA.  The
// kernel is latency-bound (tensor pipe ~50 % active at 16 warps per SM), so the
// transpose -- whose items re-gather their vector rows once per pass and carry
// more rows -- runs 8-warp CTAs on 64-row passes, three per SM (24 warps, 85
// registers): 6-7 % faster than 8 warps x 128 rows x two per SM at c3 and on
// l = 2048 order ranges; the same shape is slower for the forward.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <stdexcept>
#include <vector>

#include "wgraph_dev.hpp"

namespace bfb {

namespace {

// CTA shapes: forward 4 warps x 64-row passes, 2 stages, four CTAs per SM;
// transpose 8 warps x 64-row passes, 3 stages, three per SM
template <int W_, int MPASS_, int STAGES_, int CTAS_>
struct Shape {
    static constexpr int W = W_;                  // warps per CTA
    static constexpr int kThreads = 32 * W;
    static constexpr int MPass = MPASS_;          // output rows per pass
    static constexpr int Stages = STAGES_;        // cp.async ring depth
    static constexpr int Ctas = CTAS_;            // CTAs per SM (register budget)
    static constexpr int ATiles = MPASS_ / 16 + 1;  // matrix tiles per stage (a row block may start mid-tile)
    static constexpr int AStage = ATiles * 256;   // doubles
};
#ifndef BFB_FWD_W  // tuning builds: warps, stages, CTAs per SM of the two shapes
#define BFB_FWD_W 4
#define BFB_FWD_S 2
#define BFB_FWD_C 4
#endif
#ifndef BFB_BWD_W
#define BFB_BWD_W 8
#define BFB_BWD_M 64
#define BFB_BWD_S 3
#define BFB_BWD_C 3
#endif
using FwdShape = Shape<BFB_FWD_W, static_cast<int>(kGraphMaxRows), BFB_FWD_S, BFB_FWD_C>;  // rows per pass = the root row blocks
using BwdShape = Shape<BFB_BWD_W, BFB_BWD_M, BFB_BWD_S, BFB_BWD_C>;
constexpr int kKC = 16;                     // K chunk
constexpr int kIdxCap = 1024;               // index-list entries kept in shared memory
constexpr int kSegMax = 8;                  // root-block segments kept in shared memory

template <int NT, class SH>
struct Cfg {
    static_assert(NT == 8 || NT == 16 || NT == 32 || NT == 64, "column block");
    using Shape = SH;
    static constexpr int NTW = NT >= 16 ? 2 : 1;           // n8 tiles per warp
    static constexpr int WN = NT / (8 * NTW);              // warps along n
    static constexpr int WM = SH::W / WN;                  // warps along m
    static constexpr int MTW = (SH::MPass / 8 + WM - 1) / WM;  // m8 tiles per warp (max)
    static constexpr int LDB = NT + 4;                     // B tile row stride (4 mod 16: conflict-free)
    static constexpr int StageD = SH::AStage + kKC * LDB;
};

struct GraphArgs {
    const GraphItem* items;
    const std::uint32_t* deps;
    const RootSeg* segs;
    const WaveNode* nodes;
    const std::uint32_t* idx;
    const double* T;
    const RootStripeDesc* stripes;
    const double* S;
    double* V;
    double* u;                       // chain rows [plan][b][l][4], or (stacked) cell-major rows [row][R]
    const std::uint32_t* plan_row0;  // stacked: first row of each plan
    int stacked;
    std::uint32_t* flags;
    std::uint32_t* counter;
    std::uint32_t epoch;
    std::uint32_t n_items;
    int l, batch, R, H;
    int debug;  // BFLY_GRAPH_DEBUG (timing experiments only; wrong results): bit 0 no MMA, bit 1 no
                // accumulator init loads, bit 2 no dependency waits
};

// Per-item state in shared memory.
struct ItemSh {
    GraphItem pre[2];             // the current item and the prefetched next one (alternating)
    std::uint32_t pre_claim[2];   // their claims (item * H + column block)
    std::uint32_t item, half, smem_idx, nchunks;
    WaveNode nd[2];
    RootStripeDesc sd[kSegMax];
    std::uint32_t row_off[kSegMax];
    std::uint32_t idx[kIdxCap];
};

// ---- PTX helpers ---------------------------------------------------------------
__device__ __forceinline__ std::uint32_t sa(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
// 16-byte cp.async through L2 (the vectors are written by other CTAs); src_bytes 0 fills zeros.
__device__ __forceinline__ void cp16(void* dst, const void* src, std::uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa(dst)), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp16s(std::uint32_t dst, const void* src, std::uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ std::uint32_t ld_relaxed(const std::uint32_t* p) {
    std::uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed(std::uint32_t* p, std::uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 ldcg2(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

// A K-chunk's matrix operand: forward (TRANS = false) column tile kt, row tiles
// [t0, t1) (one contiguous run of tiles); transposed row tile kt, column tiles
// [t0, t1) (2 KB each).  aoff: first output row inside tile t0 (forward).
struct AChunk {
    const double* P;
    int nib, kt, t0, t1, aoff, kn;
};

// A K-chunk's vector operand: row k (k < kn) starts at base + row(k) * stride,
// row(k) = idx[k] (an index list) or k; a thread's column pair n, n + 1 sits
// at offset n (cell-major rows of R doubles) or, for the chain rows
// u[b][row][4] (cstride = doubles between batch members), at
// (n >> 2) * cstride + (n & 3).
struct BRows {
    const double* base;
    long long stride;
    const std::uint32_t* idx;
    long long cstride;
};

template <int NT, class SH>
struct Cta {
    using C = Cfg<NT, SH>;
    static constexpr int kThreads = SH::kThreads, kStages = SH::Stages, kMPass = SH::MPass, kAStage = SH::AStage,
                         kW = SH::W;
    const GraphArgs& a;
    ItemSh& sh;
    double* stages;
    int tid, warp, lane, wm, wn;
    int n0 = 0;

    // Stage one chunk into ring slot `slot`: the matrix tiles, the vector rows
    // k < kn and zero rows kn .. kn rounded up to 4 (the last k-step reads
    // them).  Every thread owns fixed 16-byte pieces (a column pair of the
    // vector rows, a fixed offset inside the tiles), so a piece costs an add
    // and the copy; the rows' addresses come from `br`.
    template <bool TRANS>
    __device__ __forceinline__ void stage(int slot, const AChunk& ch, const BRows& br) {
        double* As = stages + slot * C::StageD;
        const int ntile = ch.t1 - ch.t0;
        if (!TRANS) {
            const double* src = ch.P + (static_cast<long long>(ch.kt) * ch.nib + ch.t0) * 256 + 2 * tid;
            std::uint32_t dst = sa(As) + 16u * tid;
            for (int e = tid; e < ntile * 128; e += kThreads, src += 2 * kThreads, dst += 16u * kThreads)
                cp16s(dst, src, 16u);
        } else {
            constexpr int TS = kThreads / 128;  // tiles per sweep
            const int p = tid & 127;
            const double* src = ch.P + (static_cast<long long>(ch.t0 + (tid >> 7)) * ch.nib + ch.kt) * 256 + 2 * p;
            const long long sstep = static_cast<long long>(TS) * ch.nib * 256;
            std::uint32_t dst = sa(As) + 8u * (256 * (tid >> 7) + 2 * p);
            for (int t = tid >> 7; t < ntile; t += TS, src += sstep, dst += 2048u * TS) cp16s(dst, src, 16u);
        }
        constexpr int HP = NT / 2;            // pieces per row
        constexpr int KS = kThreads / HP;     // rows per sweep
        const int h = tid % HP, k0 = tid / HP;
        const int n = n0 + 2 * h;
        const bool okn = n < a.R;
        const long long noff = br.cstride ? static_cast<long long>(n >> 2) * br.cstride + (n & 3) : n;
        const int kr = (ch.kn + 3) & ~3;
        std::uint32_t dst = sa(As + kAStage) + 8u * (k0 * C::LDB + 2 * h);
        for (int k = k0; k < kr; k += KS, dst += 8u * KS * C::LDB) {
            const bool ok = okn && k < ch.kn;
            const double* src = a.V;
            if (ok) {
                const long long row = br.idx ? static_cast<long long>(br.idx[k]) : static_cast<long long>(k);
                src = br.base + row * br.stride + noff;
            }
            cp16s(dst, src, ok ? 16u : 0u);
        }
    }

    // The chunk's k-steps on this warp's first MT m8 tiles (all live: a guard
    // inside the unrolled tile loop would compile to predicated DMMAs, which
    // still take tensor-pipe cycles).
    template <int MT, bool TRANS>
    __device__ __forceinline__ void mma_chunk(double (&acc)[C::MTW][C::NTW][2], const double* As, const double* Bs,
                                              int aoff, int ksteps) {
        static_assert(MT <= C::MTW, "mma_chunk: tiles");
        const int ka = lane & 3, c3 = (lane >> 2) & 3;
        int ab[MT];
#pragma unroll
        for (int t = 0; t < MT; ++t) {
            const int r = 8 * (wm + t * C::WM) + (lane >> 2);
            if (TRANS) {
                ab[t] = (r >> 4) * 256 + (r & 15) * 16 + ka;
            } else {
                const int i = r + aoff;
                ab[t] = (i >> 4) * 256 + ((i & 15) ^ (4 * ka)) + 16 * ka;
            }
        }
        const double* bp = Bs + ka * C::LDB + 8 * wn * C::NTW + (lane >> 2);
        for (int ks = 0; ks < ksteps; ++ks) {
            double bv[C::NTW];
#pragma unroll
            for (int j = 0; j < C::NTW; ++j) bv[j] = bp[4 * ks * C::LDB + 8 * j];
#pragma unroll
            for (int t = 0; t < MT; ++t) {
                const double av = TRANS ? As[ab[t] + 4 * (ks ^ c3)] : As[ab[t] + 64 * ks];
#pragma unroll
                for (int j = 0; j < C::NTW; ++j) dmma(acc[t][j], av, bv[j]);
            }
        }
    }

    template <bool TRANS>
    __device__ __forceinline__ void mma_dispatch(double (&acc)[C::MTW][C::NTW][2], int mtw, const double* As,
                                                 const double* Bs, int aoff, int ksteps) {
        switch (mtw) {
        case 1: mma_chunk<1, TRANS>(acc, As, Bs, aoff, ksteps); break;
        case 2: mma_chunk<(2 < C::MTW ? 2 : C::MTW), TRANS>(acc, As, Bs, aoff, ksteps); break;
        case 3: mma_chunk<(3 < C::MTW ? 3 : C::MTW), TRANS>(acc, As, Bs, aoff, ksteps); break;
        case 4: mma_chunk<(4 < C::MTW ? 4 : C::MTW), TRANS>(acc, As, Bs, aoff, ksteps); break;
        case 5: mma_chunk<(5 < C::MTW ? 5 : C::MTW), TRANS>(acc, As, Bs, aoff, ksteps); break;
        case 6: mma_chunk<(6 < C::MTW ? 6 : C::MTW), TRANS>(acc, As, Bs, aoff, ksteps); break;
        case 7: mma_chunk<(7 < C::MTW ? 7 : C::MTW), TRANS>(acc, As, Bs, aoff, ksteps); break;
        case 8: mma_chunk<(8 < C::MTW ? 8 : C::MTW), TRANS>(acc, As, Bs, aoff, ksteps); break;
        default: break;
        }
    }

    // One pass: output rows [m0, m0 + mp) (mp <= kMPass) over nk chunks;
    // chunk(c) -> AChunk, brows(c) -> the vector rows of chunk c;
    // init(row, n) / store(row, n, v): double2 at columns n, n + 1.
    template <bool TRANS, class CHUNK, class BROWS, class INIT, class STORE>
    __device__ void pass(int m0, int mp, int nk, CHUNK chunk, BROWS brows, bool has_init, INIT init, STORE store) {
        double acc[C::MTW][C::NTW][2];
        const int mt = (mp + 7) >> 3;
        const int mtw = wm < mt ? (mt - wm + C::WM - 1) / C::WM : 0;
        // prologue: the first kStages - 1 chunks in flight
#pragma unroll
        for (int s = 0; s < kStages - 1; ++s) {
            if (s < nk) {
                stage<TRANS>(s, chunk(s), brows(s));
            }
            cp_commit();
        }
        // accumulator start values (their latency overlaps the staging above)
#pragma unroll
        for (int t = 0; t < C::MTW; ++t) {
            const int row = m0 + 8 * (wm + t * C::WM) + (lane >> 2);
#pragma unroll
            for (int j = 0; j < C::NTW; ++j) {
                const int n = n0 + 8 * (wn * C::NTW + j) + 2 * (lane & 3);
                double2 v = make_double2(0.0, 0.0);
                if (has_init && !(a.debug & 2) && t < mtw && row < m0 + mp && n < a.R) v = init(row, n);
                acc[t][j][0] = v.x;
                acc[t][j][1] = v.y;
            }
        }
        for (int c = 0; c < nk; ++c) {
            cp_wait<kStages - 2>();
            __syncthreads();  // chunk c landed for every thread; chunk c - 1's slot is free
            if (c + kStages - 1 < nk) {
                const int cc = c + kStages - 1;
                stage<TRANS>(cc % kStages, chunk(cc), brows(cc));
            }
            cp_commit();
            const AChunk ch = chunk(c);
            const int ksteps = (a.debug & 1) ? 0 : (ch.kn + 3) >> 2;
            if (ksteps > 0) {
                const double* As = stages + (c % kStages) * C::StageD;
                mma_dispatch<TRANS>(acc, mtw, As, As + kAStage, ch.aoff, ksteps);
            }
        }
        cp_wait<0>();
        __syncthreads();  // the ring is free for the next pass
#pragma unroll
        for (int t = 0; t < C::MTW; ++t) {
            const int row = m0 + 8 * (wm + t * C::WM) + (lane >> 2);
            if (t >= mtw || row >= m0 + mp) continue;
#pragma unroll
            for (int j = 0; j < C::NTW; ++j) {
                const int n = n0 + 8 * (wn * C::NTW + j) + 2 * (lane & 3);
                if (n < a.R) store(row, n, make_double2(acc[t][j][0], acc[t][j][1]));
            }
        }
    }

    // The next item: its 64-byte record was prefetched (cp.async, thread 0) while the
    // previous item ran; wait for its dependencies (the lanes 16.. of warp 0 poll one
    // flag each while the other threads fetch the descriptors), claim and prefetch the
    // item after it, stage the descriptors.
    __device__ bool next_item(int par) {
        if (tid == 0) asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
        const std::uint32_t claim = sh.pre_claim[par];
        const std::uint32_t item = claim / a.H, half = claim - item * a.H;
        if (item >= a.n_items) return false;
        const GraphItem it = sh.pre[par];
        std::uint32_t nxt = 0;
        if (tid == 0) {
            sh.item = item;
            sh.half = half;
            nxt = atomicAdd(a.counter, 1u);  // its latency runs under the loads below
        }
        // descriptors (16-byte pieces)
        auto copy16 = [&](void* dst, const void* src, int bytes, int t0) {
            const int p = tid - t0;
            if (p >= 0 && p < bytes / 16)
                reinterpret_cast<uint4*>(dst)[p] = __ldg(reinterpret_cast<const uint4*>(src) + p);
        };
        if (it.kind == GK_NODE_FWD || it.kind == GK_PAIR_BWD) {
            copy16(&sh.nd[0], a.nodes + it.a, sizeof(WaveNode), 0);
            if (it.kind == GK_PAIR_BWD && it.b != ~0u) copy16(&sh.nd[1], a.nodes + it.b, sizeof(WaveNode), 32);
        } else if (it.kind == GK_ROOT_BWD) {
            copy16(&sh.sd[0], a.stripes + it.a, sizeof(RootStripeDesc), 0);
        } else {
            const int ns = static_cast<int>(min(it.b, static_cast<std::uint32_t>(kSegMax)));
            for (int g = 0; g < ns; ++g) {
                const RootSeg sg = a.segs[it.a + g];
                copy16(&sh.sd[g], a.stripes + sg.stripe, sizeof(RootStripeDesc), 32 * (g % kW));
                if (tid == 32 * (g % kW) + 8) sh.row_off[g] = sg.row_off;
            }
        }
        // dependencies
        if (!(a.debug & 4) && it.ndep > 0 && tid >= 16 && tid < 32) {
            bool polled = false;
            for (std::uint32_t d = static_cast<std::uint32_t>(tid) - 16u; d < it.ndep; d += 16u) {
                const std::uint32_t dep = d < kGraphInlineDeps ? sh.pre[par].dep[d] : a.deps[it.dep0 + d];
                const std::uint32_t* f = a.flags + static_cast<std::size_t>(dep) * a.H + half;
                polled = true;
                if (ld_relaxed(f) == a.epoch) continue;
                const long long t0 = clock64();
                while (ld_relaxed(f) != a.epoch) {
                    __nanosleep(32);
                    if (clock64() - t0 > (1LL << 36)) __trap();
                }
            }
            if (polled) fence_acq_rel_gpu();  // acquire: the producers' vectors (published with a release fence)
        }
        if (tid == 0) {
            sh.pre_claim[par ^ 1] = nxt;
            const std::uint32_t ni = nxt / a.H;
            if (ni < a.n_items) {
                const char* src = reinterpret_cast<const char*>(a.items + ni);
                const std::uint32_t dst = sa(&sh.pre[par ^ 1]);
#pragma unroll
                for (int q = 0; q < 4; ++q) cp16s(dst + 16u * q, src + 16 * q, 16u);
            }
            cp_commit();
        }
        __syncthreads();
        // index lists
        if (it.kind == GK_NODE_FWD || it.kind == GK_PAIR_BWD) {
            const WaveNode n0d = sh.nd[0];
            const bool two = it.kind == GK_PAIR_BWD && it.b != ~0u;
            const std::uint32_t len0 = n0d.rank + n0d.nothers;
            const std::uint32_t len1 = two ? sh.nd[1].rank + sh.nd[1].nothers : 0;
            const bool fits = len0 + len1 <= static_cast<std::uint32_t>(kIdxCap);
            if (fits) {
                for (std::uint32_t e = tid; e < len0; e += kThreads) sh.idx[e] = __ldg(a.idx + n0d.idx + e);
                const std::uint32_t i1 = two ? sh.nd[1].idx : 0;
                for (std::uint32_t e = tid; e < len1; e += kThreads) sh.idx[len0 + e] = __ldg(a.idx + i1 + e);
            }
            if (tid == 0) sh.smem_idx = fits ? 1u : 0u;
            __syncthreads();
        }
        if (it.kind == GK_ROOT_FWD) {
            // chunk table: c -> (segment, chunk inside the segment's rank)
            const int ns = static_cast<int>(it.b);
            auto rank_of = [&](int g) {
                return static_cast<int>(g < kSegMax ? sh.sd[g].rank : a.stripes[a.segs[it.a + g].stripe].rank);
            };
            int nk = 0;
            for (int g = 0; g < ns; ++g) nk += (rank_of(g) + kKC - 1) / kKC;
            if (ns > 255 || nk > kIdxCap) __trap();
            for (int c = tid; c < nk; c += kThreads) {
                int cc = c, g = 0;
                for (; g < ns; ++g) {
                    const int n = (rank_of(g) + kKC - 1) / kKC;
                    if (cc < n) break;
                    cc -= n;
                }
                sh.idx[c] = static_cast<std::uint32_t>(g) | (static_cast<std::uint32_t>(cc) << 8);
            }
            if (tid == 0) sh.nchunks = static_cast<std::uint32_t>(nk);
            __syncthreads();
        }
        n0 = static_cast<int>(sh.half) * NT;
        return true;
    }

    __device__ void run() {
        if (tid == 0) {  // the first claim and its record
            const std::uint32_t c0 = atomicAdd(a.counter, 1u);
            sh.pre_claim[0] = c0;
            if (c0 / a.H < a.n_items) sh.pre[0] = a.items[c0 / a.H];
        }
        const int R = a.R;
        double* V = a.V;
        for (int par = 0; next_item(par); par ^= 1) {
            const GraphItem it = sh.pre[par];
            auto zero = [](int, int) { return make_double2(0.0, 0.0); };
            switch (it.kind) {
            case GK_NODE_FWD: {
                const WaveNode nd = sh.nd[0];
                const std::uint32_t* sel = sh.smem_idx ? sh.idx : a.idx + nd.idx;
                const std::uint32_t* oth = sel + nd.rank;
                const double* P = a.T + nd.t_off;
                const int M = static_cast<int>(nd.rank), K = static_cast<int>(nd.nothers), nib = static_cast<int>(nd.nib);
                const int nk = K > 0 ? (K + kKC - 1) / kKC : 0;
                double* out = V + static_cast<long long>(nd.cA) * R;
                for (int m0 = 0; m0 < M; m0 += kMPass) {
                    const int mp = min(kMPass, M - m0);
                    const int t0 = m0 >> 4, t1 = min(nib, (m0 + mp + 15) >> 4);
                    pass<false>(
                        m0, mp, nk,
                        [&](int c) { return AChunk{P, nib, c, t0, t1, 0, min(kKC, K - c * kKC)}; },
                        [&](int c) { return BRows{V, R, oth + kKC * c, 0}; }, true,
                        [&](int row, int n) { return ldcg2(V + static_cast<long long>(sel[row]) * R + n); },
                        [&](int row, int n, double2 v) { st2(out + static_cast<long long>(row) * R + n, v); });
                }
                break;
            }
            case GK_ROOT_FWD: {
                // chunks run over the block's segments (one per root group) in turn;
                // next_item left the chunk table in sh.idx: c -> segment | chunk of the segment << 8
                const int rows = static_cast<int>(it.rows);
                const int nk = static_cast<int>(sh.nchunks);
                auto seg = [&](int g, RootStripeDesc& d, std::uint32_t& off) {
                    if (g < kSegMax) {
                        d = sh.sd[g];
                        off = sh.row_off[g];
                    } else {
                        const RootSeg sg = a.segs[it.a + g];
                        d = a.stripes[sg.stripe];
                        off = sg.row_off;
                    }
                };
                auto chunk = [&](int c) {
                    const std::uint32_t e = sh.idx[c];
                    const int g = static_cast<int>(e & 255u), cc = static_cast<int>(e >> 8);
                    RootStripeDesc d;
                    std::uint32_t off;
                    seg(g, d, off);
                    const int nib = static_cast<int>(d.lds), t0 = static_cast<int>(off) >> 4;
                    return AChunk{a.S + d.s_off, nib, cc, t0, min(nib, (static_cast<int>(off) + rows + 15) >> 4),
                                  static_cast<int>(off) - 16 * t0, min(kKC, static_cast<int>(d.rank) - cc * kKC)};
                };
                auto bs = [&](int c) {
                    const std::uint32_t e = sh.idx[c];
                    const int g = static_cast<int>(e & 255u), cc = static_cast<int>(e >> 8);
                    const std::uint32_t coff = g < kSegMax ? sh.sd[g].coff : a.stripes[a.segs[it.a + g].stripe].coff;
                    return BRows{V + (static_cast<long long>(coff) + kKC * cc) * R, R, nullptr, 0};
                };
                if (a.stacked) {
                    double* Y = a.u + (static_cast<long long>(a.plan_row0[it.plan]) + it.r0) * R;
                    pass<false>(0, rows, nk, chunk, bs, false, zero, [&](int row, int n, double2 v) {
                        st2(Y + static_cast<long long>(row) * R + n, v);
                    });
                } else {
                    const long long bstride = static_cast<long long>(a.l) * 4;
                    double* U = a.u + (static_cast<long long>(it.plan) * a.batch * a.l + it.r0) * 4;
                    pass<false>(0, rows, nk, chunk, bs, false, zero, [&](int row, int n, double2 v) {
                        st2(U + (n >> 2) * bstride + static_cast<long long>(row) * 4 + (n & 3), v);
                    });
                }
                break;
            }
            case GK_PAIR_BWD: {
                std::uint32_t ioff = 0;
                for (int t = 0; t < 2; ++t) {
                    const std::uint32_t x = t == 0 ? it.a : it.b;
                    if (x == ~0u) break;
                    const bool second = t == 1;
                    const WaveNode nd = sh.nd[t];
                    const std::uint32_t* sel = sh.smem_idx ? sh.idx + ioff : a.idx + nd.idx;
                    const std::uint32_t* oth = sel + nd.rank;
                    ioff += nd.rank + nd.nothers;
                    const int M = static_cast<int>(nd.nothers), K = static_cast<int>(nd.rank),
                              nib = static_cast<int>(nd.nib);
                    const int nk = K > 0 ? (K + kKC - 1) / kKC : 0;
                    const double* P = a.T + nd.t_off;
                    const double* cv = V + static_cast<long long>(nd.cA) * R;
                    for (int m0 = 0; m0 < M; m0 += kMPass) {
                        const int mp = min(kMPass, M - m0);
                        const int t0 = m0 >> 4, t1 = (m0 + mp + 15) >> 4;
                        pass<true>(
                            m0, mp, nk, [&](int c) { return AChunk{P, nib, c, t0, t1, 0, min(kKC, K - c * kKC)}; },
                            [&](int c) { return BRows{cv + static_cast<long long>(kKC * c) * R, R, nullptr, 0}; }, second,
                            [&](int row, int n) { return ldcg2(V + static_cast<long long>(oth[row]) * R + n); },
                            [&](int row, int n, double2 v) { st2(V + static_cast<long long>(oth[row]) * R + n, v); });
                    }
                    // z[sel] (=|+=) c over this block's columns
                    // (two pieces per round, so four loads are in flight before the first store: the
                    // compiler cannot move loads over the stores, the cells could alias for all it knows)
                    const int nn = (min(NT, R - n0) + 1) / 2;
                    const int tot = static_cast<int>(nd.rank) * nn;
                    for (int e = tid; e < tot; e += 2 * kThreads) {
                        const int e1 = e + kThreads;
                        const bool two = e1 < tot;
                        const int i0 = e / nn, c0 = n0 + 2 * (e - i0 * nn);
                        const int i1 = two ? e1 / nn : i0, c1 = two ? n0 + 2 * (e1 - i1 * nn) : c0;
                        double* z0 = V + static_cast<long long>(sel[i0]) * R + c0;
                        double* z1 = V + static_cast<long long>(sel[i1]) * R + c1;
                        double2 v0 = ldcg2(cv + static_cast<long long>(i0) * R + c0);
                        double2 v1 = ldcg2(cv + static_cast<long long>(i1) * R + c1);
                        if (second) {
                            const double2 o0 = ldcg2(z0), o1 = ldcg2(z1);
                            v0.x += o0.x;
                            v0.y += o0.y;
                            v1.x += o1.x;
                            v1.y += o1.y;
                        }
                        st2(z0, v0);
                        if (two) st2(z1, v1);
                    }
                    __syncthreads();  // the second node adds onto the same z cells
                }
                break;
            }
            default: {  // GK_ROOT_BWD
                const RootStripeDesc d = sh.sd[0];
                const int M = static_cast<int>(d.rank), K = static_cast<int>(d.rows), nib = static_cast<int>(d.lds);
                const int nk = (K + kKC - 1) / kKC;
                const double* P = a.S + d.s_off;
                double* out = V + static_cast<long long>(d.coff) * R;
                auto store = [&](int row, int n, double2 v) { st2(out + static_cast<long long>(row) * R + n, v); };
                for (int m0 = 0; m0 < M; m0 += kMPass) {
                    const int mp = min(kMPass, M - m0);
                    const int t0 = m0 >> 4, t1 = (m0 + mp + 15) >> 4;
                    auto chunk = [&](int c) { return AChunk{P, nib, c, t0, t1, 0, min(kKC, K - c * kKC)}; };
                    if (a.stacked) {
                        const double* W = a.u + static_cast<long long>(d.pad[1]) * R;
                        pass<true>(
                            m0, mp, nk, chunk,
                            [&](int c) { return BRows{W + static_cast<long long>(kKC * c) * R, R, nullptr, 0}; }, false,
                            zero, store);
                    } else {
                        const double* U = a.u + (static_cast<long long>(d.plan) * a.batch * a.l + d.yin) * 4;
                        const long long bstride = static_cast<long long>(a.l) * 4;
                        pass<true>(
                            m0, mp, nk, chunk,
                            [&](int c) { return BRows{U + static_cast<long long>(kKC * c) * 4, 4, nullptr, bstride}; },
                            false, zero, store);
                    }
                }
                break;
            }
            }
            // publish: every thread's stores of this item are done
            __syncthreads();
            if (tid == 0) {
                fence_acq_rel_gpu();
                st_relaxed(a.flags + static_cast<std::size_t>(sh.item) * a.H + sh.half, a.epoch);
            }
        }
    }
};

template <int NT, class SH>
__global__ void __launch_bounds__(SH::kThreads, SH::Ctas) wgraph_kernel(const __grid_constant__ GraphArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    ItemSh& sh = *reinterpret_cast<ItemSh*>(smem);
    double* stages = reinterpret_cast<double*>(smem + ((sizeof(ItemSh) + 127) & ~std::size_t{127}));
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    Cta<NT, SH> cta{a, sh, stages, tid, warp, lane, warp / Cfg<NT, SH>::WN, warp % Cfg<NT, SH>::WN, 0};
    cta.run();
}

template <class T>
T* upload(const std::vector<T>& v) {
    T* d = nullptr;
    if (v.empty()) return nullptr;
    if (cudaMalloc(&d, v.size() * sizeof(T)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed (graph)");
    if (cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
        throw std::runtime_error("cudaMemcpy failed (graph)");
    return d;
}

}  // namespace

DeviceGraph upload_graph(const GraphProgram& g) {
    DeviceGraph d;
    d.items[0] = upload(g.fwd);
    d.items[1] = upload(g.bwd);
    d.deps[0] = upload(g.fwd_deps);
    d.deps[1] = upload(g.bwd_deps);
    d.segs = upload(g.segs);
    d.n_items[0] = static_cast<std::uint32_t>(g.fwd.size());
    d.n_items[1] = static_cast<std::uint32_t>(g.bwd.size());
    if (cudaMalloc(&d.counter, 2 * sizeof(std::uint32_t)) != cudaSuccess) throw std::runtime_error("cudaMalloc failed (graph)");
    d.groups = g.groups;
    d.ok = true;
    return d;
}

void free_graph(DeviceGraph& d) {
    for (int k = 0; k < 2; ++k) {
        cudaFree(d.items[k]);
        cudaFree(d.deps[k]);
        cudaFree(d.flags[k]);
    }
    cudaFree(d.segs);
    cudaFree(d.counter);
    d = DeviceGraph{};
}

cudaError_t launch_graph(DeviceGraph& g, const DeviceWaveSet& w, double* V, double* u, int l, int batch, bool transpose,
                         cudaStream_t st, bool stacked) {
    const int k = transpose ? 1 : 0;
    if (g.n_items[k] == 0 || batch == 0) return cudaSuccess;
    const int R = 4 * batch;
    const int nt = R <= 8 ? 8 : R <= 16 ? 16 : R <= 32 ? 32 : 64;
    const int H = (R + nt - 1) / nt;
    const std::size_t need = static_cast<std::size_t>(g.n_items[k]) * H;
    if (g.flag_cap[k] < need) {
        cudaFree(g.flags[k]);
        g.flags[k] = nullptr;
        g.flag_cap[k] = 0;
        cudaError_t e = cudaMalloc(&g.flags[k], need * sizeof(std::uint32_t));
        if (e != cudaSuccess) return e;
        e = cudaMemsetAsync(g.flags[k], 0, need * sizeof(std::uint32_t), st);
        if (e != cudaSuccess) return e;
        g.flag_cap[k] = need;
        g.epoch[k] = 0;
    }
    if (++g.epoch[k] == 0) {  // 2^32 launches: start the flags over
        cudaError_t e = cudaMemsetAsync(g.flags[k], 0, g.flag_cap[k] * sizeof(std::uint32_t), st);
        if (e != cudaSuccess) return e;
        g.epoch[k] = 1;
    }
    cudaError_t e = cudaMemsetAsync(g.counter + k, 0, sizeof(std::uint32_t), st);
    if (e != cudaSuccess) return e;
    GraphArgs a{};
    a.items = g.items[k];
    a.deps = g.deps[k];
    a.segs = g.segs;
    a.nodes = w.nodes;
    a.idx = w.idx;
    a.T = w.T;
    a.stripes = w.roots.stripes;
    a.S = w.roots.data;
    a.V = V;
    a.u = u;
    a.plan_row0 = w.plan_row0;
    a.stacked = stacked ? 1 : 0;
    a.flags = g.flags[k];
    a.counter = g.counter + k;
    a.epoch = g.epoch[k];
    a.n_items = g.n_items[k];
    a.l = l;
    a.batch = batch;
    a.R = R;
    a.H = H;
    a.debug = 0;
    if (const char* e = std::getenv("BFLY_GRAPH_DEBUG")) a.debug = static_cast<int>(std::strtol(e, nullptr, 10));
    auto go = [&](auto kern, auto cfg) -> cudaError_t {
        using CF = decltype(cfg);
        using SH = typename CF::Shape;
        const std::size_t smem = ((sizeof(ItemSh) + 127) & ~std::size_t{127}) +
                                 static_cast<std::size_t>(SH::Stages) * CF::StageD * sizeof(double);
        cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e2 != cudaSuccess) return e2;
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, SH::kThreads, smem);
        const long long want = static_cast<long long>(g.n_items[k]) * H;
        const int grid = static_cast<int>(std::max(1LL, std::min<long long>(static_cast<long long>(sms) * std::max(1, per), want)));
        kern<<<grid, SH::kThreads, smem, st>>>(a);
        return cudaGetLastError();
    };
    auto run = [&](auto sh) -> cudaError_t {
        using SH = decltype(sh);
        switch (nt) {
        case 8: return go(wgraph_kernel<8, SH>, Cfg<8, SH>{});
        case 16: return go(wgraph_kernel<16, SH>, Cfg<16, SH>{});
        case 32: return go(wgraph_kernel<32, SH>, Cfg<32, SH>{});
        default: return go(wgraph_kernel<64, SH>, Cfg<64, SH>{});
        }
    };
    return transpose ? run(BwdShape{}) : run(FwdShape{});
}

}  // namespace bfb
