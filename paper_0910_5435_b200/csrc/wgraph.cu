// Persistent graph kernel of the wave programs (wgraph.hpp): one launch runs
// a whole direction of the batched butterfly apply on the FP64 tensor cores.
//
// CTA = 16 consumer warps + a scheduler warp + a streaming warp, one CTA per SM.
//
// Producer warp (lane 0 leads):
//   * claims the next (item, column block) from an atomic counter, so items
//     start in queue order — the queue is topological, which makes the spin
//     below deadlock-free (every item an item waits for was claimed earlier
//     by a running CTA and waits only on even earlier ones);
//   * waits until the items it depends on have published (per-(item, column
//     block) flags = this launch's epoch, ld.acquire.gpu), then hands the
//     item to the consumers through a two-slot mailbox (mbarriers);
//   * copies the item's index lists into the mailbox slot (shared memory);
//   * streams the item's operands in K-chunks of 16 into a 3-stage ring: the
//     matrix (T of a node, S of a root stripe; 16 x 16 swizzled tiles,
//     packer.hpp) by cp.async.bulk (TMA bulk copies with mbarrier
//     complete_tx): a forward chunk is ONE contiguous run of tiles, a
//     transposed chunk one 2 KB copy per output tile; the vector rows
//     (gathered through the index list, or the strided chain rows u) by
//     16-byte cp.async whose completion the same mbarrier tracks
//     (cp.async.mbarrier.arrive.noinc).  Each stage carries a small header
//     (valid K, last chunk of the pass, row offset).
// Consumer warps: a 4 x 4 (NT = 64) warp grid over the output tile (up to
//   192 rows x NT columns in one pass, so a node of rank <= 192 needs one
//   pass and its gathered vectors are staged once), DMMA m8n8k4 with the
//   accumulators starting from the forward's z[sel] term / the transpose's
//   old z; epilogue straight to V / u; then the item's flag is released.
//
// Memory: the vectors V between items go through L2 (the queue is
// group-major, so a producer's output is normally still in L2 when its
// consumer runs); the matrices are read once per column block.
#include <cuda_runtime.h>

#include <algorithm>
#include <stdexcept>
#include <type_traits>

#include "wgraph_dev.hpp"

namespace bfb {

namespace {

constexpr int kKC = 16;                    // K chunk
constexpr int kMMax = static_cast<int>(kGraphMaxRows);
constexpr int kCW = 16;                    // consumer warps (one CTA per SM)
constexpr int kStreamWarp = kCW;           // producer warp: operand streaming
constexpr int kSchedWarp = kCW + 1;        // producer warp: claims, dependencies, descriptors
constexpr int kThreads = 32 * (kCW + 2);
constexpr int kSegMax = 4;                 // root-block segments kept in the mailbox
constexpr int kStages = 5;
constexpr int kATiles = kMMax / 16 + 1;    // matrix tiles per stage (a row block may start mid-tile)
constexpr int kAStage = kATiles * 256;     // doubles
constexpr int kIdxCap = 1536;              // index-list entries per mailbox slot

template <int NT>
struct Cfg {
    static_assert(NT == 8 || NT == 16 || NT == 32 || NT == 64, "column block");
    static constexpr int NTW = NT >= 16 ? 2 : 1;     // n8 tiles per warp
    static constexpr int WN = NT / (8 * NTW);        // warps along n
    static constexpr int WM = kCW / WN;              // warps along m
    static constexpr int MTW = (kMMax / 8 + WM - 1) / WM;  // m8 tiles per warp (max)
    static constexpr int LDB = NT + 4;               // B tile row stride (4 mod 16: conflict-free)
    static constexpr int StageD = kAStage + kKC * LDB;
};

struct StageHdr {
    int aoff;  // forward: row of the item's first output row inside the first tile
    int kn;    // valid K of this chunk
    int last;  // last chunk of the pass
    int pad;
};
// Mailbox slot: one item, its descriptors and index lists, written by the
// scheduler warp; read by the streaming warp and the consumers.
struct Slot {
    GraphItem it;
    std::uint32_t item, half, end, smem_idx;  // smem_idx: the index lists are in Ctrl::idx[slot]
    WaveNode nd[2];                            // NODE_FWD: nd[0]; PAIR_BWD: nd[0], nd[1]
    RootStripeDesc sd[kSegMax];                // ROOT_BWD: sd[0]; ROOT_FWD: the segments' stripes
    std::uint32_t row_off[kSegMax];            // ROOT_FWD: the segments' first rows
};
struct Ctrl {
    std::uint64_t full[kStages], empty[kStages], ifull[2], iempty[2];
    StageHdr hdr[kStages];
    Slot slot[2];
    std::uint32_t idx[2][kIdxCap];
};
constexpr std::size_t kCtrlBytes = (sizeof(Ctrl) + 127) & ~std::size_t{127};

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
    double* u;                    // chain rows [plan][b][l][4], or (stacked) cell-major rows [row][R]
    const std::uint32_t* plan_row0;  // stacked: first row of each plan
    int stacked;
    std::uint32_t* flags;
    std::uint32_t* counter;
    std::uint32_t epoch;
    std::uint32_t n_items;
    int l, batch, R, H;
};

// ---- PTX helpers ---------------------------------------------------------------
__device__ __forceinline__ std::uint32_t sa(const void* p) {
    return static_cast<std::uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(std::uint64_t* b, std::uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(std::uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(std::uint64_t* b, std::uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try(std::uint64_t* b, std::uint32_t parity) {
    std::uint32_t ok;
    asm volatile(
        "{\n.reg .pred P1;\nmbarrier.try_wait.parity.shared::cta.b64 P1, [%1], %2, %3;\nselp.u32 %0, 1, 0, P1;\n}\n"
        : "=r"(ok)
        : "r"(sa(b)), "r"(parity), "r"(1000000u)
        : "memory");
    return ok != 0;
}
// A wait beyond ~2^35 cycles (well over ten seconds) traps instead of hanging the device.
__device__ __forceinline__ void mbar_wait(std::uint64_t* b, std::uint32_t parity) {
    if (mbar_try(b, parity)) return;
    long long t0 = 0;
    for (std::uint32_t it = 1; !mbar_try(b, parity); ++it) {
        if ((it & 1023u) == 0) {
            const long long now = clock64();
            if (t0 == 0) t0 = now;
            else if (now - t0 > (1LL << 35)) __trap();
        }
    }
}
// The matrices are streamed once per launch: evict-first in L2, so they do not
// push out the vectors passed between items.
__device__ __forceinline__ std::uint64_t evict_first_policy() {
    std::uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, std::uint32_t bytes, std::uint64_t* bar,
                                          std::uint64_t pol) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            sa(dst)),
        "l"(src), "r"(bytes), "r"(sa(bar)), "l"(pol)
        : "memory");
}
// 16-byte cp.async through L2 (the vectors are written by other CTAs); src_bytes 0 fills zeros.
__device__ __forceinline__ void cp16(void* dst, const void* src, std::uint32_t src_bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa(dst)), "l"(src), "r"(src_bytes) : "memory");
}
__device__ __forceinline__ void cp_arrive_noinc(std::uint64_t* b) {
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ std::uint32_t ld_acquire(const std::uint32_t* p) {
    std::uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(std::uint32_t* p, std::uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void consumers_sync() { asm volatile("bar.sync 1, %0;" ::"n"(32 * kCW) : "memory"); }
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}
__device__ __forceinline__ double2 ldcg2(const double* p) { return __ldcg(reinterpret_cast<const double2*>(p)); }
// A warp copies a 16-byte-aligned struct from global to shared memory.
template <class T>
__device__ __forceinline__ void warp_copy(T* dst, const T* src, int lane) {
    static_assert(sizeof(T) % 16 == 0, "warp_copy: 16-byte multiples");
    constexpr int n = sizeof(T) / 16;
    if (lane < n) reinterpret_cast<uint4*>(dst)[lane] = __ldg(reinterpret_cast<const uint4*>(src) + lane);
}
__device__ __forceinline__ void st2(double* p, double2 v) { *reinterpret_cast<double2*>(p) = v; }

// ---- scheduler warp ---------------------------------------------------------------
// Claims items in queue order, waits for their dependencies, and fills the
// mailbox slot (descriptors, index lists) one item ahead of the consumers, so
// none of these dependent global round trips sits between two items.
struct Scheduler {
    const GraphArgs& a;
    Ctrl& c;
    int lane;

    __device__ void run() {
        std::uint32_t icount = 0;
        std::uint32_t next = 0;
        if (lane == 0) next = atomicAdd(a.counter, 1u);
        for (;;) {
            const std::uint32_t claim = __shfl_sync(~0u, next, 0);
            const std::uint32_t item = claim / a.H, half = claim - item * a.H;
            const bool end = item >= a.n_items;
            if (lane == 0 && !end) next = atomicAdd(a.counter, 1u);  // the claim after this one, in flight
            const std::uint32_t j = icount & 1, use = icount >> 1;
            if (use > 0) mbar_wait(&c.iempty[j], (use - 1) & 1);  // the consumers are done with item icount - 2
            Slot& sl = c.slot[j];
            bool sidx = false;
            if (!end) {
                const GraphItem it = a.items[item];
                // descriptors first (independent of the dependencies)
                if (it.kind == GK_NODE_FWD || it.kind == GK_PAIR_BWD) {
                    warp_copy(&sl.nd[0], a.nodes + it.a, lane);
                    if (it.kind == GK_PAIR_BWD && it.b != ~0u) warp_copy(&sl.nd[1], a.nodes + it.b, lane);
                } else if (it.kind == GK_ROOT_BWD) {
                    warp_copy(&sl.sd[0], a.stripes + it.a, lane);
                } else {
                    const std::uint32_t ns = min(it.b, static_cast<std::uint32_t>(kSegMax));
                    for (std::uint32_t g = 0; g < ns; ++g) {
                        const RootSeg sg = a.segs[it.a + g];
                        warp_copy(&sl.sd[g], a.stripes + sg.stripe, lane);
                        if (lane == 0) sl.row_off[g] = sg.row_off;
                    }
                }
                if (lane == 0) {
                    for (std::uint32_t d = 0; d < it.ndep; ++d) {
                        const std::uint32_t* f = a.flags + static_cast<std::size_t>(a.deps[it.dep0 + d]) * a.H + half;
                        if (ld_acquire(f) == a.epoch) continue;
                        long long t0 = clock64();
                        while (ld_acquire(f) != a.epoch) {
                            __nanosleep(64);
                            if (clock64() - t0 > (1LL << 36)) __trap();
                        }
                    }
                }
                __syncwarp();
                // index lists into the slot (when they fit)
                if (it.kind == GK_NODE_FWD || it.kind == GK_PAIR_BWD) {
                    const WaveNode n0 = sl.nd[0];
                    const bool two = it.kind == GK_PAIR_BWD && it.b != ~0u;
                    const std::uint32_t len0 = n0.rank + n0.nothers;
                    const std::uint32_t len1 = two ? sl.nd[1].rank + sl.nd[1].nothers : 0;
                    if (len0 + len1 <= static_cast<std::uint32_t>(kIdxCap)) {
                        for (std::uint32_t e = lane; e < len0; e += 32) c.idx[j][e] = __ldg(a.idx + n0.idx + e);
                        const std::uint32_t i1 = two ? sl.nd[1].idx : 0;
                        for (std::uint32_t e = lane; e < len1; e += 32) c.idx[j][len0 + e] = __ldg(a.idx + i1 + e);
                        sidx = true;
                    }
                }
                if (lane == 0) sl.it = it;
            }
            __syncwarp();
            if (lane == 0) {
                sl.item = item;
                sl.half = half;
                sl.end = end ? 1u : 0u;
                sl.smem_idx = sidx ? 1u : 0u;
                mbar_arrive(&c.ifull[j]);  // release: the slot's stores above
            }
            ++icount;
            if (end) break;
        }
    }
};

// ---- streaming warp ---------------------------------------------------------------
template <int NT>
struct Streamer {
    using C = Cfg<NT>;
    const GraphArgs& a;
    Ctrl& c;
    double* stages;
    int lane;
    std::uint32_t q = 0;  // chunks issued
    int n0 = 0;
    std::uint64_t pol = evict_first_policy();

    // One K-chunk.  Forward (TRANS = false): the matrix's column tile `kt`, row
    // tiles [t0, t1) -- one contiguous copy.  Transposed: row tile `kt`, column
    // tiles [t0, t1) -- one 2 KB copy each.  P: the tiled matrix, nib its row tiles.
    template <bool TRANS, class BSRC>
    __device__ void chunk(const double* P, int nib, int kt, int t0, int t1, int aoff, int kn, bool last, BSRC bsrc) {
        const std::uint32_t s = q % kStages, use = q / kStages;
        if (use > 0) mbar_wait(&c.empty[s], (use - 1) & 1);
        double* As = stages + s * C::StageD;
        double* Bs = As + kAStage;
        const std::uint32_t abytes = static_cast<std::uint32_t>(t1 - t0) * 2048u;
        if (lane == 0) {
            c.hdr[s] = StageHdr{aoff, kn, last ? 1 : 0, 0};
            mbar_expect_tx(&c.full[s], abytes);
        }
        __syncwarp();
        if (!TRANS) {
            if (lane == 0 && abytes)
                bulk_copy(As, P + (static_cast<long long>(kt) * nib + t0) * 256, abytes, &c.full[s], pol);
        } else {
            for (int t = t0 + lane; t < t1; t += 32)
                bulk_copy(As + (t - t0) * 256, P + (static_cast<long long>(t) * nib + kt) * 256, 2048u, &c.full[s], pol);
        }
        // vector rows: K rows x NT columns (pieces of 2 doubles); rows kn .. kn rounded
        // up to 4 are zero-filled (the last k-step), later rows are never read
        const int kr = (kn + 3) & ~3;
        for (int e = lane; e < kr * (NT / 2); e += 32) {
            const int k = e / (NT / 2), h = e - k * (NT / 2);
            const int n = n0 + 2 * h;
            const bool ok = k < kn && n < a.R;
            cp16(Bs + k * C::LDB + 2 * h, ok ? bsrc(16 * kt + k, n) : a.V, ok ? 16u : 0u);
        }
        cp_arrive_noinc(&c.full[s]);
        ++q;
    }

    __device__ void run() {
        std::uint32_t icount = 0;
        for (;;) {
            const std::uint32_t j = icount & 1;
            mbar_wait(&c.ifull[j], (icount >> 1) & 1);
            ++icount;
            const Slot& sl = c.slot[j];
            if (sl.end) break;
            // the vectors were written by other CTAs' generic stores (published to the
            // scheduler); the bulk copies below read through the async proxy
            asm volatile("fence.proxy.async.global;" ::: "memory");
            const GraphItem it = sl.it;
            n0 = static_cast<int>(sl.half) * NT;
            const int R = a.R;
            double* V = a.V;
            switch (it.kind) {
            case GK_NODE_FWD: {
                const WaveNode nd = sl.nd[0];
                const std::uint32_t* oth = (sl.smem_idx ? c.idx[j] : a.idx + nd.idx) + nd.rank;
                const double* P = a.T + nd.t_off;
                const int M = static_cast<int>(nd.rank), K = static_cast<int>(nd.nothers), nib = static_cast<int>(nd.nib);
                const int nk = K > 0 ? (K + kKC - 1) / kKC : 1;
                auto bs = [&](int kk, int n) { return V + static_cast<long long>(oth[kk]) * R + n; };
                for (int m0 = 0; m0 < M; m0 += kMMax) {
                    const int t0 = m0 >> 4, t1 = min(nib, (m0 + kMMax) >> 4);
                    for (int ch = 0; ch < nk; ++ch)
                        chunk<false>(P, nib, ch, K > 0 ? t0 : 0, K > 0 ? t1 : 0, 0, min(kKC, K - ch * kKC), ch == nk - 1,
                                     bs);
                }
                break;
            }
            case GK_ROOT_FWD: {
                const int rows = static_cast<int>(it.rows);
                if (it.b == 0) {  // no stripe with a nonzero rank covers the block: zeros
                    chunk<false>(a.S, 1, 0, 0, 0, 0, 0, true, [&](int, int) { return V; });
                    break;
                }
                for (std::uint32_t g = 0; g < it.b; ++g) {
                    RootStripeDesc d;
                    std::uint32_t row_off;
                    if (g < static_cast<std::uint32_t>(kSegMax)) {
                        d = sl.sd[g];
                        row_off = sl.row_off[g];
                    } else {
                        const RootSeg sg = a.segs[it.a + g];
                        d = a.stripes[sg.stripe];
                        row_off = sg.row_off;
                    }
                    const double* P = a.S + d.s_off;
                    const int K = static_cast<int>(d.rank), nib = static_cast<int>(d.lds);
                    const int nk = (K + kKC - 1) / kKC;
                    const int t0 = static_cast<int>(row_off) >> 4;
                    const int t1 = min(nib, (static_cast<int>(row_off) + rows + 15) >> 4);
                    const double* Cv = V + static_cast<long long>(d.coff) * R;
                    auto bs = [&](int kk, int n) { return Cv + static_cast<long long>(kk) * R + n; };
                    for (int ch = 0; ch < nk; ++ch)
                        chunk<false>(P, nib, ch, t0, t1, static_cast<int>(row_off) - 16 * t0, min(kKC, K - ch * kKC),
                                     g + 1 == it.b && ch == nk - 1, bs);
                }
                break;
            }
            case GK_PAIR_BWD: {
                for (int t = 0; t < 2; ++t) {
                    const std::uint32_t x = t == 0 ? it.a : it.b;
                    if (x == ~0u) break;
                    const WaveNode nd = sl.nd[t];
                    const int M = static_cast<int>(nd.nothers), K = static_cast<int>(nd.rank), nib = static_cast<int>(nd.nib);
                    const int nk = K > 0 ? (K + kKC - 1) / kKC : 1;
                    const double* P = a.T + nd.t_off;
                    const double* Cv = V + static_cast<long long>(nd.cA) * R;
                    auto bs = [&](int kk, int n) { return Cv + static_cast<long long>(kk) * R + n; };
                    for (int m0 = 0; m0 < M; m0 += kMMax) {
                        const int t0 = m0 >> 4, t1 = (min(M, m0 + kMMax) + 15) >> 4;
                        for (int ch = 0; ch < nk; ++ch)
                            chunk<true>(P, nib, ch, K > 0 ? t0 : 0, K > 0 ? t1 : 0, 0, min(kKC, K - ch * kKC),
                                        ch == nk - 1, bs);
                    }
                }
                break;
            }
            default: {  // GK_ROOT_BWD
                const RootStripeDesc d = sl.sd[0];
                const int M = static_cast<int>(d.rank), K = static_cast<int>(d.rows), nib = static_cast<int>(d.lds);
                const int nk = (K + kKC - 1) / kKC;
                const double* P = a.S + d.s_off;
                if (a.stacked) {
                    const double* W = a.u + static_cast<long long>(d.pad[1]) * R;
                    auto bs = [&](int kk, int n) { return W + static_cast<long long>(kk) * R + n; };
                    for (int m0 = 0; m0 < M; m0 += kMMax) {
                        const int t0 = m0 >> 4, t1 = (min(M, m0 + kMMax) + 15) >> 4;
                        for (int ch = 0; ch < nk; ++ch)
                            chunk<true>(P, nib, ch, t0, t1, 0, min(kKC, K - ch * kKC), ch == nk - 1, bs);
                    }
                } else {
                    const double* U = a.u + (static_cast<long long>(d.plan) * a.batch * a.l + d.yin) * 4;
                    const long long bstride = static_cast<long long>(a.l) * 4;
                    auto bs = [&](int kk, int n) {
                        return U + (n >> 2) * bstride + static_cast<long long>(kk) * 4 + (n & 3);
                    };
                    for (int m0 = 0; m0 < M; m0 += kMMax) {
                        const int t0 = m0 >> 4, t1 = (min(M, m0 + kMMax) + 15) >> 4;
                        for (int ch = 0; ch < nk; ++ch)
                            chunk<true>(P, nib, ch, t0, t1, 0, min(kKC, K - ch * kKC), ch == nk - 1, bs);
                    }
                }
                break;
            }
            }
        }
    }
};

// ---- consumers -------------------------------------------------------------------
template <int NT>
struct Consumer {
    using C = Cfg<NT>;
    const GraphArgs& a;
    Ctrl& c;
    double* stages;
    int warp, lane, wm, wn;
    std::uint32_t q = 0;
    int n0 = 0;

    // The chunk's k-steps on this warp's first MT m8 tiles (all live).
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

    // One pass: rows [m0, m0 + mp) of the output, every chunk the producer streams
    // for it.  TRANS: the matrix tiles hold the transposed operand (one tile per 16
    // output rows); else a run of row tiles starting hdr.aoff rows before m0.
    // init(row, n) / store(row, n, v): double2 at columns n, n + 1.
    template <bool TRANS, class INIT, class STORE>
    __device__ void pass(int m0, int mp, bool has_init, INIT init, STORE store) {
        double acc[C::MTW][C::NTW][2];
        const int mt = (mp + 7) >> 3;
        const int mtw = wm < mt ? (mt - wm + C::WM - 1) / C::WM : 0;
#pragma unroll
        for (int t = 0; t < C::MTW; ++t) {
            const int row = m0 + 8 * (wm + t * C::WM) + (lane >> 2);
#pragma unroll
            for (int j = 0; j < C::NTW; ++j) {
                const int n = n0 + 8 * (wn * C::NTW + j) + 2 * (lane & 3);
                double2 v = make_double2(0.0, 0.0);
                if (has_init && t < mtw && row < m0 + mp && n < a.R) v = init(row, n);
                acc[t][j][0] = v.x;
                acc[t][j][1] = v.y;
            }
        }
        for (;;) {
            const std::uint32_t s = q % kStages;
            mbar_wait(&c.full[s], (q / kStages) & 1);
            const StageHdr h = c.hdr[s];
            const double* As = stages + s * C::StageD;
            const double* Bs = As + kAStage;
            const int ksteps = (h.kn + 3) >> 2;
            if (ksteps > 0) {
                // exactly this warp's live m8 tiles (a guard inside the unrolled tile
                // loop compiles to predicated DMMAs, which still take tensor-pipe cycles)
                switch (mtw) {
                case 1: mma_chunk<(1 < C::MTW ? 1 : C::MTW), TRANS>(acc, As, Bs, h.aoff, ksteps); break;
                case 2: mma_chunk<(2 < C::MTW ? 2 : C::MTW), TRANS>(acc, As, Bs, h.aoff, ksteps); break;
                case 3: mma_chunk<(3 < C::MTW ? 3 : C::MTW), TRANS>(acc, As, Bs, h.aoff, ksteps); break;
                case 4: mma_chunk<(4 < C::MTW ? 4 : C::MTW), TRANS>(acc, As, Bs, h.aoff, ksteps); break;
                case 5: mma_chunk<(5 < C::MTW ? 5 : C::MTW), TRANS>(acc, As, Bs, h.aoff, ksteps); break;
                case 6: mma_chunk<(6 < C::MTW ? 6 : C::MTW), TRANS>(acc, As, Bs, h.aoff, ksteps); break;
                default: break;
                }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&c.empty[s]);
            ++q;
            if (h.last) break;
        }
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

    __device__ void run() {
        std::uint32_t icount = 0;
        const int R = a.R;
        double* V = a.V;
        for (;;) {
            const std::uint32_t j = icount & 1;
            mbar_wait(&c.ifull[j], (icount >> 1) & 1);
            const Slot& sl = c.slot[j];
            ++icount;
            if (sl.end) break;
            const GraphItem it = sl.it;
            const std::uint32_t item = sl.item;
            n0 = static_cast<int>(sl.half) * NT;
            switch (it.kind) {
            case GK_NODE_FWD: {
                const WaveNode nd = sl.nd[0];
                const std::uint32_t* sel = sl.smem_idx ? c.idx[j] : a.idx + nd.idx;
                const int M = static_cast<int>(nd.rank);
                double* out = V + static_cast<long long>(nd.cA) * R;
                for (int m0 = 0; m0 < M; m0 += kMMax)
                    pass<false>(
                        m0, min(kMMax, M - m0), true,
                        [&](int row, int n) { return ldcg2(V + static_cast<long long>(sel[row]) * R + n); },
                        [&](int row, int n, double2 v) { st2(out + static_cast<long long>(row) * R + n, v); });
                break;
            }
            case GK_ROOT_FWD: {
                auto zero = [&](int, int) { return make_double2(0.0, 0.0); };
                if (a.stacked) {
                    double* Y = a.u + (static_cast<long long>(a.plan_row0[it.plan]) + it.r0) * R;
                    pass<false>(0, static_cast<int>(it.rows), false, zero, [&](int row, int n, double2 v) {
                        st2(Y + static_cast<long long>(row) * R + n, v);
                    });
                } else {
                    const long long bstride = static_cast<long long>(a.l) * 4;
                    double* U = a.u + (static_cast<long long>(it.plan) * a.batch * a.l + it.r0) * 4;
                    pass<false>(0, static_cast<int>(it.rows), false, zero, [&](int row, int n, double2 v) {
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
                    const WaveNode nd = sl.nd[t];
                    const std::uint32_t* sel = sl.smem_idx ? c.idx[j] + ioff : a.idx + nd.idx;
                    const std::uint32_t* oth = sel + nd.rank;
                    ioff += nd.rank + nd.nothers;
                    const int M = static_cast<int>(nd.nothers);
                    for (int m0 = 0; m0 < M; m0 += kMMax)
                        pass<true>(
                            m0, min(kMMax, M - m0), second,
                            [&](int row, int n) { return ldcg2(V + static_cast<long long>(oth[row]) * R + n); },
                            [&](int row, int n, double2 v) { st2(V + static_cast<long long>(oth[row]) * R + n, v); });
                    // z[sel] (=|+=) c over this block's columns
                    const int nn = (min(NT, R - n0) + 1) / 2;
                    const double* cv = V + static_cast<long long>(nd.cA) * R;
                    for (int e = threadIdx.x; e < static_cast<int>(nd.rank) * nn; e += 32 * kCW) {
                        const int i = e / nn, n = n0 + 2 * (e - i * nn);
                        double2 v = ldcg2(cv + static_cast<long long>(i) * R + n);
                        double* z = V + static_cast<long long>(sel[i]) * R + n;
                        if (second) {
                            const double2 o = ldcg2(z);
                            v.x += o.x;
                            v.y += o.y;
                        }
                        st2(z, v);
                    }
                    consumers_sync();  // the second node adds onto the same z cells
                }
                break;
            }
            default: {  // GK_ROOT_BWD
                const RootStripeDesc d = sl.sd[0];
                const int M = static_cast<int>(d.rank);
                double* out = V + static_cast<long long>(d.coff) * R;
                for (int m0 = 0; m0 < M; m0 += kMMax)
                    pass<true>(
                        m0, min(kMMax, M - m0), false, [&](int, int) { return make_double2(0.0, 0.0); },
                        [&](int row, int n, double2 v) { st2(out + static_cast<long long>(row) * R + n, v); });
                break;
            }
            }
            // publish: every consumer warp's stores of this item are done; the slot
            // (and its index lists) can take the item after next
            const std::uint32_t half = sl.half;
            consumers_sync();
            if (lane == 0) mbar_arrive(&c.iempty[j]);
            if (threadIdx.x == 0) {
                __threadfence();
                st_release(a.flags + static_cast<std::size_t>(item) * a.H + half, a.epoch);
            }
        }
    }
};

template <int NT>
__global__ void __maxnreg__(112) wgraph_kernel(const __grid_constant__ GraphArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    Ctrl& c = *reinterpret_cast<Ctrl*>(smem);
    double* stages = reinterpret_cast<double*>(smem + kCtrlBytes);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&c.full[s], 33);  // the streaming leader's expect_tx arrival + 32 cp.async arrivals
            mbar_init(&c.empty[s], kCW);
        }
        for (int j = 0; j < 2; ++j) {
            mbar_init(&c.ifull[j], 1);
            mbar_init(&c.iempty[j], kCW);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == kSchedWarp) {
        Scheduler sch{a, c, lane};
        sch.run();
    } else if (warp == kStreamWarp) {
        Streamer<NT> p{a, c, stages, lane};
        p.run();
    } else {
        Consumer<NT> k{a, c, stages, warp, lane, warp / Cfg<NT>::WN, warp % Cfg<NT>::WN};
        k.run();
    }
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
    auto go = [&](auto kern, int stage_doubles) -> cudaError_t {
        const std::size_t smem = kCtrlBytes + static_cast<std::size_t>(kStages) * stage_doubles * sizeof(double);
        cudaError_t e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        if (e2 != cudaSuccess) return e2;
        int dev = 0, sms = 0, per = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, kThreads, smem);
        const long long want = static_cast<long long>(g.n_items[k]) * H;
        const int grid = static_cast<int>(std::max(1LL, std::min<long long>(static_cast<long long>(sms) * std::max(1, per), want)));
        kern<<<grid, kThreads, smem, st>>>(a);
        return cudaGetLastError();
    };
    switch (nt) {
    case 8: return go(wgraph_kernel<8>, Cfg<8>::StageD);
    case 16: return go(wgraph_kernel<16>, Cfg<16>::StageD);
    case 32: return go(wgraph_kernel<32>, Cfg<32>::StageD);
    default: return go(wgraph_kernel<64>, Cfg<64>::StageD);
    }
}

}  // namespace bfb
