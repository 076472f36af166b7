// Order-sharded SHT over a group of processes, one GPU each, behind the C ABI
// (include/bfly_b200.h, bfly_shard_*).
//
// Orders m are independent, so rank r holds only the plans of a contiguous
// order range [mu_r, mu_{r+1}) (cut so every rank holds about the same dense
// Legendre storage) and a latitude slab of the grid.  The one exchange per
// direction is the m <-> theta transpose between the Legendre stage (local
// orders, all 2l colatitudes) and the phi DFT (all orders, the slab's rows):
//
//   synthesis:  beta --Legendre + parity combine--> order-side buffer
//               --grouped ncclSend / ncclRecv (alltoallv)--> slab-side buffer
//               --phi DFT of the slab rows--> grid slab
//   analysis:   the reverse.
//
// The batch runs as member chunks on two streams so the exchange of chunk c
// overlaps the Legendre stage of chunk c + 1 (synthesis) / the phi DFT of
// chunk c + 1 (analysis); two buffer sets alternate between chunks.  With one
// rank the order-side buffer is the slab-side buffer (no NCCL).
//
// NCCL is loaded at run time (dlopen "libnccl.so.2": the copy a PyTorch process
// already holds, else the system's), so the library has no link-time NCCL
// dependency; only the group calls below are used, which both installed NCCL
// versions (2.27, 2.28) provide.  The partition, slab and exchange-table rules
// are the ones of paper_0910_5435_b200/sharded.py (tested against each other).
#include <cuda_runtime.h>
#include <cufft.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "../../include/bfly_b200.h"
#include "phi.hpp"

namespace {

// ---- layout ------------------------------------------------------------------------
// Contiguous order ranges with near-equal dense Legendre words l (2l - mu) per
// order; every rank gets at least one order (sharded.py partition_orders).
std::vector<std::pair<int, int>> partition_orders(int l, int world) {
    const int n = 2 * l;
    std::vector<double> cum(static_cast<std::size_t>(n) + 1, 0.0);
    for (int mu = 0; mu < n; ++mu) cum[mu + 1] = cum[mu] + static_cast<double>(l) * (2.0 * l - mu);
    std::vector<int> cuts{0};
    for (int r = 1; r < world; ++r) {
        const double target = cum[n] * r / world;
        int c = static_cast<int>(std::lower_bound(cum.begin(), cum.end(), target) - cum.begin());
        if (c > 0 && std::fabs(cum[c - 1] - target) <= std::fabs(cum[std::min(c, n)] - target)) --c;
        const int lo = cuts.back() + (n - cuts.back() > world - r ? 1 : 0);
        const int hi = n - (world - r);
        cuts.push_back(std::min(std::max(c, lo), std::max(hi, lo)));
    }
    cuts.push_back(n);
    std::vector<std::pair<int, int>> out;
    for (int r = 0; r < world; ++r) out.emplace_back(cuts[r], cuts[r + 1]);
    return out;
}

std::vector<std::pair<int, int>> latitude_slabs(int l, int world) {
    const int rows = 2 * l, base = rows / world, extra = rows % world;
    std::vector<std::pair<int, int>> out;
    int t = 0;
    for (int r = 0; r < world; ++r) {
        const int n = base + (r < extra ? 1 : 0);
        out.emplace_back(t, t + n);
        t += n;
    }
    return out;
}

// phi bins of an order range: mu for +mu, N - mu for -mu (mu > 0)
std::vector<int> order_bins(int l, int mu0, int mu1) {
    const int N = 4 * l - 1;
    std::vector<int> b;
    for (int mu = mu0; mu < mu1; ++mu) b.push_back(mu);
    for (int mu = std::max(mu0, 1); mu < mu1; ++mu) b.push_back(N - mu);
    return b;
}

// Exchange tables for `batch` members (sharded.py exchange_tables): order-side
// buffer, peer j's block = [my bin][member][row of j's slab]; slab-side buffer,
// peer r's block = [r's bin][member][row of my slab].  Sizes in complex.
struct Tables {
    std::vector<std::int64_t> row_base, bin_off;
    std::vector<std::int32_t> row_T;
    std::vector<std::int64_t> osz, ssz, ooff, soff;
};
Tables exchange_tables(int l, int world, int me, const std::vector<std::pair<int, int>>& orders,
                       const std::vector<std::pair<int, int>>& slabs, int batch) {
    const int N = 4 * l - 1;
    Tables t;
    std::vector<std::int64_t> n(world), T(world);
    for (int r = 0; r < world; ++r) {
        n[r] = static_cast<std::int64_t>(order_bins(l, orders[r].first, orders[r].second).size());
        T[r] = slabs[r].second - slabs[r].first;
    }
    t.osz.resize(world);
    t.ssz.resize(world);
    t.ooff.resize(world);
    t.soff.resize(world);
    std::int64_t oo = 0, so = 0;
    for (int j = 0; j < world; ++j) {
        t.osz[j] = n[me] * batch * T[j];
        t.ssz[j] = n[j] * batch * T[me];
        t.ooff[j] = oo;
        t.soff[j] = so;
        oo += t.osz[j];
        so += t.ssz[j];
    }
    t.row_base.resize(2 * static_cast<std::size_t>(l));
    t.row_T.resize(2 * static_cast<std::size_t>(l));
    for (int j = 0; j < world; ++j)
        for (int r = slabs[j].first; r < slabs[j].second; ++r) {
            t.row_base[r] = t.ooff[j] + (r - slabs[j].first);
            t.row_T[r] = static_cast<std::int32_t>(T[j]);
        }
    t.bin_off.assign(static_cast<std::size_t>(N), 0);
    for (int r = 0; r < world; ++r) {
        const std::vector<int> bins = order_bins(l, orders[r].first, orders[r].second);
        for (std::size_t k = 0; k < bins.size(); ++k)
            t.bin_off[bins[k]] = t.soff[r] + static_cast<std::int64_t>(k) * batch * T[me];
    }
    return t;
}

// ---- NCCL (dlopen) --------------------------------------------------------------------
struct Nccl {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
Nccl& nccl() {
    static Nccl n = [] {
        Nccl x;
        x.h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!x.h) x.h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!x.h) return x;
        auto sym = [&](auto& f, const char* name) { f = reinterpret_cast<std::remove_reference_t<decltype(f)>>(dlsym(x.h, name)); };
        sym(x.GetUniqueId, "ncclGetUniqueId");
        sym(x.CommInitRank, "ncclCommInitRank");
        sym(x.CommDestroy, "ncclCommDestroy");
        sym(x.GroupStart, "ncclGroupStart");
        sym(x.GroupEnd, "ncclGroupEnd");
        sym(x.Send, "ncclSend");
        sym(x.Recv, "ncclRecv");
        sym(x.GetErrorString, "ncclGetErrorString");
        return x;
    }();
    if (!n.h || !n.CommInitRank || !n.Send || !n.Recv || !n.GroupStart || !n.GroupEnd)
        throw std::runtime_error("shard: cannot load NCCL (libnccl.so.2)");
    return n;
}
struct NcclError : std::runtime_error {
    using std::runtime_error::runtime_error;
};
void nck(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw NcclError(std::string(what) + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "NCCL error"));
}
void cck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}
void apick(int rc, const char* what) {
    if (rc != BFLY_OK) throw std::runtime_error(std::string(what) + ": " + bfly_last_error());
}

template <class T>
struct DBuf {
    T* p = nullptr;
    std::size_t n = 0;
    void ensure(std::size_t want) {
        if (want <= n) return;
        cudaFree(p);
        p = nullptr;
        n = 0;
        cck(cudaMalloc(&p, want * sizeof(T)), "cudaMalloc (shard)");
        n = want;
    }
    ~DBuf() { cudaFree(p); }
};

thread_local std::string g_shard_err;

}  // namespace

struct bfly_shard_s {
    int l = 0, N = 0, world = 1, rank = 0, device = 0;
    std::vector<std::pair<int, int>> orders, slabs;
    bfly_sht_t sht = nullptr;  // Legendre stage of the local orders (+ the shard kernels)
    bool fused_phi = false;    // in-kernel slab DFT (else cuFFT on contiguous slab rows)
    ncclComm_t comm = nullptr;
    cudaStream_t sc = nullptr, sx = nullptr;  // compute, exchange
    cudaEvent_t ev_in = nullptr, ev_out = nullptr, ev_packed[2] = {nullptr, nullptr}, ev_moved[2] = {nullptr, nullptr};
    struct DevTables {
        DBuf<std::int64_t> row_base, bin_off;
        DBuf<std::int32_t> row_T;
        Tables host;
    };
    std::map<int, std::unique_ptr<DevTables>> tabs;
    DBuf<double> obuf[2], sbuf[2], rows;  // order-side, slab-side, cuFFT rows (complex as 2 doubles)
    std::map<int, cufftHandle> fft;       // by chunk size
    int chunk_env = 0;

    int T() const { return slabs[rank].second - slabs[rank].first; }
    int n_local_bins() const { return static_cast<int>(order_bins(l, orders[rank].first, orders[rank].second).size()); }

    DevTables& tables(int bc) {
        auto it = tabs.find(bc);
        if (it != tabs.end()) return *it->second;
        auto t = std::make_unique<DevTables>();
        t->host = exchange_tables(l, world, rank, orders, slabs, bc);
        auto up = [&](auto& d, const auto& h) {
            d.ensure(h.size());
            cck(cudaMemcpy(d.p, h.data(), h.size() * sizeof(h[0]), cudaMemcpyHostToDevice), "cudaMemcpy (shard tables)");
        };
        up(t->row_base, t->host.row_base);
        up(t->row_T, t->host.row_T);
        up(t->bin_off, t->host.bin_off);
        DevTables& ref = *t;
        tabs.emplace(bc, std::move(t));
        return ref;
    }
    cufftHandle plan(int bc) {
        auto it = fft.find(bc);
        if (it != fft.end()) return it->second;
        cufftHandle h;
        int n = N;
        if (cufftPlanMany(&h, 1, &n, nullptr, 1, N, nullptr, 1, N, CUFFT_Z2Z, bc * T()) != CUFFT_SUCCESS)
            throw std::runtime_error("shard: cufftPlanMany failed");
        cufftSetStream(h, sc);
        fft.emplace(bc, h);
        return h;
    }
    // members per pipeline chunk: one chunk for one rank; otherwise >= 2 chunks when the batch allows (overlap),
    // whole 16-member chunks for large batches (the wave programs' 64 columns)
    int chunk(int batch) const {
        if (chunk_env > 0) return std::min(chunk_env, batch);
        if (world == 1) return batch;  // nothing to overlap
        if (batch >= 32) return 16;
        if (batch >= 4) return (batch + 1) / 2;
        return batch;
    }
    // the alltoallv of one chunk on sx: send blocks `snd` (offsets/sizes so, ss), receive `rcv` (ro, rs)
    void exchange(const double* snd, const std::vector<std::int64_t>& so, const std::vector<std::int64_t>& ss, double* rcv,
                  const std::vector<std::int64_t>& ro, const std::vector<std::int64_t>& rs) {
        Nccl& x = nccl();
        nck(x.GroupStart(), "ncclGroupStart");
        for (int j = 0; j < world; ++j) {
            if (ss[j]) nck(x.Send(snd + 2 * so[j], 2 * static_cast<size_t>(ss[j]), ncclFloat64, j, comm, sx), "ncclSend");
            if (rs[j]) nck(x.Recv(rcv + 2 * ro[j], 2 * static_cast<size_t>(rs[j]), ncclFloat64, j, comm, sx), "ncclRecv");
        }
        nck(x.GroupEnd(), "ncclGroupEnd");
    }
    ~bfly_shard_s() {
        for (auto& kv : fft) cufftDestroy(kv.second);
        for (cudaEvent_t e : {ev_in, ev_out, ev_packed[0], ev_packed[1], ev_moved[0], ev_moved[1]})
            if (e) cudaEventDestroy(e);
        if (sc) cudaStreamDestroy(sc);
        if (sx) cudaStreamDestroy(sx);
        if (comm && nccl().CommDestroy) nccl().CommDestroy(comm);
        if (sht) bfly_sht_destroy(sht);
    }
};

namespace {

template <class F>
int sguard(F&& f) {
    try {
        f();
        return BFLY_OK;
    } catch (const std::invalid_argument& e) {
        g_shard_err = e.what();
        return BFLY_EINVAL;
    } catch (const NcclError& e) {
        g_shard_err = e.what();
        return BFLY_ENCCL;
    } catch (const std::exception& e) {
        g_shard_err = e.what();
        return BFLY_ERUNTIME;
    }
}

void check(bfly_shard_t s) {
    if (!s) throw std::invalid_argument("shard: null handle");
}

}  // namespace

extern "C" {

const char* bfly_shard_last_error(void) { return g_shard_err.c_str(); }

int bfly_shard_layout(int l, int world, int64_t* orders, int64_t* slabs) {
    return sguard([&] {
        if (l < 1 || world < 1 || world > 2 * l) throw std::invalid_argument("shard: bad (l, world)");
        const auto o = partition_orders(l, world);
        const auto t = latitude_slabs(l, world);
        for (int r = 0; r < world; ++r) {
            if (orders) orders[2 * r] = o[r].first, orders[2 * r + 1] = o[r].second;
            if (slabs) slabs[2 * r] = t[r].first, slabs[2 * r + 1] = t[r].second;
        }
    });
}

int bfly_shard_tables(int l, int world, int rank, int batch, int64_t* row_base, int32_t* row_T, int64_t* bin_off,
                      int64_t* order_sizes, int64_t* slab_sizes) {
    return sguard([&] {
        if (l < 1 || world < 1 || world > 2 * l || rank < 0 || rank >= world || batch < 1)
            throw std::invalid_argument("shard: bad (l, world, rank, batch)");
        const Tables t = exchange_tables(l, world, rank, partition_orders(l, world), latitude_slabs(l, world), batch);
        if (row_base) std::copy(t.row_base.begin(), t.row_base.end(), row_base);
        if (row_T) std::copy(t.row_T.begin(), t.row_T.end(), row_T);
        if (bin_off) std::copy(t.bin_off.begin(), t.bin_off.end(), bin_off);
        if (order_sizes) std::copy(t.osz.begin(), t.osz.end(), order_sizes);
        if (slab_sizes) std::copy(t.ssz.begin(), t.ssz.end(), slab_sizes);
    });
}

int bfly_shard_nccl_id(void* id) {
    return sguard([&] {
        if (!id) throw std::invalid_argument("shard: null id");
        ncclUniqueId u;
        nck(nccl().GetUniqueId(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof u);
    });
}

int bfly_shard_create(int l, double eps, int block_width, int threads, int rank, int world, const void* nccl_id,
                      int device, bfly_shard_t* out) {
    return sguard([&] {
        if (!out) throw std::invalid_argument("shard: null output");
        if (l < 1 || world < 1 || world > 2 * l || rank < 0 || rank >= world)
            throw std::invalid_argument("shard: bad (l, world, rank)");
        if (world > 1 && !nccl_id) throw std::invalid_argument("shard: world > 1 needs an NCCL unique id");
        auto s = std::make_unique<bfly_shard_s>();
        s->l = l;
        s->N = 4 * l - 1;
        s->world = world;
        s->rank = rank;
        s->device = device;
        s->orders = partition_orders(l, world);
        s->slabs = latitude_slabs(l, world);
        if (const char* e = std::getenv("BFLY_SHARD_CHUNK")) s->chunk_env = std::max(0, static_cast<int>(std::strtol(e, nullptr, 10)));
        cck(cudaSetDevice(device), "cudaSetDevice");
        // this rank's plans only
        const int mu0 = s->orders[rank].first, mu1 = s->orders[rank].second;
        int np = 0;
        apick(bfly_glrow_planset_build(l, mu0, mu1, eps, block_width, threads, nullptr, 0, &np), "shard plan count");
        std::vector<bfly_plan_t> plans(static_cast<std::size_t>(np));
        apick(bfly_glrow_planset_build(l, mu0, mu1, eps, block_width, threads, plans.data(), np, &np), "shard plan build");
        const int rc = bfly_sht_create_range(l, mu0, mu1, plans.data(), np, nullptr, device, &s->sht);
        for (bfly_plan_t p : plans) bfly_plan_destroy(p);
        apick(rc, "shard range handle");
        int ok = 0;
        apick(bfly_sht_shard_supported(s->sht, &ok), "shard supported");
        s->fused_phi = ok != 0;
        if (world > 1) {
            ncclUniqueId u;
            std::memcpy(&u, nccl_id, sizeof u);
            nck(nccl().CommInitRank(&s->comm, world, u, rank), "ncclCommInitRank");
        }
        cck(cudaStreamCreateWithFlags(&s->sc, cudaStreamNonBlocking), "cudaStreamCreate");
        cck(cudaStreamCreateWithFlags(&s->sx, cudaStreamNonBlocking), "cudaStreamCreate");
        for (cudaEvent_t* e : {&s->ev_in, &s->ev_out, &s->ev_packed[0], &s->ev_packed[1], &s->ev_moved[0], &s->ev_moved[1]})
            cck(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
        *out = s.release();
    });
}

int bfly_shard_info(bfly_shard_t s, int64_t* info) {
    return sguard([&] {
        check(s);
        if (!info) throw std::invalid_argument("shard: null argument");
        info[0] = s->orders[s->rank].first;
        info[1] = s->orders[s->rank].second;
        info[2] = s->slabs[s->rank].first;
        info[3] = s->slabs[s->rank].second;
        info[4] = s->world;
        info[5] = s->rank;
        info[6] = s->fused_phi ? 1 : 0;
    });
}

int bfly_shard_sht(bfly_shard_t s, bfly_sht_t* sht) {
    return sguard([&] {
        check(s);
        if (!sht) throw std::invalid_argument("shard: null argument");
        *sht = s->sht;
    });
}

int bfly_shard_synthesize(bfly_shard_t s, const double* beta, double* grid, int batch, void* stream) {
    return sguard([&] {
        check(s);
        if (batch < 1) throw std::invalid_argument("shard: batch must be >= 1");
        cck(cudaSetDevice(s->device), "cudaSetDevice");
        const auto user = static_cast<cudaStream_t>(stream);
        const int bc = s->chunk(batch), T = s->T(), N = s->N, l = s->l;
        const std::int64_t ncoef = 4LL * l * l;
        const std::size_t osize = static_cast<std::size_t>(s->n_local_bins()) * bc * 2 * l;
        const std::size_t ssize = static_cast<std::size_t>(N) * bc * T;
        for (int k = 0; k < 2; ++k) {
            s->obuf[k].ensure(2 * osize);
            if (s->world > 1) s->sbuf[k].ensure(2 * ssize);
        }
        cck(cudaEventRecord(s->ev_in, user), "cudaEventRecord");
        cck(cudaStreamWaitEvent(s->sc, s->ev_in, 0), "cudaStreamWaitEvent");
        cck(cudaStreamWaitEvent(s->sx, s->ev_in, 0), "cudaStreamWaitEvent");
        const int nch = (batch + bc - 1) / bc;
        auto finish = [&](int c) {  // slab DFT of chunk c (after its exchange)
            const int b0 = c * bc, nb = std::min(bc, batch - b0), k = c & 1;
            auto& tb = s->tables(nb);
            const double* rcv = s->world > 1 ? s->sbuf[k].p : s->obuf[k].p;
            if (s->world > 1) cck(cudaStreamWaitEvent(s->sc, s->ev_moved[k], 0), "cudaStreamWaitEvent");
            double* g = grid + 2 * static_cast<std::int64_t>(b0) * T * N;
            if (s->fused_phi) {
                apick(bfly_sht_shard_phi(s->sht, 1, rcv, g, tb.bin_off.p, T, nb, s->sc), "shard phi");
            } else {
                cck(bfb::launch_shard_bins_rows(true, rcv, g, reinterpret_cast<const long long*>(tb.bin_off.p), N, T, nb,
                                                s->sc),
                    "shard bins to rows");
                cufftHandle h = s->plan(nb);
                if (cufftExecZ2Z(h, reinterpret_cast<cufftDoubleComplex*>(g), reinterpret_cast<cufftDoubleComplex*>(g),
                                 CUFFT_INVERSE) != CUFFT_SUCCESS)
                    throw std::runtime_error("shard: cufftExecZ2Z failed");
            }
        };
        for (int c = 0; c <= nch; ++c) {
            if (c < nch) {
                const int b0 = c * bc, nb = std::min(bc, batch - b0), k = c & 1;
                auto& tb = s->tables(nb);
                apick(bfly_sht_shard_synthesize(s->sht, beta + 2 * b0 * ncoef, s->obuf[k].p, tb.row_base.p, tb.row_T.p,
                                                nb, s->sc),
                      "shard synthesize");
                if (s->world > 1) {
                    cck(cudaEventRecord(s->ev_packed[k], s->sc), "cudaEventRecord");
                    cck(cudaStreamWaitEvent(s->sx, s->ev_packed[k], 0), "cudaStreamWaitEvent");
                    s->exchange(s->obuf[k].p, tb.host.ooff, tb.host.osz, s->sbuf[k].p, tb.host.soff, tb.host.ssz);
                    cck(cudaEventRecord(s->ev_moved[k], s->sx), "cudaEventRecord");
                }
            }
            if (c >= 1) finish(c - 1);
        }
        cck(cudaEventRecord(s->ev_out, s->sc), "cudaEventRecord");
        cck(cudaStreamWaitEvent(user, s->ev_out, 0), "cudaStreamWaitEvent");
    });
}

int bfly_shard_analyze(bfly_shard_t s, const double* grid, double* beta, int batch, void* stream) {
    return sguard([&] {
        check(s);
        if (batch < 1) throw std::invalid_argument("shard: batch must be >= 1");
        cck(cudaSetDevice(s->device), "cudaSetDevice");
        const auto user = static_cast<cudaStream_t>(stream);
        const int bc = s->chunk(batch), T = s->T(), N = s->N, l = s->l;
        const std::int64_t ncoef = 4LL * l * l;
        const std::size_t osize = static_cast<std::size_t>(s->n_local_bins()) * bc * 2 * l;
        const std::size_t ssize = static_cast<std::size_t>(N) * bc * T;
        for (int k = 0; k < 2; ++k) {
            s->sbuf[k].ensure(2 * ssize);
            if (s->world > 1) s->obuf[k].ensure(2 * osize);
        }
        if (!s->fused_phi) s->rows.ensure(2 * ssize);
        cck(cudaEventRecord(s->ev_in, user), "cudaEventRecord");
        cck(cudaStreamWaitEvent(s->sc, s->ev_in, 0), "cudaStreamWaitEvent");
        cck(cudaStreamWaitEvent(s->sx, s->ev_in, 0), "cudaStreamWaitEvent");
        const int nch = (batch + bc - 1) / bc;
        auto finish = [&](int c) {  // parity split + transposed Legendre stage of chunk c
            const int b0 = c * bc, nb = std::min(bc, batch - b0), k = c & 1;
            auto& tb = s->tables(nb);
            const double* rcv = s->world > 1 ? s->obuf[k].p : s->sbuf[k].p;
            if (s->world > 1) cck(cudaStreamWaitEvent(s->sc, s->ev_moved[k], 0), "cudaStreamWaitEvent");
            apick(bfly_sht_shard_analyze(s->sht, rcv, beta + 2 * b0 * ncoef, tb.row_base.p, tb.row_T.p, nb, s->sc),
                  "shard analyze");
        };
        for (int c = 0; c <= nch; ++c) {
            if (c < nch) {
                const int b0 = c * bc, nb = std::min(bc, batch - b0), k = c & 1;
                auto& tb = s->tables(nb);
                const double* g = grid + 2 * static_cast<std::int64_t>(b0) * T * N;
                if (s->fused_phi) {
                    apick(bfly_sht_shard_phi(s->sht, 0, g, s->sbuf[k].p, tb.bin_off.p, T, nb, s->sc), "shard phi");
                } else {
                    cufftHandle h = s->plan(nb);
                    if (cufftExecZ2Z(h, reinterpret_cast<cufftDoubleComplex*>(const_cast<double*>(g)),
                                     reinterpret_cast<cufftDoubleComplex*>(s->rows.p), CUFFT_FORWARD) != CUFFT_SUCCESS)
                        throw std::runtime_error("shard: cufftExecZ2Z failed");
                    cck(bfb::launch_shard_bins_rows(false, s->rows.p, s->sbuf[k].p,
                                                    reinterpret_cast<const long long*>(tb.bin_off.p), N, T, nb, s->sc),
                        "shard rows to bins");
                }
                if (s->world > 1) {
                    cck(cudaEventRecord(s->ev_packed[k], s->sc), "cudaEventRecord");
                    cck(cudaStreamWaitEvent(s->sx, s->ev_packed[k], 0), "cudaStreamWaitEvent");
                    s->exchange(s->sbuf[k].p, tb.host.soff, tb.host.ssz, s->obuf[k].p, tb.host.ooff, tb.host.osz);
                    cck(cudaEventRecord(s->ev_moved[k], s->sx), "cudaEventRecord");
                }
            }
            if (c >= 1) finish(c - 1);
        }
        cck(cudaEventRecord(s->ev_out, s->sc), "cudaEventRecord");
        cck(cudaStreamWaitEvent(user, s->ev_out, 0), "cudaStreamWaitEvent");
    });
}

void bfly_shard_destroy(bfly_shard_t s) { delete s; }

}  // extern "C"
