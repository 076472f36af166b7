// C ABI (include/bfly_b200.h): host plans, device plan sets, SHT handles.
//
// Every entry point converts C++ exceptions into the BFLY_E* codes that mirror
// the reference's exception types (std::invalid_argument, std::runtime_error,
// bfly::SerializationError) and keeps the message for bfly_last_error().
#include <cuda_runtime.h>
#include <cufft.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/bfly_b200.h"
#include "builder.hpp"
#include "gpubuild.hpp"
#include "engine.hpp"
#include "packer.hpp"
#include "plan.hpp"
#include "rootmv.hpp"
#include "waves_dev.hpp"
#include "wgraph_dev.hpp"
#include "phi.hpp"

namespace {

thread_local std::string g_err;

struct CudaFailure : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaFailure(std::string(what) + ": " + cudaGetErrorString(e));
}
void ckfft(cufftResult r, const char* what) {
    if (r != CUFFT_SUCCESS) throw CudaFailure(std::string(what) + ": cufft error " + std::to_string(static_cast<int>(r)));
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return BFLY_OK;
    } catch (const bfb::SerializationError& e) {
        g_err = e.what();
        return BFLY_ESERIAL;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return BFLY_EINVAL;
    } catch (const std::length_error& e) {
        g_err = e.what();
        return BFLY_EINVAL;
    } catch (const CudaFailure& e) {
        g_err = e.what();
        return BFLY_ECUDA;
    } catch (const std::runtime_error& e) {
        g_err = e.what();
        return BFLY_ERUNTIME;
    } catch (const std::exception& e) {
        g_err = e.what();
        return BFLY_EOTHER;
    }
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    std::size_t n = 0;
    void ensure(std::size_t count) {
        if (count <= n) return;
        if (p) cudaFree(p);
        p = nullptr;
        n = 0;
        ck(cudaMalloc(&p, count * sizeof(T)), "cudaMalloc");
        n = count;
    }
    ~DevBuf() {
        if (p) cudaFree(p);
    }
};

// Makes `dev` current for the scope and restores the caller's device after.
// Never throws: a failure surfaces at the next checked CUDA call.
struct DeviceScope {
    int prev = -1;
    explicit DeviceScope(int dev) {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            prev = -1;
            return;
        }
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceScope() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};

}  // namespace

struct bfly_plan_s {
    bfb::ButterflyPlan plan;
};

struct bfly_planset_s {
    int device = 0;
    int n_plans = 0;
    bfb::DeviceProgram prog;
    std::vector<std::uint64_t> rows_prefix, cols_prefix;  // host, length n_plans + 1
    std::uint64_t* d_rows_prefix = nullptr;
    std::uint64_t* d_cols_prefix = nullptr;
    DevBuf<double> h_in, h_out;  // staging for bfly_host_apply
    // Wave programs (waves.hpp) for many right-hand sides per call: every matrix
    // word read once per launch for all of them, FP64 tensor cores.
    bool wave = false;
    int wave_min_rhs = 16;  // l = 256 GL plan set: nrhs 8 engine 0.10 vs waves 0.14 ms, 16: 0.19 vs 0.18, 64: 0.70 vs 0.40
    bfb::DeviceWaveSet wv;
    bfb::DeviceGraph graph;
    DevBuf<double> vbuf, wbuf;  // V cells; stacked rows, cell-major
    ~bfly_planset_s() {
        cudaFree(d_rows_prefix);
        cudaFree(d_cols_prefix);
        bfb::free_program(prog);
        bfb::free_waves(wv);
        bfb::free_graph(graph);
    }
};

struct bfly_sht_s {
    int l = 0, N = 0, device = 0;
    int mu_begin = 0, mu_end = 0;
    int n_plans = 0;
    bool split = false;              // event / root programs (BFLY_SPLIT=1) or whole-chain jobs (default)
    bfb::DeviceProgram prog;         // whole-chain program (split = false) or the event program
    bfb::DeviceProgram roots;        // root program (split = true, engine roots)
    bfb::DeviceRootSet root_set;     // dedicated root kernels (split = true, default)
    bool engine_roots = false;
    bool merged = false;             // split programs merged into one launch (BFLY_ROOTS=merged)
    bool whole = false;              // prog is a whole-chain program
    bool wave = false;               // wv holds the level-synchronous batched programs (waves.hpp)
    int wave_min_batch = 2;          // with both: waves from this many functions per call on (finish_sht)
    bfb::DeviceWaveSet wv;
    bfb::DeviceGraph graph;          // wave programs as one dependency-ordered launch per direction (wgraph.hpp)
    DevBuf<double> vbuf;             // wave programs: V[cell][b][4]
    DevBuf<unsigned long long> dep[2];  // merged: per (plan, member) dependency words per direction
    unsigned long long epoch[2] = {0, 0};
    int dep_batch = 0;
    std::uint32_t c_cells = 0, y_rows = 0;
    std::uint32_t* d_plan_yoff = nullptr;
    std::uint32_t* d_plan_groups = nullptr;
    DevBuf<double> cbuf, ybuf;       // C and the root partials
    std::vector<double> nodes, rho;
    double* d_isr = nullptr;
    double* d_hsr = nullptr;
    std::map<int, std::pair<cufftHandle, cufftHandle>> fft;  // per batch: (synthesis, analysis)
    DevBuf<double> gbuf;             // phi-stage buffer, [bin][b][t] complex
    DevBuf<unsigned char> fftwork;   // one cuFFT work area shared by every cached plan
    std::size_t device_mem = 0;      // total device memory (batch chunking budget)
    DevBuf<double> ubuf;             // engine staging, u[plan][b][i][4]
    DevBuf<double> h_beta, h_grid;   // staging for the host-buffer API
    // host-buffer API pipeline: copy-in, compute and copy-out streams (created on
    // first use) so member chunks overlap H2D, the transform and D2H
    cudaStream_t hst[3] = {nullptr, nullptr, nullptr};
    std::vector<cudaEvent_t> hev;
    bfb::PhiPlan phi;                // fused phi stage (full order range, N's factors <= 127)
    bool time_engine = false;        // bfly_sht_engine_time: CUDA events around every engine launch
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> engine_ev[2];
    ~bfly_sht_s() {
        for (cudaStream_t x : hst)
            if (x) cudaStreamDestroy(x);
        for (cudaEvent_t e : hev) cudaEventDestroy(e);
        for (auto& v : engine_ev)
            for (auto& e : v) {
                cudaEventDestroy(e.first);
                cudaEventDestroy(e.second);
            }
        bfb::free_phi_plan(phi);
        if (prog.trace) cudaFree(prog.trace);
        prog.trace = nullptr;
        for (auto& kv : fft) {
            cufftDestroy(kv.second.first);
            cufftDestroy(kv.second.second);
        }
        cudaFree(d_isr);
        cudaFree(d_hsr);
        cudaFree(d_plan_yoff);
        cudaFree(d_plan_groups);
        bfb::free_program(prog);
        bfb::free_program(roots);
        bfb::free_roots(root_set);
        bfb::free_waves(wv);
        bfb::free_graph(graph);
    }
    std::int64_t coeffs() const { return 4LL * l * l; }
    std::int64_t grid_points() const { return 2LL * l * N; }
    // Batched length-N DFTs between the user grid [b][t][n] and the engine's
    // [bin][b][t] layout: batch index j = b * 2l + t, element stride B * 2l.
    std::pair<cufftHandle, cufftHandle> plans_for(int batch, cudaStream_t st) {
        auto it = fft.find(batch);
        if (it == fft.end()) {
            long long n = N;
            long long nembed = N;
            const long long rows = 2LL * l * batch;
            std::size_t w_syn = 0, w_ana = 0;
            cufftHandle syn, ana;
            ckfft(cufftCreate(&syn), "cufftCreate");
            ckfft(cufftSetAutoAllocation(syn, 0), "cufftSetAutoAllocation");
            ckfft(cufftMakePlanMany64(syn, 1, &n, &nembed, rows, 1, &nembed, 1, N, CUFFT_Z2Z, rows, &w_syn),
                  "cufftMakePlanMany64 (synthesis)");
            ckfft(cufftCreate(&ana), "cufftCreate");
            ckfft(cufftSetAutoAllocation(ana, 0), "cufftSetAutoAllocation");
            ckfft(cufftMakePlanMany64(ana, 1, &n, &nembed, 1, N, &nembed, rows, 1, CUFFT_Z2Z, rows, &w_ana),
                  "cufftMakePlanMany64 (analysis)");
            it = fft.emplace(batch, std::make_pair(syn, ana)).first;
            fftwork.ensure(std::max<std::size_t>({w_syn, w_ana, 16}));
        }
        // the work area may have been reallocated for a larger plan since
        ckfft(cufftSetWorkArea(it->second.first, fftwork.p), "cufftSetWorkArea");
        ckfft(cufftSetWorkArea(it->second.second, fftwork.p), "cufftSetWorkArea");
        ckfft(cufftSetStream(it->second.first, st), "cufftSetStream");
        ckfft(cufftSetStream(it->second.second, st), "cufftSetStream");
        return it->second;
    }
    double* phi_buffer(int batch) {
        gbuf.ensure(static_cast<std::size_t>(2 * grid_points() * batch));
        return gbuf.p;
    }
    double* u_buffer(int batch) {
        ubuf.ensure(static_cast<std::size_t>(n_plans) * batch * l * 4);
        return ubuf.p;
    }
};

namespace {

// Packs with the largest stage capacity (<= 16 KiB) that still lets
// kTargetCtas engine CTAs share an SM; BFLY_STAGE_KB overrides (tuning).
constexpr int kDefaultTargetCtas = 3;
constexpr std::uint32_t kSmemPerSm = 227u * 1024u;  // opt-in max per block on B200, also usable per SM

int target_ctas() {  // BFLY_TARGET_CTAS: tuning builds with other launch bounds
    if (const char* e = std::getenv("BFLY_TARGET_CTAS")) {
        const long v = std::strtol(e, nullptr, 10);
        if (v >= 1 && v <= 8) return static_cast<int>(v);
    }
    return kDefaultTargetCtas;
}

bfb::PackedProgram pack_for_engine(const std::vector<const bfb::ButterflyPlan*>& plans,
                                   const std::vector<std::vector<int>>& jobs, const std::vector<int>& mu,
                                   const std::vector<int>& par) {
    if (const char* e = std::getenv("BFLY_STAGE_KB")) {
        const long kb = std::strtol(e, nullptr, 10);
        if (kb >= 8 && kb <= 64)
            return bfb::pack_program(plans, jobs, mu, static_cast<std::uint32_t>(kb * 1024), par);
    }
    // Largest stage (ring slot) that still lets target_ctas() engine CTAs share
    // an SM next to their arenas (measured best at c2: 2 slots x ~24 KiB, 3
    // CTAs); when the arena is too large for that (large l), one CTA fewer.
    bfb::PackedProgram p = bfb::pack_program(plans, jobs, mu, 16384, par);
    bfb::DeviceProgram d;
    d.arena_cells = p.arena_cells;
    d.stage_capacity = 0;
    const std::size_t fixed = bfb::engine_smem_bytes(d) + 1024;  // + per-CTA reservation
    std::uint32_t fit = 0;
    for (int ctas = target_ctas(); ctas >= 1; --ctas) {
        const std::size_t per_cta = kSmemPerSm / static_cast<std::size_t>(ctas);
        fit = per_cta > fixed ? static_cast<std::uint32_t>((per_cta - fixed) / bfb::kRingStages) & ~1023u : 0u;
        if (fit >= 16384) break;
    }
    fit = std::min<std::uint32_t>(std::max<std::uint32_t>(fit, bfb::kStageBytesMin), bfb::kStageBytesMax);
    if (fit != 16384) p = bfb::pack_program(plans, jobs, mu, fit, par);
    return p;
}

std::uint32_t fit_capacity(std::uint32_t arena_cells) {
    bfb::DeviceProgram d;
    d.arena_cells = arena_cells;
    d.stage_capacity = 0;
    const std::size_t fixed = bfb::engine_smem_bytes(d) + 1024;
    const std::size_t per_cta = kSmemPerSm / target_ctas();
    std::uint32_t cap = 16384;
    if (fixed + bfb::kRingStages * cap > per_cta) {
        cap = per_cta > fixed ? static_cast<std::uint32_t>((per_cta - fixed) / bfb::kRingStages) & ~1023u : 0u;
        cap = std::max<std::uint32_t>(cap, bfb::kStageBytesMin);
    }
    return cap;
}

bfb::SplitProgram pack_split_for_engine(const std::vector<const bfb::ButterflyPlan*>& plans,
                                        const std::vector<int>& mu, const std::vector<int>& par) {
    if (const char* e = std::getenv("BFLY_STAGE_KB")) {
        const long kb = std::strtol(e, nullptr, 10);
        if (kb >= 8 && kb <= 64) {
            const std::uint32_t cap = static_cast<std::uint32_t>(kb * 1024);
            return bfb::pack_split(plans, mu, par, cap, cap);
        }
    }
    bfb::SplitProgram sp = bfb::pack_split(plans, mu, par, 16384, 16384);
    const std::uint32_t ce = fit_capacity(sp.events.arena_cells), cr = fit_capacity(sp.roots.arena_cells);
    if (ce < 16384 || cr < 16384) sp = bfb::pack_split(plans, mu, par, ce, cr);
    return sp;
}

void check_plan_handle(const void* h) {
    if (!h) throw std::invalid_argument("null handle");
}

std::vector<const bfb::ButterflyPlan*> plan_ptrs(const bfly_plan_t* plans, int n) {
    if (n < 1 || !plans) throw std::invalid_argument("plan set: need at least one plan");
    std::vector<const bfb::ButterflyPlan*> v;
    for (int i = 0; i < n; ++i) {
        check_plan_handle(plans[i]);
        plans[i]->plan.validate();
        v.push_back(&plans[i]->plan);
    }
    return v;
}

// SHT jobs: one per order mu, holding its even and (if non-empty) odd plan.
// Per-colatitude scale factors and the fused phi plan (after the program is set).
void finish_sht(bfly_sht_s& s) {
    const int l = s.l;
    // measured crossovers (whole-chain engine vs waves, pairs/s): l = 256, B = 4:
    // 8.6k vs 9.9k, B = 16: 9.2k vs 17.5k; l = 1024, B = 1: 210 vs 131, B = 2: 215 vs 244
    s.wave_min_batch = l >= 512 ? 2 : 4;
    if (const char* e = std::getenv("BFLY_WAVE_MIN_BATCH"))
        s.wave_min_batch = std::max(1, static_cast<int>(std::strtol(e, nullptr, 10)));
    const char* pe = std::getenv("BFLY_PHI");  // "cufft": the unfused path (comparisons)
    // (order ranges need it too: the sharded transform's slab-side DFT rows)
    if (!(pe && std::string(pe) == "cufft")) s.phi = bfb::make_phi_plan(s.N);
    std::vector<double> isr(static_cast<std::size_t>(l)), hsr(static_cast<std::size_t>(l));
    for (int i = 0; i < l; ++i) {
        const double sr = std::sqrt(s.rho[static_cast<std::size_t>(i)]);
        isr[static_cast<std::size_t>(i)] = 1.0 / sr;
        hsr[static_cast<std::size_t>(i)] = sr / (2.0 * s.N);
    }
    ck(cudaMalloc(&s.d_isr, sizeof(double) * l), "cudaMalloc");
    ck(cudaMalloc(&s.d_hsr, sizeof(double) * l), "cudaMalloc");
    ck(cudaMemcpy(s.d_isr, isr.data(), sizeof(double) * l, cudaMemcpyHostToDevice), "cudaMemcpy");
    ck(cudaMemcpy(s.d_hsr, hsr.data(), sizeof(double) * l, cudaMemcpyHostToDevice), "cudaMemcpy");
}

// Per plan: first root-partial row and number of root groups (split / wave programs).
void upload_plan_rows(bfly_sht_s& s, const std::vector<std::uint32_t>& yoff, const std::vector<std::uint32_t>& groups) {
    const std::size_t np = yoff.size();
    ck(cudaMalloc(&s.d_plan_yoff, sizeof(std::uint32_t) * np), "cudaMalloc");
    ck(cudaMalloc(&s.d_plan_groups, sizeof(std::uint32_t) * np), "cudaMalloc");
    ck(cudaMemcpy(s.d_plan_yoff, yoff.data(), sizeof(std::uint32_t) * np, cudaMemcpyHostToDevice), "cudaMemcpy");
    ck(cudaMemcpy(s.d_plan_groups, groups.data(), sizeof(std::uint32_t) * np, cudaMemcpyHostToDevice), "cudaMemcpy");
}

// The graph program of a wave set (wgraph.hpp), which executes it.
// BFLY_GRAPH_GROUP: nodes per plan group of the queue.
bfb::DeviceGraph make_graph(const bfb::WaveSet& w) {
    std::uint32_t group = 65536;
    if (const char* e = std::getenv("BFLY_GRAPH_GROUP"))
        group = static_cast<std::uint32_t>(std::max(1L, std::strtol(e, nullptr, 10)));
    bool wavefront = false;  // BFLY_GRAPH_WAVEFRONT=1: diagonal order over small groups (wgraph.hpp)
    if (const char* e = std::getenv("BFLY_GRAPH_WAVEFRONT")) wavefront = std::strtol(e, nullptr, 10) != 0;
    return bfb::upload_graph(bfb::build_graph(w, group, wavefront));
}

void make_sht(bfly_sht_s& s, int l, int mu_begin, int mu_end, const std::vector<const bfb::ButterflyPlan*>& plans,
              const double* rho, int device, const double* nodes = nullptr) {
    if (l < 1) throw std::invalid_argument("sht: l must be >= 1");
    if (mu_begin < 0 || mu_end > 2 * l || mu_begin >= mu_end) throw std::invalid_argument("sht: bad order range");
    s.l = l;
    s.N = 4 * l - 1;
    s.device = device;
    s.mu_begin = mu_begin;
    s.mu_end = mu_end;
    std::vector<std::vector<int>> job_plans;
    std::vector<int> job_mu, job_par;
    int idx = 0;
    for (int mu = mu_begin; mu < mu_end; ++mu) {
        for (int p = 0; p < 2; ++p) {
            const std::int64_t nc = bfb::chain_cols(l, mu, p);
            if (nc == 0) continue;
            if (idx >= static_cast<int>(plans.size()))
                throw std::invalid_argument("sht: fewer plans than non-empty chains");
            const bfb::ButterflyPlan& pl = *plans[static_cast<std::size_t>(idx)];
            if (pl.n_rows != static_cast<std::uint64_t>(l) || pl.n_cols != static_cast<std::uint64_t>(nc))
                throw std::invalid_argument("sht: plan " + std::to_string(idx) + " has shape " +
                                            std::to_string(pl.n_rows) + "x" + std::to_string(pl.n_cols) +
                                            ", expected " + std::to_string(l) + "x" + std::to_string(nc) +
                                            " for (mu=" + std::to_string(mu) + ", parity=" + std::to_string(p) + ")");
            job_plans.push_back({idx++});  // one degree chain per job
            job_mu.push_back(mu);
            job_par.push_back(p);
        }
    }
    if (idx != static_cast<int>(plans.size())) throw std::invalid_argument("sht: more plans than non-empty chains");
    s.n_plans = idx;
    const bfb::GlRule rule = (rho && nodes) ? bfb::GlRule{} : bfb::gauss_legendre_positive(l);
    s.nodes = nodes ? std::vector<double>(nodes, nodes + l) : rule.nodes;
    s.rho = rho ? std::vector<double>(rho, rho + l) : rule.rho;
    DeviceScope ds(device);
    // Programs: level-synchronous wave programs (waves.hpp; every matrix word
    // read once per launch for the whole batch, FP64 tensor cores) from l = 128
    // on — batches of functions — next to the whole-chain engine
    // program (one function's four right-hand sides in shared memory; faster
    // for small batches), which is dropped where it stops fitting shared memory.
    // Each call takes the waves from wave_min_batch functions on (use_waves).
    // BFLY_WAVES=0: whole-chain (or split) only; 1: waves only; 2: both.
    int wmode = l >= 128 ? 2 : 0;
    if (const char* e = std::getenv("BFLY_WAVES")) wmode = static_cast<int>(std::strtol(e, nullptr, 10));
    if (wmode != 0) {
        const bool verbose = std::getenv("BFLY_BUILD_VERBOSE") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        const bfb::WaveSet w = bfb::build_waves(plans, job_mu, job_par);
        const auto t1 = std::chrono::steady_clock::now();
        s.wave = true;
        s.wv = bfb::upload_waves(w);
        const auto t2 = std::chrono::steady_clock::now();
        s.graph = make_graph(w);
        if (verbose) {
            const auto t3 = std::chrono::steady_clock::now();
            auto sec = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
            std::fprintf(stderr, "sht programs: l=%d wave compile + tiling %.2f s, upload %.2f s (%.1f GB), graph queue %.2f s\n", l,
                         sec(t0, t1), sec(t1, t2), 8e-9 * static_cast<double>(w.T.size() + w.roots.data.size()), sec(t2, t3));
        }
        s.prog.stored_words = w.event_words + w.root_words;
        s.prog.fetched_bytes = 8 * (w.T.size() + w.roots.data.size());
        if (wmode == 1) {
            finish_sht(s);
            return;
        }
    }
    if (const char* e = std::getenv("BFLY_SPLIT")) s.split = std::strtol(e, nullptr, 10) != 0;
    bfb::PackedProgram whole;
    if (!s.split) {
        // Whole-chain jobs keep a chain's rows (l cells) and its root blocks in
        // the CTA's arena (~3.2 l cells).  When that leaves less than 16 KiB
        // stages even at one CTA per SM (l ~ 2048: measured 79 ms vs 59 ms per
        // pair) or does not fit at all, the split programs (root vectors through
        // global memory) take over.
        if (s.wave && !std::getenv("BFLY_STAGE_KB")) {
            // The whole-chain arena holds at least 3.2 l cells (measured 3.2-3.4 l): where even that
            // leaves no 16 KiB stages at one CTA per SM (l ~ 1940 on), do not pack the program (two
            // passes over every matrix word, 41 GB and 110 s at l = 2048) just to drop it.
            bfb::DeviceProgram d0;
            d0.arena_cells = static_cast<std::uint32_t>(3.2 * l);
            d0.stage_capacity = 0;
            const std::size_t fixed0 = bfb::engine_smem_bytes(d0) + 1024;
            if (fixed0 + bfb::kRingStages * 16384u > kSmemPerSm) {
                finish_sht(s);
                return;
            }
        }
        whole = pack_for_engine(plans, job_plans, job_mu, job_par);
        bfb::DeviceProgram d;
        d.arena_cells = whole.arena_cells;
        d.stage_capacity = whole.stage_capacity;
        int max_smem = 0;
        ck(cudaDeviceGetAttribute(&max_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, device), "cudaDeviceGetAttribute");
        if (whole.stage_capacity < 16384 || bfb::engine_smem_bytes(d) > static_cast<std::size_t>(max_smem)) {
            whole = bfb::PackedProgram{};
            if (s.wave) {  // the wave programs serve every batch
                finish_sht(s);
                return;
            }
            s.split = true;
        }
    }
    if (s.split) {
        const bfb::SplitProgram sp = pack_split_for_engine(plans, job_mu, job_par);
        s.prog = bfb::upload_program(sp.events, device);
        if (const char* e = std::getenv("BFLY_ROOTS")) {
            s.engine_roots = std::string(e) == "engine";
            s.merged = std::string(e) == "merged";
        }
        if (s.merged) {
            bfb::free_program(s.prog);
            s.prog = bfb::upload_program(bfb::merge_split(sp, plans.size()), device);
        } else if (s.engine_roots) {
            s.roots = bfb::upload_program(sp.roots, device);
        } else {
            // tensor-core root kernels (all right-hand sides per skeleton read)
            // unless BFLY_ROOTS=rootmv asks for the per-member matrix-vector ones
            const char* e = std::getenv("BFLY_ROOTS");
            s.root_set = bfb::upload_roots(sp.root_set, !(e && std::string(e) == "rootmv"));
        }
        s.prog.stored_words = sp.events.stored_words + sp.roots.stored_words;
        s.prog.fetched_bytes = sp.events.fetched_bytes + sp.roots.fetched_bytes;
        s.c_cells = sp.c_cells;
        s.y_rows = sp.y_rows;
        upload_plan_rows(s, sp.plan_yoff, sp.plan_groups);
    } else {
        s.prog = bfb::upload_program(whole, device);
        s.whole = true;
    }
    finish_sht(s);
}

// Engine launch with optional event timing on the launching stream.
template <class F>
void timed_engine(bfly_sht_s& s, bool transpose, cudaStream_t st, F&& launch) {
    if (!s.time_engine) {
        launch();
        return;
    }
    cudaEvent_t a, b;
    ck(cudaEventCreate(&a), "cudaEventCreate");
    ck(cudaEventCreate(&b), "cudaEventCreate");
    ck(cudaEventRecord(a, st), "cudaEventRecord");
    launch();
    ck(cudaEventRecord(b, st), "cudaEventRecord");
    s.engine_ev[transpose].emplace_back(a, b);
}

bfb::ShtIO sht_io(const bfly_sht_s& s) {
    bfb::ShtIO io;
    io.isr = s.d_isr;
    io.hsr = s.d_hsr;
    io.l = s.l;
    io.N = s.N;
    io.beta_stride = 2 * s.coeffs();
    return io;
}

void check_batch(int batch) {
    if (batch < 1) throw std::invalid_argument("sht: batch must be >= 1");
}

void split_buffers(bfly_sht_s& s, bfb::ShtIO& io, int batch) {
    s.cbuf.ensure(static_cast<std::size_t>(s.c_cells) * batch * 4 + 4);
    s.ybuf.ensure(static_cast<std::size_t>(s.y_rows) * batch * 4 + 4);
    io.c = s.cbuf.p;
    io.ypart = s.ybuf.p;
    io.c_cells = s.c_cells;
    io.y_rows = s.y_rows;
    io.plan_yoff = s.d_plan_yoff;
    io.plan_groups = s.d_plan_groups;
    io.cell_major = s.root_set.mma ? 1 : 0;
}

// Dependency words of the merged program for one direction: zeroed whenever
// the batch (and so the word layout) changes, then reused with a rising epoch.
void merged_deps(bfly_sht_s& s, bfb::ShtIO& io, int batch, bool transpose, cudaStream_t st) {
    const std::size_t words = static_cast<std::size_t>(s.n_plans) * batch;
    if (s.dep_batch != batch) {
        for (int d = 0; d < 2; ++d) {
            s.dep[d].ensure(words);
            ck(cudaMemsetAsync(s.dep[d].p, 0, words * sizeof(unsigned long long), st), "cudaMemsetAsync");
            s.epoch[d] = 0;
        }
        s.dep_batch = batch;
    }
    io.dep = s.dep[transpose].p;
    io.plan_roots = s.prog.plan_roots;
    io.epoch = ++s.epoch[transpose];
}

cudaError_t launch_root_set(const bfly_sht_s& s, const bfb::ShtIO& io, bool transpose, cudaStream_t st);

bfb::RootArgs root_args(const bfly_sht_s& s, const bfb::ShtIO& io, bool transpose) {
    bfb::RootArgs a;
    a.data = s.root_set.data;
    a.stripes = s.root_set.stripes;
    a.items = transpose ? s.root_set.bwd_items : s.root_set.fwd_items;
    a.n_items = transpose ? s.root_set.n_bwd : s.root_set.n_fwd;
    a.C = io.c;
    a.ypart = io.ypart;
    a.u = io.u;
    a.c_cells = io.c_cells;
    a.y_rows = io.y_rows;
    a.l = io.l;
    a.batch = io.batch;
    return a;
}

cudaError_t launch_root_set(const bfly_sht_s& s, const bfb::ShtIO& io, bool transpose, cudaStream_t st) {
    if (!s.root_set.mma) return bfb::launch_roots(root_args(s, io, transpose), transpose, st);
    bfb::RootMmaArgs a;
    a.data = s.root_set.data;
    a.stripes = s.root_set.stripes;
    a.fwd_items = s.root_set.mma_fwd;
    a.bwd_items = s.root_set.mma_bwd;
    a.n_fwd = s.root_set.n_mma_fwd;
    a.n_bwd = s.root_set.n_mma_bwd;
    a.C = io.c;
    a.ypart = io.ypart;
    a.u = io.u;
    a.l = io.l;
    a.batch = io.batch;
    return bfb::launch_roots_mma(a, transpose, st);
}

// Which program serves a call of `batch` functions (c3, l = 1024: the whole-chain
// engine streams the plans once per function, 4.8 ms per pair; the waves cost
// ~17 ms + ~1 ms per function).
bool use_waves(const bfly_sht_s& s, int batch) {
    if (!s.wave) return false;
    if (!s.whole) return true;
    return batch >= s.wave_min_batch;
}

// Wave programs, one direction of the Legendre stage for all members at once.
// Synthesis: beta -> V input cells, levels 1..L, roots -> chain rows u.
// Analysis: u -> roots^T -> levels L..1 -> beta.
void wave_legendre(bfly_sht_s& s, bfb::ShtIO& io, int batch, bool transpose, cudaStream_t st) {
    const bfb::DeviceWaveSet& w = s.wv;
    s.vbuf.ensure(static_cast<std::size_t>(w.v_cells) * batch * 4 + 4);
    bfb::WaveArgs a = bfb::wave_args(w, s.vbuf.p, s.l, batch, io.beta_stride);
    if (io.real_per_task > 0) a.real_members = io.real_members;  // batch = pairs of fields
    if (!transpose) {
        ck(bfb::launch_wave_gather(w, a, io.beta_in, st), "wave gather");
        ck(bfb::launch_graph(s.graph, w, s.vbuf.p, io.u, s.l, batch, false, st), "graph launch (synthesis)");
    } else {
        ck(bfb::launch_graph(s.graph, w, s.vbuf.p, io.u, s.l, batch, true, st), "graph launch (analysis)");
        ck(bfb::launch_wave_scatter(w, a, io.beta_out, st), "wave scatter");
    }
}

// Legendre stage between the coefficients and the chain rows u (the fused phi
// kernels' and the shard exchange's operand): wave programs or the engine.
void legendre_u(bfly_sht_s& s, bfb::ShtIO& io, int batch, bool transpose, cudaStream_t st, bool pdl) {
    if (use_waves(s, batch))
        wave_legendre(s, io, batch, transpose, st);
    else
        ck(bfb::launch_sht(s.prog, transpose, io, batch, st, pdl),
           transpose ? "engine launch (analysis)" : "engine launch (synthesis)");
}

void legendre_synth(bfly_sht_s& s, const double* beta, double* gbins, int batch, cudaStream_t st) {
    bfb::ShtIO io = sht_io(s);
    io.beta_in = beta;
    io.g_out = gbins;
    io.u = s.u_buffer(batch);
    io.batch = batch;
    if (use_waves(s, batch)) {
        timed_engine(s, false, st, [&] { wave_legendre(s, io, batch, false, st); });
    } else if (s.split) {
        split_buffers(s, io, batch);
        if (s.merged) {
            merged_deps(s, io, batch, false, st);
            ck(bfb::launch_sht_merged(s.prog, false, io, batch, st), "engine launch (synthesis, merged)");
        } else {
            ck(bfb::launch_sht_events(s.prog, false, io, batch, st), "engine launch (synthesis events)");
            if (s.engine_roots)
                ck(bfb::launch_sht_roots(s.roots, false, io, batch, st), "engine launch (synthesis roots)");
            else
                ck(launch_root_set(s, io, false, st), "root kernel (synthesis)");
        }
    } else {
        timed_engine(s, false, st, [&] { ck(bfb::launch_sht(s.prog, false, io, batch, st), "engine launch (synthesis)"); });
    }
    ck(bfb::launch_sht_combine(io, s.mu_begin, s.mu_end, st), "parity combine");
}

void legendre_anal(bfly_sht_s& s, const double* gdft, double* beta, int batch, cudaStream_t st) {
    bfb::ShtIO io = sht_io(s);
    io.g_in = gdft;
    io.beta_out = beta;
    io.u = s.u_buffer(batch);
    io.batch = batch;
    ck(bfb::launch_sht_split(io, s.mu_begin, s.mu_end, st), "parity split");
    if (use_waves(s, batch)) {
        timed_engine(s, true, st, [&] { wave_legendre(s, io, batch, true, st); });
    } else if (s.split) {
        split_buffers(s, io, batch);
        if (s.merged) {
            merged_deps(s, io, batch, true, st);
            ck(bfb::launch_sht_merged(s.prog, true, io, batch, st), "engine launch (analysis, merged)");
        } else {
            if (s.engine_roots)
                ck(bfb::launch_sht_roots(s.roots, true, io, batch, st), "engine launch (analysis roots)");
            else
                ck(launch_root_set(s, io, true, st), "root kernel (analysis)");
            ck(bfb::launch_sht_events(s.prog, true, io, batch, st), "engine launch (analysis events)");
        }
    } else {
        timed_engine(s, true, st, [&] { ck(bfb::launch_sht(s.prog, true, io, batch, st), "engine launch (analysis)"); });
    }
}

// Full transforms.  Default (whole-chain program, fused phi plan available):
// engine -> fused combine + inverse DFT, and fused DFT + split -> engine, with
// the weighted chain values u as the only intermediate.  Otherwise the
// Legendre stage writes the [bin][b][t] buffer and cuFFT does the DFTs.
bool fused_phi(const bfly_sht_s& s) { return (s.phi.ok || s.phi.rader) && !s.split; }
// The real-field kernels and the sharded slab DFT exist for the Stockham plans only.
bool fused_phi_stockham(const bfly_sht_s& s) { return s.phi.ok && !s.split; }

// The order-side steps (Legendre stage + parity combine / split into the
// exchange layout) need whole-chain or wave programs; the fused slab DFT also
// the in-kernel phi plan.
void check_shard_orders(const bfly_sht_s& s) {
    if (s.split) throw std::invalid_argument("sht shard: needs whole-chain or wave programs");
}
void check_shard(const bfly_sht_s& s) {
    if (s.split || !s.phi.ok)
        throw std::invalid_argument("sht shard: needs whole-chain or wave programs and the fused phi stage");
}

// Batch chunking of the full transforms: the scratch (u, and on the stage-wise
// path the bin buffer, cuFFT work area and split-program partials) grows with
// the batch, the user's beta [b][4l^2] and grid [b][2l][N] are member-major,
// so large batches (c4: l = 2048, B = 64) run as consecutive member chunks
// whose scratch fits BFLY_SCRATCH_GB (default: a quarter of device memory).
// Every member streams the plans once either way (R = 4 per task).
int batch_chunk(bfly_sht_s& s, int batch) {
    double per = 32.0 * s.n_plans * s.l;  // u
    if (!fused_phi(s)) per += 2.0 * 16.0 * s.grid_points();  // bins + cuFFT work area
    if (s.split) per += 32.0 * (static_cast<double>(s.c_cells) + s.y_rows);
    const bool waves = use_waves(s, batch);
    if (waves) per += 32.0 * static_cast<double>(s.wv.v_cells);
    double budget = 0;
    if (const char* e = std::getenv("BFLY_SCRATCH_GB")) budget = std::strtod(e, nullptr) * 1e9;
    if (budget <= 0) {
        if (s.device_mem == 0) {  // queried once per handle: cudaMemGetInfo costs tens of microseconds
            std::size_t fr = 0, tot = 0;
            s.device_mem = cudaMemGetInfo(&fr, &tot) == cudaSuccess ? tot : static_cast<std::size_t>(64e9);
        }
        budget = 0.25 * static_cast<double>(s.device_mem);
    }
    double c = std::floor(budget / per);
    if (c >= batch) return batch;
    if (waves && c >= 16) return 16 * static_cast<int>(c / 16);  // whole 64-column chunks (R = 4B)
    // equal chunks: no small tail chunk (for the waves a lone member costs
    // about as much as sixteen)
    const int cmax = std::max(1, static_cast<int>(c));
    const int n = (batch + cmax - 1) / cmax;
    return (batch + n - 1) / n;
}

void sht_synth_chunk(bfly_sht_s& s, const double* beta, double* grid, int batch, cudaStream_t st);
void sht_anal_chunk(bfly_sht_s& s, const double* grid, double* beta, int batch, cudaStream_t st);

void sht_synth(bfly_sht_s& s, const double* beta, double* grid, int batch, cudaStream_t st) {
    const int bc = batch_chunk(s, batch);
    for (int b0 = 0; b0 < batch; b0 += bc)
        sht_synth_chunk(s, beta + 2 * s.coeffs() * b0, grid + 2 * s.grid_points() * b0, std::min(bc, batch - b0), st);
}

void sht_anal(bfly_sht_s& s, const double* grid, double* beta, int batch, cudaStream_t st) {
    const int bc = batch_chunk(s, batch);
    for (int b0 = 0; b0 < batch; b0 += bc)
        sht_anal_chunk(s, grid + 2 * s.grid_points() * b0, beta + 2 * s.coeffs() * b0, std::min(bc, batch - b0), st);
}

void sht_synth_chunk(bfly_sht_s& s, const double* beta, double* grid, int batch, cudaStream_t st) {
    if (fused_phi(s)) {
        bfb::ShtIO io = sht_io(s);
        io.beta_in = beta;
        io.u = s.u_buffer(batch);
        io.batch = batch;
        // programmatic dependent of whatever precedes on the stream: the
        // producers stream the (read-only) plan while it finishes; consumers
        // wait for it before touching the coefficients
        timed_engine(s, false, st, [&] {
            legendre_u(s, io, batch, false, st, !s.time_engine);
        });
        ck(bfb::launch_phi_synth_fused(s.phi, io, grid, st), "phi synthesis");
        return;
    }
    double* gb = s.phi_buffer(batch);
    legendre_synth(s, beta, gb, batch, st);
    ckfft(cufftExecZ2Z(s.plans_for(batch, st).first, reinterpret_cast<cufftDoubleComplex*>(gb),
                       reinterpret_cast<cufftDoubleComplex*>(grid), CUFFT_INVERSE),
          "cufftExecZ2Z");
}

void sht_anal_chunk(bfly_sht_s& s, const double* grid, double* beta, int batch, cudaStream_t st) {
    if (fused_phi(s)) {
        bfb::ShtIO io = sht_io(s);
        io.beta_out = beta;
        io.u = s.u_buffer(batch);
        io.batch = batch;
        ck(bfb::launch_phi_anal_fused(s.phi, io, grid, st), "phi analysis");
        // programmatic dependent: the engine's producers stream plan stages
        // while the phi kernel finishes (not with event timing, which would
        // sit between the two launches)
        timed_engine(s, true, st, [&] {
            legendre_u(s, io, batch, true, st, !s.time_engine);
        });
        return;
    }
    double* gb = s.phi_buffer(batch);
    ckfft(cufftExecZ2Z(s.plans_for(batch, st).second, reinterpret_cast<cufftDoubleComplex*>(const_cast<double*>(grid)),
                       reinterpret_cast<cufftDoubleComplex*>(gb), CUFFT_FORWARD),
          "cufftExecZ2Z");
    legendre_anal(s, gb, beta, batch, st);
}

void full_range(const bfly_sht_s& s) {
    if (s.mu_begin != 0 || s.mu_end != 2 * s.l)
        throw std::invalid_argument("sht: a partial order range has no phi stage; use the legendre_* entry points");
}

}  // namespace

// ---- device-ready program cache ("BFLYSHT1") -------------------------------
// The packed device program of a whole-chain SHT, byte for byte, plus what
// make_sht derived from the plans: loading skips the
// host plan build and the packer.  Little-endian, all counts u64 unless noted.
namespace {
constexpr char kShtMagic[8] = {'B', 'F', 'L', 'Y', 'S', 'H', 'T', '1'};
struct ShtFileHeader {
    char magic[8];
    std::uint32_t version, l, mu_begin, mu_end, n_plans, arena_cells, zo_cells, stage_capacity, chunk_rows, pad;
    std::uint64_t stored_words, fetched_bytes, n_stages, n_jobs, stream_bytes;
};
template <class T>
void dev_to_file(std::FILE* f, const T* d, std::size_t n) {
    std::vector<T> h(n);
    if (n) ck(cudaMemcpy(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
    if (n && std::fwrite(h.data(), sizeof(T), n, f) != n) throw std::runtime_error("sht save: write failed");
}
template <class T>
std::vector<T> from_file(std::FILE* f, std::size_t n) {
    std::vector<T> h(n);
    if (n && std::fread(h.data(), sizeof(T), n, f) != n) throw std::runtime_error("sht load: truncated file");
    return h;
}
struct FileCloser {
    std::FILE* f;
    ~FileCloser() {
        if (f) std::fclose(f);
    }
};
// Wave programs in the program cache: header version 2, then rho, nodes, the
// counts below and every array of the WaveSet (the S-only root set included).
struct WaveFileCounts {
    std::uint64_t n_T, n_idx, n_nodes, n_fwd, n_pairs, n_stripes, n_sdata, event_words, root_words;
    std::uint32_t levels, v_cells, n_plans, pad;
    std::uint64_t n_src, n_pnb;  // producer records (graph programs)
};

void save_wave_file(const bfly_sht_s& s, std::FILE* f) {
    const bfb::DeviceWaveSet& w = s.wv;
    WaveFileCounts c{};
    c.n_T = w.n_T;
    c.n_idx = w.n_idx;
    c.n_nodes = w.n_nodes;
    c.n_fwd = w.n_fwd;
    c.n_pairs = w.n_pairs;
    c.n_stripes = w.roots.n_stripes;
    c.n_sdata = w.roots.bytes / sizeof(double);
    c.event_words = w.event_words;
    c.root_words = w.root_words;
    c.levels = static_cast<std::uint32_t>(w.levels);
    c.v_cells = w.v_cells;
    c.n_plans = static_cast<std::uint32_t>(w.n_plans);
    c.n_src = w.node_src.size();
    c.n_pnb = w.plan_node_begin.size();
    if (std::fwrite(&c, sizeof c, 1, f) != 1) throw std::runtime_error("sht save: write failed");
    auto put = [&](const auto& v) {
        if (!v.empty() && std::fwrite(v.data(), sizeof(v[0]), v.size(), f) != v.size())
            throw std::runtime_error("sht save: write failed");
    };
    put(w.fwd_begin);
    put(w.bwd_begin);
    dev_to_file(f, w.T, c.n_T);
    dev_to_file(f, w.idx, c.n_idx);
    dev_to_file(f, w.nodes, c.n_nodes);
    dev_to_file(f, w.fwd, c.n_fwd);
    dev_to_file(f, w.pairs, c.n_pairs);
    for (const std::uint32_t* a : {w.plan_in, w.plan_mu, w.plan_parity, w.plan_cols}) dev_to_file(f, a, c.n_plans);
    dev_to_file(f, w.roots.stripes, c.n_stripes);
    dev_to_file(f, w.roots.data, c.n_sdata);
    put(w.node_src);
    put(w.plan_node_begin);
}

// The wave section of a program cache file into s (rho / nodes already read).
void load_wave_file(bfly_sht_s& s, std::FILE* f) {
    WaveFileCounts c{};
    if (std::fread(&c, sizeof c, 1, f) != 1) throw std::runtime_error("sht load: truncated file");
    bfb::WaveSet w;
    w.levels = static_cast<int>(c.levels);
    w.v_cells = c.v_cells;
    w.event_words = c.event_words;
    w.root_words = c.root_words;
    w.fwd_begin = from_file<std::uint32_t>(f, c.levels + 1);
    w.bwd_begin = from_file<std::uint32_t>(f, c.levels + 1);
    w.T = from_file<double>(f, c.n_T);
    w.idx = from_file<std::uint32_t>(f, c.n_idx);
    w.nodes = from_file<bfb::WaveNode>(f, c.n_nodes);
    w.fwd = from_file<std::uint32_t>(f, c.n_fwd);
    w.pairs = from_file<std::uint32_t>(f, c.n_pairs);
    w.plan_in = from_file<std::uint32_t>(f, c.n_plans);
    w.plan_mu = from_file<std::uint32_t>(f, c.n_plans);
    w.plan_parity = from_file<std::uint32_t>(f, c.n_plans);
    w.plan_cols = from_file<std::uint32_t>(f, c.n_plans);
    w.roots.stripes = from_file<bfb::RootStripeDesc>(f, c.n_stripes);
    w.roots.data = from_file<double>(f, c.n_sdata);
    w.roots.stored_words = c.root_words;
    w.node_src = from_file<std::uint32_t>(f, c.n_src);
    w.plan_node_begin = from_file<std::uint32_t>(f, c.n_pnb);
    s.wv = bfb::upload_waves(w);
    s.wave = true;
    s.graph = make_graph(w);
}

}  // namespace

extern "C" {

const char* bfly_last_error(void) { return g_err.c_str(); }
const char* bfly_version(void) { return "bfly_b200 0.1 (sm_100a)"; }

int bfly_plan_from_bfly1(const uint8_t* bytes, size_t n, bfly_plan_t* out) {
    return guard([&] {
        if (!bytes || !out) throw std::invalid_argument("bfly_plan_from_bfly1: null argument");
        auto p = std::make_unique<bfly_plan_s>();
        p->plan = bfb::load_bfly1(bytes, n);
        *out = p.release();
    });
}

int bfly_plan_to_bfly1(bfly_plan_t plan, uint8_t* buf, size_t cap, size_t* size) {
    return guard([&] {
        check_plan_handle(plan);
        const std::vector<std::uint8_t> b = bfb::save_bfly1(plan->plan);
        if (size) *size = b.size();
        if (buf && cap >= b.size()) std::memcpy(buf, b.data(), b.size());
    });
}

int bfly_plan_build_glrow(int l, int mu, int parity, double eps, int block_width, bfly_plan_t* out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null output");
        if (l < 1 || mu < 0 || mu >= 2 * l || (parity != 0 && parity != 1))
            throw std::invalid_argument("bfly_plan_build_glrow: bad (l, mu, parity)");
        if (bfb::chain_cols(l, mu, parity) < 1) throw std::invalid_argument("build_plan: empty source");
        auto p = std::make_unique<bfly_plan_s>();
        p->plan = bfb::build_glrow_plan(l, mu, parity, eps, block_width, bfb::gauss_legendre_positive(l));
        *out = p.release();
    });
}

int bfly_plan_build_dense(const double* a, int64_t rows, int64_t cols, double eps, int block_width,
                          bfly_plan_t* out) {
    return guard([&] {
        if (!out || (!a && rows * cols > 0)) throw std::invalid_argument("null argument");
        bfb::Mat m(rows, cols);
        if (rows * cols > 0) std::memcpy(m.a.data(), a, sizeof(double) * static_cast<std::size_t>(rows * cols));
        std::int64_t next = 0;
        auto feed = [&](bfb::Mat& o) {
            if (next + o.cols > cols) throw std::out_of_range("dense source: past the last column");
            std::memcpy(o.a.data(), m.col(next), sizeof(double) * static_cast<std::size_t>(rows * o.cols));
            next += o.cols;
        };
        auto p = std::make_unique<bfly_plan_s>();
        p->plan = bfb::build_plan(rows, cols, feed, eps, block_width);
        *out = p.release();
    });
}

int bfly_plan_info(bfly_plan_t plan, int64_t* info, double* kstat) {
    return guard([&] {
        check_plan_handle(plan);
        const auto& p = plan->plan;
        const bfb::PlanStats st = bfb::plan_stats(p);
        if (info) {
            info[0] = static_cast<int64_t>(p.n_rows);
            info[1] = static_cast<int64_t>(p.n_cols);
            info[2] = static_cast<int64_t>(p.levels);
            info[3] = static_cast<int64_t>(p.stored_words);
            info[4] = static_cast<int64_t>(p.m_max_words);
            info[5] = static_cast<int64_t>(p.events.size());
            info[6] = static_cast<int64_t>(p.root_groups.size());
            info[7] = static_cast<int64_t>(st.k_max);
            info[8] = static_cast<int64_t>(st.id_count);
            info[9] = static_cast<int64_t>(p.block_width);
        }
        if (kstat) {
            kstat[0] = st.k_avg;
            kstat[1] = st.k_sigma;
        }
    });
}

void bfly_plan_destroy(bfly_plan_t plan) { delete plan; }

int bfly_dev_planset_create(const bfly_plan_t* plans, int n, int device, bfly_planset_t* out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null output");
        const auto ptrs = plan_ptrs(plans, n);
        auto s = std::make_unique<bfly_planset_s>();
        s->device = device;
        s->n_plans = n;
        std::vector<std::vector<int>> jobs;
        s->rows_prefix.assign(static_cast<std::size_t>(n) + 1, 0);
        s->cols_prefix.assign(static_cast<std::size_t>(n) + 1, 0);
        for (int i = 0; i < n; ++i) {
            jobs.push_back({i});
            s->rows_prefix[i + 1] = s->rows_prefix[i] + ptrs[i]->n_rows;
            s->cols_prefix[i + 1] = s->cols_prefix[i] + ptrs[i]->n_cols;
        }
        const bfb::PackedProgram packed = pack_for_engine(ptrs, jobs, {}, {});
        DeviceScope ds(device);
        s->prog = bfb::upload_program(packed, device);
        ck(cudaMalloc(&s->d_rows_prefix, sizeof(std::uint64_t) * (n + 1)), "cudaMalloc");
        ck(cudaMalloc(&s->d_cols_prefix, sizeof(std::uint64_t) * (n + 1)), "cudaMalloc");
        ck(cudaMemcpy(s->d_rows_prefix, s->rows_prefix.data(), sizeof(std::uint64_t) * (n + 1), cudaMemcpyHostToDevice),
           "cudaMemcpy");
        ck(cudaMemcpy(s->d_cols_prefix, s->cols_prefix.data(), sizeof(std::uint64_t) * (n + 1), cudaMemcpyHostToDevice),
           "cudaMemcpy");
        // BFLY_WAVES=0: engine only; BFLY_WAVE_MIN_RHS: smallest nrhs served by the waves
        const char* we = std::getenv("BFLY_WAVES");
        if (!(we && std::strtol(we, nullptr, 10) == 0)) {
            const std::vector<int> zeros(static_cast<std::size_t>(n), 0);
            const bfb::WaveSet w = bfb::build_waves(ptrs, zeros, zeros);
            s->wv = bfb::upload_waves(w);
            s->graph = make_graph(w);
            s->wave = true;
            if (const char* e = std::getenv("BFLY_WAVE_MIN_RHS"))
                s->wave_min_rhs = std::max(1, static_cast<int>(std::strtol(e, nullptr, 10)));
        }
        *out = s.release();
    });
}

namespace {
void check_lengths(const bfly_planset_s& s, int transpose, int64_t in_len, int64_t out_len, int nrhs) {
    if (nrhs < 1) throw std::invalid_argument("apply: nrhs must be >= 1");
    const std::uint64_t rows = s.rows_prefix.back(), cols = s.cols_prefix.back();
    const std::int64_t want_in = static_cast<std::int64_t>((transpose ? rows : cols) * nrhs);
    const std::int64_t want_out = static_cast<std::int64_t>((transpose ? cols : rows) * nrhs);
    const char* who = transpose ? "apply_transpose" : "apply";
    if (in_len != want_in)
        throw std::invalid_argument(std::string(who) + ": vector length " + std::to_string(in_len) + ", expected " +
                                    std::to_string(want_in));
    if (out_len != want_out)
        throw std::invalid_argument(std::string(who) + ": output length " + std::to_string(out_len) + ", expected " +
                                    std::to_string(want_out));
}

// Plan-set apply on the wave programs: stacked reference-layout vectors <->
// cell-major V / rows (R = nrhs rounded up to 4), one graph launch.
void dev_apply_waves(bfly_planset_s& s, int transpose, const double* in, double* out, int nrhs, cudaStream_t st) {
    const bfb::DeviceWaveSet& w = s.wv;
    const int n = s.n_plans;
    const std::size_t rows = s.rows_prefix.back();
    // at most kChunk right-hand sides per pass: the cell-major scratch grows with R
    constexpr int kChunk = 256;
    for (int r0 = 0; r0 < nrhs; r0 += kChunk) {
        const int nr = std::min(kChunk, nrhs - r0);
        const int batch = (nr + 3) / 4, R = 4 * batch;
        s.vbuf.ensure(static_cast<std::size_t>(w.v_cells) * R + 4);
        s.wbuf.ensure(rows * R + 4);
        if (!transpose) {
            ck(bfb::launch_plan_cells_in(in, s.vbuf.p, s.d_cols_prefix, w.plan_in, n, nr, R, st, r0, nrhs),
               "plan cells in");
            ck(cudaMemsetAsync(s.wbuf.p, 0, rows * R * sizeof(double), st), "cudaMemsetAsync");  // rows of empty plans
            ck(bfb::launch_graph(s.graph, w, s.vbuf.p, s.wbuf.p, 0, batch, false, st, true), "graph launch (apply)");
            ck(bfb::launch_plan_cells_out(s.wbuf.p, out, s.d_rows_prefix, nullptr, n, nr, R, st, r0, nrhs),
               "plan rows out");
        } else {
            ck(bfb::launch_plan_cells_in(in, s.wbuf.p, s.d_rows_prefix, nullptr, n, nr, R, st, r0, nrhs), "plan rows in");
            ck(bfb::launch_graph(s.graph, w, s.vbuf.p, s.wbuf.p, 0, batch, true, st, true),
               "graph launch (apply_transpose)");
            ck(bfb::launch_plan_cells_out(s.vbuf.p, out, s.d_cols_prefix, w.plan_in, n, nr, R, st, r0, nrhs),
               "plan cells out");
        }
    }
}

void dev_apply(bfly_planset_s& s, int transpose, const double* in, double* out, int nrhs, cudaStream_t st) {
    if (s.wave && nrhs >= s.wave_min_rhs) {
        dev_apply_waves(s, transpose, in, out, nrhs, st);
        return;
    }
    bfb::GenericIO io;
    io.in = in;
    io.out = out;
    io.nrhs = nrhs;
    io.in_prefix = transpose ? s.d_rows_prefix : s.d_cols_prefix;
    io.out_prefix = transpose ? s.d_cols_prefix : s.d_rows_prefix;
    ck(bfb::launch_generic(s.prog, transpose != 0, io, st), "engine launch");
}
}  // namespace

int bfly_dev_apply(bfly_planset_t set, int transpose, const double* in, int64_t in_len, double* out,
                   int64_t out_len, int nrhs, void* stream) {
    return guard([&] {
        check_plan_handle(set);
        check_lengths(*set, transpose, in_len, out_len, nrhs);
        DeviceScope ds(set->device);
        dev_apply(*set, transpose, in, out, nrhs, static_cast<cudaStream_t>(stream));
    });
}

int bfly_host_apply(bfly_planset_t set, int transpose, const double* in, int64_t in_len, double* out,
                    int64_t out_len, int nrhs) {
    return guard([&] {
        check_plan_handle(set);
        check_lengths(*set, transpose, in_len, out_len, nrhs);
        DeviceScope ds(set->device);
        set->h_in.ensure(static_cast<std::size_t>(std::max<int64_t>(in_len, 1)));
        set->h_out.ensure(static_cast<std::size_t>(std::max<int64_t>(out_len, 1)));
        ck(cudaMemcpy(set->h_in.p, in, sizeof(double) * in_len, cudaMemcpyHostToDevice), "cudaMemcpy H2D");
        dev_apply(*set, transpose, set->h_in.p, set->h_out.p, nrhs, nullptr);
        ck(cudaMemcpy(out, set->h_out.p, sizeof(double) * out_len, cudaMemcpyDeviceToHost), "cudaMemcpy D2H");
    });
}

int bfly_dev_planset_info(bfly_planset_t set, int64_t* info) {
    return guard([&] {
        check_plan_handle(set);
        info[0] = set->n_plans;
        info[1] = set->prog.n_jobs;
        info[2] = static_cast<int64_t>(set->prog.stored_words);
        info[3] = static_cast<int64_t>(set->prog.fetched_bytes);
        info[4] = static_cast<int64_t>(set->prog.stream_bytes);
        info[5] = set->prog.arena_cells;
        info[6] = static_cast<int64_t>(bfb::engine_smem_bytes(set->prog));
        info[7] = static_cast<int64_t>(set->rows_prefix.back());
    });
}

void bfly_dev_planset_destroy(bfly_planset_t set) {
    if (!set) return;
    DeviceScope ds(set->device);
    delete set;
}

int bfly_waves_inspect(const bfly_plan_t* plans, int n, int64_t* sizes, double* T, uint32_t* idx, uint32_t* nodes,
                       uint32_t* fwd, uint32_t* pairs, uint32_t* fwd_begin, uint32_t* bwd_begin, uint32_t* plan_in,
                       uint64_t* stripes, double* S) {
    return guard([&] {
        const auto ptrs = plan_ptrs(plans, n);
        const std::vector<int> zeros(static_cast<std::size_t>(n), 0);
        const bfb::WaveSet w = bfb::build_waves(ptrs, zeros, zeros);
        if (sizes) {
            sizes[0] = static_cast<int64_t>(w.T.size());
            sizes[1] = static_cast<int64_t>(w.idx.size());
            sizes[2] = static_cast<int64_t>(w.nodes.size());
            sizes[3] = static_cast<int64_t>(w.fwd.size());
            sizes[4] = static_cast<int64_t>(w.pairs.size() / 2);
            sizes[5] = w.levels;
            sizes[6] = w.v_cells;
            sizes[7] = static_cast<int64_t>(w.roots.stripes.size());
            sizes[8] = static_cast<int64_t>(w.roots.data.size());
            sizes[9] = static_cast<int64_t>(w.aliased_leaves);
        }
        auto put = [](auto* dst, const auto& v) {
            if (dst && !v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
        };
        put(T, w.T);
        put(idx, w.idx);
        if (nodes)
            for (std::size_t i = 0; i < w.nodes.size(); ++i) {
                const bfb::WaveNode& d = w.nodes[i];
                const uint32_t row[8] = {static_cast<uint32_t>(d.t_off), static_cast<uint32_t>(d.t_off >> 32), d.rank,
                                         d.nothers, d.idx, d.cA, d.level, d.nib};
                std::memcpy(nodes + 8 * i, row, sizeof row);
            }
        put(fwd, w.fwd);
        put(pairs, w.pairs);
        put(fwd_begin, w.fwd_begin);
        put(bwd_begin, w.bwd_begin);
        put(plan_in, w.plan_in);
        if (stripes)  // per stripe: s_off, rows, rank, lds, coff, plan, group, first stacked row
            for (std::size_t i = 0; i < w.roots.stripes.size(); ++i) {
                const bfb::RootStripeDesc& d = w.roots.stripes[i];
                const uint64_t row[8] = {d.s_off, d.rows, d.rank, d.lds, d.coff, d.plan, d.pad[0], d.pad[1]};
                std::memcpy(stripes + 8 * i, row, sizeof row);
            }
        put(S, w.roots.data);
    });
}

int bfly_pack_inspect(const bfly_plan_t* plans, int n, uint8_t* stream, uint64_t* stage_off, uint32_t* stage_bytes,
                      void* jobs, int64_t* sizes) {
    return guard([&] {
        const auto ptrs = plan_ptrs(plans, n);
        std::vector<std::vector<int>> jp;
        for (int i = 0; i < n; ++i) jp.push_back({i});
        const bfb::PackedProgram p = bfb::pack_program(ptrs, jp, {});
        if (sizes) {
            sizes[0] = static_cast<int64_t>(p.stream.size());
            sizes[1] = static_cast<int64_t>(p.stage_off.size());
            sizes[2] = static_cast<int64_t>(p.jobs.size());
            sizes[3] = p.arena_cells;
            sizes[4] = p.zo_cells;
            bfb::DeviceProgram d;
            d.arena_cells = p.arena_cells;
            d.zo_cells = p.zo_cells;
            d.stage_capacity = p.stage_capacity;
            sizes[5] = static_cast<int64_t>(bfb::engine_smem_bytes(d));
        }
        if (stream) std::memcpy(stream, p.stream.data(), p.stream.size());
        if (stage_off) std::memcpy(stage_off, p.stage_off.data(), p.stage_off.size() * sizeof(std::uint64_t));
        if (stage_bytes) std::memcpy(stage_bytes, p.stage_bytes.data(), p.stage_bytes.size() * sizeof(std::uint32_t));
        if (jobs) std::memcpy(jobs, p.jobs.data(), p.jobs.size() * sizeof(bfb::Job));
    });
}

int bfly_pack_inspect_split(const bfly_plan_t* plans, int n, const int* parity, int which, uint8_t* stream,
                            uint64_t* stage_off, uint32_t* stage_bytes, void* jobs, int64_t* sizes,
                            uint32_t* plan_yoff, uint32_t* plan_groups) {
    return guard([&] {
        const auto ptrs = plan_ptrs(plans, n);
        std::vector<int> mu(static_cast<std::size_t>(n), 0), par(parity, parity + n);
        const bfb::SplitProgram sp = bfb::pack_split(ptrs, mu, par, 16384, 16384);
        const bfb::PackedProgram& p = which == 0 ? sp.events : sp.roots;
        if (sizes) {
            sizes[0] = static_cast<int64_t>(p.stream.size());
            sizes[1] = static_cast<int64_t>(p.stage_off.size());
            sizes[2] = static_cast<int64_t>(p.jobs.size());
            sizes[3] = p.arena_cells;
            sizes[4] = p.zo_cells;
            bfb::DeviceProgram d;
            d.arena_cells = p.arena_cells;
            d.stage_capacity = p.stage_capacity;
            sizes[5] = static_cast<int64_t>(bfb::engine_smem_bytes(d));
            sizes[6] = sp.c_cells;
            sizes[7] = sp.y_rows;
        }
        if (stream) std::memcpy(stream, p.stream.data(), p.stream.size());
        if (stage_off) std::memcpy(stage_off, p.stage_off.data(), p.stage_off.size() * sizeof(std::uint64_t));
        if (stage_bytes) std::memcpy(stage_bytes, p.stage_bytes.data(), p.stage_bytes.size() * sizeof(std::uint32_t));
        if (jobs) std::memcpy(jobs, p.jobs.data(), p.jobs.size() * sizeof(bfb::Job));
        if (plan_yoff) std::memcpy(plan_yoff, sp.plan_yoff.data(), sp.plan_yoff.size() * sizeof(std::uint32_t));
        if (plan_groups) std::memcpy(plan_groups, sp.plan_groups.data(), sp.plan_groups.size() * sizeof(std::uint32_t));
    });
}

int bfly_phi_time(int l, int batch, int iters, double* ms) {
    return guard([&] {
        if (l < 1 || batch < 1 || iters < 1 || !ms) throw std::invalid_argument("phi time: bad arguments");
        bfb::PhiPlan p = bfb::make_phi_plan(4 * l - 1);
        if (!p.ok && !p.rader) throw std::invalid_argument("phi time: no fused phi plan for N = 4l - 1");
        DevBuf<double> u, grid, isr;
        const std::size_t nu = static_cast<std::size_t>(4 * l) * batch * l * 4;
        const std::size_t ng = static_cast<std::size_t>(batch) * 2 * l * (4 * l - 1) * 2;
        u.ensure(nu);
        grid.ensure(ng);
        isr.ensure(static_cast<std::size_t>(l));
        ck(cudaMemset(u.p, 0, nu * sizeof(double)), "cudaMemset");
        std::vector<double> ones(static_cast<std::size_t>(l), 1.0);
        ck(cudaMemcpy(isr.p, ones.data(), ones.size() * sizeof(double), cudaMemcpyHostToDevice), "cudaMemcpy");
        bfb::ShtIO io;
        io.u = u.p;
        io.isr = isr.p;
        io.hsr = isr.p;
        io.l = l;
        io.N = 4 * l - 1;
        io.batch = batch;
        io.mu0 = 0;
        io.mu_end = 2 * l;
        cudaEvent_t e[3];
        for (auto& x : e) ck(cudaEventCreate(&x), "cudaEventCreate");
        for (int w = 0; w < 2; ++w) {
            ck(bfb::launch_phi_synth_fused(p, io, grid.p, nullptr), "phi synthesis");
            ck(bfb::launch_phi_anal_fused(p, io, grid.p, nullptr), "phi analysis");
        }
        float t[2] = {0.f, 0.f};
        for (int it = 0; it < iters; ++it) {
            cudaEventRecord(e[0]);
            ck(bfb::launch_phi_synth_fused(p, io, grid.p, nullptr), "phi synthesis");
            cudaEventRecord(e[1]);
            ck(bfb::launch_phi_anal_fused(p, io, grid.p, nullptr), "phi analysis");
            cudaEventRecord(e[2]);
            ck(cudaEventSynchronize(e[2]), "cudaEventSynchronize");
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, e[0], e[1]);
            cudaEventElapsedTime(&b, e[1], e[2]);
            t[0] += a;
            t[1] += b;
        }
        for (auto& x : e) cudaEventDestroy(x);
        bfb::free_phi_plan(p);
        ms[0] = t[0] / iters;
        ms[1] = t[1] / iters;
    });
}

int bfly_gl_rule(int l, double* nodes, double* rho) {
    return guard([&] {
        const bfb::GlRule r = bfb::gauss_legendre_positive(l);
        if (nodes) std::memcpy(nodes, r.nodes.data(), sizeof(double) * r.nodes.size());
        if (rho) std::memcpy(rho, r.rho.data(), sizeof(double) * r.rho.size());
    });
}

int bfly_glrow_planset_build(int l, int mu_begin, int mu_end, double eps, int block_width, int threads,
                             bfly_plan_t* plans_out, int cap, int* n_out) {
    return bfly_glrow_planset_build_rule(l, mu_begin, mu_end, eps, block_width, threads, nullptr, nullptr, plans_out,
                                         cap, n_out);
}

int bfly_glrow_planset_build_rule(int l, int mu_begin, int mu_end, double eps, int block_width, int threads,
                                  const double* nodes, const double* rho, bfly_plan_t* plans_out, int cap, int* n_out) {
    return guard([&] {
        if (l < 1 || mu_begin < 0 || mu_end > 2 * l || mu_begin >= mu_end)
            throw std::invalid_argument("planset: bad (l, mu range)");
        if ((nodes == nullptr) != (rho == nullptr)) throw std::invalid_argument("planset: give both nodes and rho, or neither");
        bfb::GlRule rule;
        if (nodes) {
            rule.nodes.assign(nodes, nodes + l);
            rule.rho.assign(rho, rho + l);
        }
        if (!plans_out) {  // count only: the non-empty chains of the range (nothing is built)
            int n = 0;
            for (int mu = mu_begin; mu < mu_end; ++mu)
                for (int p = 0; p < 2; ++p) n += bfb::chain_cols(l, mu, p) > 0 ? 1 : 0;
            if (n_out) *n_out = n;
            return;
        }
        std::vector<bfb::PlanKey> keys;
        std::vector<bfb::ButterflyPlan> plans = bfb::build_glrow_planset_auto(l, mu_begin, mu_end, eps, block_width, threads,
                                                                         &keys, nodes ? &rule : nullptr);
        if (n_out) *n_out = static_cast<int>(plans.size());
        if (cap < static_cast<int>(plans.size())) throw std::invalid_argument("planset: output capacity too small");
        for (std::size_t i = 0; i < plans.size(); ++i) {
            auto p = std::make_unique<bfly_plan_s>();
            p->plan = std::move(plans[i]);
            plans_out[i] = p.release();
        }
    });
}

int bfly_sht_create(int l, double eps, int block_width, int threads, int device, bfly_sht_t* out) {
    return bfly_sht_create_rule(l, eps, block_width, threads, nullptr, nullptr, device, out);
}

int bfly_sht_create_rule(int l, double eps, int block_width, int threads, const double* nodes, const double* rho,
                         int device, bfly_sht_t* out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null output");
        if (l < 1) throw std::invalid_argument("sht: l must be >= 1");
        if ((nodes == nullptr) != (rho == nullptr)) throw std::invalid_argument("sht: give both nodes and rho, or neither");
        bfb::GlRule rule;
        if (nodes) {
            rule.nodes.assign(nodes, nodes + l);
            rule.rho.assign(rho, rho + l);
        }
        const bool verbose = std::getenv("BFLY_BUILD_VERBOSE") != nullptr;
        const auto t0 = std::chrono::steady_clock::now();
        auto since = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
        std::vector<bfb::PlanKey> keys;
        std::vector<bfb::ButterflyPlan> plans =
            bfb::build_glrow_planset_auto(l, 0, 2 * l, eps, block_width, threads, &keys, nodes ? &rule : nullptr);
        if (verbose) std::fprintf(stderr, "sht create: plans built at %.2f s\n", since());
        std::vector<const bfb::ButterflyPlan*> ptrs;
        for (const auto& p : plans) ptrs.push_back(&p);
        auto s = std::make_unique<bfly_sht_s>();
        make_sht(*s, l, 0, 2 * l, ptrs, rho, device, nodes);
        if (verbose) std::fprintf(stderr, "sht create: programs on the device at %.2f s\n", since());
        *out = s.release();
        plans.clear();
        plans.shrink_to_fit();
        if (verbose) std::fprintf(stderr, "sht create: host plans released at %.2f s\n", since());
    });
}

int bfly_sht_create_from_plans(int l, const bfly_plan_t* plans, int n, const double* rho, int device,
                               bfly_sht_t* out) {
    return bfly_sht_create_range(l, 0, 2 * l, plans, n, rho, device, out);
}

int bfly_sht_create_range(int l, int mu_begin, int mu_end, const bfly_plan_t* plans, int n, const double* rho,
                          int device, bfly_sht_t* out) {
    return guard([&] {
        if (!out) throw std::invalid_argument("null output");
        const auto ptrs = plan_ptrs(plans, n);
        auto s = std::make_unique<bfly_sht_s>();
        make_sht(*s, l, mu_begin, mu_end, ptrs, rho, device);
        *out = s.release();
    });
}

int bfly_sht_legendre_synthesize(bfly_sht_t sht, const double* beta, double* gbins, int batch, void* stream) {
    return guard([&] {
        check_plan_handle(sht);
        check_batch(batch);
        DeviceScope ds(sht->device);
        legendre_synth(*sht, beta, gbins, batch, static_cast<cudaStream_t>(stream));
    });
}

int bfly_sht_legendre_analyze(bfly_sht_t sht, const double* gdft, double* beta, int batch, void* stream) {
    return guard([&] {
        check_plan_handle(sht);
        check_batch(batch);
        DeviceScope ds(sht->device);
        legendre_anal(*sht, gdft, beta, batch, static_cast<cudaStream_t>(stream));
    });
}

int bfly_sht_synthesize(bfly_sht_t sht, const double* beta, double* grid, int batch, void* stream) {
    return guard([&] {
        check_plan_handle(sht);
        check_batch(batch);
        full_range(*sht);
        DeviceScope ds(sht->device);
        sht_synth(*sht, beta, grid, batch, static_cast<cudaStream_t>(stream));
    });
}

int bfly_sht_analyze(bfly_sht_t sht, const double* grid, double* beta, int batch, void* stream) {
    return guard([&] {
        check_plan_handle(sht);
        check_batch(batch);
        full_range(*sht);
        DeviceScope ds(sht->device);
        sht_anal(*sht, grid, beta, batch, static_cast<cudaStream_t>(stream));
    });
}

int bfly_sht_shard_supported(bfly_sht_t sht, int* ok) {
    return guard([&] {
        check_plan_handle(sht);
        if (!ok) throw std::invalid_argument("sht shard: null argument");
        *ok = (!sht->split && sht->phi.ok) ? 1 : 0;
    });
}

int bfly_sht_shard_synthesize(bfly_sht_t sht, const double* beta, double* send, const int64_t* row_base,
                              const int32_t* row_T, int batch, void* stream) {
    return guard([&] {
        check_plan_handle(sht);
        check_batch(batch);
        check_shard_orders(*sht);
        DeviceScope ds(sht->device);
        const auto st = static_cast<cudaStream_t>(stream);
        bfb::ShtIO io = sht_io(*sht);
        io.beta_in = beta;
        io.u = sht->u_buffer(batch);
        io.batch = batch;
        timed_engine(*sht, false, st, [&] { legendre_u(*sht, io, batch, false, st, !sht->time_engine); });
        ck(bfb::launch_shard_pack(io, send, reinterpret_cast<const long long*>(row_base), row_T, sht->mu_begin,
                                  sht->mu_end, st),
           "shard pack");
    });
}

int bfly_sht_shard_phi(bfly_sht_t sht, int synthesis, const double* src, double* dst, const int64_t* bin_off,
                       int n_rows, int batch, void* stream) {
    return guard([&] {
        check_plan_handle(sht);
        check_batch(batch);
        check_shard(*sht);
        if (n_rows < 0 || n_rows > 2 * sht->l) throw std::invalid_argument("sht shard: bad slab row count");
        DeviceScope ds(sht->device);
        ck(bfb::launch_shard_phi(sht->phi, synthesis != 0, src, dst, reinterpret_cast<const long long*>(bin_off),
                                 n_rows, batch, static_cast<cudaStream_t>(stream)),
           "shard phi");
    });
}

int bfly_sht_shard_analyze(bfly_sht_t sht, const double* recv, double* beta, const int64_t* row_base,
                           const int32_t* row_T, int batch, void* stream) {
    return guard([&] {
        check_plan_handle(sht);
        check_batch(batch);
        check_shard_orders(*sht);
        DeviceScope ds(sht->device);
        const auto st = static_cast<cudaStream_t>(stream);
        bfb::ShtIO io = sht_io(*sht);
        io.beta_out = beta;
        io.u = sht->u_buffer(batch);
        io.batch = batch;
        ck(bfb::launch_shard_unpack(io, recv, reinterpret_cast<const long long*>(row_base), row_T, sht->mu_begin,
                                    sht->mu_end, st),
           "shard unpack");
        timed_engine(*sht, true, st, [&] { legendre_u(*sht, io, batch, true, st, false); });
    });
}

int bfly_sht_synthesize_real(bfly_sht_t sht, const double* beta_half, double* grid, int batch, void* stream) {
    return guard([&] {
        check_plan_handle(sht);
        check_batch(batch);
        full_range(*sht);
        if (!fused_phi_stockham(*sht))
            throw std::invalid_argument("sht: real transforms need the fused phi stage (prime factors of 4l-1 "
                                        "<= 127) and whole-chain or wave programs");
        DeviceScope ds(sht->device);
        const auto st = static_cast<cudaStream_t>(stream);
        // One field: 2 right-hand sides (RC = 2).  Several: two fields per task
        // share the four right-hand sides, so the plan streams once per pair.
        bfb::ShtIO io = sht_io(*sht);
        io.beta_in = beta_half;
        io.beta_stride = 2LL * sht->l * (2LL * sht->l + 1);
        io.u = sht->u_buffer(batch);
        io.real_members = batch;
        const bool waves = use_waves(*sht, (batch + 1) / 2);
        io.real_per_task = (batch > 1 || waves) ? 2 : 1;
        const int tasks = (batch + io.real_per_task - 1) / io.real_per_task;
        io.batch = tasks;
        if (waves)
            wave_legendre(*sht, io, tasks, false, st);
        else
            ck(bfb::launch_sht(sht->prog, false, io, tasks, st, true, io.real_per_task == 1),
               "engine launch (real synthesis)");
        io.batch = batch;
        ck(bfb::launch_phi_synth_real(sht->phi, io, grid, st), "phi synthesis (real)");
    });
}

int bfly_sht_analyze_real(bfly_sht_t sht, const double* grid, double* beta_half, int batch, void* stream) {
    return guard([&] {
        check_plan_handle(sht);
        check_batch(batch);
        full_range(*sht);
        if (!fused_phi_stockham(*sht))
            throw std::invalid_argument("sht: real transforms need the fused phi stage (prime factors of 4l-1 "
                                        "<= 127) and whole-chain or wave programs");
        DeviceScope ds(sht->device);
        const auto st = static_cast<cudaStream_t>(stream);
        bfb::ShtIO io = sht_io(*sht);
        io.beta_out = beta_half;
        io.beta_stride = 2LL * sht->l * (2LL * sht->l + 1);
        io.u = sht->u_buffer(batch);
        io.real_members = batch;
        const bool waves = use_waves(*sht, (batch + 1) / 2);
        io.real_per_task = (batch > 1 || waves) ? 2 : 1;
        const int tasks = (batch + io.real_per_task - 1) / io.real_per_task;
        io.batch = batch;
        ck(bfb::launch_phi_anal_real(sht->phi, io, grid, st), "phi analysis (real)");
        io.batch = tasks;
        if (waves)
            wave_legendre(*sht, io, tasks, true, st);
        else
            ck(bfb::launch_sht(sht->prog, true, io, tasks, st, true, io.real_per_task == 1),
               "engine launch (real analysis)");
    });
}

int bfly_sht_phi_synthesize(bfly_sht_t sht, const double* gbins, double* grid, int batch, void* stream) {
    return guard([&] {
        check_plan_handle(sht);
        check_batch(batch);
        DeviceScope ds(sht->device);
        const auto st = static_cast<cudaStream_t>(stream);
        ckfft(cufftExecZ2Z(sht->plans_for(batch, st).first,
                           reinterpret_cast<cufftDoubleComplex*>(const_cast<double*>(gbins)),
                           reinterpret_cast<cufftDoubleComplex*>(grid), CUFFT_INVERSE),
              "cufftExecZ2Z");
    });
}

int bfly_sht_phi_analyze(bfly_sht_t sht, const double* grid, double* gdft, int batch, void* stream) {
    return guard([&] {
        check_plan_handle(sht);
        check_batch(batch);
        DeviceScope ds(sht->device);
        const auto st = static_cast<cudaStream_t>(stream);
        ckfft(cufftExecZ2Z(sht->plans_for(batch, st).second,
                           reinterpret_cast<cufftDoubleComplex*>(const_cast<double*>(grid)),
                           reinterpret_cast<cufftDoubleComplex*>(gdft), CUFFT_FORWARD),
              "cufftExecZ2Z");
    });
}

namespace {

// Host-buffer transforms: the batch runs as member chunks through three streams
// (H2D of chunk k + 1 and D2H of chunk k - 1 overlap the transform of chunk k;
// the two copy directions also overlap each other).  BFLY_HOST_CHUNKS overrides.
void host_pipeline(bfly_sht_s& s, const double* in, double* out, int batch, bool synthesis) {
    const std::size_t pb = static_cast<std::size_t>(2 * s.coeffs()), pg = static_cast<std::size_t>(2 * s.grid_points());
    const std::size_t pin = synthesis ? pb : pg, pout = synthesis ? pg : pb;  // doubles per function
    s.h_beta.ensure(pb * batch);
    s.h_grid.ensure(pg * batch);
    double* din = synthesis ? s.h_beta.p : s.h_grid.p;
    double* dout = synthesis ? s.h_grid.p : s.h_beta.p;
    // chunks as small as the program still runs efficiently (the wave programs'
    // smallest batch), at most 8 (c3: 2 chunks 139, 4 chunks 160, 8 chunks 173 e2e pairs/s)
    const int cmin = s.wave ? s.wave_min_batch : 1;
    int chunks = std::max(1, std::min(8, batch / cmin));
    if (const char* e = std::getenv("BFLY_HOST_CHUNKS")) chunks = std::max(1, static_cast<int>(std::strtol(e, nullptr, 10)));
    chunks = std::min(chunks, batch);
    if (chunks == 1) {
        ck(cudaMemcpyAsync(din, in, pin * batch * sizeof(double), cudaMemcpyHostToDevice, nullptr), "H2D");
        if (synthesis)
            sht_synth(s, din, dout, batch, nullptr);
        else
            sht_anal(s, din, dout, batch, nullptr);
        ck(cudaMemcpyAsync(out, dout, pout * batch * sizeof(double), cudaMemcpyDeviceToHost, nullptr), "D2H");
        ck(cudaStreamSynchronize(nullptr), "synchronize");
        return;
    }
    for (cudaStream_t& x : s.hst)
        if (!x) ck(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking), "cudaStreamCreate");
    while (static_cast<int>(s.hev.size()) < 2 * chunks) {
        cudaEvent_t e;
        ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
        s.hev.push_back(e);
    }
    // the device buffers may still be read by an earlier call's work on the legacy stream
    ck(cudaStreamSynchronize(nullptr), "synchronize");
    const int cb = (batch + chunks - 1) / chunks;
    for (int c = 0, b0 = 0; b0 < batch; ++c, b0 += cb) {
        const int n = std::min(cb, batch - b0);
        ck(cudaMemcpyAsync(din + pin * b0, in + pin * b0, pin * n * sizeof(double), cudaMemcpyHostToDevice, s.hst[0]),
           "H2D");
        ck(cudaEventRecord(s.hev[2 * c], s.hst[0]), "cudaEventRecord");
        ck(cudaStreamWaitEvent(s.hst[1], s.hev[2 * c], 0), "cudaStreamWaitEvent");
        if (synthesis)
            sht_synth(s, din + pin * b0, dout + pout * b0, n, s.hst[1]);
        else
            sht_anal(s, din + pin * b0, dout + pout * b0, n, s.hst[1]);
        ck(cudaEventRecord(s.hev[2 * c + 1], s.hst[1]), "cudaEventRecord");
        ck(cudaStreamWaitEvent(s.hst[2], s.hev[2 * c + 1], 0), "cudaStreamWaitEvent");
        ck(cudaMemcpyAsync(out + pout * b0, dout + pout * b0, pout * n * sizeof(double), cudaMemcpyDeviceToHost,
                           s.hst[2]),
           "D2H");
    }
    ck(cudaStreamSynchronize(s.hst[2]), "synchronize");
    ck(cudaStreamSynchronize(s.hst[1]), "synchronize");
}

}  // namespace

int bfly_sht_synthesize_host(bfly_sht_t sht, const double* beta, double* grid, int batch) {
    return guard([&] {
        check_plan_handle(sht);
        check_batch(batch);
        full_range(*sht);
        DeviceScope ds(sht->device);
        host_pipeline(*sht, beta, grid, batch, true);
    });
}

int bfly_sht_analyze_host(bfly_sht_t sht, const double* grid, double* beta, int batch) {
    return guard([&] {
        check_plan_handle(sht);
        check_batch(batch);
        full_range(*sht);
        DeviceScope ds(sht->device);
        host_pipeline(*sht, grid, beta, batch, false);
    });
}

int bfly_sht_debug(bfly_sht_t sht, int flags) {
    return guard([&] {
        check_plan_handle(sht);
        sht->prog.debug = flags;
    });
}

int bfly_sht_engine_time(bfly_sht_t sht, int enable, double* ms, int64_t* launches) {
    return guard([&] {
        check_plan_handle(sht);
        DeviceScope ds(sht->device);
        for (int d = 0; d < 2; ++d) {
            double total = 0.0;
            for (auto& e : sht->engine_ev[d]) {
                ck(cudaEventSynchronize(e.second), "cudaEventSynchronize");
                float t = 0.f;
                ck(cudaEventElapsedTime(&t, e.first, e.second), "cudaEventElapsedTime");
                total += t;
                cudaEventDestroy(e.first);
                cudaEventDestroy(e.second);
            }
            if (ms) ms[d] = total;
            if (launches) launches[d] = static_cast<int64_t>(sht->engine_ev[d].size());
            sht->engine_ev[d].clear();
        }
        sht->time_engine = enable != 0;
    });
}

int bfly_sht_trace(bfly_sht_t sht, int max_tasks) {
    return guard([&] {
        check_plan_handle(sht);
        DeviceScope ds(sht->device);
        if (sht->prog.trace) cudaFree(sht->prog.trace);
        sht->prog.trace = nullptr;
        if (max_tasks > 0) {
            ck(cudaMalloc(&sht->prog.trace, sizeof(unsigned long long) * 4 * max_tasks), "cudaMalloc");
            ck(cudaMemset(sht->prog.trace, 0, sizeof(unsigned long long) * 4 * max_tasks), "cudaMemset");
        }
    });
}

int bfly_sht_trace_read(bfly_sht_t sht, uint64_t* out, int max_tasks) {
    return guard([&] {
        check_plan_handle(sht);
        if (!sht->prog.trace) throw std::invalid_argument("trace not enabled");
        DeviceScope ds(sht->device);
        ck(cudaMemcpy(out, sht->prog.trace, sizeof(unsigned long long) * 4 * max_tasks, cudaMemcpyDeviceToHost),
           "cudaMemcpy");
    });
}

int bfly_sht_program_info(bfly_sht_t sht, int64_t* info) {
    return guard([&] {
        check_plan_handle(sht);
        if (!info) throw std::invalid_argument("sht program info: null argument");
        const bfb::DeviceWaveSet& w = sht->wv;
        info[0] = sht->whole ? 1 : 0;
        info[1] = sht->wave ? 1 : 0;
        info[2] = sht->wave ? w.levels : 0;
        info[3] = sht->wave ? static_cast<int64_t>(w.root_groups) : 0;
        info[4] = sht->wave ? static_cast<int64_t>(w.v_cells) : 0;
        info[5] = sht->wave ? static_cast<int64_t>(w.n_nodes) : 0;
        info[6] = sht->wave ? static_cast<int64_t>(w.event_words) : 0;
        info[7] = sht->wave_min_batch;
        info[8] = sht->graph.ok ? 1 : 0;  // (always, with wave programs)
        info[9] = sht->graph.ok ? static_cast<int64_t>(sht->graph.groups) : 0;
    });
}

int bfly_sht_info(bfly_sht_t sht, int64_t* info) {
    return guard([&] {
        check_plan_handle(sht);
        info[0] = sht->l;
        info[1] = sht->n_plans;
        info[2] = static_cast<int64_t>(sht->prog.stored_words);
        info[3] = static_cast<int64_t>(sht->prog.fetched_bytes);
        info[4] = sht->prog.n_jobs;
        info[5] = static_cast<int64_t>(std::max(bfb::engine_smem_bytes(sht->prog),
                                                sht->split ? bfb::engine_smem_bytes(sht->roots) : std::size_t{0}));
        info[6] = sht->coeffs();
        info[7] = sht->grid_points();
    });
}

int bfly_sht_rule(bfly_sht_t sht, double* nodes, double* rho) {
    return guard([&] {
        check_plan_handle(sht);
        if (nodes) std::memcpy(nodes, sht->nodes.data(), sizeof(double) * sht->nodes.size());
        if (rho) std::memcpy(rho, sht->rho.data(), sizeof(double) * sht->rho.size());
    });
}

int bfly_sht_save(bfly_sht_t sht, const char* path) {
    return guard([&] {
        check_plan_handle(sht);
        if (!path) throw std::invalid_argument("sht save: null path");
        if (sht->split) throw std::invalid_argument("sht save: split programs are not cached (whole-chain and wave programs are)");
        DeviceScope ds(sht->device);
        FileCloser fc{std::fopen(path, "wb")};
        if (!fc.f) throw std::runtime_error(std::string("sht save: cannot open ") + path);
        const bfb::DeviceProgram& d = sht->prog;
        ShtFileHeader h{};
        std::memcpy(h.magic, kShtMagic, 8);
        // version 1: whole-chain program only; 5: flags (bit 0 whole-chain
        // program, bit 1 wave section after it; matrices in 16 x 16 tiles)
        h.version = sht->wave ? 5 : 1;
        h.pad = (sht->whole ? 1u : 0u) | (sht->wave ? 2u : 0u);
        h.l = static_cast<std::uint32_t>(sht->l);
        h.mu_begin = static_cast<std::uint32_t>(sht->mu_begin);
        h.mu_end = static_cast<std::uint32_t>(sht->mu_end);
        h.n_plans = static_cast<std::uint32_t>(sht->n_plans);
        h.arena_cells = d.arena_cells;
        h.zo_cells = d.zo_cells;
        h.stage_capacity = d.stage_capacity;
        h.chunk_rows = static_cast<std::uint32_t>(bfb::kChunkRows);
        h.stored_words = d.stored_words;
        h.fetched_bytes = d.fetched_bytes;
        h.n_stages = d.n_stages;
        h.n_jobs = static_cast<std::uint64_t>(d.n_jobs);
        h.stream_bytes = d.stream_bytes;
        if (std::fwrite(&h, sizeof h, 1, fc.f) != 1) throw std::runtime_error("sht save: write failed");
        if (std::fwrite(sht->rho.data(), sizeof(double), sht->rho.size(), fc.f) != sht->rho.size() ||
            std::fwrite(sht->nodes.data(), sizeof(double), sht->nodes.size(), fc.f) != sht->nodes.size())
            throw std::runtime_error("sht save: write failed");
        if (sht->whole) {
            dev_to_file(fc.f, d.stage_off, d.n_stages);
            dev_to_file(fc.f, d.stage_bytes, d.n_stages);
            dev_to_file(fc.f, d.jobs, static_cast<std::size_t>(d.n_jobs));
            dev_to_file(fc.f, d.stream, d.stream_bytes);
        }
        if (sht->wave) save_wave_file(*sht, fc.f);
    });
}

int bfly_sht_load(const char* path, int device, bfly_sht_t* out) {
    return guard([&] {
        if (!path || !out) throw std::invalid_argument("sht load: null argument");
        FileCloser fc{std::fopen(path, "rb")};
        if (!fc.f) throw std::runtime_error(std::string("sht load: cannot open ") + path);
        ShtFileHeader h{};
        if (std::fread(&h, sizeof h, 1, fc.f) != 1 || std::memcmp(h.magic, kShtMagic, 8) != 0 ||
            (h.version != 1 && h.version != 5))
            throw bfb::SerializationError("sht load: not a BFLYSHT1 file", 0);
        const unsigned flags = h.version == 1 ? 1u : h.pad;
        if (h.chunk_rows != static_cast<std::uint32_t>(bfb::kChunkRows))
            throw bfb::SerializationError("sht load: program packed for " + std::to_string(h.chunk_rows) +
                                              "-row chunks, this build uses " + std::to_string(bfb::kChunkRows),
                                          0);
        auto s = std::make_unique<bfly_sht_s>();
        s->l = static_cast<int>(h.l);
        s->N = 4 * s->l - 1;
        s->device = device;
        s->mu_begin = static_cast<int>(h.mu_begin);
        s->mu_end = static_cast<int>(h.mu_end);
        s->n_plans = static_cast<int>(h.n_plans);
        s->rho = from_file<double>(fc.f, h.l);
        s->nodes = from_file<double>(fc.f, h.l);
        DeviceScope ds(device);
        if (flags & 1u) {
            bfb::PackedProgram p;
            p.stage_off = from_file<std::uint64_t>(fc.f, h.n_stages);
            p.stage_bytes = from_file<std::uint32_t>(fc.f, h.n_stages);
            p.jobs = from_file<bfb::Job>(fc.f, h.n_jobs);
            p.stream = from_file<std::uint8_t>(fc.f, h.stream_bytes);
            p.arena_cells = h.arena_cells;
            p.zo_cells = h.zo_cells;
            p.stage_capacity = h.stage_capacity;
            p.stored_words = h.stored_words;
            p.fetched_bytes = h.fetched_bytes;
            s->prog = bfb::upload_program(p, device);
            s->whole = true;
        }
        if (flags & 2u) load_wave_file(*s, fc.f);
        s->prog.stored_words = h.stored_words;
        s->prog.fetched_bytes = h.fetched_bytes;
        finish_sht(*s);
        *out = s.release();
    });
}

void bfly_sht_destroy(bfly_sht_t sht) {
    if (!sht) return;
    DeviceScope ds(sht->device);
    delete sht;
}

}  // extern "C"
