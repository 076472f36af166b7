// oracle/ref_capi.cpp — TEST INFRASTRUCTURE (the CPU oracle), never shipped.
//
// A thin C ABI around the UNMODIFIED reference library compiled from
// /root/reference/proj/src/{butterfly,id,legendre,quadrature,transform,
// serialize}.cpp against oracle/eigen_shim (see oracle/Makefile).  Only
// tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg load the
// resulting oracle/_ref/libbfly_ref.so.
//
// What it exposes, each a direct call into the reference:
//   * plan construction: bfly::build_plan over a DenseColumnSource
//     (include/bfly/column_source.hpp:21-40), over the reference's own
//     transform::build_transform (src/transform.cpp:62-81), and over GL rows
//     (the north_star's rows: LegendreColumnSource(mu, p, build_rule(0, l,
//     even)) truncated to n_p(mu) columns);
//   * bfly::apply / bfly::apply_transpose (src/butterfly.cpp:384-513), one
//     right-hand side per call exactly as the reference API takes them;
//   * save_plan / load_plan (src/serialize.cpp:125-232) so plans cross into the
//     product as the reference's own BFLY1 bytes;
//   * build_rule (src/quadrature.cpp:206-255) and dense materialisation;
//   * a std::thread pool over plans for the whole-transform CPU baseline.
#include <atomic>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <sstream>
#include <string>
#include <thread>
#include <vector>

#include "bfly/butterfly.hpp"
#include "bfly/column_source.hpp"
#include "bfly/quadrature.hpp"
#include "bfly/serialize.hpp"
#include "bfly/transform.hpp"

namespace {

thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
    if (dynamic_cast<const bfly::SerializationError*>(&e)) return 3;
    if (dynamic_cast<const std::runtime_error*>(&e)) return 2;
    return 4;
}

bfly::legendre::Parity par(int p) {
    return p ? bfly::legendre::Parity::odd : bfly::legendre::Parity::even;
}

// Column count of chain p at order mu for bandlimit l (SURVEY.md §8 defs).
std::int64_t chain_cols(int l, int mu, int p) {
    const std::int64_t n = p == 0 ? (2LL * l - mu + 1) / 2 : (2LL * l - 1 - mu + 1) / 2;
    return n < 0 ? 0 : n;
}

// The reference's LegendreColumnSource over the m = 0 even rule (the l
// positive Gauss-Legendre nodes, weights rho_i = 2 w_GL,i), reporting only the
// first n_p(mu) columns.  The reference constructor takes m separately from
// rule.m (include/bfly/transform.hpp:24), so this is its intended use.
class GlRowSource final : public bfly::ColumnSource {
public:
    GlRowSource(int mu, int p, const bfly::quadrature::QuadratureRule& rule,
                Eigen::Index cols)
        : inner_(mu, par(p), rule), cols_(cols) {}
    Eigen::Index rows() const override { return inner_.rows(); }
    Eigen::Index cols() const override { return cols_; }
    void next_columns(Eigen::Ref<Eigen::MatrixXd> out) override { inner_.next_columns(out); }
    void reset() override { inner_.reset(); }

private:
    bfly::transform::LegendreColumnSource inner_;
    Eigen::Index cols_;
};

struct PlanSet {
    int l = 0;
    std::vector<int> mu, parity;
    std::vector<bfly::ButterflyPlan> plans;
};

template <class F>
void parallel_for(std::int64_t n, int nthreads, F&& f) {
    if (nthreads <= 1 || n <= 1) {
        for (std::int64_t i = 0; i < n; ++i) f(i);
        return;
    }
    std::atomic<std::int64_t> next{0};
    std::vector<std::thread> pool;
    std::exception_ptr err;
    std::mutex mu;
    for (int t = 0; t < nthreads; ++t)
        pool.emplace_back([&] {
            for (;;) {
                const std::int64_t i = next.fetch_add(1);
                if (i >= n) return;
                try {
                    f(i);
                } catch (...) {
                    std::lock_guard<std::mutex> lk(mu);
                    if (!err) err = std::current_exception();
                }
            }
        });
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
}

}  // namespace

extern "C" {

const char* bref_last_error() { return g_err.c_str(); }

std::int64_t bref_chain_cols(int l, int mu, int p) { return chain_cols(l, mu, p); }

void* bref_plan_glrow(int l, int mu, int p, double eps, int bw) {
    try {
        const auto rule = bfly::quadrature::build_rule(0, l, bfly::legendre::Parity::even);
        GlRowSource src(mu, p, rule, chain_cols(l, mu, p));
        return new bfly::ButterflyPlan(bfly::build_plan(src, eps, bw));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void* bref_plan_dense(const double* a, std::int64_t rows, std::int64_t cols,
                      double eps, int bw) {
    try {
        Eigen::MatrixXd m(rows, cols);
        std::memcpy(m.data(), a, sizeof(double) * static_cast<std::size_t>(rows * cols));
        bfly::DenseColumnSource src(std::move(m));
        return new bfly::ButterflyPlan(bfly::build_plan(src, eps, bw));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// The reference's own square Gauss-Jacobi transform plan (build_transform).
void* bref_plan_transform(int m, int n, int p, double eps, int bw) {
    try {
        auto tp = bfly::transform::build_transform(m, n, par(p), eps, bw);
        return new bfly::ButterflyPlan(std::move(tp.plan));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void* bref_plan_load(const std::uint8_t* bytes, std::int64_t n) {
    try {
        std::istringstream is(std::string(reinterpret_cast<const char*>(bytes),
                                          static_cast<std::size_t>(n)),
                              std::ios::binary);
        return new bfly::ButterflyPlan(bfly::load_plan(is));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// BFLY1 bytes of the plan; returns the size, copies only if cap suffices.
std::int64_t bref_plan_save(void* h, std::uint8_t* buf, std::int64_t cap) {
    try {
        std::ostringstream os(std::ios::binary);
        bfly::save_plan(*static_cast<bfly::ButterflyPlan*>(h), os);
        const std::string s = os.str();
        if (buf && cap >= static_cast<std::int64_t>(s.size()))
            std::memcpy(buf, s.data(), s.size());
        return static_cast<std::int64_t>(s.size());
    } catch (const std::exception& e) {
        fail(e);
        return -1;
    }
}

void bref_plan_free(void* h) { delete static_cast<bfly::ButterflyPlan*>(h); }

// info[0..9] = n_rows, n_cols, levels, stored_words, m_max_words, events,
// root_groups, k_max, id_count, block_width;  kstat[0..1] = k_avg, k_sigma.
void bref_plan_info(void* h, std::int64_t* info, double* kstat) {
    const auto& p = *static_cast<bfly::ButterflyPlan*>(h);
    const bfly::PlanStats st = bfly::plan_stats(p);
    info[0] = static_cast<std::int64_t>(p.n_rows);
    info[1] = static_cast<std::int64_t>(p.n_cols);
    info[2] = static_cast<std::int64_t>(p.levels);
    info[3] = static_cast<std::int64_t>(p.stored_words);
    info[4] = static_cast<std::int64_t>(p.m_max_words);
    info[5] = static_cast<std::int64_t>(p.events.size());
    info[6] = static_cast<std::int64_t>(p.root_groups.size());
    info[7] = static_cast<std::int64_t>(st.k_max);
    info[8] = static_cast<std::int64_t>(st.id_count);
    info[9] = static_cast<std::int64_t>(p.block_width);
    kstat[0] = st.k_avg;
    kstat[1] = st.k_sigma;
}

// nrhs reference calls, one vector each.  Column r of `in` starts at
// in + r * ld_in (column-major, like Eigen).
int bref_apply(void* h, int transpose, const double* in, std::int64_t ld_in,
               double* out, std::int64_t ld_out, int nrhs) {
    try {
        const auto& p = *static_cast<bfly::ButterflyPlan*>(h);
        const Eigen::Index n_in = static_cast<Eigen::Index>(transpose ? p.n_rows : p.n_cols);
        for (int r = 0; r < nrhs; ++r) {
            Eigen::VectorXd v(n_in);
            std::memcpy(v.data(), in + r * ld_in, sizeof(double) * static_cast<std::size_t>(n_in));
            const Eigen::VectorXd y = transpose ? bfly::apply_transpose(p, v) : bfly::apply(p, v);
            std::memcpy(out + r * ld_out, y.data(), sizeof(double) * static_cast<std::size_t>(y.size()));
        }
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Apply with an explicit input length, so callers can exercise the reference's
// length checks (std::invalid_argument) through the C ABI.
int bref_apply_len(void* h, int transpose, const double* in, std::int64_t n_in,
                   double* out) {
    try {
        const auto& p = *static_cast<bfly::ButterflyPlan*>(h);
        Eigen::VectorXd v(static_cast<Eigen::Index>(n_in));
        if (n_in) std::memcpy(v.data(), in, sizeof(double) * static_cast<std::size_t>(n_in));
        const Eigen::VectorXd y = transpose ? bfly::apply_transpose(p, v) : bfly::apply(p, v);
        std::memcpy(out, y.data(), sizeof(double) * static_cast<std::size_t>(y.size()));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

int bref_rule(int m, int n, int p, double* nodes, double* weights, double* center) {
    try {
        const auto rule = bfly::quadrature::build_rule(m, n, par(p));
        std::memcpy(nodes, rule.nodes.data(), sizeof(double) * rule.nodes.size());
        std::memcpy(weights, rule.weights.data(), sizeof(double) * rule.weights.size());
        if (center) *center = rule.center_weight.value_or(0.0);
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Dense l x n_p(mu) GL-row matrix, column-major, via the reference source.
int bref_dense_glrow(int l, int mu, int p, double* out) {
    try {
        const auto rule = bfly::quadrature::build_rule(0, l, bfly::legendre::Parity::even);
        GlRowSource src(mu, p, rule, chain_cols(l, mu, p));
        const Eigen::MatrixXd a = bfly::materialize(src);
        std::memcpy(out, a.data(), sizeof(double) * static_cast<std::size_t>(a.size()));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Dense n x n matrix of the reference's own transform (Gauss-Jacobi rows).
int bref_dense_transform(int m, int n, int p, double* out, double* nodes, double* weights) {
    try {
        const auto rule = bfly::quadrature::build_rule(m, n, par(p));
        bfly::transform::LegendreColumnSource src(m, par(p), rule);
        const Eigen::MatrixXd a = bfly::materialize(src);
        std::memcpy(out, a.data(), sizeof(double) * static_cast<std::size_t>(a.size()));
        if (nodes) std::memcpy(nodes, rule.nodes.data(), sizeof(double) * rule.nodes.size());
        if (weights) std::memcpy(weights, rule.weights.data(), sizeof(double) * rule.weights.size());
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// ---- whole plan sets (every |m| and parity of one bandlimit) --------------

// Plans for (mu, p) over mu in [mu_begin, mu_end) with n_p(mu) >= 1, built on
// nthreads host threads.  Plan order: mu ascending, even before odd.
void* bref_planset_glrow(int l, int mu_begin, int mu_end, double eps, int bw, int nthreads) {
    try {
        auto set = std::make_unique<PlanSet>();
        set->l = l;
        for (int mu = mu_begin; mu < mu_end; ++mu)
            for (int p = 0; p < 2; ++p)
                if (chain_cols(l, mu, p) > 0) {
                    set->mu.push_back(mu);
                    set->parity.push_back(p);
                }
        set->plans.resize(set->mu.size());
        const auto rule = bfly::quadrature::build_rule(0, l, bfly::legendre::Parity::even);
        parallel_for(static_cast<std::int64_t>(set->plans.size()), nthreads, [&](std::int64_t i) {
            GlRowSource src(set->mu[i], set->parity[i], rule,
                            chain_cols(l, set->mu[i], set->parity[i]));
            set->plans[i] = bfly::build_plan(src, eps, bw);
        });
        return set.release();
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

std::int64_t bref_planset_size(void* s) {
    return static_cast<std::int64_t>(static_cast<PlanSet*>(s)->plans.size());
}

void* bref_planset_plan(void* s, std::int64_t i) { return &static_cast<PlanSet*>(s)->plans[i]; }

void bref_planset_free(void* s) { delete static_cast<PlanSet*>(s); }

// For each plan i: nrhs[i] reference apply calls.  Input of plan i is the
// column-major block in + in_off[i] with leading dimension = the plan's input
// length; output likewise at out + out_off[i].  Returns the wall seconds.
double bref_planset_apply(void* s, int transpose, const double* in, const std::int64_t* in_off,
                          double* out, const std::int64_t* out_off, const int* nrhs,
                          int nthreads) {
    try {
        auto& set = *static_cast<PlanSet*>(s);
        const auto t0 = std::chrono::steady_clock::now();
        parallel_for(static_cast<std::int64_t>(set.plans.size()), nthreads, [&](std::int64_t i) {
            const auto& p = set.plans[i];
            const Eigen::Index n_in = static_cast<Eigen::Index>(transpose ? p.n_rows : p.n_cols);
            const Eigen::Index n_out = static_cast<Eigen::Index>(transpose ? p.n_cols : p.n_rows);
            for (int r = 0; r < nrhs[i]; ++r) {
                Eigen::VectorXd v(n_in);
                std::memcpy(v.data(), in + in_off[i] + r * n_in, sizeof(double) * static_cast<std::size_t>(n_in));
                const Eigen::VectorXd y = transpose ? bfly::apply_transpose(p, v) : bfly::apply(p, v);
                std::memcpy(out + out_off[i] + r * n_out, y.data(), sizeof(double) * static_cast<std::size_t>(n_out));
            }
        });
        return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    } catch (const std::exception& e) {
        fail(e);
        return -1.0;
    }
}

}  // extern "C"
