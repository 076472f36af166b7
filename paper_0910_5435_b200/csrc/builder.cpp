// Host precompute for GL-row butterfly plans (see builder.hpp).
#include "builder.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <exception>
#include <limits>
#include <mutex>
#include <numeric>
#include <thread>

namespace bfb {

// ---------------------------------------------------------------------------
// Gauss-Legendre nodes: Newton on P_{2l} from Tricomi-style initial guesses.
// The l positive nodes of the degree-2l rule, with rho = 2 w.
GlRule gauss_legendre_positive(int l) {
    if (l < 1) throw std::invalid_argument("gauss_legendre_positive: l must be >= 1");
    const int n = 2 * l;
    GlRule r;
    r.nodes.resize(static_cast<std::size_t>(l));
    r.rho.resize(static_cast<std::size_t>(l));
    const double pi = 3.14159265358979323846;
    for (int i = 0; i < l; ++i) {
        // i-th positive root counted from the pole: theta_i ~ pi (i + 3/4) / (n + 1/2).
        double x = std::cos(pi * (i + 0.75) / (n + 0.5));
        double dp = 0.0;
        for (int it = 0; it < 100; ++it) {
            double p0 = 1.0, p1 = x;
            for (int k = 1; k < n; ++k) {
                const double p2 = ((2.0 * k + 1.0) * x * p1 - k * p0) / (k + 1.0);
                p0 = p1;
                p1 = p2;
            }
            dp = n * (x * p1 - p0) / (x * x - 1.0);
            const double dx = p1 / dp;
            x -= dx;
            if (std::abs(dx) <= 1e-17 * std::max(1.0, std::abs(x)) && it > 1) break;
        }
        // Derivative at the converged node for the weight.
        double p0 = 1.0, p1 = x;
        for (int k = 1; k < n; ++k) {
            const double p2 = ((2.0 * k + 1.0) * x * p1 - k * p0) / (k + 1.0);
            p0 = p1;
            p1 = p2;
        }
        dp = n * (x * p1 - p0) / (x * x - 1.0);
        const double w = 2.0 / ((1.0 - x) * (1.0 + x) * dp * dp);
        // Stored ascending: the root nearest the pole is the largest.
        r.nodes[static_cast<std::size_t>(l - 1 - i)] = x;
        r.rho[static_cast<std::size_t>(l - 1 - i)] = 2.0 * w;
    }
    return r;
}

// ---------------------------------------------------------------------------
// Legendre columns with per-row binary exponents.
namespace {

constexpr double kBig = 0x1p+256;
constexpr double kSmall = 0x1p-256;

// mantissa * 2^exp with |mantissa| in [0.5, 1)
struct Wide {
    double m = 0.0;
    std::int64_t e = 0;
    static Wide of(double v) {
        Wide w;
        if (v != 0.0) {
            int ee;
            w.m = std::frexp(v, &ee);
            w.e = ee;
        }
        return w;
    }
    Wide operator*(const Wide& o) const {
        if (m == 0.0 || o.m == 0.0) return Wide{};
        Wide w = of(m * o.m);
        w.e += e + o.e;
        return w;
    }
};

Wide wide_pow(Wide b, std::int64_t p) {
    Wide r = Wide::of(1.0);
    while (p > 0) {
        if (p & 1) r = r * b;
        b = b * b;
        p >>= 1;
    }
    return r;
}

}  // namespace

LegendreColumns::LegendreColumns(int mu, int parity, const GlRule& rule, std::int64_t n_cols)
    : mu_(mu), parity_(parity), n_cols_(n_cols), x_(rule.nodes) {
    if (mu < 0) throw std::invalid_argument("LegendreColumns: order must be nonnegative");
    sqrt_rho_.reserve(rule.rho.size());
    for (double r : rule.rho) sqrt_rho_.push_back(std::sqrt(r));
    // c_mu = (1/sqrt 2) prod_{k=1..mu} sqrt((2k+1)/(2k)), kept wide.
    Wide c = Wide::of(1.0 / std::sqrt(2.0));
    for (int k = 1; k <= mu; ++k) c = c * Wide::of(std::sqrt((2.0 * k + 1.0) / (2.0 * k)));
    st_.resize(x_.size());
    for (std::size_t i = 0; i < x_.size(); ++i) {
        const double x = x_[i];
        // Pbar^mu_mu(x) = c_mu (1 - x^2)^{mu/2}
        const double s2 = (1.0 - x) * (1.0 + x);
        Wide seed = c * wide_pow(Wide::of(s2), mu / 2);
        if (mu & 1) seed = seed * Wide::of(std::sqrt(s2));
        Row& r = st_[i];
        r.prev = 0.0;
        r.cur = seed.m;
        r.exp = seed.e;
    }
    degree_ = mu;
}

// Pbar_{k+1} = (x Pbar_k - alpha_k Pbar_{k-1}) / alpha_{k+1},
// alpha_k = sqrt((k^2 - mu^2) / (4k^2 - 1)).
void LegendreColumns::step(Row& r, double x, int k) const {
    const double kk = static_cast<double>(k), m2 = static_cast<double>(mu_) * mu_;
    const double a_k = (k == mu_) ? 0.0 : std::sqrt((kk * kk - m2) / (4.0 * kk * kk - 1.0));
    const double k1 = kk + 1.0;
    const double inv_a_k1 = std::sqrt((4.0 * k1 * k1 - 1.0) / (k1 * k1 - m2));
    const double nxt = (x * r.cur - a_k * r.prev) * inv_a_k1;
    r.prev = r.cur;
    r.cur = nxt;
    const double mag = std::max(std::abs(nxt), std::abs(r.prev));
    if (mag > kBig) {
        r.prev *= kSmall;
        r.cur *= kSmall;
        r.exp += 256;
    } else if (mag < kSmall && mag != 0.0) {
        r.prev *= kBig;
        r.cur *= kBig;
        r.exp -= 256;
    }
}

void LegendreColumns::next(Mat& out) {
    if (out.rows != rows() || next_col_ + out.cols > n_cols_)
        throw std::out_of_range("LegendreColumns: past the last column");
    for (std::int64_t j = 0; j < out.cols; ++j) {
        const int target = mu_ + 2 * static_cast<int>(next_col_ + j) + parity_;
        const int steps = target - degree_;
        for (std::size_t i = 0; i < x_.size(); ++i) {
            Row& r = st_[i];
            for (int s = 0; s < steps; ++s) step(r, x_[i], degree_ + s);
            const double v = (r.exp < -1200) ? 0.0 : std::ldexp(r.cur, static_cast<int>(std::max<std::int64_t>(r.exp, -1200)));
            out(static_cast<std::int64_t>(i), j) = sqrt_rho_[i] * v;
        }
        degree_ = target;
    }
    next_col_ += out.cols;
}

// ---------------------------------------------------------------------------
// Interpolative decomposition by column-pivoted Householder QR.
namespace {

double sq_norm(const double* v, std::int64_t n) {
    double s = 0.0;
    for (std::int64_t i = 0; i < n; ++i) s += v[i] * v[i];
    return s;
}

// Apply the reflector (I - beta v v^T), v = [1-alpha..; tail], to columns
// [c0, c1) of w restricted to rows [j, m).
void reflect(Mat& w, std::int64_t j, const std::vector<double>& v, double beta, std::int64_t c0,
             std::int64_t c1) {
    const std::int64_t len = w.rows - j;
    for (std::int64_t c = c0; c < c1; ++c) {
        double* col = w.col(c) + j;
        double d = 0.0;
        for (std::int64_t i = 0; i < len; ++i) d += v[static_cast<std::size_t>(i)] * col[i];
        d *= beta;
        for (std::int64_t i = 0; i < len; ++i) col[i] -= d * v[static_cast<std::size_t>(i)];
    }
}

// One Householder step on column j of w (rows j..m): zero below the diagonal
// and update columns j+1..n-1.
void householder_step(Mat& w, std::int64_t j, std::vector<double>& v) {
    const std::int64_t len = w.rows - j;
    double* cj = w.col(j) + j;
    const double sigma = std::sqrt(sq_norm(cj, len));
    if (sigma == 0.0) return;
    const double alpha = cj[0] >= 0.0 ? -sigma : sigma;
    v.assign(cj, cj + len);
    v[0] -= alpha;
    const double vn2 = sq_norm(v.data(), len);
    if (vn2 > 0.0) reflect(w, j, v, 2.0 / vn2, j + 1, w.cols);
    cj[0] = alpha;
    std::fill(cj + 1, cj + len, 0.0);
}

// R11^{-1} R12 from the top k rows of the factored w (zero pivots -> 0 rows).
Mat solve_upper(const Mat& w, std::int64_t k) {
    Mat t(k, w.cols - k);
    for (std::int64_t c = 0; c < t.cols; ++c) {
        const double* rhs = w.col(k + c);
        for (std::int64_t i = k - 1; i >= 0; --i) {
            double s = rhs[i];
            for (std::int64_t q = i + 1; q < k; ++q) s -= w(i, q) * t(q, c);
            const double d = w(i, i);
            t(i, c) = d == 0.0 ? 0.0 : s / d;
        }
    }
    return t;
}

Mat permuted(const Mat& block, const std::vector<std::int64_t>& perm) {
    Mat w(block.rows, block.cols);
    for (std::int64_t j = 0; j < block.cols; ++j)
        std::copy(block.col(perm[static_cast<std::size_t>(j)]),
                  block.col(perm[static_cast<std::size_t>(j)]) + block.rows, w.col(j));
    return w;
}

}  // namespace

IdResult interpolative_decomposition(const Mat& block, double eps) {
    if (!(eps > 0.0)) throw std::invalid_argument("id_adaptive: epsilon must be positive");
    const std::int64_t m = block.rows, n = block.cols;
    if (m < 1 || n < 1) throw std::invalid_argument("id_adaptive: empty block");
    IdResult res;
    const double fro = std::sqrt(sq_norm(block.a.data(), m * n));
    if (fro == 0.0) {
        res.selected = {0};
        res.t = Mat(1, n - 1);
        return res;
    }
    const double threshold = eps * fro / std::sqrt(static_cast<double>(n));
    const double limit = eps * fro;

    Mat w = block;
    std::vector<std::int64_t> perm(static_cast<std::size_t>(n));
    std::iota(perm.begin(), perm.end(), 0);
    std::vector<double> cn(static_cast<std::size_t>(n)), cref(static_cast<std::size_t>(n));
    for (std::int64_t j = 0; j < n; ++j) cn[j] = cref[j] = std::sqrt(sq_norm(w.col(j), m));
    std::vector<double> v;

    auto argmax_from = [&](std::int64_t j) {
        std::int64_t p = j;
        for (std::int64_t q = j + 1; q < n; ++q)
            if (cn[q] > cn[p]) p = q;
        return p;
    };

    const std::int64_t kcap = std::min(m, n);
    std::int64_t k = 0;
    while (k < kcap) {
        std::int64_t piv = argmax_from(k);
        if (cn[piv] <= threshold && k > 0) {
            // Candidate stop: certify with exactly recomputed trailing norms.
            double tail2 = 0.0;
            for (std::int64_t q = k; q < n; ++q) {
                const double t = std::sqrt(sq_norm(w.col(q) + k, m - k));
                cn[q] = cref[q] = t;
                tail2 += t * t;
            }
            if (std::sqrt(tail2) <= limit) break;
            piv = argmax_from(k);
        }
        if (piv != k) {
            std::swap_ranges(w.col(k), w.col(k) + m, w.col(piv));
            std::swap(cn[k], cn[piv]);
            std::swap(cref[k], cref[piv]);
            std::swap(perm[k], perm[piv]);
        }
        householder_step(w, k, v);
        // Downdate the remaining column norms (LAPACK-style cancellation guard).
        for (std::int64_t q = k + 1; q < n; ++q) {
            if (cn[q] == 0.0) continue;
            double t = w(k, q) / cn[q];
            t = std::max(0.0, (1.0 - t) * (1.0 + t));
            const double ratio = cn[q] / cref[q];
            if (t * ratio * ratio <= 1e-14) {
                cn[q] = cref[q] = std::sqrt(sq_norm(w.col(q) + k + 1, m - k - 1));
            } else {
                cn[q] *= std::sqrt(t);
            }
        }
        ++k;
    }

    Mat t = solve_upper(w, k);
    // Refine toward |T| <= 2 by exchanging a skeleton column with the
    // non-skeleton column of the largest coefficient (bounded passes).
    for (int pass = 0; pass < 64 && t.cols > 0; ++pass) {
        std::int64_t bi = 0, bj = 0;
        double worst = -1.0;
        for (std::int64_t c = 0; c < t.cols; ++c)
            for (std::int64_t i = 0; i < t.rows; ++i) {
                const double a = std::abs(t(i, c));
                if (a > worst) {
                    worst = a;
                    bi = i;
                    bj = c;
                }
            }
        if (worst <= 2.0) break;
        std::swap(perm[static_cast<std::size_t>(bi)], perm[static_cast<std::size_t>(k + bj)]);
        w = permuted(block, perm);
        for (std::int64_t j = 0; j < k; ++j) householder_step(w, j, v);
        t = solve_upper(w, k);
    }

    res.selected.assign(perm.begin(), perm.begin() + k);
    // Columns of T in ascending input order.
    std::vector<std::int64_t> order(static_cast<std::size_t>(n - k));
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(),
              [&](std::int64_t a, std::int64_t b) { return perm[k + a] < perm[k + b]; });
    res.t = Mat(k, n - k);
    for (std::int64_t c = 0; c < n - k; ++c)
        std::copy(t.col(order[c]), t.col(order[c]) + k, res.t.col(c));
    return res;
}

// ---------------------------------------------------------------------------
// Depth-first butterfly construction.
namespace {

struct Span {
    std::int64_t begin, count;
};

struct StripeData {
    Mat skeleton;                  // stripe rows x rank, verbatim source columns
    std::vector<double> col_norm;  // full-column norms behind each skeleton column
};

struct PendingBlock {
    int level = 1;
    std::vector<StripeData> stripes;
};

Mat take_rows(const Mat& a, std::int64_t r0, std::int64_t nr) {
    Mat out(nr, a.cols);
    for (std::int64_t j = 0; j < a.cols; ++j) std::copy(a.col(j) + r0, a.col(j) + r0 + nr, out.col(j));
    return out;
}

Mat take_cols(const Mat& a, const std::vector<std::uint64_t>& idx) {
    Mat out(a.rows, static_cast<std::int64_t>(idx.size()));
    for (std::size_t j = 0; j < idx.size(); ++j)
        std::copy(a.col(static_cast<std::int64_t>(idx[j])), a.col(static_cast<std::int64_t>(idx[j])) + a.rows,
                  out.col(static_cast<std::int64_t>(j)));
    return out;
}

class DepthFirstBuilder {
public:
    DepthFirstBuilder(std::int64_t rows, std::int64_t cols, double eps, std::int64_t width)
        : rows_(rows), cols_(cols), eps_(eps), width_(width) {
        levels_.push_back({});
        levels_.push_back({Span{0, rows}});
    }

    ButterflyPlan run(const ColumnFeed& feed) {
        const auto t0 = std::chrono::steady_clock::now();
        plan_.n_rows = static_cast<std::uint64_t>(rows_);
        plan_.n_cols = static_cast<std::uint64_t>(cols_);
        plan_.epsilon = eps_;
        plan_.block_width = static_cast<std::uint64_t>(width_);
        for (std::int64_t c = 0; c < cols_; c += width_) {
            add_leaf(feed, c, std::min(width_, cols_ - c));
            while (stack_.size() >= 2 && stack_[stack_.size() - 2].level == stack_.back().level)
                if (!combine(false)) break;
        }
        // Ragged tail: promote the shallower block until levels align, merge.
        while (stack_.size() >= 2) {
            const bool aligned = stack_[stack_.size() - 2].level == stack_.back().level;
            if (!combine(!aligned)) break;
        }
        close();
        plan_.t_comp_seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return std::move(plan_);
    }

private:
    const std::vector<Span>& rows_at(int level) {
        while (static_cast<int>(levels_.size()) <= level) {
            std::vector<Span> nxt;
            for (const Span& s : levels_.back()) {
                const std::int64_t top = (s.count + 1) / 2;
                nxt.push_back(Span{s.begin, top});
                nxt.push_back(Span{s.begin + top, s.count - top});
            }
            levels_.push_back(std::move(nxt));
        }
        return levels_[static_cast<std::size_t>(level)];
    }

    void peak(std::uint64_t transient) {
        peak_ = std::max(peak_, plan_words_ + pending_words_ + transient);
    }

    void add_leaf(const ColumnFeed& feed, std::int64_t c0, std::int64_t nc) {
        Mat raw(rows_, nc);
        feed(raw);
        peak(raw.words());
        IdResult id = interpolative_decomposition(raw, eps_);
        PendingBlock blk;
        StripeData sd;
        sd.skeleton = take_cols(raw, id.selected);
        for (auto s : id.selected)
            sd.col_norm.push_back(std::sqrt(sq_norm(raw.col(static_cast<std::int64_t>(s)), rows_)));
        PlanEvent ev;
        ev.kind = EventKind::leaf;
        ev.col_begin = static_cast<std::uint64_t>(c0);
        ev.col_count = static_cast<std::uint64_t>(nc);
        plan_words_ += id.t.words();
        pending_words_ += sd.skeleton.words();
        peak(raw.words());
        ev.ids.push_back(StripeId{std::move(id.selected), std::move(id.t)});
        blk.stripes.push_back(std::move(sd));
        plan_.events.push_back(std::move(ev));
        stack_.push_back(std::move(blk));
    }

    struct Trial {
        PlanEvent ev;
        PendingBlock out;
        std::uint64_t skel_words = 0, interp_words = 0;
    };

    // Compress one row half; false when its rank crowds its rows (>90 %).
    bool compress_half(Trial& tr, const Mat& half, const std::vector<double>& norms) {
        const double bn = std::sqrt(sq_norm(half.a.data(), half.rows * half.cols));
        double eps = eps_;
        if (bn > 0.0) {
            double nn = 0.0;
            for (double v : norms) nn += v * v;
            eps = std::min(0.5, std::max(eps_, eps_ * std::sqrt(nn) / bn));
        }
        IdResult id = interpolative_decomposition(half, eps);
        if (10 * static_cast<std::int64_t>(id.selected.size()) > 9 * half.rows) return false;
        StripeData sd;
        sd.skeleton = take_cols(half, id.selected);
        for (auto s : id.selected) sd.col_norm.push_back(norms[s]);
        tr.interp_words += id.t.words();
        tr.skel_words += sd.skeleton.words();
        peak(tr.skel_words + tr.interp_words);
        tr.ev.ids.push_back(StripeId{std::move(id.selected), std::move(id.t)});
        tr.out.stripes.push_back(std::move(sd));
        return true;
    }

    bool combine(bool promote) {
        PendingBlock& top = stack_.back();
        const int lv = top.level + 1;
        if (lv > cap_) return false;
        const std::vector<Span>& part = rows_at(lv);
        std::int64_t thinnest = rows_;
        for (const Span& s : part) thinnest = std::min(thinnest, s.count);
        if (thinnest < width_) {
            cap_ = top.level;
            return false;
        }
        const PendingBlock& a = promote ? top : stack_[stack_.size() - 2];
        const PendingBlock* b = promote ? nullptr : &top;

        Trial tr;
        tr.ev.kind = promote ? EventKind::promote : EventKind::merge;
        tr.out.level = lv;
        bool ok = true;
        for (std::size_t s = 0; s < a.stripes.size() && ok; ++s) {
            const StripeData& sa = a.stripes[s];
            Mat cat;
            std::vector<double> norms = sa.col_norm;
            if (b) {
                const StripeData& sb = b->stripes[s];
                tr.ev.left_ranks.push_back(static_cast<std::uint64_t>(sa.skeleton.cols));
                cat = Mat(sa.skeleton.rows, sa.skeleton.cols + sb.skeleton.cols);
                std::copy(sa.skeleton.a.begin(), sa.skeleton.a.end(), cat.a.begin());
                std::copy(sb.skeleton.a.begin(), sb.skeleton.a.end(), cat.a.begin() + sa.skeleton.a.size());
                norms.insert(norms.end(), sb.col_norm.begin(), sb.col_norm.end());
                peak(tr.skel_words + tr.interp_words + cat.words());
            } else {
                cat = sa.skeleton;
            }
            const std::int64_t top_rows = part[2 * s].count;
            ok = compress_half(tr, take_rows(cat, 0, top_rows), norms) &&
                 compress_half(tr, take_rows(cat, top_rows, cat.rows - top_rows), norms);
        }
        std::uint64_t freed = 0;
        for (const auto& sd : a.stripes) freed += sd.skeleton.words();
        if (b)
            for (const auto& sd : b->stripes) freed += sd.skeleton.words();
        if (!ok || 10 * (tr.skel_words + tr.interp_words) > 17 * freed) {
            cap_ = top.level;
            return false;
        }
        pending_words_ += tr.skel_words;
        peak(tr.interp_words);
        pending_words_ -= freed;
        plan_words_ += tr.interp_words;
        stack_.pop_back();
        if (!promote) stack_.pop_back();
        plan_.events.push_back(std::move(tr.ev));
        stack_.push_back(std::move(tr.out));
        return true;
    }

    void close() {
        plan_.levels = 0;
        for (PendingBlock& blk : stack_) {
            plan_.levels = std::max<std::uint64_t>(plan_.levels, static_cast<std::uint64_t>(blk.level));
            const std::vector<Span>& part = rows_at(blk.level);
            std::vector<RootStripe> group;
            for (std::size_t s = 0; s < blk.stripes.size(); ++s) {
                RootStripe rs;
                rs.row_begin = static_cast<std::uint64_t>(part[s].begin);
                rs.row_count = static_cast<std::uint64_t>(part[s].count);
                rs.skeleton = std::move(blk.stripes[s].skeleton);
                group.push_back(std::move(rs));
            }
            plan_.root_groups.push_back(std::move(group));
        }
        stack_.clear();
        plan_.stored_words = plan_.count_stored_words();
        plan_.m_max_words = std::max(peak_, plan_.stored_words);
    }

    std::int64_t rows_, cols_;
    double eps_;
    std::int64_t width_;
    ButterflyPlan plan_;
    std::vector<PendingBlock> stack_;
    std::vector<std::vector<Span>> levels_;
    int cap_ = std::numeric_limits<int>::max();
    std::uint64_t plan_words_ = 0, pending_words_ = 0, peak_ = 0;
};

}  // namespace

ButterflyPlan build_plan(std::int64_t n_rows, std::int64_t n_cols, const ColumnFeed& feed, double eps,
                         std::int64_t block_width) {
    if (!(eps > 0.0)) throw std::invalid_argument("build_plan: epsilon must be positive");
    if (block_width < 2) throw std::invalid_argument("build_plan: block_width must be >= 2");
    if (n_rows < 1 || n_cols < 1) throw std::invalid_argument("build_plan: empty source");
    return DepthFirstBuilder(n_rows, n_cols, eps, block_width).run(feed);
}

ButterflyPlan build_glrow_plan(int l, int mu, int parity, double eps, std::int64_t block_width,
                               const GlRule& rule) {
    const std::int64_t nc = chain_cols(l, mu, parity);
    LegendreColumns cols(mu, parity, rule, nc);
    return build_plan(cols.rows(), nc, [&](Mat& out) { cols.next(out); }, eps, block_width);
}

std::vector<ButterflyPlan> build_glrow_planset(int l, int mu_begin, int mu_end, double eps,
                                               std::int64_t block_width, int threads,
                                               std::vector<PlanKey>* keys_out, const GlRule* rule_in) {
    std::vector<PlanKey> keys;
    for (int mu = mu_begin; mu < mu_end; ++mu)
        for (int p = 0; p < 2; ++p)
            if (chain_cols(l, mu, p) > 0) keys.push_back(PlanKey{mu, p});
    const GlRule rule = rule_in ? *rule_in : gauss_legendre_positive(l);
    if (static_cast<int>(rule.nodes.size()) != l || static_cast<int>(rule.rho.size()) != l)
        throw std::invalid_argument("planset: the rule must have l nodes and weights");
    std::vector<ButterflyPlan> plans(keys.size());
    // Largest plans first (cost falls with mu) for a balanced pool.
    std::atomic<std::size_t> next{0};
    std::exception_ptr err;
    std::mutex mu_err;
    auto worker = [&] {
        for (;;) {
            const std::size_t i = next.fetch_add(1);
            if (i >= keys.size()) return;
            try {
                plans[i] = build_glrow_plan(l, keys[i].mu, keys[i].parity, eps, block_width, rule);
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu_err);
                if (!err) err = std::current_exception();
            }
        }
    };
    threads = std::max(1, threads);
    std::vector<std::thread> pool;
    for (int t = 1; t < threads; ++t) pool.emplace_back(worker);
    worker();
    for (auto& th : pool) th.join();
    if (err) std::rethrow_exception(err);
    if (keys_out) *keys_out = std::move(keys);
    return plans;
}

}  // namespace bfb
