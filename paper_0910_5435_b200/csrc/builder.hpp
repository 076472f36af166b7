// Host precompute: Gauss-Legendre rows, Legendre columns, interpolative
// decompositions and the depth-first butterfly construction.
//
// Provenance.  gauss_legendre_positive and LegendreColumns are this library's
// own code.  The interpolative decomposition (builder.cpp, "Interpolative
// decomposition") is a PORT of the reference's id.cpp:31-235 (pivoted_qr,
// interpolation_coefficients, refactor, finish_id, id_adaptive) from Eigen to
// the plain column-major Mat of plan.hpp, and DepthFirstBuilder is a PORT of
// the reference PlanBuilder (src/butterfly.cpp:95-382) with the same
// tolerance rule, refusal rules and ragged-tail handling: the precompute may
// stay the reference's algorithm (north_star), and the port exists so the
// library can build GL-row plan sets threaded and without Eigen.  Plans it
// produces have the reference's structure (same ranks / pivots; checked
// against reference-built plans in tests/test_capi.py
// test_own_builder_matches_reference_structure).  The GPU plan builder
// (gpubuild.cu) is the B200-native replacement for the column generation and
// the IDs.
#pragma once

#include <cstdint>
#include <functional>
#include <vector>

#include "plan.hpp"

namespace bfb {

// The l positive Gauss-Legendre nodes of degree 2l (ascending) and
// rho_i = 2 * w_GL,i — what the reference's build_rule(0, l, even) returns
// (reference src/quadrature.cpp:206-255; tests/test_quadrature.cpp:160-168).
struct GlRule {
    std::vector<double> nodes;
    std::vector<double> rho;
};
GlRule gauss_legendre_positive(int l);

// Number of columns of chain p (0 even, 1 odd) at order mu, bandlimit l.
inline std::int64_t chain_cols(int l, int mu, int p) {
    const std::int64_t n = p == 0 ? (2LL * l - mu + 1) / 2 : (2LL * l - mu) / 2;
    return n < 0 ? 0 : n;
}

// Streams the columns A(i, j) = sqrt(rho_i) * Pbar^mu_{mu+2j+p}(x_i) of one
// GL-row plan, a block of columns at a time, with per-row exponent tracking
// so orders in the thousands neither underflow nor overflow.
class LegendreColumns {
public:
    LegendreColumns(int mu, int parity, const GlRule& rule, std::int64_t n_cols);
    std::int64_t rows() const { return static_cast<std::int64_t>(x_.size()); }
    std::int64_t cols() const { return n_cols_; }
    // Fills `out` (rows x out.cols) with the next out.cols columns.
    void next(Mat& out);

private:
    struct Row {
        double prev, cur;   // Pbar_{k-1}, Pbar_k scaled by 2^-exp
        std::int64_t exp;
    };
    void step(Row& r, double x, int k) const;  // advance one degree: k -> k+1
    int mu_, parity_;
    std::int64_t n_cols_, next_col_ = 0;
    int degree_ = 0;  // degree held in Row::cur
    std::vector<double> x_, sqrt_rho_;
    std::vector<Row> st_;
};

// Interpolative decomposition of `block` (reference semantics of id_adaptive,
// include/bfly/id.hpp:35-45): smallest rank whose certified Frobenius residual
// is within eps * ||block||_F, skeleton columns chosen by column-pivoted
// Householder QR, interpolation entries refined toward |T| <= 2.
struct IdResult {
    std::vector<std::uint64_t> selected;  // pivot order
    Mat t;                                // rank x (n - rank), columns in ascending input order
};
IdResult interpolative_decomposition(const Mat& block, double eps);

// Depth-first plan construction over a column stream (the reference's
// build_plan policy, include/bfly/butterfly.hpp:86-91).
using ColumnFeed = std::function<void(Mat& out)>;
ButterflyPlan build_plan(std::int64_t n_rows, std::int64_t n_cols, const ColumnFeed& feed,
                         double eps, std::int64_t block_width);

// GL-row plan for (mu, parity) at bandlimit l.
ButterflyPlan build_glrow_plan(int l, int mu, int parity, double eps, std::int64_t block_width,
                               const GlRule& rule);

// Every non-empty (mu, parity) plan with mu in [mu_begin, mu_end), built on
// `threads` host threads; order: mu ascending, even before odd.  `rule`: the
// caller's quadrature (e.g. the reference's build_rule(0, l, even), so the
// plans sit on exactly the reference's grid); default gauss_legendre_positive.
struct PlanKey {
    int mu, parity;
};
std::vector<ButterflyPlan> build_glrow_planset(int l, int mu_begin, int mu_end, double eps,
                                               std::int64_t block_width, int threads,
                                               std::vector<PlanKey>* keys, const GlRule* rule = nullptr);

}  // namespace bfb
