// Reference-side drop-in check: code written against the
// reference's bfly:: API builds plans with the reference (oracle/_ref, its own
// sources) and applies them through include/bfly_b200.hpp.
//   dropin_check cpu : BFLY1 hand-over and plan statistics (no device needed)
//   dropin_check gpu : DevicePlan::apply / apply_transpose vs bfly::apply on
//                      the same plans, plus the reference's error behaviour
#include <cmath>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "bfly/column_source.hpp"
#include "bfly/rng.hpp"
#include "bfly/transform.hpp"
#include "bfly_b200.hpp"

namespace {

int failures = 0;

void expect(bool ok, const std::string& what) {
    std::printf("%s %s\n", ok ? "ok  " : "FAIL", what.c_str());
    if (!ok) ++failures;
}

Eigen::MatrixXd kernel_matrix(Eigen::Index n) {
    Eigen::MatrixXd a(n, n);
    for (Eigen::Index j = 0; j < n; ++j)
        for (Eigen::Index i = 0; i < n; ++i)
            a(i, j) = std::cos(8.0 * M_PI * (i + 0.5) * (j + 0.5) / static_cast<double>(n)) / std::sqrt(double(n));
    return a;
}

double rel(const Eigen::VectorXd& a, const Eigen::VectorXd& b) { return (a - b).norm() / b.norm(); }

}  // namespace

int main(int argc, char** argv) {
    const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
    bfly::DenseColumnSource src(kernel_matrix(300));
    const bfly::ButterflyPlan dense = bfly::build_plan(src, 1e-13, 60);
    const auto tp = bfly::transform::build_transform(3, 64, bfly::legendre::Parity::even, 1e-12);

    // BFLY1 hand-over: the product parses the reference's bytes and agrees on the statistics.
    for (const bfly::ButterflyPlan* p : {&dense, &tp.plan}) {
        const std::string bytes = bfly::b200::to_bfly1(*p);
        bfly_plan_t h = nullptr;
        bfly::b200::check(bfly_plan_from_bfly1(reinterpret_cast<const std::uint8_t*>(bytes.data()), bytes.size(), &h));
        std::int64_t info[10] = {};
        bfly::b200::check(bfly_plan_info(h, info, nullptr));
        const bfly::PlanStats st = bfly::plan_stats(*p);
        expect(info[0] == p->n_rows && info[1] == p->n_cols, "shape after BFLY1 hand-over");
        expect(static_cast<std::uint64_t>(info[3]) == st.stored_words, "stored words match plan_stats");
        std::vector<std::uint8_t> back(bytes.size());
        std::size_t n = 0;
        bfly::b200::check(bfly_plan_to_bfly1(h, back.data(), back.size(), &n));
        expect(n == bytes.size() && std::memcmp(back.data(), bytes.data(), n) == 0, "BFLY1 round trip byte-exact");
        bfly_plan_destroy(h);
    }

    if (gpu) {
        bfly::CounterRng rng(17);
        for (const bfly::ButterflyPlan* p : {&dense, &tp.plan}) {
            bfly::b200::DevicePlan dp(*p);
            const Eigen::VectorXd v = rng.vector(p->n_cols);
            const Eigen::VectorXd w = rng.vector(p->n_rows);
            expect(rel(dp.apply(v), bfly::apply(*p, v)) <= 1e-14, "apply matches bfly::apply");
            expect(rel(dp.apply_transpose(w), bfly::apply_transpose(*p, w)) <= 1e-14,
                   "apply_transpose matches bfly::apply_transpose");
            Eigen::MatrixXd X(p->n_cols, 5);
            for (int c = 0; c < 5; ++c) X.col(c) = rng.vector(p->n_cols);
            const Eigen::MatrixXd Y = dp.apply(X, false);
            double err = 0;
            for (int c = 0; c < 5; ++c) err = std::max(err, rel(Y.col(c), bfly::apply(*p, X.col(c))));
            expect(err <= 1e-14, "batched apply matches column by column");
            std::string ref_msg, our_msg;
            try {
                bfly::apply(*p, Eigen::VectorXd::Zero(p->n_cols - 1));
            } catch (const std::invalid_argument& e) {
                ref_msg = e.what();
            }
            try {
                dp.apply(Eigen::VectorXd::Zero(p->n_cols - 1));
            } catch (const std::invalid_argument& e) {
                our_msg = e.what();
            }
            expect(!ref_msg.empty() && ref_msg == our_msg, "length error: same type and message (" + our_msg + ")");
            std::string ref_tmsg, our_tmsg;
            try {
                bfly::apply_transpose(*p, Eigen::VectorXd::Zero(p->n_rows + 1));
            } catch (const std::invalid_argument& e) {
                ref_tmsg = e.what();
            }
            try {
                dp.apply_transpose(Eigen::VectorXd::Zero(p->n_rows + 1));
            } catch (const std::invalid_argument& e) {
                our_tmsg = e.what();
            }
            expect(!ref_tmsg.empty() && ref_tmsg == our_tmsg,
                   "transpose length error: same type and message (" + our_tmsg + ")");
            std::string our_bmsg;
            try {
                dp.apply(Eigen::MatrixXd::Zero(p->n_rows + 1, 2), true);
            } catch (const std::invalid_argument& e) {
                our_bmsg = e.what();
            }
            expect(our_bmsg.rfind("apply_transpose: vector length", 0) == 0,
                   "batched transpose length error names apply_transpose (" + our_bmsg + ")");
        }
    }
    std::printf("%s\n", failures ? "FAILED" : "PASSED");
    return failures ? 1 : 0;
}
