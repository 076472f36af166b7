// bfly_b200.hpp — the reference-side binding: C++ adapters over the C ABI in
// bfly_b200.h for code written against the reference's bfly:: API
// (/root/reference/proj/include/bfly).  Header-only; needs the reference's
// headers (bfly/butterfly.hpp, bfly/serialize.hpp) and Eigen on the include
// path, and links libbfly_b200.so.  See INTEGRATION.md.
//
//   reference call (include/bfly/butterfly.hpp:93-96)      drop-in
//   bfly::apply(plan, v)                                 bfly::b200::DevicePlan(plan).apply(v)
//   bfly::apply_transpose(plan, w)                       bfly::b200::DevicePlan(plan).apply_transpose(w)
//   transform::forward / inverse (transform.hpp:60-66)   same, on tp.plan
//
// A DevicePlan uploads the plan once (as the reference's own BFLY1 bytes,
// serialize.hpp:44-45) and keeps it resident; error codes are rethrown as the
// reference's exception types (std::invalid_argument with the reference's
// messages, bfly::SerializationError, std::runtime_error).
#ifndef BFLY_B200_HPP
#define BFLY_B200_HPP

#include <Eigen/Dense>

#include <cstdint>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "bfly/butterfly.hpp"
#include "bfly/serialize.hpp"
#include "bfly_b200.h"

namespace bfly {
namespace b200 {

inline void check(int rc) {
    if (rc == BFLY_OK) return;
    const std::string msg = bfly_last_error();
    if (rc == BFLY_EINVAL) throw std::invalid_argument(msg);
    if (rc == BFLY_ESERIAL) throw bfly::SerializationError(msg, 0);
    throw std::runtime_error(msg);
}

inline std::string to_bfly1(const ButterflyPlan& plan) {
    std::ostringstream os(std::ios::binary);
    save_plan(plan, os);
    return os.str();
}

// One reference plan, resident on a GPU.
class DevicePlan {
public:
    explicit DevicePlan(const ButterflyPlan& plan, int device = 0) {
        const std::string bytes = to_bfly1(plan);
        check(bfly_plan_from_bfly1(reinterpret_cast<const std::uint8_t*>(bytes.data()), bytes.size(), &plan_));
        const int rc = bfly_dev_planset_create(&plan_, 1, device, &set_);
        if (rc != BFLY_OK) {
            bfly_plan_destroy(plan_);
            check(rc);
        }
        std::int64_t info[10] = {};
        check(bfly_plan_info(plan_, info, nullptr));
        rows_ = info[0];
        cols_ = info[1];
    }
    DevicePlan(const DevicePlan&) = delete;
    DevicePlan& operator=(const DevicePlan&) = delete;
    ~DevicePlan() {
        bfly_dev_planset_destroy(set_);
        bfly_plan_destroy(plan_);
    }

    std::int64_t rows() const { return rows_; }
    std::int64_t cols() const { return cols_; }

    // bfly::apply: A v (host vectors; copies to and from the device inside).
    Eigen::VectorXd apply(const Eigen::Ref<const Eigen::VectorXd>& v) const { return run(v, false); }
    // bfly::apply_transpose: A^T w.
    Eigen::VectorXd apply_transpose(const Eigen::Ref<const Eigen::VectorXd>& w) const { return run(w, true); }

    // Batched: columns of X are independent right-hand sides.
    Eigen::MatrixXd apply(const Eigen::MatrixXd& X, bool transpose) const {
        const std::int64_t n_in = transpose ? rows_ : cols_, n_out = transpose ? cols_ : rows_;
        if (X.rows() != n_in)
            throw std::invalid_argument(std::string(transpose ? "apply_transpose" : "apply") + ": vector length " +
                                        std::to_string(X.rows()) + ", expected " + std::to_string(n_in));
        Eigen::MatrixXd Y(n_out, X.cols());
        check(bfly_host_apply(set_, transpose ? 1 : 0, X.data(), n_in * X.cols(), Y.data(), n_out * X.cols(),
                              static_cast<int>(X.cols())));
        return Y;
    }

private:
    Eigen::VectorXd run(const Eigen::Ref<const Eigen::VectorXd>& v, bool transpose) const {
        const std::int64_t n_in = transpose ? rows_ : cols_, n_out = transpose ? cols_ : rows_;
        // same type and message as the reference (src/butterfly.cpp:386-389, :446-449)
        if (v.size() != n_in)
            throw std::invalid_argument(std::string(transpose ? "apply_transpose" : "apply") + ": vector length " +
                                        std::to_string(v.size()) + ", expected " + std::to_string(n_in));
        const Eigen::VectorXd in = v;  // contiguous copy
        Eigen::VectorXd out(n_out);
        check(bfly_host_apply(set_, transpose ? 1 : 0, in.data(), n_in, out.data(), n_out, 1));
        return out;
    }

    bfly_plan_t plan_ = nullptr;
    bfly_planset_t set_ = nullptr;
    std::int64_t rows_ = 0, cols_ = 0;
};

}  // namespace b200
}  // namespace bfly

#endif
