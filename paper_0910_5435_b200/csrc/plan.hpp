// Host-side butterfly plan: the reference's data structure, held without Eigen.
//
// Field-for-field this is bfly::ButterflyPlan and friends from the reference
// (/root/reference/proj/include/bfly/butterfly.hpp:18-74): a depth-first list
// of leaf / merge / promote events, each carrying the non-identity part of its
// interpolation matrices, followed by the root skeleton groups.  Matrices are
// column-major double arrays exactly as the reference stores them, so a plan
// built by the reference and handed over as BFLY1 bytes (serialize.hpp:14-31)
// and a plan built by this library's own builder are interchangeable.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace bfb {

// Column-major dense matrix.
struct Mat {
    std::int64_t rows = 0;
    std::int64_t cols = 0;
    std::vector<double> a;

    Mat() = default;
    Mat(std::int64_t r, std::int64_t c) : rows(r), cols(c), a(static_cast<std::size_t>(r * c), 0.0) {}
    double& operator()(std::int64_t i, std::int64_t j) { return a[static_cast<std::size_t>(i + j * rows)]; }
    double operator()(std::int64_t i, std::int64_t j) const { return a[static_cast<std::size_t>(i + j * rows)]; }
    double* col(std::int64_t j) { return a.data() + j * rows; }
    const double* col(std::int64_t j) const { return a.data() + j * rows; }
    std::uint64_t words() const { return static_cast<std::uint64_t>(rows * cols); }
};

// One interpolation step: out = z[selected] + interpolation * z[others], with
// `others` the ascending complement of `selected` in [0, inputs).
// (reference include/bfly/butterfly.hpp:18-27)
struct StripeId {
    std::vector<std::uint64_t> selected;  // reference: column_indices (pivot order)
    Mat interpolation;                    // rank x (inputs - rank)

    std::int64_t rank() const { return static_cast<std::int64_t>(selected.size()); }
    std::int64_t inputs() const { return rank() + interpolation.cols; }
    std::vector<std::uint32_t> others() const;
};

enum class EventKind : std::uint8_t { leaf = 0, merge = 1, promote = 2 };

// (reference include/bfly/butterfly.hpp:38-46)
struct PlanEvent {
    EventKind kind = EventKind::leaf;
    std::uint64_t col_begin = 0;            // leaf
    std::uint64_t col_count = 0;            // leaf
    std::vector<std::uint64_t> left_ranks;  // merge: per input stripe
    std::vector<StripeId> ids;              // leaf: 1, merge/promote: 2 per input stripe
};

// (reference include/bfly/butterfly.hpp:48-52)
struct RootStripe {
    std::uint64_t row_begin = 0;
    std::uint64_t row_count = 0;
    Mat skeleton;  // row_count x rank
};

// (reference include/bfly/butterfly.hpp:59-74)
struct ButterflyPlan {
    std::uint64_t n_rows = 0;
    std::uint64_t n_cols = 0;
    double epsilon = 0.0;
    std::uint64_t block_width = 0;
    std::uint64_t levels = 0;
    std::vector<PlanEvent> events;
    std::vector<std::vector<RootStripe>> root_groups;
    std::uint64_t m_max_words = 0;
    std::uint64_t stored_words = 0;
    double t_comp_seconds = 0.0;

    std::uint64_t count_stored_words() const;
    // Structural validation (replays the event stack without arithmetic);
    // throws std::runtime_error with the reference's wording on mismatch.
    void validate() const;
};

struct PlanStats {
    std::uint64_t k_max = 0;
    double k_avg = 0.0;
    double k_sigma = 0.0;
    std::uint64_t id_count = 0;
    std::uint64_t levels = 0;
    std::uint64_t stored_words = 0;
    std::uint64_t m_max_words = 0;
    double t_comp_seconds = 0.0;
};

// Rank statistics (reference src/butterfly.cpp:515-541).
PlanStats plan_stats(const ButterflyPlan& plan);

// ---- BFLY1 container (reference include/bfly/serialize.hpp:14-31) --------
class SerializationError : public std::runtime_error {
public:
    SerializationError(const std::string& what, std::uint64_t offset)
        : std::runtime_error(what + " at byte offset " + std::to_string(offset)), offset_(offset) {}
    std::uint64_t offset() const { return offset_; }

private:
    std::uint64_t offset_;
};

std::vector<std::uint8_t> save_bfly1(const ButterflyPlan& plan);
// Parses one plan starting at bytes[0]; *consumed receives the plan's length.
ButterflyPlan load_bfly1(const std::uint8_t* bytes, std::size_t n, std::size_t* consumed = nullptr);

}  // namespace bfb
