// Plan utilities: complement maps, statistics, structural validation and the
// BFLY1 container.  The BFLY1 layout is the reference's documented format
// (/root/reference/proj/include/bfly/serialize.hpp:14-31): little-endian u64
// integers, IEEE binary64 reals, column-major matrices, errors reported with a
// byte offset.  Reading a reference-written file here and writing it back
// reproduces the same bytes.
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>

namespace bfb {

std::vector<std::uint32_t> StripeId::others() const {
    const std::int64_t n = inputs();
    std::vector<char> taken(static_cast<std::size_t>(n), 0);
    for (std::uint64_t s : selected) {
        if (s >= static_cast<std::uint64_t>(n)) throw std::runtime_error("plan: selected index out of range");
        taken[s] = 1;
    }
    std::vector<std::uint32_t> out;
    out.reserve(static_cast<std::size_t>(interpolation.cols));
    for (std::int64_t j = 0; j < n; ++j)
        if (!taken[static_cast<std::size_t>(j)]) out.push_back(static_cast<std::uint32_t>(j));
    if (static_cast<std::int64_t>(out.size()) != interpolation.cols)
        throw std::runtime_error("plan: duplicate selected index");
    return out;
}

std::uint64_t ButterflyPlan::count_stored_words() const {
    std::uint64_t w = 0;
    for (const auto& ev : events)
        for (const auto& id : ev.ids) w += id.interpolation.words();
    for (const auto& g : root_groups)
        for (const auto& rs : g) w += rs.skeleton.words();
    return w;
}

void ButterflyPlan::validate() const {
    // Each stack entry records its per-stripe coefficient lengths.
    std::vector<std::vector<std::int64_t>> stack;
    for (const auto& ev : events) {
        switch (ev.kind) {
        case EventKind::leaf: {
            if (ev.ids.size() != 1) throw std::runtime_error("plan: leaf with != 1 id");
            if (ev.ids[0].inputs() != static_cast<std::int64_t>(ev.col_count) ||
                ev.col_begin + ev.col_count > n_cols)
                throw std::runtime_error("plan: leaf columns disagree with its id");
            stack.push_back({ev.ids[0].rank()});
            break;
        }
        case EventKind::merge:
        case EventKind::promote: {
            const bool merge = ev.kind == EventKind::merge;
            if (stack.size() < (merge ? 2u : 1u)) throw std::runtime_error("plan: event stack underflow");
            std::vector<std::int64_t> right;
            if (merge) {
                right = std::move(stack.back());
                stack.pop_back();
            }
            std::vector<std::int64_t> left = std::move(stack.back());
            stack.pop_back();
            if (ev.ids.size() != 2 * left.size() || (merge && right.size() != left.size()) ||
                (merge && ev.left_ranks.size() != left.size()))
                throw std::runtime_error("plan: stripe counts disagree");
            std::vector<std::int64_t> out;
            for (std::size_t s = 0; s < left.size(); ++s) {
                const std::int64_t inputs = left[s] + (merge ? right[s] : 0);
                if (merge && static_cast<std::int64_t>(ev.left_ranks[s]) != left[s])
                    throw std::runtime_error("plan: left rank disagrees");
                for (int h = 0; h < 2; ++h) {
                    const StripeId& id = ev.ids[2 * s + h];
                    if (id.inputs() != inputs) throw std::runtime_error("plan: id inputs disagree");
                    out.push_back(id.rank());
                }
            }
            stack.push_back(std::move(out));
            break;
        }
        }
    }
    if (stack.size() != root_groups.size())
        throw std::runtime_error("apply: plan events and root groups disagree");
    for (std::size_t g = 0; g < stack.size(); ++g) {
        if (stack[g].size() != root_groups[g].size())
            throw std::runtime_error("plan: root group stripe count disagrees");
        std::uint64_t covered = 0;
        for (std::size_t s = 0; s < stack[g].size(); ++s) {
            const RootStripe& rs = root_groups[g][s];
            if (rs.skeleton.cols != stack[g][s] || rs.skeleton.rows != static_cast<std::int64_t>(rs.row_count) ||
                rs.row_begin != covered)
                throw std::runtime_error("plan: root stripe shape disagrees");
            covered += rs.row_count;
        }
        if (covered != n_rows) throw std::runtime_error("plan: root group does not cover the rows");
    }
}

PlanStats plan_stats(const ButterflyPlan& plan) {
    PlanStats st;
    st.levels = plan.levels;
    st.stored_words = plan.stored_words;
    st.m_max_words = plan.m_max_words;
    st.t_comp_seconds = plan.t_comp_seconds;
    double s1 = 0.0, s2 = 0.0;
    for (const auto& ev : plan.events)
        for (const auto& id : ev.ids) {
            const auto k = static_cast<std::uint64_t>(id.rank());
            st.k_max = std::max(st.k_max, k);
            s1 += static_cast<double>(k);
            s2 += static_cast<double>(k) * static_cast<double>(k);
            ++st.id_count;
        }
    if (st.id_count) {
        const double n = static_cast<double>(st.id_count);
        st.k_avg = s1 / n;
        st.k_sigma = std::sqrt(std::max(0.0, s2 / n - st.k_avg * st.k_avg));
    }
    return st;
}

// ---- BFLY1 ----------------------------------------------------------------

namespace {

class ByteSink {
public:
    void raw(const void* p, std::size_t n) {
        const auto* b = static_cast<const std::uint8_t*>(p);
        buf.insert(buf.end(), b, b + n);
    }
    void u8(std::uint8_t v) { buf.push_back(v); }
    void u64(std::uint64_t v) {
        for (int k = 0; k < 8; ++k) buf.push_back(static_cast<std::uint8_t>(v >> (8 * k)));
    }
    void f64(double v) {
        std::uint64_t u;
        std::memcpy(&u, &v, 8);
        u64(u);
    }
    void mat(const Mat& m) {
        for (double v : m.a) f64(v);
    }
    std::vector<std::uint8_t> buf;
};

constexpr std::uint64_t kCountLimit = 1ull << 40;

class ByteSource {
public:
    ByteSource(const std::uint8_t* p, std::size_t n) : p_(p), n_(n) {}
    std::size_t pos() const { return pos_; }

    void need(std::size_t k) {
        if (n_ - pos_ < k) throw SerializationError("truncated input", pos_);
    }
    std::uint8_t u8() {
        need(1);
        return p_[pos_++];
    }
    std::uint64_t u64() {
        need(8);
        std::uint64_t v = 0;
        for (int k = 0; k < 8; ++k) v |= static_cast<std::uint64_t>(p_[pos_ + k]) << (8 * k);
        pos_ += 8;
        return v;
    }
    double f64() {
        const std::uint64_t u = u64();
        double v;
        std::memcpy(&v, &u, 8);
        return v;
    }
    std::uint64_t count() {
        const std::uint64_t v = u64();
        if (v > kCountLimit) throw SerializationError("implausible count " + std::to_string(v), pos_ - 8);
        return v;
    }
    Mat mat(std::uint64_t r, std::uint64_t c) {
        // Guard against counts that pass the limit but overrun the buffer.
        if (r && c > (n_ - pos_) / 8 / r) throw SerializationError("truncated input", pos_);
        Mat m(static_cast<std::int64_t>(r), static_cast<std::int64_t>(c));
        for (double& v : m.a) v = f64();
        return m;
    }
    void magic(const char* tag, std::size_t k) {
        const std::size_t at = pos_;
        need(k);
        if (std::memcmp(p_ + pos_, tag, k) != 0) throw SerializationError("bad magic", at);
        pos_ += k;
    }

private:
    const std::uint8_t* p_;
    std::size_t n_;
    std::size_t pos_ = 0;
};

}  // namespace

std::vector<std::uint8_t> save_bfly1(const ButterflyPlan& plan) {
    ByteSink w;
    w.raw("BFLY1", 5);
    w.u64(plan.n_rows);
    w.u64(plan.n_cols);
    w.f64(plan.epsilon);
    w.u64(plan.block_width);
    w.u64(plan.levels);
    w.u64(plan.events.size());
    for (const auto& ev : plan.events) {
        w.u8(static_cast<std::uint8_t>(ev.kind));
        if (ev.kind == EventKind::leaf) {
            w.u64(ev.col_begin);
            w.u64(ev.col_count);
        } else if (ev.kind == EventKind::merge) {
            w.u64(ev.left_ranks.size());
            for (auto k : ev.left_ranks) w.u64(k);
        }
        w.u64(ev.ids.size());
        for (const auto& id : ev.ids) {
            w.u64(static_cast<std::uint64_t>(id.rank()));
            w.u64(static_cast<std::uint64_t>(id.interpolation.cols));
            for (auto s : id.selected) w.u64(s);
            w.mat(id.interpolation);
        }
    }
    w.u64(plan.root_groups.size());
    for (const auto& g : plan.root_groups) {
        w.u64(g.size());
        for (const auto& rs : g) {
            w.u64(rs.row_begin);
            w.u64(rs.row_count);
            w.u64(static_cast<std::uint64_t>(rs.skeleton.cols));
            w.mat(rs.skeleton);
        }
    }
    return std::move(w.buf);
}

ButterflyPlan load_bfly1(const std::uint8_t* bytes, std::size_t n, std::size_t* consumed) {
    ByteSource r(bytes, n);
    ButterflyPlan plan;
    r.magic("BFLY1", 5);
    plan.n_rows = r.count();
    plan.n_cols = r.count();
    plan.epsilon = r.f64();
    plan.block_width = r.count();
    plan.levels = r.count();
    const std::uint64_t n_events = r.count();
    plan.events.reserve(static_cast<std::size_t>(std::min<std::uint64_t>(n_events, 1u << 20)));
    for (std::uint64_t e = 0; e < n_events; ++e) {
        PlanEvent ev;
        const std::uint8_t kind = r.u8();
        if (kind > 2) throw SerializationError("unknown event kind", r.pos() - 1);
        ev.kind = static_cast<EventKind>(kind);
        if (ev.kind == EventKind::leaf) {
            ev.col_begin = r.u64();
            ev.col_count = r.u64();
        } else if (ev.kind == EventKind::merge) {
            const std::uint64_t s = r.count();
            for (std::uint64_t i = 0; i < s; ++i) ev.left_ranks.push_back(r.u64());
        }
        const std::uint64_t n_ids = r.count();
        for (std::uint64_t i = 0; i < n_ids; ++i) {
            StripeId id;
            const std::uint64_t rank = r.count();
            const std::uint64_t others = r.count();
            for (std::uint64_t k = 0; k < rank; ++k) id.selected.push_back(r.u64());
            id.interpolation = r.mat(rank, others);
            ev.ids.push_back(std::move(id));
        }
        plan.events.push_back(std::move(ev));
    }
    const std::uint64_t n_groups = r.count();
    for (std::uint64_t g = 0; g < n_groups; ++g) {
        const std::uint64_t n_stripes = r.count();
        std::vector<RootStripe> group;
        for (std::uint64_t s = 0; s < n_stripes; ++s) {
            RootStripe rs;
            rs.row_begin = r.u64();
            rs.row_count = r.count();
            const std::uint64_t rank = r.count();
            rs.skeleton = r.mat(rs.row_count, rank);
            group.push_back(std::move(rs));
        }
        plan.root_groups.push_back(std::move(group));
    }
    plan.stored_words = plan.count_stored_words();
    plan.m_max_words = 0;  // BFLY1 carries no peak-memory or timing fields
    plan.t_comp_seconds = 0.0;
    if (consumed) *consumed = r.pos();
    return plan;
}

}  // namespace bfb
