// Host compiler of the level-synchronous wave programs (see waves.hpp).
#include "waves.hpp"

#include "hostpar.hpp"

#include <algorithm>
#include <numeric>
#include <stdexcept>

namespace bfb {

namespace {

// A coefficient vector: the V cell of each element (contiguous for node
// outputs, a permutation of input cells for aliased full-rank leaves).
struct Vec {
    std::vector<std::uint32_t> cells;
    std::uint32_t level = 0;
    std::uint32_t node = ~0u;  // the node that writes these cells (~0u: coefficient cells)
    std::uint32_t len() const { return static_cast<std::uint32_t>(cells.size()); }
    bool contiguous() const {
        for (std::size_t k = 1; k < cells.size(); ++k)
            if (cells[k] != cells[0] + k) return false;
        return true;
    }
};

Vec range_vec(std::uint32_t cell, std::uint32_t len, std::uint32_t level, std::uint32_t node = ~0u) {
    Vec v;
    v.cells.resize(len);
    for (std::uint32_t k = 0; k < len; ++k) v.cells[k] = cell + k;
    v.level = level;
    v.node = node;
    return v;
}

}  // namespace

WaveSet build_waves(const std::vector<const ButterflyPlan*>& plans, const std::vector<int>& plan_mu,
                    const std::vector<int>& plan_parity) {
    WaveSet w;
    const std::size_t np = plans.size();
    std::uint64_t cells = 0;
    auto take = [&](std::uint64_t n) {
        const std::uint64_t c = cells;
        cells += n;
        if (cells >= (1ull << 32)) throw std::length_error("waves: more than 2^32 vector cells");
        return static_cast<std::uint32_t>(c);
    };
    struct Pair {
        std::uint32_t a, b;
    };
    std::vector<Pair> pairs;
    // The matrices are tiled after the symbolic pass: one allocation, the tiles
    // written by host threads (l = 2048: 41 GB).
    struct TileFill {
        const double* src;  // column-major rows x cols
        std::uint64_t off;
        std::uint32_t rows, cols, nib;
    };
    std::vector<TileFill> t_fill, s_fill;
    std::uint64_t t_words = 0, s_words = 0;
    // A node: c = z[sel] + T z[others], z = [A; B] (cells of two input vectors).
    auto add_node = [&](const StripeId& id, const Vec& A, const Vec& B) -> std::uint32_t {
        const std::uint32_t inputs = A.len() + B.len();
        if (static_cast<std::int64_t>(inputs) != id.inputs())
            throw std::runtime_error("waves: StripeId inputs disagree with the event stack");
        auto zc = [&](std::uint64_t k) { return k < A.len() ? A.cells[k] : B.cells[k - A.len()]; };
        WaveNode n{};
        n.rank = static_cast<std::uint32_t>(id.rank());
        n.nothers = static_cast<std::uint32_t>(id.interpolation.cols);
        n.level = std::max(A.len() ? A.level : 0u, B.len() ? B.level : 0u) + 1;
        n.cA = take(n.rank);
        n.idx = static_cast<std::uint32_t>(w.idx.size());
        for (std::uint64_t s : id.selected) w.idx.push_back(zc(s));
        for (std::uint32_t o : id.others()) w.idx.push_back(zc(o));
        n.nib = tiles16(n.rank);
        n.t_off = t_words;  // a multiple of 256 doubles (2 KB tiles); filled after the symbolic pass
        t_words += tiled_size(n.rank, n.nothers);
        if (n.rank > 0 && n.nothers > 0) t_fill.push_back(TileFill{id.interpolation.a.data(), n.t_off, n.rank, n.nothers, n.nib});
        w.event_words += id.interpolation.words();
        w.nodes.push_back(n);
        w.node_src.push_back(A.len() ? A.node : ~0u);
        w.node_src.push_back(B.len() ? B.node : ~0u);
        return static_cast<std::uint32_t>(w.nodes.size() - 1);
    };

    w.plan_in.resize(np);
    w.plan_yoff.resize(np);
    w.plan_groups.resize(np);
    std::uint32_t row_base = 0;  // rows of the earlier plans (stacked row vectors)
    for (std::size_t i = 0; i < np; ++i) {
        const ButterflyPlan& p = *plans[i];
        w.plan_node_begin.push_back(static_cast<std::uint32_t>(w.nodes.size()));
        if (i > 0) row_base += static_cast<std::uint32_t>(plans[i - 1]->n_rows);
        w.plan_row0.push_back(row_base);
        w.plan_mu.push_back(static_cast<std::uint32_t>(plan_mu[i]));
        w.plan_parity.push_back(static_cast<std::uint32_t>(plan_parity[i]));
        w.plan_cols.push_back(static_cast<std::uint32_t>(p.n_cols));
        w.plan_in[i] = take(p.n_cols);
        std::vector<std::vector<Vec>> stack;
        for (const PlanEvent& ev : p.events) {
            switch (ev.kind) {
            case EventKind::leaf: {
                const Vec z = range_vec(w.plan_in[i] + static_cast<std::uint32_t>(ev.col_begin),
                                        static_cast<std::uint32_t>(ev.col_count), 0);
                const StripeId& id = ev.ids.at(0);
                if (id.interpolation.cols == 0) {
                    // full-rank leaf (c = z[sel], e.g. every leaf of l >= 1024 at
                    // block width 60): no node, c aliases the coefficient cells.
                    // Its transpose needs nothing either: whatever consumes c
                    // writes those cells, all of them.
                    Vec c;
                    for (std::uint64_t s : id.selected) c.cells.push_back(z.cells.at(s));
                    stack.push_back({std::move(c)});
                    ++w.aliased_leaves;
                    break;
                }
                const std::uint32_t a = add_node(id, z, Vec{});
                pairs.push_back({a, ~0u});
                const WaveNode& n = w.nodes[a];
                stack.push_back({range_vec(n.cA, n.rank, n.level, a)});
                break;
            }
            case EventKind::merge: {
                if (stack.size() < 2) throw std::runtime_error("waves: merge on a short stack");
                std::vector<Vec> right = std::move(stack.back());
                stack.pop_back();
                std::vector<Vec> left = std::move(stack.back());
                stack.pop_back();
                std::vector<Vec> out;
                for (std::size_t s = 0; s < left.size(); ++s) {
                    const std::uint32_t a = add_node(ev.ids.at(2 * s), left[s], right.at(s));
                    const std::uint32_t b = add_node(ev.ids.at(2 * s + 1), left[s], right[s]);
                    pairs.push_back({a, b});
                    out.push_back(range_vec(w.nodes[a].cA, w.nodes[a].rank, w.nodes[a].level, a));
                    out.push_back(range_vec(w.nodes[b].cA, w.nodes[b].rank, w.nodes[b].level, b));
                }
                stack.push_back(std::move(out));
                break;
            }
            case EventKind::promote: {
                if (stack.empty()) throw std::runtime_error("waves: promote on an empty stack");
                std::vector<Vec> parent = std::move(stack.back());
                stack.pop_back();
                std::vector<Vec> out;
                for (std::size_t s = 0; s < parent.size(); ++s) {
                    const std::uint32_t a = add_node(ev.ids.at(2 * s), parent[s], Vec{});
                    const std::uint32_t b = add_node(ev.ids.at(2 * s + 1), parent[s], Vec{});
                    pairs.push_back({a, b});
                    out.push_back(range_vec(w.nodes[a].cA, w.nodes[a].rank, w.nodes[a].level, a));
                    out.push_back(range_vec(w.nodes[b].cA, w.nodes[b].rank, w.nodes[b].level, b));
                }
                stack.push_back(std::move(out));
                break;
            }
            }
        }
        if (stack.size() != p.root_groups.size()) throw std::runtime_error("apply: plan events and root groups disagree");
        // root stripes: S only (column-major, ld = rows rounded up to even), C = V
        w.plan_yoff[i] = w.y_rows;
        w.plan_groups[i] = static_cast<std::uint32_t>(p.root_groups.size());
        w.y_rows += static_cast<std::uint32_t>(p.root_groups.size() * p.n_rows);
        for (std::size_t g = 0; g < p.root_groups.size(); ++g) {
            if (stack[g].size() != p.root_groups[g].size()) throw std::runtime_error("waves: root group size mismatch");
            for (std::size_t s = 0; s < p.root_groups[g].size(); ++s) {
                const RootStripe& rs = p.root_groups[g][s];
                RootStripeDesc d{};
                d.rows = static_cast<std::uint32_t>(rs.row_count);
                d.rank = static_cast<std::uint32_t>(rs.skeleton.cols);
                Vec& cv = stack[g][s];
                if (d.rank != cv.len()) throw std::runtime_error("waves: root rank mismatch");
                if (!cv.contiguous()) {
                    // an aliased leaf feeding a root: the root kernels read
                    // contiguous cells, so copy it (a node without T)
                    WaveNode n{};
                    n.rank = cv.len();
                    n.level = cv.level + 1;
                    n.cA = take(n.rank);
                    n.idx = static_cast<std::uint32_t>(w.idx.size());
                    w.idx.insert(w.idx.end(), cv.cells.begin(), cv.cells.end());
                    n.t_off = t_words;
                    n.nib = tiles16(n.rank);
                    w.nodes.push_back(n);
                    w.node_src.push_back(cv.node);
                    w.node_src.push_back(~0u);
                    const std::uint32_t cn = static_cast<std::uint32_t>(w.nodes.size() - 1);
                    pairs.push_back({cn, ~0u});
                    cv = range_vec(n.cA, n.rank, n.level, cn);
                }
                d.lds = tiles16(d.rows);  // row tiles of S
                d.yout = w.plan_yoff[i] + static_cast<std::uint32_t>(g * p.n_rows + rs.row_begin);
                d.yin = static_cast<std::uint32_t>(rs.row_begin);
                d.coff = cv.len() ? cv.cells[0] : 0;
                d.plan = static_cast<std::uint32_t>(i);
                d.st_off = cv.node;  // waves: the node writing the stripe's coefficient cells (~0u: none)
                d.pad[0] = static_cast<std::uint32_t>(g);  // root group
                d.pad[1] = row_base + static_cast<std::uint32_t>(rs.row_begin);  // stacked row (plan-set apply)
                d.s_off = s_words;
                s_words += tiled_size(d.rows, d.rank);
                if (d.rows > 0 && d.rank > 0) s_fill.push_back(TileFill{rs.skeleton.a.data(), d.s_off, d.rows, d.rank, d.lds});
                w.roots.stored_words += rs.skeleton.words();
                w.roots.stripes.push_back(d);
            }
        }
    }
    w.plan_node_begin.push_back(static_cast<std::uint32_t>(w.nodes.size()));
    // fill the tiles (every job owns its whole tiled region; the padding stays zero)
    w.T.resize(t_words);
    w.roots.data.resize(s_words);
    auto fill = [](std::vector<double>& dst, const std::vector<TileFill>& jobs) {
        parallel_for(jobs.size(), [&](std::size_t k) {
            const TileFill& f = jobs[k];
            double* out = dst.data() + f.off;
            for (std::uint32_t q = 0; q < f.cols; ++q) {
                const double* col = f.src + static_cast<std::size_t>(q) * f.rows;
                for (std::uint32_t r = 0; r < f.rows; ++r) out[tiled_index(r, q, f.nib)] = col[r];
            }
        });
    };
    fill(w.T, t_fill);
    fill(w.roots.data, s_fill);
    w.root_words = w.roots.stored_words;

    w.v_cells = static_cast<std::uint32_t>(cells);
    // by root group (the forward sums groups into the chain rows, one launch per
    // group), largest stripes first (the hardware schedules CTAs roughly in order)
    std::stable_sort(w.roots.stripes.begin(), w.roots.stripes.end(), [](const RootStripeDesc& a, const RootStripeDesc& b) {
        if (a.pad[0] != b.pad[0]) return a.pad[0] < b.pad[0];
        return static_cast<std::uint64_t>(a.rows) * a.rank > static_cast<std::uint64_t>(b.rows) * b.rank;
    });

    for (const WaveNode& n : w.nodes) w.levels = std::max(w.levels, static_cast<int>(n.level));
    auto work = [&](std::uint32_t i) { return static_cast<std::uint64_t>(w.nodes[i].rank) * (w.nodes[i].nothers + 1); };
    // forward items: nodes with rank > 0, by level, then largest first
    for (std::uint32_t i = 0; i < w.nodes.size(); ++i)
        if (w.nodes[i].rank > 0) w.fwd.push_back(i);
    std::stable_sort(w.fwd.begin(), w.fwd.end(), [&](std::uint32_t a, std::uint32_t b) {
        if (w.nodes[a].level != w.nodes[b].level) return w.nodes[a].level < w.nodes[b].level;
        return work(a) > work(b);
    });
    // transposed items: a pair's level is its nodes' level (both share z)
    auto plevel = [&](const Pair& p) {
        return std::max(w.nodes[p.a].level, p.b == ~0u ? 0u : w.nodes[p.b].level);
    };
    auto pwork = [&](const Pair& p) { return work(p.a) + (p.b == ~0u ? 0 : work(p.b)); };
    std::stable_sort(pairs.begin(), pairs.end(), [&](const Pair& a, const Pair& b) {
        if (plevel(a) != plevel(b)) return plevel(a) < plevel(b);
        return pwork(a) > pwork(b);
    });
    for (const Pair& p : pairs) {
        w.pairs.push_back(p.a);
        w.pairs.push_back(p.b);
    }
    w.fwd_begin.assign(static_cast<std::size_t>(w.levels) + 1, 0);
    w.bwd_begin.assign(static_cast<std::size_t>(w.levels) + 1, 0);
    for (int L = 1; L <= w.levels; ++L) {
        w.fwd_begin[L] = static_cast<std::uint32_t>(
            std::count_if(w.fwd.begin(), w.fwd.end(), [&](std::uint32_t i) { return static_cast<int>(w.nodes[i].level) <= L; }));
        w.bwd_begin[L] = static_cast<std::uint32_t>(
            std::count_if(pairs.begin(), pairs.end(), [&](const Pair& p) { return static_cast<int>(plevel(p)) <= L; }));
    }
    return w;
}

}  // namespace bfb
