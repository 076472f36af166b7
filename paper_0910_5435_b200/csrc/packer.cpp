// Host packer: compiles butterfly plans into the engine's stage stream.
//
// For every job the packer replays the reference's event stack
// (src/butterfly.cpp:384-442) once, symbolically: it assigns every
// coefficient vector a region of the job's shared-memory arena (first-fit,
// lifetimes = the stack discipline, identical in both directions), emits the
// records that realise each StripeId / root stripe, and cuts the matrices into
// panels that fill the stages.  Assign-vs-accumulate and barrier flags are
// decided here for both traversal orders, so the kernel never branches on
// plan structure.
#include "packer.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <numeric>
#include <stdexcept>

namespace bfb {

namespace {

constexpr std::uint32_t align16(std::uint32_t x) { return (x + 15u) & ~15u; }
constexpr int kMaxChunkRows = 1536;  // a single column of any panel fits a stage
constexpr int kMinPanelCols = 4;

class CellAllocator {
public:
    std::uint32_t alloc(std::uint32_t n) {
        if (n == 0) return 0;
        for (auto it = free_.begin(); it != free_.end(); ++it) {
            if (it->second >= n) {
                const std::uint32_t at = it->first, len = it->second;
                free_.erase(it);
                if (len > n) free_[at + n] = len - n;
                return at;
            }
        }
        const std::uint32_t at = top_;
        top_ += n;
        high_ = std::max(high_, top_);
        return at;
    }
    void release(std::uint32_t at, std::uint32_t n) {
        if (n == 0) return;
        auto it = free_.emplace(at, n).first;
        // coalesce with the successor
        auto nx = std::next(it);
        if (nx != free_.end() && it->first + it->second == nx->first) {
            it->second += nx->second;
            free_.erase(nx);
        }
        // coalesce with the predecessor
        if (it != free_.begin()) {
            auto pv = std::prev(it);
            if (pv->first + pv->second == it->first) {
                pv->second += it->second;
                free_.erase(it);
                it = pv;
            }
        }
        // give back a trailing block
        if (it->first + it->second == top_) {
            top_ = it->first;
            free_.erase(it);
        }
    }
    std::uint32_t high() const { return high_; }

private:
    std::map<std::uint32_t, std::uint32_t> free_;
    std::uint32_t top_ = 0, high_ = 0;
};

struct ZMap {
    std::uint32_t zA = 0, kl = 0, zB = 0;
};

class StageWriter {
public:
    explicit StageWriter(PackedProgram& out) : out_(out) {}

    std::uint32_t room_for_payload() const {
        const std::uint32_t used = fixed_used() + static_cast<std::uint32_t>(sizeof(Rec));
        return used >= static_cast<std::uint32_t>(kStageBytes) ? 0u : kStageBytes - used;
    }
    bool empty() const { return recs_.empty(); }

    void add(Rec r, std::vector<std::uint8_t> payload) {
        if (align16(static_cast<std::uint32_t>(payload.size())) > room_for_payload()) close();
        if (align16(static_cast<std::uint32_t>(payload.size())) > room_for_payload())
            throw std::logic_error("packer: record larger than a stage");
        payload_bytes_ += align16(static_cast<std::uint32_t>(payload.size()));
        recs_.push_back(r);
        payloads_.push_back(std::move(payload));
    }

    void close() {
        if (recs_.empty()) return;
        const std::uint32_t n = static_cast<std::uint32_t>(recs_.size());
        const std::uint32_t bytes = fixed_used();
        std::uint64_t at = out_.stream.size();
        out_.stream.resize(at + bytes, 0);
        std::uint8_t* base = out_.stream.data() + at;
        StageHeader h{n, bytes, job_, 0};
        std::memcpy(base, &h, sizeof h);
        std::uint32_t p = static_cast<std::uint32_t>(sizeof(StageHeader) + n * sizeof(Rec));
        for (std::uint32_t i = 0; i < n; ++i) {
            recs_[i].data = p;
            std::memcpy(base + sizeof(StageHeader) + i * sizeof(Rec), &recs_[i], sizeof(Rec));
            if (!payloads_[i].empty()) std::memcpy(base + p, payloads_[i].data(), payloads_[i].size());
            p += align16(static_cast<std::uint32_t>(payloads_[i].size()));
        }
        out_.stage_off.push_back(at);
        out_.stage_bytes.push_back(bytes);
        out_.fetched_bytes += bytes;
        recs_.clear();
        payloads_.clear();
        payload_bytes_ = 0;
    }

    void set_job(std::uint32_t j) { job_ = j; }

private:
    std::uint32_t fixed_used() const {
        return static_cast<std::uint32_t>(sizeof(StageHeader) + recs_.size() * sizeof(Rec)) + payload_bytes_;
    }
    PackedProgram& out_;
    std::vector<Rec> recs_;
    std::vector<std::vector<std::uint8_t>> payloads_;
    std::uint32_t payload_bytes_ = 0;
    std::uint32_t job_ = 0;
};

Rec blank(RecOp op, std::uint16_t pslot) {
    Rec r{};
    r.op = op;
    r.pslot = pslot;
    return r;
}

void put_u16s(std::vector<std::uint8_t>& p, const std::uint32_t* v, std::size_t n) {
    const std::size_t at = p.size();
    p.resize(at + 2 * n);
    for (std::size_t i = 0; i < n; ++i) {
        if (v[i] > 0xffffu) throw std::length_error("packer: index exceeds 16 bits");
        const std::uint16_t x = static_cast<std::uint16_t>(v[i]);
        std::memcpy(p.data() + at + 2 * i, &x, 2);
    }
    p.resize(align16(static_cast<std::uint32_t>(p.size())), 0);
}

// Columns of an (nr x ld)-panel with an nidx-per-column u16 prefix that fit.
std::uint32_t cols_that_fit(std::uint32_t room, std::uint32_t ld, bool with_idx) {
    std::uint32_t lo = 0, hi = 65535;
    while (lo < hi) {
        const std::uint32_t mid = (lo + hi + 1) / 2;
        const std::uint64_t need = (with_idx ? align16(2 * mid) : 0u) + 8ull * ld * mid;
        if (need <= room) lo = mid; else hi = mid - 1;
    }
    return lo;
}

class JobPacker {
public:
    JobPacker(StageWriter& w) : w_(w) {}

    // Emits a matrix as panels.  TPANEL: m = T (rank x others), idx = others.
    // SPANEL: m = skeleton (rows x rank), idx = nullptr.
    void matrix(RecOp op, const Mat& m, const std::uint32_t* idx, ZMap z, std::uint32_t c, std::uint32_t y,
                bool assign_fwd_first_cols, bool assign_bwd, bool sync_fwd_first, bool sync_bwd_last,
                std::uint16_t pslot) {
        const std::int64_t R = m.rows, Q = m.cols;
        bool first = true;
        for (std::int64_t r0 = 0; r0 < R; r0 += kMaxChunkRows) {
            const std::uint32_t nr = static_cast<std::uint32_t>(std::min<std::int64_t>(kMaxChunkRows, R - r0));
            const std::uint32_t ld = nr | 1u;
            const bool last_chunk = r0 + nr == R;
            std::int64_t q = 0;
            while (q < Q) {
                std::uint32_t fit = cols_that_fit(w_.room_for_payload(), ld, idx != nullptr);
                const std::uint32_t want = static_cast<std::uint32_t>(std::min<std::int64_t>(Q - q, kMinPanelCols));
                if (fit < want) {
                    w_.close();
                    fit = cols_that_fit(w_.room_for_payload(), ld, idx != nullptr);
                    if (fit == 0) throw std::logic_error("packer: panel column does not fit a stage");
                }
                const std::uint32_t nc = static_cast<std::uint32_t>(std::min<std::int64_t>(fit, Q - q));
                const bool last = last_chunk && q + nc == Q;
                Rec r = blank(op, pslot);
                r.nr = static_cast<std::uint16_t>(nr);
                r.nc = static_cast<std::uint16_t>(nc);
                r.ld = static_cast<std::uint16_t>(ld);
                std::uint8_t f = 0;
                if (first && sync_fwd_first) f |= F_SYNC_FWD;
                if (last && sync_bwd_last) f |= F_SYNC_BWD;
                std::vector<std::uint8_t> pay;
                if (op == OP_TPANEL) {
                    r.zA = z.zA;
                    r.kl = z.kl;
                    r.zB = z.zB;
                    r.cA = c + static_cast<std::uint32_t>(r0);
                    r.q0 = static_cast<std::uint16_t>(q);
                    if (q > 0xffff) throw std::length_error("packer: panel column offset exceeds 16 bits");
                    if (assign_bwd && last_chunk) f |= F_ASSIGN_BWD;
                    put_u16s(pay, idx + q, nc);
                } else {
                    r.zA = y + static_cast<std::uint32_t>(r0);
                    r.cA = c + static_cast<std::uint32_t>(q);
                    if (assign_fwd_first_cols && q == 0) f |= F_ASSIGN_FWD;
                    if (last_chunk) f |= F_ASSIGN_BWD;
                }
                r.flags = f;
                const std::size_t at = pay.size();
                pay.resize(at + 8ull * ld * nc, 0);
                double* dst = reinterpret_cast<double*>(pay.data() + at);
                for (std::uint32_t j = 0; j < nc; ++j)
                    std::memcpy(dst + static_cast<std::size_t>(j) * ld, m.col(q + j) + r0, 8ull * nr);
                w_.add(r, std::move(pay));
                first = false;
                q += nc;
            }
        }
    }

    // One StripeId: SEL then the T panels.
    void stripe_id(const StripeId& id, std::uint32_t c, ZMap z, bool first_writer_bwd, bool sync_fwd_first,
                   std::uint16_t pslot) {
        const std::uint32_t rank = static_cast<std::uint32_t>(id.rank());
        if (rank > 0xffff) throw std::length_error("packer: rank exceeds 16 bits");
        const bool has_t = id.interpolation.cols > 0;
        Rec s = blank(OP_SEL, pslot);
        s.nr = static_cast<std::uint16_t>(rank);
        s.zA = z.zA;
        s.kl = z.kl;
        s.zB = z.zB;
        s.cA = c;
        std::uint8_t f = F_ASSIGN_FWD;
        if (first_writer_bwd) f |= F_ASSIGN_BWD;
        if (sync_fwd_first) f |= F_SYNC_FWD;
        if (!has_t) f |= F_SYNC_BWD;
        s.flags = f;
        std::vector<std::uint32_t> sel(id.selected.begin(), id.selected.end());
        std::vector<std::uint8_t> pay;
        put_u16s(pay, sel.data(), sel.size());
        w_.add(s, std::move(pay));
        if (has_t) {
            const std::vector<std::uint32_t> oth = id.others();
            matrix(OP_TPANEL, id.interpolation, oth.data(), z, c, 0, false, first_writer_bwd, false, true, pslot);
        }
    }

    void loadz(std::uint32_t zcells, std::uint64_t row0, std::uint32_t n, std::uint16_t pslot) {
        Rec r = blank(OP_LOADZ, pslot);
        r.nr = static_cast<std::uint16_t>(n);
        r.zA = zcells;
        r.zB = static_cast<std::uint32_t>(row0);
        r.flags = F_SYNC_FWD | F_SYNC_BWD;
        w_.add(r, {});
    }

private:
    StageWriter& w_;
};

struct Slot {
    std::uint32_t at, n;
};

// Emits one plan of a job.  y = cells of the plan's row vector.
void pack_plan(JobPacker& jp, CellAllocator& arena, const ButterflyPlan& plan, std::uint32_t y,
               std::uint16_t pslot) {
    std::vector<std::vector<Slot>> stack;
    for (const PlanEvent& ev : plan.events) {
        switch (ev.kind) {
        case EventKind::leaf: {
            const StripeId& id = ev.ids[0];
            const std::uint32_t n = static_cast<std::uint32_t>(ev.col_count);
            if (n > 0xffff) throw std::length_error("packer: leaf wider than 16 bits");
            const std::uint32_t zt = arena.alloc(n);
            const std::uint32_t c = arena.alloc(static_cast<std::uint32_t>(id.rank()));
            jp.loadz(zt, ev.col_begin, n, pslot);
            jp.stripe_id(id, c, ZMap{zt, n, 0}, true, true, pslot);
            arena.release(zt, n);
            stack.push_back({Slot{c, static_cast<std::uint32_t>(id.rank())}});
            break;
        }
        case EventKind::merge:
        case EventKind::promote: {
            const bool merge = ev.kind == EventKind::merge;
            std::vector<Slot> right;
            if (merge) {
                right = std::move(stack.back());
                stack.pop_back();
            }
            std::vector<Slot> left = std::move(stack.back());
            stack.pop_back();
            std::vector<Slot> out;
            bool first_rec = true;
            for (std::size_t s = 0; s < left.size(); ++s) {
                const ZMap z = merge ? ZMap{left[s].at, left[s].n, right[s].at} : ZMap{left[s].at, left[s].n, 0};
                for (int h = 0; h < 2; ++h) {
                    const StripeId& id = ev.ids[2 * s + h];
                    const std::uint32_t c = arena.alloc(static_cast<std::uint32_t>(id.rank()));
                    // Transpose order visits bottom (h = 1) first: it assigns z.
                    jp.stripe_id(id, c, z, h == 1, first_rec, pslot);
                    first_rec = false;
                    out.push_back(Slot{c, static_cast<std::uint32_t>(id.rank())});
                }
            }
            for (const Slot& sl : left) arena.release(sl.at, sl.n);
            for (const Slot& sl : right) arena.release(sl.at, sl.n);
            stack.push_back(std::move(out));
            break;
        }
        }
    }
    if (stack.size() != plan.root_groups.size())
        throw std::runtime_error("apply: plan events and root groups disagree");
    bool first_rec = true;
    const Mat* last_mat = nullptr;
    for (std::size_t g = 0; g < plan.root_groups.size(); ++g)
        for (std::size_t s = 0; s < plan.root_groups[g].size(); ++s) last_mat = &plan.root_groups[g][s].skeleton;
    for (std::size_t g = 0; g < plan.root_groups.size(); ++g) {
        const auto& group = plan.root_groups[g];
        if (group.size() != stack[g].size()) throw std::runtime_error("apply: plan events and root groups disagree");
        for (std::size_t s = 0; s < group.size(); ++s) {
            const RootStripe& rs = group[s];
            if (rs.skeleton.cols == 0) continue;
            jp.matrix(OP_SPANEL, rs.skeleton, nullptr, ZMap{}, stack[g][s].at,
                      y + static_cast<std::uint32_t>(rs.row_begin), g == 0, false, first_rec,
                      &rs.skeleton == last_mat, pslot);
            first_rec = false;
        }
    }
    for (const auto& blk : stack)
        for (const Slot& sl : blk) arena.release(sl.at, sl.n);
}

}  // namespace

PackedProgram pack_program(const std::vector<const ButterflyPlan*>& plans,
                           const std::vector<std::vector<int>>& job_plans, const std::vector<int>& job_mu) {
    PackedProgram out;
    for (const auto* p : plans) out.stored_words += p->stored_words;
    // Largest jobs first: the persistent grid then drains them LPT-style.
    std::vector<std::uint64_t> cost(job_plans.size(), 0);
    for (std::size_t j = 0; j < job_plans.size(); ++j)
        for (int pi : job_plans[j]) cost[j] += plans[static_cast<std::size_t>(pi)]->stored_words + plans[static_cast<std::size_t>(pi)]->n_rows;
    std::vector<std::size_t> order(job_plans.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) { return cost[a] > cost[b]; });

    StageWriter w(out);
    for (std::size_t jj = 0; jj < order.size(); ++jj) {
        const std::size_t j = order[jj];
        const auto& pl = job_plans[j];
        if (pl.empty() || pl.size() > 2) throw std::invalid_argument("pack: a job holds 1 or 2 plans");
        Job job{};
        job.n_plans = static_cast<std::uint16_t>(pl.size());
        job.mu = static_cast<std::uint16_t>(job_mu.empty() ? 0 : job_mu[j]);
        job.n_rows = static_cast<std::uint32_t>(plans[static_cast<std::size_t>(pl[0])]->n_rows);
        out.max_rows = std::max(out.max_rows, job.n_rows);
        CellAllocator arena;
        for (std::size_t k = 0; k < pl.size(); ++k) {
            const ButterflyPlan& p = *plans[static_cast<std::size_t>(pl[k])];
            if (p.n_rows != job.n_rows) throw std::invalid_argument("pack: plans of a job must share n_rows");
            job.plan[k] = static_cast<std::uint32_t>(pl[k]);
            job.n_cols[k] = static_cast<std::uint32_t>(p.n_cols);
            job.yA[k] = arena.alloc(job.n_rows);
        }
        w.set_job(static_cast<std::uint32_t>(jj));
        job.stage0 = out.stage_off.size();
        JobPacker jp(w);
        for (std::size_t k = 0; k < pl.size(); ++k)
            pack_plan(jp, arena, *plans[static_cast<std::size_t>(pl[k])], job.yA[k], static_cast<std::uint16_t>(k));
        w.close();
        job.n_stages = static_cast<std::uint32_t>(out.stage_off.size() - job.stage0);
        out.arena_cells = std::max(out.arena_cells, arena.high());
        out.jobs.push_back(job);
    }
    return out;
}

}  // namespace bfb
