// Host packer: compiles butterfly plans into the engine's stage stream.
//
// For every job the packer replays the reference's event stack
// (src/butterfly.cpp:384-442) once, symbolically: it assigns every
// coefficient vector a region of the job's shared-memory arena (first-fit,
// lifetimes = the stack discipline, identical in both directions), turns each
// StripeId / root stripe into records, hoists every leaf's input load one
// event ahead so it overlaps the previous event, and cuts matrices into
// row chunks (units) and column panels that fill the stages.  Assign-vs-
// accumulate and barrier flags are decided here for both traversal orders, so
// the kernel never branches on plan structure.
#include "packer.hpp"

#include <algorithm>
#include <cstring>
#include <map>
#include <numeric>
#include <stdexcept>

namespace bfb {

namespace {

constexpr std::uint32_t align16(std::uint32_t x) { return (x + 15u) & ~15u; }
constexpr std::uint32_t align8(std::uint32_t x) { return (x + 7u) & ~7u; }
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
        auto nx = std::next(it);
        if (nx != free_.end() && it->first + it->second == nx->first) {
            it->second += nx->second;
            free_.erase(nx);
        }
        if (it != free_.begin()) {
            auto pv = std::prev(it);
            if (pv->first + pv->second == it->first) {
                pv->second += it->second;
                free_.erase(it);
                it = pv;
            }
        }
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

// A logical record before panel splitting.
struct Item {
    RecOp op = OP_LOADZ;
    std::uint16_t pslot = 0;
    // LOADZ
    std::uint32_t cells = 0, row0 = 0, n = 0;
    // SEL / TPANEL
    const StripeId* id = nullptr;
    ZMap z;
    std::uint32_t c = 0;
    bool first_writer = false;
    // SPANEL
    const Mat* S = nullptr;
    std::uint32_t y = 0;
    bool group0 = false;
    // CXCH
    std::uint32_t c_off = 0;
    bool cload_fwd = false;
    // barriers
    bool sync_fwd_first = false;  // barrier before the item (forward)
    bool sync_bwd_last = false;   // barrier before the item's last record (transpose)
    bool sync_bwd_item = true;    // ... also before its first chunk in that order (false: only between chunks)
};

class StageWriter {
public:
    StageWriter(PackedProgram& out, std::uint32_t cap) : out_(out), cap_(cap) {}

    std::uint32_t room_for_payload() const {
        const std::uint32_t used = fixed_used() + static_cast<std::uint32_t>(sizeof(Rec));
        return used >= cap_ ? 0u : cap_ - used;
    }
    bool fits(std::size_t payload) const {
        return fixed_used() + sizeof(Rec) + align16(static_cast<std::uint32_t>(payload)) <= cap_;
    }

    void add(Rec r, std::vector<std::uint8_t> payload) {
        if (!fits(payload.size())) close();
        if (!fits(payload.size())) throw std::logic_error("packer: record larger than a stage");
        payload_bytes_ += align16(static_cast<std::uint32_t>(payload.size()));
        recs_.push_back(r);
        payloads_.push_back(std::move(payload));
    }

    void close() {
        if (recs_.empty()) return;
        const std::uint32_t n = static_cast<std::uint32_t>(recs_.size());
        const std::uint32_t bytes = fixed_used();
        if (bytes > cap_) throw std::logic_error("packer: stage overflow");
        const std::uint64_t at = out_.stream.size();
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
    std::uint32_t cap_;
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
    p.resize(align8(static_cast<std::uint32_t>(p.size())), 0);
}

// Columns of an (nr-row) panel that fit `room`, given the u16 index bytes.
std::uint32_t cols_that_fit(std::uint32_t room, std::uint32_t nr, bool with_idx, std::uint32_t extra) {
    std::uint32_t lo = 0, hi = 65535;
    while (lo < hi) {
        const std::uint32_t mid = (lo + hi + 1) / 2;
        const std::uint64_t need = (with_idx ? align8(2 * mid) : 0u) + extra + 8ull * nr * mid;
        if (need <= room) lo = mid; else hi = mid - 1;
    }
    return lo;
}

class Layout {
public:
    explicit Layout(StageWriter& w) : w_(w) {}
    std::uint32_t zo_max() const { return zo_max_; }

    void emit(const Item& it) {
        switch (it.op) {
        case OP_LOADZ: {
            Rec r = blank(OP_LOADZ, it.pslot);
            if (it.n > 0xffff) throw std::length_error("packer: leaf wider than 16 bits");
            r.nr = static_cast<std::uint16_t>(it.n);
            r.zA = it.cells;
            r.zB = it.row0;
            r.flags = F_SYNC_BWD | (it.sync_fwd_first ? F_SYNC_FWD : 0);
            w_.add(r, {});
            break;
        }
        case OP_SEL: {
            const std::uint32_t rank = static_cast<std::uint32_t>(it.id->rank());
            if (rank > 0xffff) throw std::length_error("packer: rank exceeds 16 bits");
            Rec r = blank(OP_SEL, it.pslot);
            r.nr = static_cast<std::uint16_t>(rank);
            r.zA = it.z.zA;
            r.kl = it.z.kl;
            r.zB = it.z.zB;
            r.cA = it.c;
            std::uint8_t f = 0;
            if (it.first_writer) f |= F_ASSIGN_BWD;
            if (it.sync_fwd_first) f |= F_SYNC_FWD;
            if (it.sync_bwd_last) f |= F_SYNC_BWD;
            r.flags = f;
            std::vector<std::uint32_t> sel(it.id->selected.begin(), it.id->selected.end());
            std::vector<std::uint8_t> pay;
            put_u16s(pay, sel.data(), sel.size());
            w_.add(r, std::move(pay));
            break;
        }
        case OP_TPANEL: {
            const Mat& T = it.id->interpolation;
            const std::vector<std::uint32_t> oth = it.id->others();
            const std::vector<std::uint32_t> sel(it.id->selected.begin(), it.id->selected.end());
            matrix(it, T, oth.data(), sel.data());
            break;
        }
        case OP_SPANEL:
            matrix(it, *it.S, nullptr, nullptr);
            break;
        case OP_CXCH: {
            Rec r = blank(OP_CXCH, it.pslot);
            if (it.n > 0xffff) throw std::length_error("packer: coefficient vector wider than 16 bits");
            r.nr = static_cast<std::uint16_t>(it.n);
            r.zA = it.cells;
            r.zB = it.c_off;
            std::uint8_t f = it.cload_fwd ? F_CLOAD_FWD : 0;
            if (it.sync_fwd_first) f |= F_SYNC_FWD;
            if (it.sync_bwd_last) f |= F_SYNC_BWD;
            r.flags = f;
            w_.add(r, {});
            break;
        }
        }
    }

private:
    // Row chunks (units) of <= kChunkRows rows, each cut into column panels.
    void matrix(const Item& it, const Mat& m, const std::uint32_t* others, const std::uint32_t* sel) {
        const bool tp = it.op == OP_TPANEL;
        const std::int64_t R = m.rows, Q = m.cols;
        bool first_rec = true;
        for (std::int64_t r0 = 0; r0 < R; r0 += kChunkRows) {
            const std::uint32_t nr = static_cast<std::uint32_t>(std::min<std::int64_t>(kChunkRows, R - r0));
            const bool last_chunk = r0 + nr == R;
            std::int64_t q = 0;
            while (q < Q) {
                const bool begin = q == 0;
                const std::uint32_t sel_bytes = (tp && begin) ? align8(2 * nr) : 0u;
                const std::uint32_t ld = nr | 1u;
                std::uint32_t fit = cols_that_fit(w_.room_for_payload(), ld, tp, sel_bytes);
                const std::uint32_t want = static_cast<std::uint32_t>(std::min<std::int64_t>(Q - q, kMinPanelCols));
                if (fit < want) {
                    w_.close();
                    fit = cols_that_fit(w_.room_for_payload(), ld, tp, sel_bytes);
                    if (fit == 0) throw std::logic_error("packer: panel column does not fit a stage");
                }
                const std::uint32_t nc = static_cast<std::uint32_t>(std::min<std::int64_t>(fit, Q - q));
                const bool end = q + nc == Q;
                Rec r = blank(it.op, it.pslot);
                r.nr = static_cast<std::uint16_t>(nr);
                r.nc = static_cast<std::uint16_t>(nc);
                r.ld = static_cast<std::uint16_t>(ld);
                std::uint8_t f = 0;
                if (begin) f |= F_BEGIN;
                if (end) f |= F_END;
                if (first_rec && it.sync_fwd_first) f |= F_SYNC_FWD;
                // transpose: a chunk accumulates into the outputs the chunk before it
                // (in that order) wrote, so every chunk but the first processed one
                // waits; the first one only if the item reads earlier items' outputs
                if (end && it.sync_bwd_last && (!last_chunk || it.sync_bwd_item)) f |= F_SYNC_BWD;
                std::vector<std::uint8_t> pay;
                if (tp) {
                    r.zA = it.z.zA;
                    r.kl = it.z.kl;
                    r.zB = it.z.zB;
                    r.cA = it.c + static_cast<std::uint32_t>(r0);
                    if (it.first_writer && last_chunk) f |= F_ASSIGN_BWD;
                    if (it.first_writer) f |= F_ASSIGN_SEL_BWD;
                    put_u16s(pay, others + q, nc);
                    if (begin) put_u16s(pay, sel + r0, nr);
                } else {
                    r.zA = it.y + static_cast<std::uint32_t>(r0);
                    r.cA = it.c + static_cast<std::uint32_t>(q);
                    if (it.group0) f |= F_ASSIGN_FWD;
                    if (last_chunk) f |= F_ASSIGN_BWD;
                }
                r.flags = f;
                r.moff = static_cast<std::uint16_t>(pay.size());
                const std::size_t at = pay.size();
                pay.resize(at + 8ull * ld * nc, 0);
                double* dst = reinterpret_cast<double*>(pay.data() + at);
                for (std::uint32_t j = 0; j < nc; ++j)
                    std::memcpy(dst + static_cast<std::size_t>(j) * ld, m.col(q + j) + r0, 8ull * nr);
                w_.add(r, std::move(pay));
                first_rec = false;
                q += nc;
            }
        }
    }

    StageWriter& w_;
    std::uint32_t zo_max_ = 0;
};

struct Slot {
    std::uint32_t at, n;
};

// Events of all plans of a job, plus one "root" pseudo-event per plan.
struct JobEvent {
    int plan_slot;
    int event;  // index into plan.events, or -1 for the plan's root stage
};

// Global C offsets of one plan's surviving-block stripes, [group][stripe].
using COffsets = std::vector<std::vector<std::uint32_t>>;

class JobBuilder {
public:
    // split_c != nullptr: the root stage is not emitted; instead the surviving
    // blocks' vectors are stored to C from *split_c on (offsets recorded in
    // split_out[plan slot]).
    JobBuilder(const std::vector<const ButterflyPlan*>& plans, const std::vector<std::uint32_t>& y,
               std::uint32_t* split_c = nullptr, std::vector<COffsets>* split_out = nullptr)
        : plans_(plans), y_(y), split_c_(split_c), split_out_(split_out) {
        for (std::size_t p = 0; p < plans.size(); ++p) {
            for (std::size_t e = 0; e < plans[p]->events.size(); ++e)
                seq_.push_back(JobEvent{static_cast<int>(p), static_cast<int>(e)});
            seq_.push_back(JobEvent{static_cast<int>(p), -1});
        }
    }

    std::vector<Item> build(CellAllocator& arena) {
        stacks_.assign(plans_.size(), {});
        std::vector<Item> items;
        std::uint32_t zt_next = 0;  // prefetched z cells of the upcoming leaf
        bool have_next = false;
        for (std::size_t k = 0; k < seq_.size(); ++k) {
            const JobEvent je = seq_[k];
            // The z cells of this event's leaf were allocated one event ago.
            std::uint32_t zt_mine = zt_next;
            const bool prefetched = have_next;
            have_next = false;
            // Allocate (and later prefetch) the next event's leaf input now.
            const PlanEvent* nxt = nullptr;
            if (k + 1 < seq_.size() && seq_[k + 1].event >= 0) {
                const auto& ev = plans_[seq_[k + 1].plan_slot]->events[seq_[k + 1].event];
                if (ev.kind == EventKind::leaf) nxt = &ev;
            }
            std::vector<Item> ev_items;
            if (je.event >= 0) {
                const PlanEvent& ev = plans_[je.plan_slot]->events[je.event];
                if (ev.kind == EventKind::leaf && !prefetched) {
                    zt_mine = arena.alloc(static_cast<std::uint32_t>(ev.col_count));
                    Item lz;
                    lz.op = OP_LOADZ;
                    lz.pslot = static_cast<std::uint16_t>(je.plan_slot);
                    lz.cells = zt_mine;
                    lz.row0 = static_cast<std::uint32_t>(ev.col_begin);
                    lz.n = static_cast<std::uint32_t>(ev.col_count);
                    lz.sync_fwd_first = true;
                    items.push_back(lz);
                }
            }
            // The next leaf's input cells are allocated before this event's
            // outputs and releases, so they never alias anything it touches.
            if (nxt) {
                zt_next = arena.alloc(static_cast<std::uint32_t>(nxt->col_count));
                have_next = true;
            }
            if (je.event < 0)
                (split_c_ ? store_c(arena, je.plan_slot, ev_items) : root(arena, je.plan_slot, ev_items));
            else
                event(arena, je.plan_slot, plans_[je.plan_slot]->events[je.event], zt_mine, ev_items);
            // Emit: first item, then the prefetch of the next leaf, then the rest.
            for (std::size_t i = 0; i < ev_items.size(); ++i) {
                items.push_back(ev_items[i]);
                if (i == 0 && have_next) {
                    const JobEvent jn = seq_[k + 1];
                    Item lz;
                    lz.op = OP_LOADZ;
                    lz.pslot = static_cast<std::uint16_t>(jn.plan_slot);
                    lz.cells = zt_next;
                    lz.row0 = static_cast<std::uint32_t>(nxt->col_begin);
                    lz.n = static_cast<std::uint32_t>(nxt->col_count);
                    items.push_back(lz);
                }
            }
        }
        return items;
    }

private:
    void event(CellAllocator& arena, int ps, const PlanEvent& ev, std::uint32_t zt, std::vector<Item>& out) {
        auto& stack = stacks_[static_cast<std::size_t>(ps)];
        switch (ev.kind) {
        case EventKind::leaf: {
            const StripeId& id = ev.ids[0];
            const std::uint32_t c = arena.alloc(static_cast<std::uint32_t>(id.rank()));
            stripe_id(id, c, ZMap{zt, static_cast<std::uint32_t>(ev.col_count), 0}, true, true, ps, out);
            arena.release(zt, static_cast<std::uint32_t>(ev.col_count));
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
            std::vector<Slot> outs;
            bool first = true;
            for (std::size_t s = 0; s < left.size(); ++s) {
                const ZMap z = merge ? ZMap{left[s].at, left[s].n, right[s].at} : ZMap{left[s].at, left[s].n, 0};
                for (int h = 0; h < 2; ++h) {
                    const StripeId& id = ev.ids[2 * s + h];
                    const std::uint32_t c = arena.alloc(static_cast<std::uint32_t>(id.rank()));
                    // The transpose visits the bottom id (h = 1) first: it assigns z.
                    stripe_id(id, c, z, h == 1, first, ps, out);
                    first = false;
                    outs.push_back(Slot{c, static_cast<std::uint32_t>(id.rank())});
                }
            }
            for (const Slot& sl : left) arena.release(sl.at, sl.n);
            for (const Slot& sl : right) arena.release(sl.at, sl.n);
            stack.push_back(std::move(outs));
            break;
        }
        }
    }

    void stripe_id(const StripeId& id, std::uint32_t c, ZMap z, bool first_writer, bool sync_fwd_first, int ps,
                   std::vector<Item>& out) {
        Item it;
        it.op = id.interpolation.cols > 0 ? OP_TPANEL : OP_SEL;
        it.pslot = static_cast<std::uint16_t>(ps);
        it.id = &id;
        it.z = z;
        it.c = c;
        it.first_writer = first_writer;
        it.sync_fwd_first = sync_fwd_first;
        it.sync_bwd_last = true;
        out.push_back(it);
    }

    void root(CellAllocator& arena, int ps, std::vector<Item>& out) {
        const ButterflyPlan& plan = *plans_[static_cast<std::size_t>(ps)];
        auto& stack = stacks_[static_cast<std::size_t>(ps)];
        if (stack.size() != plan.root_groups.size())
            throw std::runtime_error("apply: plan events and root groups disagree");
        for (std::size_t g = 0; g < plan.root_groups.size(); ++g) {
            const auto& group = plan.root_groups[g];
            if (group.size() != stack[g].size()) throw std::runtime_error("apply: plan events and root groups disagree");
            for (std::size_t s = 0; s < group.size(); ++s) {
                const RootStripe& rs = group[s];
                if (rs.skeleton.cols == 0) throw std::runtime_error("plan: empty root skeleton");
                Item it;
                it.op = OP_SPANEL;
                it.pslot = static_cast<std::uint16_t>(ps);
                it.S = &rs.skeleton;
                it.c = stack[g][s].at;
                it.y = y_[static_cast<std::size_t>(ps)] + static_cast<std::uint32_t>(rs.row_begin);
                it.group0 = g == 0;
                it.sync_fwd_first = s == 0;  // groups overlap in rows: barrier per group
                it.sync_bwd_last = true;
                // Transpose: stripes read the (synced) row cells and write their own
                // coefficient cells, so only their chunks need barriers between them.
                it.sync_bwd_item = false;
                out.push_back(it);
            }
        }
        for (const auto& blk : stack)
            for (const Slot& sl : blk) arena.release(sl.at, sl.n);
        stack.clear();
    }

    void store_c(CellAllocator& arena, int ps, std::vector<Item>& out) {
        const ButterflyPlan& plan = *plans_[static_cast<std::size_t>(ps)];
        auto& stack = stacks_[static_cast<std::size_t>(ps)];
        if (stack.size() != plan.root_groups.size())
            throw std::runtime_error("apply: plan events and root groups disagree");
        COffsets offs;
        bool first = true;
        for (std::size_t g = 0; g < stack.size(); ++g) {
            if (plan.root_groups[g].size() != stack[g].size())
                throw std::runtime_error("apply: plan events and root groups disagree");
            std::vector<std::uint32_t> go;
            for (const Slot& sl : stack[g]) {
                Item it;
                it.op = OP_CXCH;
                it.pslot = static_cast<std::uint16_t>(ps);
                it.cells = sl.at;
                it.n = sl.n;
                it.c_off = *split_c_;
                it.cload_fwd = false;  // forward stores, transpose loads
                it.sync_fwd_first = first;
                it.sync_bwd_last = false;
                first = false;
                go.push_back(*split_c_);
                *split_c_ += sl.n;
                out.push_back(it);
            }
            offs.push_back(std::move(go));
        }
        (*split_out_)[static_cast<std::size_t>(ps)] = std::move(offs);
        for (const auto& blk : stack)
            for (const Slot& sl : blk) arena.release(sl.at, sl.n);
        stack.clear();
    }

    const std::vector<const ButterflyPlan*>& plans_;
    const std::vector<std::uint32_t>& y_;
    std::uint32_t* split_c_;
    std::vector<COffsets>* split_out_;
    std::vector<JobEvent> seq_;
    std::vector<std::vector<std::vector<Slot>>> stacks_;
};

}  // namespace

PackedProgram pack_program(const std::vector<const ButterflyPlan*>& plans,
                           const std::vector<std::vector<int>>& job_plans, const std::vector<int>& job_mu,
                           std::uint32_t stage_capacity, const std::vector<int>& job_parity) {
    if (stage_capacity < static_cast<std::uint32_t>(kStageBytesMin) || stage_capacity > 65536u ||
        stage_capacity % 16 != 0)
        throw std::invalid_argument("pack: stage capacity must be a multiple of 16 in [8 KiB, 64 KiB]");
    PackedProgram out;
    out.stage_capacity = stage_capacity;
    for (const auto* p : plans) out.stored_words += p->stored_words;
    // Largest jobs first: the persistent grid then drains them LPT-style.
    std::vector<std::uint64_t> cost(job_plans.size(), 0);
    for (std::size_t j = 0; j < job_plans.size(); ++j)
        for (int pi : job_plans[j])
            cost[j] += plans[static_cast<std::size_t>(pi)]->stored_words + plans[static_cast<std::size_t>(pi)]->n_rows;
    std::vector<std::size_t> order(job_plans.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) { return cost[a] > cost[b]; });

    StageWriter w(out, stage_capacity);
    Layout lay(w);
    for (std::size_t jj = 0; jj < order.size(); ++jj) {
        const std::size_t j = order[jj];
        const auto& pl = job_plans[j];
        if (pl.empty() || pl.size() > 2) throw std::invalid_argument("pack: a job holds 1 or 2 plans");
        Job job{};
        job.n_plans = static_cast<std::uint16_t>(pl.size());
        job.mu = static_cast<std::uint16_t>(job_mu.empty() ? 0 : job_mu[j]);
        job.parity = static_cast<std::uint32_t>(job_parity.empty() ? 0 : job_parity[j]);
        job.n_rows = static_cast<std::uint32_t>(plans[static_cast<std::size_t>(pl[0])]->n_rows);
        out.max_rows = std::max(out.max_rows, job.n_rows);
        CellAllocator arena;
        std::vector<const ButterflyPlan*> jp;
        std::vector<std::uint32_t> ys;
        for (std::size_t k = 0; k < pl.size(); ++k) {
            const ButterflyPlan& p = *plans[static_cast<std::size_t>(pl[k])];
            if (p.n_rows != job.n_rows) throw std::invalid_argument("pack: plans of a job must share n_rows");
            job.plan[k] = static_cast<std::uint32_t>(pl[k]);
            job.n_cols[k] = static_cast<std::uint32_t>(p.n_cols);
            job.yA[k] = arena.alloc(job.n_rows);
            jp.push_back(&p);
            ys.push_back(job.yA[k]);
        }
        w.set_job(static_cast<std::uint32_t>(jj));
        job.stage0 = out.stage_off.size();
        JobBuilder jb(jp, ys);
        for (const Item& it : jb.build(arena)) lay.emit(it);
        w.close();
        job.n_stages = static_cast<std::uint32_t>(out.stage_off.size() - job.stage0);
        out.arena_cells = std::max(out.arena_cells, arena.high());
        out.jobs.push_back(job);
    }
    out.zo_cells = lay.zo_max();
    return out;
}

PackedProgram merge_split(const SplitProgram& sp, std::size_t n_plans) {
    const PackedProgram& e = sp.events;
    const PackedProgram& r = sp.roots;
    if (e.stage_capacity != r.stage_capacity) throw std::invalid_argument("merge: stage capacities differ");
    PackedProgram m;
    m.stage_capacity = e.stage_capacity;
    m.stream = e.stream;
    m.stream.insert(m.stream.end(), r.stream.begin(), r.stream.end());
    m.stage_off = e.stage_off;
    for (std::uint64_t o : r.stage_off) m.stage_off.push_back(o + e.stream.size());
    m.stage_bytes = e.stage_bytes;
    m.stage_bytes.insert(m.stage_bytes.end(), r.stage_bytes.begin(), r.stage_bytes.end());
    m.jobs = e.jobs;
    for (Job j : r.jobs) {
        j.stage0 += e.stage_off.size();
        j.kind = 1;
        m.jobs.push_back(j);
    }
    m.arena_cells = std::max(e.arena_cells, r.arena_cells);
    m.zo_cells = std::max(e.zo_cells, r.zo_cells);
    m.stored_words = e.stored_words + r.stored_words;
    m.fetched_bytes = e.fetched_bytes + r.fetched_bytes;
    m.max_rows = std::max(e.max_rows, r.max_rows);
    const std::uint32_t ne = static_cast<std::uint32_t>(e.jobs.size()), nr = static_cast<std::uint32_t>(r.jobs.size());
    for (std::uint32_t i = 0; i < ne + nr; ++i) m.order_fwd.push_back(i);
    for (std::uint32_t i = 0; i < nr; ++i) m.order_bwd.push_back(ne + i);
    for (std::uint32_t i = 0; i < ne; ++i) m.order_bwd.push_back(i);
    m.plan_roots.assign(n_plans, 0);
    for (const Job& j : r.jobs) ++m.plan_roots[j.plan[0]];
    return m;
}

SplitProgram pack_split(const std::vector<const ButterflyPlan*>& plans, const std::vector<int>& plan_mu,
                        const std::vector<int>& plan_parity, std::uint32_t event_cap, std::uint32_t root_cap) {
    for (std::uint32_t cap : {event_cap, root_cap})
        if (cap < static_cast<std::uint32_t>(kStageBytesMin) || cap > 65536u || cap % 16 != 0)
            throw std::invalid_argument("pack: stage capacity must be a multiple of 16 in [8 KiB, 64 KiB]");
    SplitProgram sp;
    const std::size_t np = plans.size();

    // ---- event program: one job per plan, largest first --------------------
    std::vector<std::uint64_t> cost(np);
    for (std::size_t i = 0; i < np; ++i) {
        std::uint64_t w = 0;
        for (const auto& ev : plans[i]->events)
            for (const auto& id : ev.ids) w += id.interpolation.words() + static_cast<std::uint64_t>(id.rank());
        cost[i] = w;
        sp.events.stored_words += w;
    }
    std::vector<std::size_t> order(np);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](std::size_t a, std::size_t b) { return cost[a] > cost[b]; });
    std::vector<COffsets> coffs(np);
    {
        sp.events.stage_capacity = event_cap;
        StageWriter w(sp.events, event_cap);
        Layout lay(w);
        for (std::size_t jj = 0; jj < np; ++jj) {
            const std::size_t i = order[jj];
            const ButterflyPlan& p = *plans[i];
            Job job{};
            job.n_plans = 1;
            job.mu = static_cast<std::uint16_t>(plan_mu[i]);
            job.parity = static_cast<std::uint32_t>(plan_parity[i]);
            job.plan[0] = static_cast<std::uint32_t>(i);
            job.n_rows = static_cast<std::uint32_t>(p.n_rows);
            job.n_cols[0] = static_cast<std::uint32_t>(p.n_cols);
            CellAllocator arena;
            std::vector<const ButterflyPlan*> jp{&p};
            std::vector<std::uint32_t> ys{0};
            std::vector<COffsets> one(1);
            w.set_job(static_cast<std::uint32_t>(jj));
            job.stage0 = sp.events.stage_off.size();
            JobBuilder jb(jp, ys, &sp.c_cells, &one);
            for (const Item& it : jb.build(arena)) lay.emit(it);
            w.close();
            job.n_stages = static_cast<std::uint32_t>(sp.events.stage_off.size() - job.stage0);
            sp.events.arena_cells = std::max(sp.events.arena_cells, arena.high());
            sp.events.max_rows = std::max(sp.events.max_rows, job.n_rows);
            sp.events.jobs.push_back(job);
            coffs[i] = std::move(one[0]);
        }
    }

    // ---- root program: one job per root stripe, largest first ----------------
    sp.plan_yoff.resize(np);
    sp.plan_groups.resize(np);
    struct RootJob {
        std::size_t plan, g, s;
        std::uint64_t words;
    };
    std::vector<RootJob> rj;
    for (std::size_t i = 0; i < np; ++i) {
        const ButterflyPlan& p = *plans[i];
        sp.plan_yoff[i] = sp.y_rows;
        sp.plan_groups[i] = static_cast<std::uint32_t>(p.root_groups.size());
        sp.y_rows += static_cast<std::uint32_t>(p.root_groups.size() * p.n_rows);
        for (std::size_t g = 0; g < p.root_groups.size(); ++g)
            for (std::size_t s = 0; s < p.root_groups[g].size(); ++s) {
                rj.push_back(RootJob{i, g, s, p.root_groups[g][s].skeleton.words()});
                sp.roots.stored_words += p.root_groups[g][s].skeleton.words();
            }
    }
    std::stable_sort(rj.begin(), rj.end(), [](const RootJob& a, const RootJob& b) { return a.words > b.words; });
    {
        // dedicated root kernels: S and S^T per stripe, work items per 32 rows / columns
        RootSet& rs_out = sp.root_set;
        for (const RootJob& r : rj) {
            const ButterflyPlan& p = *plans[r.plan];
            const RootStripe& rs = p.root_groups[r.g][r.s];
            RootStripeDesc d{};
            d.rows = static_cast<std::uint32_t>(rs.row_count);
            d.rank = static_cast<std::uint32_t>(rs.skeleton.cols);
            if (d.rows > 64u * 255u || d.rank > 64u * 255u)
                throw std::length_error("packer: root stripe too large for the root kernels");
            d.yout = sp.plan_yoff[r.plan] + static_cast<std::uint32_t>(r.g * p.n_rows + rs.row_begin);
            d.yin = static_cast<std::uint32_t>(rs.row_begin);
            d.coff = coffs[r.plan][r.g][r.s];
            d.plan = static_cast<std::uint32_t>(r.plan);
            const std::size_t n = static_cast<std::size_t>(d.rows) * d.rank;
            d.lds = (d.rows + 1) & ~1u;
            d.ldt = (d.rank + 1) & ~1u;
            d.s_off = rs_out.data.size();
            rs_out.data.resize(rs_out.data.size() + static_cast<std::size_t>(d.lds) * d.rank, 0.0);
            for (std::uint32_t j = 0; j < d.rank; ++j)
                std::copy(rs.skeleton.col(j), rs.skeleton.col(j) + d.rows,
                          rs_out.data.begin() + static_cast<std::ptrdiff_t>(d.s_off + static_cast<std::size_t>(j) * d.lds));
            rs_out.data.resize((rs_out.data.size() + 3) & ~std::size_t{3}, 0.0);
            d.st_off = rs_out.data.size();
            rs_out.data.resize(rs_out.data.size() + static_cast<std::size_t>(d.ldt) * d.rows, 0.0);
            double* st = rs_out.data.data() + d.st_off;
            for (std::uint32_t j = 0; j < d.rank; ++j)
                for (std::uint32_t i = 0; i < d.rows; ++i) st[j + static_cast<std::size_t>(i) * d.ldt] = rs.skeleton(i, j);
            rs_out.data.resize((rs_out.data.size() + 3) & ~std::size_t{3}, 0.0);
            rs_out.stored_words += n;
            const std::uint32_t si = static_cast<std::uint32_t>(rs_out.stripes.size());
            if (si >= (1u << 24)) throw std::length_error("packer: too many root stripes");
            rs_out.stripes.push_back(d);
            for (std::uint32_t b = 0; b < (d.rows + 63) / 64; ++b) rs_out.fwd_items.push_back((si << 8) | b);
            for (std::uint32_t b = 0; b < (d.rank + 63) / 64; ++b) rs_out.bwd_items.push_back((si << 8) | b);
        }
    }
    {
        sp.roots.stage_capacity = root_cap;
        StageWriter w(sp.roots, root_cap);
        Layout lay(w);
        for (std::size_t jj = 0; jj < rj.size(); ++jj) {
            const RootJob& r = rj[jj];
            const ButterflyPlan& p = *plans[r.plan];
            const RootStripe& rs = p.root_groups[r.g][r.s];
            Job job{};
            job.n_plans = 1;
            job.mu = static_cast<std::uint16_t>(plan_mu[r.plan]);
            job.parity = static_cast<std::uint32_t>(plan_parity[r.plan]);
            job.plan[0] = static_cast<std::uint32_t>(r.plan);
            job.n_rows = static_cast<std::uint32_t>(rs.row_count);
            job.yin = static_cast<std::uint32_t>(rs.row_begin);
            job.yout = sp.plan_yoff[r.plan] + static_cast<std::uint32_t>(r.g * p.n_rows + rs.row_begin);
            CellAllocator arena;
            job.yA[0] = arena.alloc(job.n_rows);
            const std::uint32_t rank = static_cast<std::uint32_t>(rs.skeleton.cols);
            const std::uint32_t c = arena.alloc(rank);
            w.set_job(static_cast<std::uint32_t>(jj));
            job.stage0 = sp.roots.stage_off.size();
            Item cx;
            cx.op = OP_CXCH;
            cx.cells = c;
            cx.n = rank;
            cx.c_off = coffs[r.plan][r.g][r.s];
            cx.cload_fwd = true;       // forward loads, transpose stores
            cx.sync_bwd_last = true;   // transpose: after the panels wrote c
            lay.emit(cx);
            Item sm;
            sm.op = OP_SPANEL;
            sm.S = &rs.skeleton;
            sm.c = c;
            sm.y = job.yA[0];
            sm.group0 = true;          // each job owns its partial rows
            sm.sync_fwd_first = true;  // forward: after c arrived
            sm.sync_bwd_last = true;   // transpose: row chunks all write c
            lay.emit(sm);
            w.close();
            job.n_stages = static_cast<std::uint32_t>(sp.roots.stage_off.size() - job.stage0);
            sp.roots.arena_cells = std::max(sp.roots.arena_cells, arena.high());
            sp.roots.max_rows = std::max(sp.roots.max_rows, job.n_rows);
            sp.roots.jobs.push_back(job);
        }
    }
    return sp;
}

}  // namespace bfb
