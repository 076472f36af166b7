// Host compiler of the graph programs (see wgraph.hpp).
#include "wgraph.hpp"

#include <algorithm>
#include <stdexcept>

namespace bfb {

GraphProgram build_graph(const WaveSet& w, std::uint32_t group_nodes, bool wavefront) {
    const std::size_t nn = w.nodes.size(), np = w.plan_in.size();
    if (w.node_src.size() != 2 * nn || w.plan_node_begin.size() != np + 1)
        throw std::runtime_error("graph: wave set without producer records");
    constexpr std::uint32_t kNone = ~0u;
    GraphProgram g;

    std::vector<std::uint32_t> node_plan(nn);
    for (std::size_t p = 0; p < np; ++p)
        for (std::uint32_t n = w.plan_node_begin[p]; n < w.plan_node_begin[p + 1]; ++n)
            node_plan[n] = static_cast<std::uint32_t>(p);
    auto live = [&](std::uint32_t n) { return n != kNone && w.nodes[n].rank > 0; };

    // Plan groups: consecutive plans of about group_nodes nodes.
    std::vector<std::uint32_t> plan_group(np);
    {
        std::uint32_t grp = 0, count = 0;
        for (std::size_t p = 0; p < np; ++p) {
            plan_group[p] = grp;
            count += w.plan_node_begin[p + 1] - w.plan_node_begin[p];
            if (count >= group_nodes && p + 1 < np) {
                ++grp;
                count = 0;
            }
        }
        g.groups = np ? grp + 1 : 0;
    }
    const std::vector<RootStripeDesc>& st = w.roots.stripes;
    std::vector<std::vector<std::uint32_t>> plan_stripes(np);
    for (std::uint32_t s = 0; s < st.size(); ++s) plan_stripes[st[s].plan].push_back(s);
    auto work = [&](std::uint32_t n) { return static_cast<std::uint64_t>(w.nodes[n].rank) * (w.nodes[n].nothers + 1); };

    // ---- forward -----------------------------------------------------------
    // Buckets (plan group, level) and (plan group, roots); emitted group-major (a group's levels,
    // then its roots) or, wavefront, along the diagonals group + level = const: a bucket's consumers
    // follow one diagonal (a few thousand items) later -- far enough that their producers have
    // finished, near enough that the vectors are still in L2.
    int max_level = 0;
    for (std::uint32_t n = 0; n < nn; ++n)
        if (w.nodes[n].rank > 0) max_level = std::max(max_level, static_cast<int>(w.nodes[n].level));
    std::vector<std::uint32_t> node_item(nn, kNone);
    {
        std::vector<std::vector<std::vector<std::uint32_t>>> bucket(
            g.groups, std::vector<std::vector<std::uint32_t>>(static_cast<std::size_t>(max_level) + 1));
        for (std::uint32_t n = 0; n < nn; ++n)
            if (w.nodes[n].rank > 0) bucket[plan_group[node_plan[n]]][w.nodes[n].level].push_back(n);
        std::vector<std::size_t> grp_plan0(g.groups + 1, np);
        for (std::size_t p = np; p-- > 0;) grp_plan0[plan_group[p]] = p;
        auto emit_nodes = [&](std::vector<std::uint32_t>& ns) {
            std::stable_sort(ns.begin(), ns.end(), [&](std::uint32_t a, std::uint32_t b) { return work(a) > work(b); });
            for (std::uint32_t n : ns) {
                GraphItem it{};
                it.kind = GK_NODE_FWD;
                it.a = n;
                it.b = kNone;
                it.dep0 = static_cast<std::uint32_t>(g.fwd_deps.size());
                for (int k = 0; k < 2; ++k) {
                    const std::uint32_t src = w.node_src[2 * n + k];
                    if (!live(src)) continue;
                    if (node_item[src] == kNone) throw std::runtime_error("graph: forward order is not topological");
                    if (k == 1 && src == w.node_src[2 * n]) continue;
                    g.fwd_deps.push_back(node_item[src]);
                }
                it.ndep = static_cast<std::uint32_t>(g.fwd_deps.size()) - it.dep0;
                node_item[n] = static_cast<std::uint32_t>(g.fwd.size());
                g.fwd.push_back(it);
            }
        };
        auto emit_roots = [&](std::uint32_t grp) {
            // the group's root row blocks: the union of every root group's stripe
            // boundaries, cut to at most kGraphMaxRows rows
            std::vector<GraphItem> roots;
            for (std::size_t p0 = grp_plan0[grp]; p0 < np && plan_group[p0] == grp; ++p0) {
                const std::vector<std::uint32_t>& ss = plan_stripes[p0];
                if (ss.empty()) continue;
                std::vector<std::uint32_t> cuts;
                for (std::uint32_t s : ss) {
                    cuts.push_back(st[s].yin);
                    cuts.push_back(st[s].yin + st[s].rows);
                }
                std::sort(cuts.begin(), cuts.end());
                cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
                for (std::size_t c = 0; c + 1 < cuts.size(); ++c) {
                    for (std::uint32_t r0 = cuts[c]; r0 < cuts[c + 1]; r0 += kGraphMaxRows) {
                        const std::uint32_t r1 = std::min(cuts[c + 1], r0 + kGraphMaxRows);
                        GraphItem it{};
                        it.kind = GK_ROOT_FWD;
                        it.a = static_cast<std::uint32_t>(g.segs.size());
                        it.plan = static_cast<std::uint32_t>(p0);
                        it.r0 = r0;
                        it.rows = r1 - r0;
                        it.dep0 = kNone;  // filled below (item indices known after sorting)
                        for (std::uint32_t s : ss)
                            if (st[s].yin <= r0 && r1 <= st[s].yin + st[s].rows && st[s].rank > 0)
                                g.segs.push_back(RootSeg{s, r0 - st[s].yin});
                        it.b = static_cast<std::uint32_t>(g.segs.size()) - it.a;
                        roots.push_back(it);
                    }
                }
            }
            auto rwork = [&](const GraphItem& it) {
                std::uint64_t k = 0;
                for (std::uint32_t i = 0; i < it.b; ++i) k += st[g.segs[it.a + i].stripe].rank;
                return k * it.rows;
            };
            std::stable_sort(roots.begin(), roots.end(),
                             [&](const GraphItem& a, const GraphItem& b) { return rwork(a) > rwork(b); });
            for (GraphItem& it : roots) {
                it.dep0 = static_cast<std::uint32_t>(g.fwd_deps.size());
                for (std::uint32_t i = 0; i < it.b; ++i) {
                    const std::uint32_t src = static_cast<std::uint32_t>(st[g.segs[it.a + i].stripe].st_off);
                    if (!live(src)) continue;
                    if (node_item[src] == kNone) throw std::runtime_error("graph: root before its producer");
                    g.fwd_deps.push_back(node_item[src]);
                }
                it.ndep = static_cast<std::uint32_t>(g.fwd_deps.size()) - it.dep0;
                g.fwd.push_back(it);
            }
        };
        if (!wavefront) {
            for (std::uint32_t grp = 0; grp < g.groups; ++grp) {
                for (int L = 1; L <= max_level; ++L) emit_nodes(bucket[grp][static_cast<std::size_t>(L)]);
                emit_roots(grp);
            }
        } else {
            // diagonal t: (group t, level 1), (group t - 1, level 2), ..., (group t - max_level, roots)
            for (long long t = 0; t < static_cast<long long>(g.groups) + max_level; ++t)
                for (int L = 1; L <= max_level + 1; ++L) {
                    const long long grp = t - (L - 1);
                    if (grp < 0 || grp >= static_cast<long long>(g.groups)) continue;
                    if (L <= max_level)
                        emit_nodes(bucket[static_cast<std::size_t>(grp)][static_cast<std::size_t>(L)]);
                    else
                        emit_roots(static_cast<std::uint32_t>(grp));
                }
        }
    }

    // ---- transpose ---------------------------------------------------------
    // who reads a node's output in the forward = who writes it in the transpose
    const std::size_t npairs = w.pairs.size() / 2;
    std::vector<std::uint32_t> cons_pair(nn, kNone), cons_stripe(nn, kNone);
    for (std::size_t P = 0; P < npairs; ++P)
        for (int k = 0; k < 2; ++k) {
            const std::uint32_t x = w.pairs[2 * P + k];
            if (x == kNone) continue;
            for (int j = 0; j < 2; ++j) {
                const std::uint32_t src = w.node_src[2 * x + j];
                if (src != kNone) cons_pair[src] = static_cast<std::uint32_t>(P);
            }
        }
    for (std::uint32_t s = 0; s < st.size(); ++s) {
        const std::uint32_t src = static_cast<std::uint32_t>(st[s].st_off);
        if (src != kNone) cons_stripe[src] = s;
    }
    {
        std::vector<std::uint32_t> pair_item(npairs, kNone), stripe_item(st.size(), kNone);
        std::vector<std::vector<std::uint32_t>> grp_pairs(g.groups), grp_stripes(g.groups);
        for (std::uint32_t P = 0; P < npairs; ++P) grp_pairs[plan_group[node_plan[w.pairs[2 * P]]]].push_back(P);
        for (std::uint32_t s = 0; s < st.size(); ++s) grp_stripes[plan_group[st[s].plan]].push_back(s);
        auto plevel = [&](std::uint32_t P) {
            const std::uint32_t a = w.pairs[2 * P], b = w.pairs[2 * P + 1];
            return std::max(w.nodes[a].level, b == kNone ? 0u : w.nodes[b].level);
        };
        auto pwork = [&](std::uint32_t P) {
            const std::uint32_t b = w.pairs[2 * P + 1];
            return work(w.pairs[2 * P]) + (b == kNone ? 0 : work(b));
        };
        auto emit_stripes = [&](std::uint32_t grp) {
            std::vector<std::uint32_t>& ss = grp_stripes[grp];
            std::stable_sort(ss.begin(), ss.end(), [&](std::uint32_t a, std::uint32_t b) {
                return static_cast<std::uint64_t>(st[a].rows) * st[a].rank > static_cast<std::uint64_t>(st[b].rows) * st[b].rank;
            });
            for (std::uint32_t s : ss) {
                GraphItem it{};
                it.kind = GK_ROOT_BWD;
                it.a = s;
                it.b = kNone;
                it.dep0 = static_cast<std::uint32_t>(g.bwd_deps.size());
                it.ndep = 0;
                stripe_item[s] = static_cast<std::uint32_t>(g.bwd.size());
                g.bwd.push_back(it);
            }
        };
        // pairs of one group at one level (level < 0: all, deepest level first)
        auto emit_pairs = [&](std::uint32_t grp, int level) {
            std::vector<std::uint32_t> ps;
            for (std::uint32_t P : grp_pairs[grp])
                if (level < 0 || static_cast<int>(plevel(P)) == level) ps.push_back(P);
            std::stable_sort(ps.begin(), ps.end(), [&](std::uint32_t a, std::uint32_t b) {
                if (plevel(a) != plevel(b)) return plevel(a) > plevel(b);
                return pwork(a) > pwork(b);
            });
            for (std::uint32_t P : ps) {
                GraphItem it{};
                it.kind = GK_PAIR_BWD;
                it.a = w.pairs[2 * P];
                it.b = w.pairs[2 * P + 1];
                it.dep0 = static_cast<std::uint32_t>(g.bwd_deps.size());
                for (int k = 0; k < 2; ++k) {
                    const std::uint32_t x = k == 0 ? it.a : it.b;
                    if (!live(x)) continue;
                    std::uint32_t d = kNone;
                    if (cons_pair[x] != kNone)
                        d = pair_item[cons_pair[x]];
                    else if (cons_stripe[x] != kNone)
                        d = stripe_item[cons_stripe[x]];
                    else
                        throw std::runtime_error("graph: a node output nobody reads");
                    if (d == kNone) throw std::runtime_error("graph: transpose order is not topological");
                    if (it.ndep == 1 && g.bwd_deps.back() == d) continue;
                    g.bwd_deps.push_back(d);
                    it.ndep = static_cast<std::uint32_t>(g.bwd_deps.size()) - it.dep0;
                }
                it.ndep = static_cast<std::uint32_t>(g.bwd_deps.size()) - it.dep0;
                pair_item[P] = static_cast<std::uint32_t>(g.bwd.size());
                g.bwd.push_back(it);
            }
        };
        if (!wavefront) {
            for (std::uint32_t grp = 0; grp < g.groups; ++grp) {
                emit_stripes(grp);
                emit_pairs(grp, -1);
            }
        } else {
            // diagonal t: (group t, root stripes), (group t - 1, level max), ..., (group t - max, level 1);
            // level 0 holds the pairs without a live node level (copies)
            int pmax = 0;
            for (std::uint32_t P = 0; P < npairs; ++P) pmax = std::max(pmax, static_cast<int>(plevel(P)));
            for (long long t = 0; t < static_cast<long long>(g.groups) + pmax + 1; ++t)
                for (int k = 0; k <= pmax + 1; ++k) {
                    const long long grp = t - k;
                    if (grp < 0 || grp >= static_cast<long long>(g.groups)) continue;
                    if (k == 0)
                        emit_stripes(static_cast<std::uint32_t>(grp));
                    else
                        emit_pairs(static_cast<std::uint32_t>(grp), pmax + 1 - k);
                }
        }
    }
    for (int k = 0; k < 2; ++k) {
        std::vector<GraphItem>& items = k ? g.bwd : g.fwd;
        const std::vector<std::uint32_t>& deps = k ? g.bwd_deps : g.fwd_deps;
        for (GraphItem& it : items)
            for (std::uint32_t d = 0; d < kGraphInlineDeps; ++d) it.dep[d] = d < it.ndep ? deps[it.dep0 + d] : ~0u;
    }
    // every dependency precedes its item (the kernel's deadlock freedom rests on it)
    for (int k = 0; k < 2; ++k) {
        const std::vector<GraphItem>& items = k ? g.bwd : g.fwd;
        const std::vector<std::uint32_t>& deps = k ? g.bwd_deps : g.fwd_deps;
        for (std::size_t i = 0; i < items.size(); ++i)
            for (std::uint32_t d = 0; d < items[i].ndep; ++d)
                if (deps[items[i].dep0 + d] >= i) throw std::runtime_error("graph: a dependency after its item");
    }
    return g;
}

}  // namespace bfb
