// Dependency-ordered ("graph") execution of the wave programs (waves.hpp).
//
// The level-synchronous wave programs launch one kernel per butterfly level
// and one per root group, so every level's coefficient vectors make a round
// trip through HBM (at c3 the DRAM traffic was 2.3x the algorithmic bytes)
// and every launch drains to a tail.  The graph program instead lists every
// unit of work of one direction in ONE queue, in an order that is topological
// (every item after the items that write its inputs) and group-major: the
// plans are cut into groups of about `group_nodes` nodes, and a group's items
// run level by level (then its roots) before the next group's.  One persistent
// kernel (wgraph.cu) claims items in queue order from an atomic counter and
// waits, per item, until the items it depends on have published their
// outputs; the window of items in flight then spans one or two groups, whose
// vectors stay in L2 between producer and consumer.
//
// Items (one direction):
//   forward  (bfly::apply, reference src/butterfly.cpp:384-442)
//     NODE_FWD  node n:           c = z[sel] + T z[others]        deps: the nodes writing z
//     ROOT_FWD  plan, row block:  u[rows] = sum over root groups of S_g[rows, :] c_g
//                                 (the groups' stripes covering the block;
//                                 :430-440; the sum stays in registers, so the
//                                 groups need no ordering)           deps: the nodes writing c_g
//   transpose (bfly::apply_transpose, :444-513)
//     ROOT_BWD  stripe s:         c = S^T u[rows]                  no deps
//     PAIR_BWD  nodes a (, b):    z (=|+=) T_a^T c_a (+ T_b^T c_b), z[sel] (=|+=) c
//                                 (the one or two StripeIds sharing one z)
//                                 deps: the items that wrote c_a, c_b
#pragma once

#include <cstdint>
#include <vector>

#include "waves.hpp"

namespace bfb {

enum GraphKind : std::uint32_t { GK_NODE_FWD = 0, GK_ROOT_FWD = 1, GK_PAIR_BWD = 2, GK_ROOT_BWD = 3 };

constexpr std::uint32_t kGraphInlineDeps = 8;
struct alignas(16) GraphItem {
    std::uint32_t kind;
    std::uint32_t a;     // NODE_FWD: node; PAIR_BWD: first node; ROOT_BWD: stripe; ROOT_FWD: first segment
    std::uint32_t b;     // PAIR_BWD: second node (~0u: none); ROOT_FWD: number of segments
    std::uint32_t dep0;  // dependencies: deps[dep0 .. dep0 + ndep) (item indices, same queue)
    std::uint32_t ndep;
    std::uint32_t plan;  // ROOT_FWD: plan
    std::uint32_t r0;    // ROOT_FWD: first row of the block
    std::uint32_t rows;  // ROOT_FWD: rows of the block (<= kGraphMaxRows)
    std::uint32_t dep[kGraphInlineDeps];  // the first dependencies again (the kernel prefetches the item as one 64-byte record)
};
static_assert(sizeof(GraphItem) == 64, "GraphItem layout");

// A root stripe's share of a forward row block: rows [row_off, row_off + rows) of the stripe.
struct RootSeg {
    std::uint32_t stripe;
    std::uint32_t row_off;
};

#ifndef BFB_GRAPH_MAXROWS
#define BFB_GRAPH_MAXROWS 64
#endif
constexpr std::uint32_t kGraphMaxRows = BFB_GRAPH_MAXROWS;  // output rows per pass of the graph kernel (root blocks are cut to it)

struct GraphProgram {
    std::vector<GraphItem> fwd, bwd;
    std::vector<std::uint32_t> fwd_deps, bwd_deps;
    std::vector<RootSeg> segs;
    std::uint32_t groups = 0;
};

// Needs the producer records of build_waves (WaveSet::node_src, plan_node_begin,
// RootStripeDesc::st_off).
// wavefront: emit the (plan group, level) buckets along the diagonals group + level = const instead of
// group by group (small groups then keep producer and consumer a few thousand items apart).
GraphProgram build_graph(const WaveSet& w, std::uint32_t group_nodes, bool wavefront = false);

}  // namespace bfb
