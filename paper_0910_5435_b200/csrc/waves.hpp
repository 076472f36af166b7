// Level-synchronous ("wave") programs: the batched butterfly apply.
//
// The whole-chain engine (engine.cu) runs one plan per CTA with every
// coefficient vector in shared memory, which is the right shape for a single
// function (4 right-hand sides: +-m x re/im) but streams the plans once per
// batch member.  With a batch of B functions (R = 4B right-hand sides) the
// apply becomes a sequence of small dense contractions, so the wave program
// replays every plan's event stack symbolically on the host (reference
// bfly::apply, src/butterfly.cpp:384-442) and gives every coefficient vector a
// place in one global, cell-major buffer V[cell][R]:
//
//   * each StripeId becomes a NODE: c[rank] = z[sel] + T * z[others], with z
//     the concatenation of its input vectors (leaf: the chain's coefficient
//     columns, merge: [left[s]; right[s]], promote: parent[s]), written as
//     absolute V cells;
//   * nodes are grouped into LEVELS (a node's level = 1 + the largest level of
//     its inputs; the chain coefficients are level 0), and one launch per level
//     applies every node of every plan for all R right-hand sides (FP64 DMMA,
//     wavekern.cu);
//   * the transpose (bfly::apply_transpose, :444-513) walks the levels
//     backwards; the two StripeIds that share one z (a merge or promote pair)
//     form one transposed work item, so the '+=' into z needs no atomics;
//   * the root stage is the tensor-core root kernel (rootmma.cu) with C = V.
//
// Every matrix word is read from HBM once per launch for all R right-hand
// sides; the vectors travel through HBM / L2 between levels.
#pragma once

#include <cstdint>
#include <vector>

#include "packer.hpp"
#include "plan.hpp"

namespace bfb {

struct alignas(16) WaveNode {
    std::uint64_t t_off;    // doubles: T (rank x nothers), 16 x 16 tiles (packer.hpp tiled_index)
    std::uint32_t rank;     // output cells
    std::uint32_t nothers;  // interpolation columns
    std::uint32_t idx;      // u32 index array: sel cells [rank], then others cells [nothers]
    std::uint32_t cA;       // first output cell (c = V[cA .. cA + rank))
    std::uint32_t level;
    std::uint32_t nib;      // row tiles of T: tiles16(rank)
};
static_assert(sizeof(WaveNode) == 32, "WaveNode layout");

struct WaveSet {
    std::vector<double> T;               // interpolation matrices, back to back
    std::vector<std::uint32_t> idx;      // absolute V cells
    std::vector<WaveNode> nodes;         // every StripeId of every plan
    std::vector<std::uint32_t> fwd;      // forward items (nodes with rank > 0), by level, largest first
    std::vector<std::uint32_t> fwd_begin;  // items of level L (1-based): [fwd_begin[L-1], fwd_begin[L])
    std::vector<std::uint32_t> pairs;    // transposed items: (node a, node b or ~0u) sharing one z, by level
    std::vector<std::uint32_t> bwd_begin;  // pairs of level L: [bwd_begin[L-1], bwd_begin[L])
    int levels = 0;
    std::uint32_t v_cells = 0;
    std::vector<std::uint32_t> plan_in;  // per plan: V cell of its coefficient column 0
    std::vector<std::uint32_t> plan_mu, plan_parity, plan_cols;
    RootSet roots;                       // S only (tiled, lds = row tiles); coff = V cells; pad[0] root group,
                                         // pad[1] stacked first row;
                                         // st_off = the node writing the coefficient cells (~0u: none)
    std::uint32_t y_rows = 0;
    std::vector<std::uint32_t> plan_yoff, plan_groups;
    std::vector<std::uint32_t> plan_row0;  // per plan: first stacked row (plan-set apply)
    std::vector<std::uint32_t> node_src;         // per node: the two nodes writing its inputs (~0u: coefficients / none)
    std::vector<std::uint32_t> plan_node_begin;  // nodes of plan p: [plan_node_begin[p], plan_node_begin[p + 1])
    std::uint64_t aliased_leaves = 0;    // full-rank leaves folded into their consumers
    std::uint64_t event_words = 0;       // interpolation words (read once per launch)
    std::uint64_t root_words = 0;        // skeleton words
};

WaveSet build_waves(const std::vector<const ButterflyPlan*>& plans, const std::vector<int>& plan_mu,
                    const std::vector<int>& plan_parity);

}  // namespace bfb
