// GPU plan construction for GL-row butterfly plan sets (SURVEY.md §8(f)
// rank 1): the Legendre matrices are generated on the device, and every
// interpolative decomposition of the build runs as a batched thread-block-
// cluster kernel; the host only schedules.
//
// What a plan is (and so what must come out) is the reference's: the events /
// StripeId / RootStripe structure of include/bfly/butterfly.hpp:18-74, built
// by the depth-first policy of src/butterfly.cpp:194-382 (leaf per block of
// `block_width` columns, merge of equal-level neighbours with the row halves
// of the next level partition, the adaptive epsilon of a half, the
// rank-crowding and storage refusals that freeze the level, the promote /
// merge tail) with IDs of the id_adaptive kind (src/id.cpp:31-235: column-
// pivoted Householder QR stopped at the first rank whose trailing columns
// are all within eps ||block||_F / sqrt(n), T = R11^-1 R12 moved toward
// |T| <= 2 by exchanging a skeleton column with the worst non-skeleton one).
//
// How it is computed is this library's own design:
//  * the plan set's dense matrices A(mu, p) live in HBM for a group of plans
//    (one recurrence thread per (order, node) writes both parities);
//  * skeletons are never copied: a stripe is (row span, list of source
//    columns), so an ID request names its block by row range + column list;
//  * every plan of the group advances its depth-first build as a resumable
//    state machine; a round collects the ID requests of every plan (all of a
//    plan's leaf IDs in the first round, then one merge / promote attempt per
//    plan), runs them in ONE batched launch per cluster size, and feeds the
//    results back;
//  * an ID request is factorised by a cluster of C CTAs (C = 1..16, chosen so
//    each CTA's row slice of the block fits shared memory): rows are split
//    over the cluster, every trailing column norm is recomputed exactly each
//    step (no downdating), and the cross-CTA sums (norms, the pivot row,
//    the reflector products) go through distributed shared memory with one
//    cluster barrier per reduction;
//  * T = R11^-1 R12 by a column-parallel back substitution kernel, written
//    compactly and read back once per round.
#pragma once

#include <cstdint>
#include <vector>

#include "builder.hpp"

namespace bfb {

// Same contract as build_glrow_planset (builder.hpp): every non-empty (mu, p)
// plan with mu in [mu_begin, mu_end), mu ascending, even before odd.  Runs on
// the current CUDA device.  `stats` (optional) receives timings.
struct GpuBuildStats {
    double seconds = 0.0, columns_s = 0.0, ids_s = 0.0, host_s = 0.0;
    long long id_tasks = 0, rounds = 0, refinements = 0, groups = 0;
};
std::vector<ButterflyPlan> build_glrow_planset_gpu(int l, int mu_begin, int mu_end, double eps,
                                                   std::int64_t block_width, std::vector<PlanKey>* keys,
                                                   const GlRule* rule = nullptr, GpuBuildStats* stats = nullptr);

// The default plan builder of the library: the GPU builder when a CUDA device
// is present (BFLY_BUILDER=host selects the threaded host builder).
std::vector<ButterflyPlan> build_glrow_planset_auto(int l, int mu_begin, int mu_end, double eps,
                                                    std::int64_t block_width, int threads, std::vector<PlanKey>* keys,
                                                    const GlRule* rule = nullptr);

}  // namespace bfb
