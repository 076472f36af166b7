// Host packer: butterfly plans -> device program (see engine_format.hpp).
#pragma once

#include <cstddef>
#include <cstdint>
#include <vector>

#include "engine_format.hpp"
#include "plan.hpp"

namespace bfb {

struct PackedProgram {
    std::vector<std::uint8_t> stream;        // all stages back to back
    std::vector<std::uint64_t> stage_off;    // byte offset of each stage (16-aligned)
    std::vector<std::uint32_t> stage_bytes;  // bytes to fetch per stage (multiple of 16)
    std::vector<Job> jobs;                   // sorted by decreasing stream bytes
    std::uint32_t arena_cells = 0;           // max over jobs
    std::uint32_t zo_cells = 0;              // widest interpolation matrix (gathered z block)
    std::uint64_t stored_words = 0;          // sum of plan.stored_words (algorithmic)
    std::uint64_t fetched_bytes = 0;         // sum of stage_bytes (what one apply streams)
    std::uint32_t max_rows = 0;
    std::uint32_t stage_capacity = kStageBytesMax;  // ring slot size the stages were cut for
    // Task order per direction (empty = job order); merged SHT programs run
    // event jobs first forward and root jobs first in the transpose.
    std::vector<std::uint32_t> order_fwd, order_bwd;
    std::vector<std::uint32_t> plan_roots;  // merged programs: root jobs per plan
};

// job_plans[j] lists the plan indices (1 or 2) executed by job j; for the SHT
// job_mu[j] / job_parity[j] are its order and degree parity.  Plans within a
// job share n_rows.
PackedProgram pack_program(const std::vector<const ButterflyPlan*>& plans,
                           const std::vector<std::vector<int>>& job_plans,
                           const std::vector<int>& job_mu,
                           std::uint32_t stage_capacity = kStageBytesMax,
                           const std::vector<int>& job_parity = {});

// Split compilation of single-chain jobs (the SHT): an event program (one job
// per plan: leaves, merges, promotes; the surviving blocks' coefficient
// vectors are exchanged with the global buffer C) and a root program (one job
// per root stripe: the dense skeleton product, writing a per-group partial of
// the plan's rows).  plan_yoff[p] / plan_groups[p] locate plan p's partials:
// rows yoff + g * n_rows + i, g < groups.
// Root skeletons for the dedicated root kernels: every stripe stored twice,
// S (rows x rank) and S^T (rank x rows), both column-major, 32-byte aligned.
// Storage of the wave programs' matrices (T of a node, S of a root stripe):
// 16 x 16 tiles, tile (ib, qb) of a matrix with nib row tiles at doubles
// (qb * nib + ib) * 256, each tile column-major with the row index XOR-swizzled
// by 4 (q & 3).  So the 16 columns of a forward K-chunk are ONE contiguous run
// of tiles and the 16 rows of a transposed K-chunk are whole 2 KB tiles (TMA
// bulk copies either way), and the DMMA fragment loads of both directions hit
// 16 distinct double slots per half-warp (no bank conflicts).  Padding rows and
// columns are zero.
constexpr std::uint32_t kTileDim = 16;
inline std::uint32_t tiles16(std::uint64_t n) { return static_cast<std::uint32_t>((n + 15) / 16); }
inline std::size_t tiled_index(std::uint32_t i, std::uint32_t q, std::uint32_t nib) {
    return (static_cast<std::size_t>(q >> 4) * nib + (i >> 4)) * 256 + (q & 15) * 16 + ((i & 15) ^ (4 * (q & 3)));
}
inline std::size_t tiled_size(std::uint64_t rows, std::uint64_t cols) {
    return static_cast<std::size_t>(tiles16(rows)) * tiles16(cols) * 256;
}

struct alignas(16) RootStripeDesc {
    std::uint64_t s_off;   // doubles: S, leading dimension lds (rows rounded up to even)
    std::uint64_t st_off;  // doubles: S^T, leading dimension ldt (rank rounded up to even)
    std::uint32_t rows, rank;
    std::uint32_t lds, ldt;
    std::uint32_t yout;    // forward: first partial row (plan_yoff + g * n_rows + row_begin)
    std::uint32_t yin;     // transpose: first input row (row_begin)
    std::uint32_t coff;    // C offset of the stripe's coefficient vector
    std::uint32_t plan;    // plan index (input rows u[plan])
    std::uint32_t pad[2];
};
static_assert(sizeof(RootStripeDesc) == 64, "RootStripeDesc layout");

struct RootSet {
    std::vector<double> data;
    std::vector<RootStripeDesc> stripes;
    std::vector<std::uint32_t> fwd_items;  // (stripe << 8) | 64-row block, largest stripes first
    std::vector<std::uint32_t> bwd_items;  // (stripe << 8) | 64-column block
    std::uint64_t stored_words = 0;        // sum rows * rank (read once per direction)
};

struct SplitProgram {
    PackedProgram events;
    PackedProgram roots;
    RootSet root_set;
    std::uint32_t c_cells = 0;  // size of C (cells per right-hand-side chunk)
    std::uint32_t y_rows = 0;   // rows of the partial-output buffer
    std::vector<std::uint32_t> plan_yoff, plan_groups;
};
// One program holding both job kinds of a split compilation (the root stages
// appended after the event stages); jobs wait on per-plan flags at run time.
PackedProgram merge_split(const SplitProgram& sp, std::size_t n_plans);

SplitProgram pack_split(const std::vector<const ButterflyPlan*>& plans, const std::vector<int>& plan_mu,
                        const std::vector<int>& plan_parity, std::uint32_t event_stage_capacity,
                        std::uint32_t root_stage_capacity);

}  // namespace bfb
