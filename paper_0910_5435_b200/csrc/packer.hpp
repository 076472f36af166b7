// Host packer: butterfly plans -> device program (see engine_format.hpp).
#pragma once

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
};

// job_plans[j] lists the plan indices (1 or 2) executed by job j; for the SHT
// job_mu[j] / job_parity[j] are its order and degree parity.  Plans within a
// job share n_rows.
PackedProgram pack_program(const std::vector<const ButterflyPlan*>& plans,
                           const std::vector<std::vector<int>>& job_plans,
                           const std::vector<int>& job_mu,
                           std::uint32_t stage_capacity = kStageBytesMax,
                           const std::vector<int>& job_parity = {});

}  // namespace bfb
