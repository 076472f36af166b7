// Device program format of the butterfly engine (shared by packer and kernel).
//
// A plan set is compiled into JOBS.  A job is the complete apply of one or
// two butterfly plans (for the SHT: the even and odd degree chains of one
// order mu) for a chunk of right-hand sides, executed by ONE CTA with every
// intermediate coefficient vector held in shared memory.  What the CTA
// streams from HBM is the job's byte stream: a sequence of STAGES (at most
// kStageBytes each), each a self-describing packet
//
//     [StageHeader][Rec x n_rec][payloads ...]
//
// fetched by one producer thread with cp.async.bulk (TMA bulk copy) into a
// shared-memory ring and consumed by four consumer warps.  Stages are stored
// back to back in HBM (16-byte aligned) and fetched with their exact byte
// counts, so packing slack inside a ring slot costs no HBM traffic.  The
// forward apply (reference bfly::apply, src/butterfly.cpp:384-442) walks the
// stages and their records in order; the transpose (bfly::apply_transpose,
// src/butterfly.cpp:444-513) walks the same stages and records backwards, so
// one copy of every matrix serves both directions.
//
// Records (all coefficient addresses are in "cells" = RC doubles, one value
// per right-hand side; z(k) = cell(k < kl ? zA + k : zB + k - kl)):
//   LOADZ   fwd: cell(zA + k) = input row (zB + k)          k < nr
//           bwd: output row (zB + k) = cell(zA + k)
//   SEL     fwd: cell(cA + i) = z(sel[i])                   i < nr
//           bwd: z(sel[i]) (=|+=) cell(cA + i)
//   TPANEL  fwd: cell(cA + i) += sum_q T[i, q] z(others[q]) i < nr, q < nc
//           bwd: z(others[q]) (=|+=) sum_i T[i, q] cell(cA + i)
//   SPANEL  fwd: cell(zA + i) (=|+=) sum_q S[i, q] cell(cA + q)
//           bwd: cell(cA + q) (=|+=) sum_i S[i, q] cell(zA + i)
// T / S panels are column-major with an ODD leading dimension ld >= nr, so
// both thread-per-row (forward) and thread-per-column (transpose) reads of
// 8-byte words are shared-memory bank-conflict free.
#pragma once

#include <cstdint>

namespace bfb {

constexpr int kStageBytes = 16384;
constexpr int kRingStages = 4;
constexpr int kConsumerThreads = 128;
constexpr int kEngineThreads = kConsumerThreads + 32;  // + one producer warp

enum RecOp : std::uint8_t { OP_LOADZ = 0, OP_SEL = 1, OP_TPANEL = 2, OP_SPANEL = 3 };

enum RecFlag : std::uint8_t {
    F_ASSIGN_FWD = 1,  // forward: '=' instead of '+=' on the written cells
    F_ASSIGN_BWD = 2,  // transpose: '=' instead of '+='
    F_SYNC_FWD = 4,    // consumer barrier before this record (forward order)
    F_SYNC_BWD = 8,    // consumer barrier before this record (transpose order)
};

struct alignas(16) Rec {
    std::uint8_t op;
    std::uint8_t flags;
    std::uint16_t nr;     // rows of the panel / count for LOADZ, SEL
    std::uint16_t nc;     // columns of the panel
    std::uint16_t ld;     // leading dimension of the panel (doubles, odd)
    std::uint32_t data;   // byte offset of the payload inside the stage
    std::uint32_t zA;     // z part 0 cells | SPANEL: y cells (row offset folded) | LOADZ: z cells
    std::uint32_t zB;     // z part 1 cells | LOADZ: first input row (col_begin)
    std::uint32_t kl;     // length of z part 0
    std::uint32_t cA;     // coefficient cells (panel row / column offset folded)
    std::uint16_t q0;     // TPANEL: absolute first column (transpose thread mapping)
    std::uint16_t pslot;  // plan slot inside the job (0 or 1), for I/O records
};
static_assert(sizeof(Rec) == 32, "Rec layout");

struct alignas(16) StageHeader {
    std::uint32_t n_rec;
    std::uint32_t bytes;  // bytes used in this stage (multiple of 16)
    std::uint32_t job;
    std::uint32_t pad;
};
static_assert(sizeof(StageHeader) == 16, "StageHeader layout");

// One job = one CTA's unit of work (times the number of RHS chunks).
struct alignas(16) Job {
    std::uint64_t stage0;      // index of the job's first stage
    std::uint32_t n_stages;
    std::uint16_t n_plans;     // 1 or 2
    std::uint16_t mu;          // SHT: order |m|
    std::uint32_t plan[2];     // plan indices (generic I/O offsets)
    std::uint32_t yA[2];       // cells of each plan's row vector (n_rows cells)
    std::uint32_t n_rows;
    std::uint32_t n_cols[2];
    std::uint32_t pad;
};
static_assert(sizeof(Job) == 48, "Job layout");

}  // namespace bfb
