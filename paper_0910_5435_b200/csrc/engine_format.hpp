// Device program format of the butterfly engine (shared by packer and kernel).
//
// A plan set is compiled into JOBS.  A job is the complete apply of one (or
// two) butterfly plans (for the SHT: one degree chain of one order mu) for a
// chunk of right-hand sides, executed by ONE CTA with every
// intermediate coefficient vector held in shared memory.  What the CTA
// streams from HBM is the job's byte stream: a sequence of STAGES (at most
// the program's stage capacity each), each a self-describing packet
//
//     [StageHeader][Rec x n_rec][payloads ...]
//
// fetched by one producer thread with cp.async.bulk (TMA bulk copy) into a
// shared-memory ring and consumed by a few consumer warps; several such
// CTAs (jobs) share each SM, so independent dependency chains overlap.  Stages are stored
// back to back in HBM (16-byte aligned) and fetched with their exact byte
// counts, so packing slack inside a ring slot costs no HBM traffic.  The
// forward apply (reference bfly::apply, src/butterfly.cpp:384-442) walks the
// stages and their records in order; the transpose (bfly::apply_transpose,
// src/butterfly.cpp:444-513) walks the same stages and records backwards, so
// one copy of every matrix serves both directions.
//
// Cells: every coefficient vector element is a "cell" of RC doubles, one per
// right-hand side.  z(k) = cell(k < kl ? zA + k : zB + k - kl) is the input
// of a StripeId (the reference's [left[s]; right[s]] concatenation).
//
// Records:
//   LOADZ   fwd: cells zA..zA+nr = input rows zB..zB+nr (cp.async prefetch)
//           bwd: output rows zB.. = cells zA..            (the leaf's output)
//   SEL     a StripeId without interpolation columns (full-rank leaf):
//           fwd: cell(cA + i) = z(sel[i]);  bwd: z(sel[i]) (=|+=) cell(cA + i)
//   TPANEL  columns of a StripeId's interpolation matrix T (rows = one chunk
//           of <= kChunkRows of the rank).  A UNIT is the run of panels of
//           one chunk, from the BEGIN record to the END record.
//           fwd: cell(cA + i) = z(sel[i]) + sum_q T[i, q] z(others[q])
//                (accumulated in registers across the unit, written at END)
//           bwd: z(others[q]) (=|+=) sum_i T[i, q] cell(cA + i)  per panel,
//                and at BEGIN z(sel[i]) (=|+=) cell(cA + i)
//   SPANEL  columns of a root skeleton S (rows = one chunk of the stripe):
//           fwd: cell(zA + i) (=|+=) sum_q S[i, q] cell(cA + q)   at END
//           bwd: cell(cA + q) (=|+=) sum_i S[i, q] cell(zA + i)   per panel
//   CXCH    cells zA..zA+nr <-> global coefficient buffer C at zB (split
//           programs: the event program hands the surviving blocks' vectors
//           to the root program through C).
// Panel payload: [u16 others[nc] (TPANEL)][u16 sel[nr] (TPANEL BEGIN only)]
//                [f64 panel, column-major, odd leading dimension ld >= nr]
//                at data + moff.  The odd ld keeps the transpose's
//                lane-per-column reads free of shared-memory bank conflicts.
#pragma once

#include <cstdint>

namespace bfb {

constexpr int kStageBytesMax = 49152;  // largest stage capacity (ring slot size)
constexpr int kStageBytesMin = 8192;
#ifndef BFB_RING_STAGES
#define BFB_RING_STAGES 2
#endif
constexpr int kRingStages = BFB_RING_STAGES;  // ring slots per CTA
#ifndef BFB_CONSUMER_WARPS
#define BFB_CONSUMER_WARPS 4
#endif
constexpr int kConsumerWarps = BFB_CONSUMER_WARPS;
constexpr int kConsumerThreads = 32 * kConsumerWarps;
constexpr int kEngineThreads = kConsumerThreads + 32;  // + one producer warp
#ifndef BFB_CHUNK_ROWS
#define BFB_CHUNK_ROWS 128
#endif
constexpr int kChunkRows = BFB_CHUNK_ROWS;            // rows per unit

enum RecOp : std::uint8_t { OP_LOADZ = 0, OP_SEL = 1, OP_TPANEL = 2, OP_SPANEL = 3, OP_CXCH = 4 };

enum RecFlag : std::uint8_t {
    F_ASSIGN_FWD = 1,      // forward: '=' instead of '+=' on the written cells (SPANEL END)
    F_ASSIGN_BWD = 2,      // transpose: '=' on the panel's outputs
    F_SYNC_FWD = 4,        // consumer barrier before this record (forward order)
    F_SYNC_BWD = 8,        // consumer barrier before this record (transpose order)
    F_BEGIN = 16,          // first record of a unit (forward order)
    F_END = 32,            // last record of a unit (forward order)
    F_ASSIGN_SEL_BWD = 64, // transpose: '=' for the z(sel) scatter at BEGIN
    F_CLOAD_FWD = 128,     // CXCH: forward loads cells from C (transpose stores); else the reverse
};

struct alignas(16) Rec {
    std::uint8_t op;
    std::uint8_t flags;
    std::uint16_t nr;     // unit rows (panels) / count (LOADZ, SEL)
    std::uint16_t nc;     // panel columns
    std::uint16_t moff;   // offset of the f64 panel from data
    std::uint32_t data;   // byte offset of the payload inside the stage
    std::uint32_t zA;     // z part 0 | SPANEL: y cells (chunk row offset folded) | LOADZ: cells
    std::uint32_t zB;     // z part 1 | LOADZ: first input row
    std::uint32_t kl;     // length of z part 0
    std::uint32_t cA;     // coefficient cells (chunk row / panel column offset folded)
    std::uint16_t ld;     // panels: leading dimension (odd, >= nr)
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
    std::uint32_t parity;      // SHT: degree parity of the (single) plan
    std::uint32_t yin;         // root jobs: first row of the stripe (input rows)
    std::uint32_t yout;        // root jobs: row offset of the partial output
    std::uint32_t kind;        // merged SHT programs: 0 event job, 1 root job
    std::uint32_t pad;
};
static_assert(sizeof(Job) == 64, "Job layout");

}  // namespace bfb
