// Butterfly engine: device program + launch interface (host side).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "engine_format.hpp"
#include "packer.hpp"

namespace bfb {

// Right-hand sides per CTA job (cells of RC doubles).
constexpr int kRC = 4;

// Device-resident program (uploaded once).
struct DeviceProgram {
    std::uint8_t* stream = nullptr;
    std::uint64_t* stage_off = nullptr;
    std::uint32_t* stage_bytes = nullptr;
    Job* jobs = nullptr;
    unsigned* counters = nullptr;  // [2] persistent-scheduler work counter (never reset)
    mutable unsigned claimed = 0;  // host: increments the counter has seen (sum of n_tasks)
    int n_jobs = 0;
    std::uint64_t n_stages = 0;
    std::uint32_t arena_cells = 0;
    std::uint32_t zo_cells = 0;
    std::uint32_t stage_capacity = kStageBytesMax;
    std::uint64_t stream_bytes = 0;
    std::uint64_t fetched_bytes = 0;
    std::uint64_t stored_words = 0;
    int device = 0;
    std::uint32_t* order[2] = {nullptr, nullptr};  // task -> job per direction (merged programs)
    std::uint32_t* plan_roots = nullptr;           // merged programs: root jobs per plan
    unsigned long long* trace = nullptr;  // optional: 4 u64 per task (start ns, end ns, smid, stages)
    int debug = 0;                        // diagnostics: bit 0 = stream stages only (no arithmetic)
};

DeviceProgram upload_program(const PackedProgram& p, int device);
void free_program(DeviceProgram& d);

// Generic I/O: plan p's input is the column-major block at
// in + nrhs * in_prefix[p] (n_in x nrhs, ld = n_in); output likewise.
struct GenericIO {
    const double* in = nullptr;
    double* out = nullptr;
    const std::uint64_t* in_prefix = nullptr;   // device, per plan: sum of n_in of earlier plans
    const std::uint64_t* out_prefix = nullptr;  // device, per plan: sum of n_out of earlier plans
    int nrhs = 0;
};

// SHT I/O (see include/bfly_b200.h for the layouts).  The phi-stage buffers
// g_in / g_out are [bin][b][t] complex: bin = m mod (4l-1), b = batch member,
// t = latitude row (cos(theta_t) increasing), so every job's rows are
// contiguous.
struct ShtIO {
    double* u = nullptr;              // staging: weighted chain values u[plan][b][i][4]
    double* c = nullptr;              // split programs: coefficient buffer C[b][c_cells][4]
    double* ypart = nullptr;          // split programs: root partials [b][y_rows][4]
    const std::uint32_t* plan_yoff = nullptr;    // per plan: first partial row
    const std::uint32_t* plan_groups = nullptr;  // per plan: number of root groups
    std::uint32_t c_cells = 0;
    std::uint32_t y_rows = 0;
    // 1: C[c_cells][b][4] and ypart[y_rows][b][4] (the tensor-core root kernels'
    // layout, rootmma.cu); 0: member-major as above
    int cell_major = 0;
    // merged programs: per (plan, batch member) dependency words and the
    // launch epoch (forward: event job publishes C; transpose: root jobs count)
    unsigned long long* dep = nullptr;
    const std::uint32_t* plan_roots = nullptr;
    unsigned long long epoch = 0;
    const double* beta_in = nullptr;  // synthesis input (packed complex coefficients)
    double* beta_out = nullptr;       // analysis output
    const double* g_in = nullptr;     // analysis input: unnormalised forward DFT over phi
    double* g_out = nullptr;          // synthesis output: g_m(theta_t)
    const double* isr = nullptr;      // 1 / sqrt(rho_i)
    const double* hsr = nullptr;      // sqrt(rho_i) / (2 N)
    int l = 0;
    int N = 0;                        // 4l - 1
    int batch = 0;
    int mu0 = 0;                      // first order of the plan set (plan index 0)
    int mu_end = 0;                   // sharded kernels: end of the order range
    // Real fields: members per engine task (1: RC = 2; 2: two fields share the
    // four right-hand sides of RC = 4) and the number of fields.
    int real_per_task = 0;
    int real_members = 0;
    long long beta_stride = 0;        // doubles between batch members
};

// Launches one apply over every job (x chunks).  Returns cudaGetLastError().
cudaError_t launch_generic(const DeviceProgram& prog, bool transpose, const GenericIO& io, cudaStream_t st);
// pdl: launch as a programmatic dependent of the previous kernel on the stream
// (its producer warps start streaming the plan before that kernel finishes).
// real_field: 2 right-hand sides per function (re / im of +m; coefficients in
// the half layout, u[chain][b][i][2]) instead of 4.
cudaError_t launch_sht(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st,
                       bool pdl = false, bool real_field = false);
// Split SHT programs: events (leaves / merges / promotes) and roots.
cudaError_t launch_sht_events(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st);
cudaError_t launch_sht_roots(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st);
// Merged event + root program (one launch, per-plan dependency flags).
cudaError_t launch_sht_merged(const DeviceProgram& prog, bool transpose, const ShtIO& io, int batch, cudaStream_t st);
// Parity combine (synthesis: u -> g_out) and split (analysis: g_in -> u) for
// orders [0, mu_end); io.batch must be set.
cudaError_t launch_sht_combine(const ShtIO& io, int mu_begin, int mu_end, cudaStream_t st);
cudaError_t launch_sht_split(const ShtIO& io, int mu_begin, int mu_end, cudaStream_t st);

// Dynamic shared memory the engine needs for this program.
std::size_t engine_smem_bytes(const DeviceProgram& prog, int rc = kRC);

}  // namespace bfb
