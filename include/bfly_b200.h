/*
 * bfly_b200.h — C ABI of the B200 butterfly associated-Legendre engine.
 *
 * The drop-in boundary for the reference's hot path (arXiv 0910.5435
 * reference, /root/reference/proj).  The reference exposes C++ only; each
 * entry point below names the reference interface it replaces:
 *
 *   bfly_plan_from_bfly1 / bfly_plan_to_bfly1
 *       <- bfly::load_plan / bfly::save_plan  (include/bfly/serialize.hpp:44-45,
 *          format serialize.hpp:14-31).  A reference ButterflyPlan crosses the
 *          boundary as its own BFLY1 bytes, unchanged.
 *   bfly_plan_build_glrow / bfly_plan_build_dense
 *       <- bfly::build_plan over a ColumnSource (include/bfly/butterfly.hpp:90-91;
 *          column_source.hpp:11-40), rows = the l positive Gauss-Legendre nodes.
 *   bfly_plan_info
 *       <- bfly::plan_stats (include/bfly/butterfly.hpp:100).
 *   bfly_dev_planset_create + bfly_dev_apply(transpose = 0 / 1)
 *       <- bfly::apply / bfly::apply_transpose (include/bfly/butterfly.hpp:93-96;
 *          src/butterfly.cpp:384-513) and transform::forward / transform::inverse
 *          (include/bfly/transform.hpp:60-66), batched over plans and
 *          right-hand sides; the plan set is uploaded once.
 *   bfly_sht_* — the full spherical-harmonic transform pair the north_star
 *       asks for (no reference counterpart; the reference stops at one (m,
 *       parity) per call).
 *
 * Conventions: every function returns 0 on success or a BFLY_E* code; the
 * message of the last failure on the calling thread is bfly_last_error().
 * BFLY_EINVAL corresponds to the reference's std::invalid_argument (for
 * example "apply: vector length X, expected Y"), BFLY_ERUNTIME to
 * std::runtime_error, BFLY_ESERIAL to bfly::SerializationError.  Device
 * pointers are CUDA device memory on the handle's device; `stream` is a
 * cudaStream_t (NULL = legacy default stream).  Work is stream-ordered; one
 * handle must not run on two streams concurrently.  Host pointers are never
 * retained after a call returns.
 */
#ifndef BFLY_B200_H
#define BFLY_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    BFLY_OK = 0,
    BFLY_EINVAL = 1,   /* std::invalid_argument */
    BFLY_ERUNTIME = 2, /* std::runtime_error */
    BFLY_ESERIAL = 3,  /* bfly::SerializationError */
    BFLY_ECUDA = 4,
    BFLY_ENCCL = 5,
    BFLY_EOTHER = 6
};

typedef struct bfly_plan_s* bfly_plan_t;       /* host ButterflyPlan */
typedef struct bfly_planset_s* bfly_planset_t; /* device-resident compiled plan set */
typedef struct bfly_sht_s* bfly_sht_t;         /* spherical harmonic transform */

const char* bfly_last_error(void);
const char* bfly_version(void);

/* ---- host plans --------------------------------------------------------- */

/* Parse one reference BFLY1 plan (bfly::save_plan bytes). */
int bfly_plan_from_bfly1(const uint8_t* bytes, size_t n, bfly_plan_t* out);
/* Serialise; *size receives the byte count, bytes copied only if cap suffices. */
int bfly_plan_to_bfly1(bfly_plan_t plan, uint8_t* buf, size_t cap, size_t* size);
/* GL-row plan: A(i, j) = sqrt(rho_i) Pbar^mu_{mu+2j+parity}(x_i), x_i the l
 * positive Gauss-Legendre nodes of degree 2l, j < n_parity(mu). */
int bfly_plan_build_glrow(int l, int mu, int parity, double eps, int block_width, bfly_plan_t* out);
/* Plan of an explicit column-major rows x cols matrix (DenseColumnSource). */
int bfly_plan_build_dense(const double* a, int64_t rows, int64_t cols, double eps, int block_width,
                          bfly_plan_t* out);
/* info[0..9] = n_rows, n_cols, levels, stored_words, m_max_words, events,
 * root_groups, k_max, id_count, block_width; kstat[0..1] = k_avg, k_sigma. */
int bfly_plan_info(bfly_plan_t plan, int64_t* info, double* kstat);
void bfly_plan_destroy(bfly_plan_t plan);

/* ---- device plan sets (upload once, apply many) --------------------------- */

int bfly_dev_planset_create(const bfly_plan_t* plans, int n, int device, bfly_planset_t* out);
/* Apply every plan of the set to nrhs right-hand sides.  Stacked layout:
 * plan p's input is the column-major block (n_in(p) x nrhs, leading dim
 * n_in(p)) at in + nrhs * sum_{q<p} n_in(q); outputs likewise.  transpose=0:
 * n_in = n_cols, out = A v (bfly::apply); transpose=1: n_in = n_rows,
 * out = A^T w (bfly::apply_transpose).  in_len / out_len are the buffer
 * lengths in doubles; a mismatch is BFLY_EINVAL with the reference's message
 * ("apply: vector length X, expected Y"). */
int bfly_dev_apply(bfly_planset_t set, int transpose, const double* in, int64_t in_len, double* out,
                   int64_t out_len, int nrhs, void* stream);
/* Same with host buffers: copies in, applies, copies out, synchronises. */
int bfly_host_apply(bfly_planset_t set, int transpose, const double* in, int64_t in_len, double* out,
                    int64_t out_len, int nrhs);
/* info[0..7] = n_plans, n_jobs, stored_words, fetched_bytes, stream_bytes,
 * arena_cells, smem_bytes, total n_rows */
int bfly_dev_planset_info(bfly_planset_t set, int64_t* info);
void bfly_dev_planset_destroy(bfly_planset_t set);

/* ---- spherical harmonic transforms --------------------------------------- */
/*
 * Bandlimit l: degrees k = 0..2l-1, orders |m| <= k, 4 l^2 complex
 * coefficients per function; grid 2l Gauss-Legendre colatitudes x (4l-1)
 * longitudes phi_n = 2 pi n / (4l-1).
 *   f(theta, phi) = sum_{k, m} beta_k^m Pbar_k^{|m|}(cos theta) e^{i m phi}
 * (Pbar orthonormal on [-1, 1]; arXiv 0910.5435 eq. "expansion").
 * Coefficient layout (complex128, interleaved re/im), per function:
 *   m = 0: k = 0..2l-1; then for mu = 1..2l-1: m = +mu, k = mu..2l-1,
 *   followed by m = -mu, k = mu..2l-1.   (batch stride 4 l^2 complex)
 * Grid layout (complex128): [t][n], t = 0..2l-1 with cos(theta_t) increasing,
 *   n = 0..4l-2.  (batch stride 2l (4l-1) complex)
 * synthesize: coefficients -> grid values (the paper's "inverse transform",
 *   the reference's transform::forward per (m, parity)).
 * analyze:    grid values -> coefficients (the paper's "forward transform",
 *   transform::inverse per (m, parity)); exact for bandlimited data.
 */
int bfly_sht_create(int l, double eps, int block_width, int threads, int device, bfly_sht_t* out);
/* The same on a caller's quadrature: `nodes` (the l positive nodes, ascending)
 * and `rho` (= 2 w_GL) of length l, e.g. the reference's
 * quadrature::build_rule(0, l, even) (reference include/bfly/quadrature.hpp,
 * src/quadrature.cpp), so the grid and the plans are exactly the reference's.
 * NULL, NULL = this library's rule (bfly_gl_rule). */
int bfly_sht_create_rule(int l, double eps, int block_width, int threads, const double* nodes, const double* rho,
                         int device, bfly_sht_t* out);
/* Build from caller-supplied plans in (mu ascending, even then odd) order,
 * one per non-empty chain (4l - 1 plans); rho (length l, may be NULL) are
 * the weights rho_i = 2 w_GL,i to use for the +-x combine. */
int bfly_sht_create_from_plans(int l, const bfly_plan_t* plans, int n, const double* rho, int device,
                               bfly_sht_t* out);
int bfly_sht_synthesize(bfly_sht_t sht, const double* beta, double* grid, int batch, void* stream);
int bfly_sht_analyze(bfly_sht_t sht, const double* grid, double* beta, int batch, void* stream);
/* Legendre stage only (no phi DFT).  The phi-stage buffers are complex
 * [bin][b][t]: bin = m mod (4l-1), b = batch member, t = latitude row.
 * legendre_synthesize writes g_m(theta_t); legendre_analyze reads the
 * unnormalised forward DFT over phi, G = sum_n f e^{-2 pi i bin n / (4l-1)}. */
int bfly_sht_legendre_synthesize(bfly_sht_t sht, const double* beta, double* gbins, int batch, void* stream);
int bfly_sht_legendre_analyze(bfly_sht_t sht, const double* gbins_scaled, double* beta, int batch,
                              void* stream);
/* phi stage only (cuFFT Z2Z, length 4l-1) between the grid [b][t][n] and
 * the [bin][b][t] phi-stage buffer (out of place). */
int bfly_sht_phi_synthesize(bfly_sht_t sht, const double* gbins, double* grid, int batch, void* stream);
/* Real fields: beta^{-m}_k = conj(beta^m_k) and Im beta^0_k = 0,
 * so only m >= 0 is stored ("half" layout: order blocks m = 0..2l-1 of 2l - m
 * complex coefficients each, l(2l+1) per function) and the grid is real,
 * [b][t][n] doubles.  Two right-hand sides per chain instead of four, and one
 * complex DFT per colatitude pair.  Needs the fused phi stage. */
int bfly_sht_synthesize_real(bfly_sht_t sht, const double* beta_half, double* grid, int batch, void* stream);
int bfly_sht_analyze_real(bfly_sht_t sht, const double* grid, double* beta_half, int batch, void* stream);
int bfly_sht_phi_analyze(bfly_sht_t sht, const double* grid, double* gdft, int batch, void* stream);
/* Host-buffer versions: H2D copy, transform, D2H copy, synchronise. */
int bfly_sht_synthesize_host(bfly_sht_t sht, const double* beta, double* grid, int batch);
int bfly_sht_analyze_host(bfly_sht_t sht, const double* grid, double* beta, int batch);
/* info[0..7] = l, n_plans, stored_words, fetched_bytes, n_jobs, smem_bytes,
 * coeffs per function (complex), grid points per function (complex) */
int bfly_sht_info(bfly_sht_t sht, int64_t* info);
/* Which programs the handle holds and how a call is served (no reference
 * counterpart; the reference has one CPU apply).  info[10]: has whole-chain
 * program, has wave programs (batched functions, FP64 tensor cores), wave
 * levels, root groups, wave vector cells per function, wave nodes,
 * interpolation words, smallest batch served by the waves when both exist,
 * wave programs run as the graph program (one persistent launch per
 * direction; else one launch per level and root group), graph plan groups. */
int bfly_sht_program_info(bfly_sht_t sht, int64_t* info);
/* Diagnostics: record per-task (start ns, end ns, SM id, stages) of the next
 * engine launches into a device buffer of max_tasks entries (0 disables). */
int bfly_sht_trace(bfly_sht_t sht, int max_tasks);
/* Diagnostics: flags bit 0 = engine streams the stages but skips arithmetic. */
int bfly_sht_debug(bfly_sht_t sht, int flags);
/* Engine timing: returns (and clears) the summed CUDA-event durations of the
 * engine launches since the last call, per direction (ms[0] synthesis, ms[1]
 * analysis) and their counts; then enables (enable != 0) or disables timing.
 * Events are recorded on the launching stream. */
int bfly_sht_engine_time(bfly_sht_t sht, int enable, double* ms, int64_t* launches);
int bfly_sht_trace_read(bfly_sht_t sht, uint64_t* out, int max_tasks);
/* The l positive nodes (ascending) and rho_i used by the handle. */
int bfly_sht_rule(bfly_sht_t sht, double* nodes, double* rho);
void bfly_sht_destroy(bfly_sht_t sht);

/* Device-ready program cache: bfly_sht_save writes the
 * packed device program of a whole-chain SHT (plus rule and shape) to `path`
 * ("BFLYSHT1"); bfly_sht_load recreates the SHT on `device` without building
 * or packing plans.  Loading a file packed by a build with other chunk rows
 * fails with BFLY_ESERIAL. */
int bfly_sht_save(bfly_sht_t sht, const char* path);
int bfly_sht_load(const char* path, int device, bfly_sht_t* out);

/* The l positive Gauss-Legendre nodes of degree 2l (ascending) and
 * rho_i = 2 w_i — the rows every GL-row plan uses. */
int bfly_gl_rule(int l, double* nodes, double* rho);
/* Diagnostics: the fused phi stage alone (plan for N = 4l - 1, zero chain
 * values) for `batch` functions, mean ms per direction over `iters` launches:
 * ms[0] synthesis, ms[1] analysis. */
int bfly_phi_time(int l, int batch, int iters, double* ms);

/* Host-only introspection of the device program a plan set compiles to (one
 * job per plan): stage bytes / offsets / jobs / header fields, for
 * validation tooling.  Any output pointer may be NULL; sizes[0..5] receives
 * stream bytes, n_stages, n_jobs, arena_cells, zo_cells, smem_bytes. */
/* Diagnostics / tests: the host-compiled wave program of a plan set (waves.hpp),
 * two-call pattern (null buffers: sizes only).  sizes[10] = T words, index
 * entries, nodes, forward items, transposed pairs, levels, V cells, root
 * stripes, S words, aliased full-rank leaves.  nodes: 8 u32 each (t_off lo/hi,
 * rank, nothers, idx, cA, level, 0); stripes: 8 u64 each (s_off, rows, rank,
 * lds, coff, plan, group, first stacked row); fwd_begin / bwd_begin: levels + 1. */
int bfly_waves_inspect(const bfly_plan_t* plans, int n, int64_t* sizes, double* T, uint32_t* idx, uint32_t* nodes,
                       uint32_t* fwd, uint32_t* pairs, uint32_t* fwd_begin, uint32_t* bwd_begin, uint32_t* plan_in,
                       uint64_t* stripes, double* S);
int bfly_pack_inspect(const bfly_plan_t* plans, int n, uint8_t* stream, uint64_t* stage_off,
                      uint32_t* stage_bytes, void* jobs, int64_t* sizes);

/* Same for the split compilation used by the SHT (plans = one degree chain
 * each, parities given): which = 0 event program, 1 root program.  sizes as
 * above plus sizes[6] = C cells, sizes[7] = partial rows; plan_yoff /
 * plan_groups (length n) may be NULL. */
int bfly_pack_inspect_split(const bfly_plan_t* plans, int n, const int* parity, int which, uint8_t* stream,
                            uint64_t* stage_off, uint32_t* stage_bytes, void* jobs, int64_t* sizes,
                            uint32_t* plan_yoff, uint32_t* plan_groups);

/* Host builder of a whole GL-row plan set, for callers that shard orders
 * (mu in [mu_begin, mu_end)) across devices.  Plans in (mu, parity) order. */
int bfly_glrow_planset_build(int l, int mu_begin, int mu_end, double eps, int block_width, int threads,
                             bfly_plan_t* plans_out, int cap, int* n_out);
/* The same on a caller's quadrature (see bfly_sht_create_rule). */
int bfly_glrow_planset_build_rule(int l, int mu_begin, int mu_end, double eps, int block_width, int threads,
                                  const double* nodes, const double* rho, bfly_plan_t* plans_out, int cap, int* n_out);
int bfly_sht_create_range(int l, int mu_begin, int mu_end, const bfly_plan_t* plans, int n, const double* rho,
                          int device, bfly_sht_t* out);

/* Order-sharded transform steps for an order-range SHT (one process per GPU;
 * paper_0910_5435_b200/sharded.py computes the tables and runs the NCCL
 * all-to-all between them).  Exchange buffers of this rank (local bins: +mu of
 * the range, then -mu) with peer j (slab of T_j rows) are
 * [local bin][member][slab row] complex, back to back by peer; row_base[t] /
 * row_T[t] (2l entries) locate grid row t in this rank's order-side buffer,
 * bin_off[bin] (4l-1 entries) a bin in its slab-side buffer (member stride =
 * n_rows, this rank's slab).  All pointers are device memory.
 *   synthesize: engine + parity combine -> order-side send buffer
 *   phi:        synthesis: slab-side receive buffer -> grid slab [b][row][n];
 *               analysis: grid slab -> slab-side send buffer (forward DFT)
 *   analyze:    order-side receive buffer -> parity split -> engine -> beta
 * bfly_sht_shard_supported sets *ok = 1 when this handle can run all three
 * (an in-kernel DFT plan for N = 4l-1); synthesize / analyze (the order side)
 * need only whole-chain or wave programs, and callers without the in-kernel
 * slab DFT run cuFFT on the slab rows (bfly_shard_*). */
int bfly_sht_shard_supported(bfly_sht_t sht, int* ok);
int bfly_sht_shard_synthesize(bfly_sht_t sht, const double* beta, double* send, const int64_t* row_base,
                              const int32_t* row_T, int batch, void* stream);
int bfly_sht_shard_phi(bfly_sht_t sht, int synthesis, const double* src, double* dst, const int64_t* bin_off,
                       int n_rows, int batch, void* stream);
int bfly_sht_shard_analyze(bfly_sht_t sht, const double* recv, double* beta, const int64_t* row_base,
                           const int32_t* row_T, int batch, void* stream);

/* ---- Order-sharded SHT over processes, one GPU each (no reference
 * counterpart).  Rank r holds the plans of its order range
 * (contiguous ranges with near-equal dense Legendre words) and the latitude
 * slab [t0, t1) of the grid; the m <-> theta transpose between the Legendre
 * stage and the phi DFT is a grouped ncclSend / ncclRecv alltoallv (NCCL loaded
 * at run time), overlapped with the next member chunk's Legendre stage / DFT on
 * a second stream.  Coefficients keep the packed 4 l^2 layout per member (only
 * the rank's orders are read; analysis writes only them); the grid is the
 * rank's slab, [member][t1 - t0][4l - 1] complex.  Device pointers, stream-
 * ordered on `stream`.  Errors: bfly_shard_last_error(); BFLY_ENCCL for NCCL. */
typedef struct bfly_shard_s* bfly_shard_t;
const char* bfly_shard_last_error(void);
/* Partition and slabs: orders[2r], orders[2r+1] = [mu_begin, mu_end) of rank r;
 * slabs[2r], slabs[2r+1] = its grid rows (each array 2 * world entries). */
int bfly_shard_layout(int l, int world, int64_t* orders, int64_t* slabs);
/* Host copy of rank `rank`'s exchange tables for `batch` members (the operands
 * of bfly_sht_shard_*): row_base / row_T (2l), bin_off (4l-1), per-peer block
 * sizes in complex (world each); any pointer may be NULL. */
int bfly_shard_tables(int l, int world, int rank, int batch, int64_t* row_base, int32_t* row_T, int64_t* bin_off,
                      int64_t* order_sizes, int64_t* slab_sizes);
/* ncclGetUniqueId into id[128] (rank 0; the caller broadcasts it). */
int bfly_shard_nccl_id(void* id);
/* Builds this rank's plans (host threads), uploads them, joins the NCCL group
 * (world > 1). */
int bfly_shard_create(int l, double eps, int block_width, int threads, int rank, int world, const void* nccl_id,
                      int device, bfly_shard_t* out);
/* info[7] = mu_begin, mu_end, slab t0, t1, world, rank, fused slab DFT (else cuFFT) */
int bfly_shard_info(bfly_shard_t s, int64_t* info);
/* The rank's order-range SHT handle (owned by the shard handle). */
int bfly_shard_sht(bfly_shard_t s, bfly_sht_t* sht);
int bfly_shard_synthesize(bfly_shard_t s, const double* beta, double* grid_slab, int batch, void* stream);
int bfly_shard_analyze(bfly_shard_t s, const double* grid_slab, double* beta, int batch, void* stream);
void bfly_shard_destroy(bfly_shard_t s);

#ifdef __cplusplus
}
#endif

#endif /* BFLY_B200_H */
