// Fused phi stage of the SHT (see phi.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>

#include "engine.hpp"

namespace bfb {

constexpr int kPhiMaxPasses = 24;
constexpr int kPhiMaxRadix = 127;  // largest prime factor handled by the in-SM DFT
constexpr int kRaderMaxStages = 16;  // prime N (Rader, phi_rader.cu): FFT stages of N - 1

struct PhiPlan {
    int N = 0;
    int n_pass = 0;
    int radix[kPhiMaxPasses] = {};
    double* W = nullptr;  // device: e^{+2 pi i k / N}, k = 0..N-1 (re, im)
    int dbg = 0;          // BFLY_PHI_DEBUG (diagnostics)
    bool stage_w = false; // twiddle table copied to shared memory per CTA
    bool big = false;     // rows too long for 4 N complex: one row at a time per CTA (3 N)
    bool ok = false;      // false: N has a prime factor > kPhiMaxRadix or does not fit shared memory
    std::size_t smem_synth = 0, smem_anal = 0;
    std::size_t smem_real_synth = 0, smem_real_anal = 0;
    std::size_t smem_big_synth = 0;  // large-row synthesis: A + aligned TMA staging
    bool tma = true;                 // small synthesis kernel: TMA chain gather (BFLY_PHI_TMA=0: cp.async)
    // TMA tensor map of the engine staging u (large-row synthesis gather),
    // rebuilt when the buffer or its shape changes
    mutable CUtensorMap umap{};
    mutable const double* umap_u = nullptr;
    mutable int umap_batch = 0, umap_l = 0;
    // Prime N whose N - 1 has only factors <= 13 (phi_rader.cu): Rader's
    // algorithm, one M = N - 1 complex buffer per CTA (c4: N = 8191).
    bool rader = false;
    int r_stages = 0;
    int r_radix[kRaderMaxStages] = {};
    double *r_bsyn = nullptr, *r_banal = nullptr;  // digit-reversed spectra of b (synthesis / analysis)
    double *r_tlo = nullptr, *r_thi = nullptr;     // two-level twiddle tables of length M
    std::uint32_t* r_pos = nullptr;                // log_g m
    std::size_t smem_rader = 0;
};

// Factorises N (odd) and uploads the twiddle table on the current device.
// Prime N that the Stockham kernels cannot take get the Rader plan instead
// (p.rader; p.ok stays false, so the real-field and sharded paths keep the
// stage-wise route).
PhiPlan make_phi_plan(int N);
void free_phi_plan(PhiPlan& p);
bool make_rader_plan(PhiPlan& p);
void free_rader_plan(PhiPlan& p);
cudaError_t launch_phi_synth_rader(const PhiPlan& p, const ShtIO& io, double* grid, cudaStream_t st);
cudaError_t launch_phi_anal_rader(const PhiPlan& p, const ShtIO& io, const double* grid, cudaStream_t st);

// Synthesis: engine staging u[plan][b][i][4] -> grid[b][t][n]
// (parity combine, 1/sqrt(rho), then the length-N inverse DFT over m per row).
cudaError_t launch_phi_synth_fused(const PhiPlan& p, const ShtIO& io, double* grid, cudaStream_t st);
// Analysis: grid[b][t][n] -> u[plan][b][i][4] (forward DFT per row, then the
// parity split with sqrt(rho)/(2N)).
cudaError_t launch_phi_anal_fused(const PhiPlan& p, const ShtIO& io, const double* grid, cudaStream_t st);

// Real fields: u[chain][b][i][2] (+m only) <-> real grid[b][t][n]; the two
// rows of a colatitude pair share one complex DFT.
cudaError_t launch_phi_synth_real(const PhiPlan& p, const ShtIO& io, double* grid, cudaStream_t st);
cudaError_t launch_phi_anal_real(const PhiPlan& p, const ShtIO& io, const double* grid, cudaStream_t st);

// Order-sharded transforms (see phi.cu): engine u <-> exchange buffers with the
// parity combine / split, and the slab-side DFT rows.
cudaError_t launch_shard_pack(const ShtIO& io, double* send, const long long* row_base, const int* row_T, int mu_begin,
                              int mu_end, cudaStream_t st);
cudaError_t launch_shard_unpack(const ShtIO& io, const double* recv, const long long* row_base, const int* row_T,
                                int mu_begin, int mu_end, cudaStream_t st);
cudaError_t launch_shard_phi(const PhiPlan& p, bool synthesis, const double* src, double* dst,
                             const long long* bin_off, int n_rows, int batch, cudaStream_t st);
// Slab side without an in-kernel DFT (N with a prime factor above the Stockham
// radices, e.g. 8191, 16383 = 3 43 127 rows too long for shared memory): the
// bins of the slab's rows move between the exchange layout (bin_off, as above)
// and contiguous rows [member][row][N] on which cuFFT runs.
//   to_rows: rows[(b n_rows + t) N + bin] = src[bin_off[bin] + b n_rows + t]
//   else:    dst[bin_off[bin] + b n_rows + t] = rows[(b n_rows + t) N + bin]
cudaError_t launch_shard_bins_rows(bool to_rows, const double* src, double* dst, const long long* bin_off, int N,
                                   int n_rows, int batch, cudaStream_t st);

}  // namespace bfb
