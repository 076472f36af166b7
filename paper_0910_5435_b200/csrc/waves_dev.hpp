// Device wave programs (wavekern.cu): upload and per-level launches.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <vector>

#include "rootmv.hpp"
#include "waves.hpp"

namespace bfb {

struct DeviceWaveSet {
    double* T = nullptr;
    std::uint32_t* idx = nullptr;
    WaveNode* nodes = nullptr;
    std::uint32_t* fwd = nullptr;
    std::uint32_t* pairs = nullptr;
    std::uint32_t *plan_in = nullptr, *plan_mu = nullptr, *plan_parity = nullptr, *plan_cols = nullptr;
    std::uint32_t* order_plan = nullptr;
    int n_orders = 0, mu0 = 0;
    std::vector<std::uint32_t> fwd_begin, bwd_begin;  // host copies (launch sizes)
    std::size_t n_T = 0, n_idx = 0, n_nodes = 0, n_fwd = 0, n_pairs = 0;  // element counts (program cache)
    int levels = 0;
    int n_plans = 0;
    std::uint32_t v_cells = 0;
    DeviceRootSet roots;  // data (tiled S) and stripes only
    int root_groups = 0;
    std::uint32_t* plan_row0 = nullptr;  // per plan: first stacked row (plan-set apply)
    std::uint64_t event_words = 0, root_words = 0;
    std::vector<std::uint32_t> node_src, plan_node_begin;  // host copies (program cache)
};

struct WaveArgs {
    const double* T = nullptr;
    const std::uint32_t* idx = nullptr;
    const WaveNode* nodes = nullptr;
    const std::uint32_t* fwd = nullptr;
    const std::uint32_t* pairs = nullptr;
    const std::uint32_t *plan_in = nullptr, *plan_mu = nullptr, *plan_parity = nullptr, *plan_cols = nullptr;
    const std::uint32_t* order_plan = nullptr;
    int mu0 = 0;
    double* V = nullptr;  // [v_cells][batch][4]
    int l = 0;
    int batch = 0;
    long long beta_stride = 0;  // doubles between batch members of the coefficients
    int real_members = 0;       // > 0: real fields in the half layout, two per batch slot
};

DeviceWaveSet upload_waves(const WaveSet& w);
void free_waves(DeviceWaveSet& d);
WaveArgs wave_args(const DeviceWaveSet& d, double* V, int l, int batch, long long beta_stride);
// beta (packed complex coefficients, member stride beta_stride) -> input cells of V
cudaError_t launch_wave_gather(const DeviceWaveSet& d, const WaveArgs& a, const double* beta, cudaStream_t st);
// input cells of V -> beta (every coefficient of the set's orders is written)
cudaError_t launch_wave_scatter(const DeviceWaveSet& d, const WaveArgs& a, double* beta, cudaStream_t st);
// Plan-set apply (reference layout: plan p, rhs r, entry k at prefix[p] * nrhs +
// r * n(p) + k): stacked vectors -> cell-major cells (cell0[p], or prefix[p] when
// cell0 is null; R doubles per cell, zero past nrhs), and the reverse.
// (r0, nrhs_total: the columns r0 .. r0 + nrhs of a layout with nrhs_total columns)
cudaError_t launch_plan_cells_in(const double* src, double* V, const std::uint64_t* prefix, const std::uint32_t* cell0,
                                 int n_plans, int nrhs, int R, cudaStream_t st, int r0 = 0, int nrhs_total = 0);
cudaError_t launch_plan_cells_out(const double* V, double* dst, const std::uint64_t* prefix, const std::uint32_t* cell0,
                                  int n_plans, int nrhs, int R, cudaStream_t st, int r0 = 0, int nrhs_total = 0);
}  // namespace bfb
