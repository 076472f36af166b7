// Root-stage kernels of the split SHT programs (see rootmv.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <vector>

#include "packer.hpp"

namespace bfb {

struct DeviceRootSet {
    double* data = nullptr;
    RootStripeDesc* stripes = nullptr;
    std::uint32_t* fwd_items = nullptr;
    std::uint32_t* bwd_items = nullptr;
    int n_fwd = 0, n_bwd = 0;
    std::uint32_t* mma_fwd = nullptr;  // tensor-core kernels: (stripe, first row) pairs
    std::uint32_t* mma_bwd = nullptr;
    int n_mma_fwd = 0, n_mma_bwd = 0;
    std::vector<int> mma_fwd_group;    // first forward item per root group (+ end)
    bool mma = false;                  // S only (no S^T copy), for launch_roots_mma
    std::size_t n_stripes = 0;
    std::uint64_t stored_words = 0;
    std::uint64_t bytes = 0;
};

// mma = true: upload S only (the tensor-core kernels read S in both
// directions) plus their work items; false: S and S^T for launch_roots.
DeviceRootSet upload_roots(const RootSet& r, bool mma = false);
void free_roots(DeviceRootSet& d);

struct RootArgs {
    const double* data = nullptr;
    const RootStripeDesc* stripes = nullptr;
    const std::uint32_t* items = nullptr;
    int n_items = 0;
    double* C = nullptr;       // [b][c_cells][4]
    double* ypart = nullptr;   // [b][y_rows][4]   (forward output)
    const double* u = nullptr; // [plan][b][l][4]  (transpose input)
    std::uint32_t c_cells = 0, y_rows = 0;
    int l = 0;
    int batch = 0;
};

cudaError_t launch_roots(const RootArgs& args, bool transpose, cudaStream_t st);

// Batched root stage on the FP64 tensor cores (rootmma.cu): all 4 * batch
// right-hand sides per skeleton read.  Cell-major C / ypart.
struct RootMmaArgs {
    const double* data = nullptr;
    const RootStripeDesc* stripes = nullptr;
    const std::uint32_t* fwd_items = nullptr;
    const std::uint32_t* bwd_items = nullptr;
    const std::uint32_t* items = nullptr;  // set by the launcher
    int n_fwd = 0, n_bwd = 0;
    double* C = nullptr;        // [c_cells][batch][4]
    double* ypart = nullptr;    // [y_rows][batch][4]   (forward output)
    const double* u = nullptr;  // [plan][batch][l][4]  (transpose input)
    double* u_out = nullptr;    // forward output when to_u (chain rows, summed over root groups)
    const double* rows_cm = nullptr;  // transpose input when set: stacked rows, cell-major [row][4 batch]
                                      // (row of a stripe = RootStripeDesc::pad[1] + i; plan-set apply)
    int to_u = 0;
    int accumulate = 0;         // forward: '+=' (root groups after the first)
    int l = 0;
    int batch = 0;
};

// Items [item0, item0 + n_items) of the direction's list (n_items < 0: to the end).
cudaError_t launch_roots_mma(const RootMmaArgs& args, bool transpose, cudaStream_t st, int item0 = 0,
                             int n_items = -1);
// Stripes with RootStripeDesc::pad[0] = root group, sorted by group: fwd_group
// receives the first forward item of each group.
void root_mma_items(const std::vector<RootStripeDesc>& stripes, std::vector<std::uint32_t>& fwd,
                    std::vector<std::uint32_t>& bwd, std::vector<int>* fwd_group = nullptr);

}  // namespace bfb
