// Root-stage kernels of the split SHT programs (see rootmv.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>

#include "packer.hpp"

namespace bfb {

struct DeviceRootSet {
    double* data = nullptr;
    RootStripeDesc* stripes = nullptr;
    std::uint32_t* fwd_items = nullptr;
    std::uint32_t* bwd_items = nullptr;
    int n_fwd = 0, n_bwd = 0;
    std::uint64_t stored_words = 0;
    std::uint64_t bytes = 0;
};

DeviceRootSet upload_roots(const RootSet& r);
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

}  // namespace bfb
