// Device side of the graph programs (wgraph.hpp): upload and the persistent launch.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "waves_dev.hpp"
#include "wgraph.hpp"

namespace bfb {

struct DeviceGraph {
    GraphItem* items[2] = {nullptr, nullptr};      // [0] forward, [1] transpose
    std::uint32_t* deps[2] = {nullptr, nullptr};
    std::uint32_t n_items[2] = {0, 0};
    RootSeg* segs = nullptr;
    std::uint32_t* flags[2] = {nullptr, nullptr};  // per (item, column block): epoch of the last completion
    std::size_t flag_cap[2] = {0, 0};
    std::uint32_t* counter = nullptr;              // claim counters, one per direction (reset per launch)
    std::uint32_t epoch[2] = {0, 0};
    std::uint32_t groups = 0;
    bool ok = false;
};

DeviceGraph upload_graph(const GraphProgram& g);
void free_graph(DeviceGraph& d);

// One direction of the Legendre stage of the wave program `w` for `batch`
// functions (R = 4 batch right-hand sides): forward reads the coefficient
// cells of V (launch_wave_gather) and writes the chain rows u [plan][b][l][4];
// the transpose reads u and writes the coefficient cells of V (then
// launch_wave_scatter).  One persistent launch.  stacked: u is instead the
// plan set's stacked rows, cell-major [row][R] (plan-set apply; l unused).
cudaError_t launch_graph(DeviceGraph& g, const DeviceWaveSet& w, double* V, double* u, int l, int batch, bool transpose,
                         cudaStream_t st, bool stacked = false);

}  // namespace bfb
