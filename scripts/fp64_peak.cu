// FP64 peak microbenchmark for the roofline denominators of the batched
// (wave) Legendre stage: FP64 tensor-core MMA (mma.sync ... .f64 -> SASS
// DMMA) and plain FP64 FMA (DFMA) throughput of this B200, measured with CUDA
// events over register-resident loops (no memory traffic).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
//   ./fp64_peak  -> one JSON line (TFLOP/s per shape, best of several grids)
#include <cuda_runtime.h>

#include <cstdio>
#include <algorithm>

#define CK(x)                                                                            \
    do {                                                                                 \
        cudaError_t e_ = (x);                                                            \
        if (e_ != cudaSuccess) {                                                         \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

constexpr int kChains = 8;  // independent accumulator chains per warp

// m8n8k4: 512 flops per instruction per warp
__global__ void dmma_m8n8k4(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-4;
    double d[kChains][2];
#pragma unroll
    for (int c = 0; c < kChains; ++c) d[c][0] = d[c][1] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                         : "+d"(d[c][0]), "+d"(d[c][1])
                         : "d"(a), "d"(b));
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += d[c][0] + d[c][1];
    if (s == 12345.678) out[threadIdx.x] = s;
}

// m16n8k16: 4096 flops per instruction per warp (sm_90+ shape)
__global__ void dmma_m16n8k16(double* out, int iters) {
    double a[8], b[4];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
#pragma unroll
    for (int i = 0; i < 4; ++i) b[i] = 1.0 + i * 1e-4;
    double d[kChains / 2][4];
#pragma unroll
    for (int c = 0; c < kChains / 2; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains / 2; ++c)
            asm volatile(
                "mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5, %6, %7, %8, %9, %10, "
                "%11}, {%12, %13, %14, %15}, {%0, %1, %2, %3};"
                : "+d"(d[c][0]), "+d"(d[c][1]), "+d"(d[c][2]), "+d"(d[c][3])
                : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]), "d"(b[0]),
                  "d"(b[1]), "d"(b[2]), "d"(b[3]));
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains / 2; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
    if (s == 12345.678) out[threadIdx.x] = s;
}

// DFMA: 2 flops per FMA per thread
__global__ void dfma(double* out, int iters) {
    double x[kChains];
    const double a = 1.0 + threadIdx.x * 1e-9, b = 1e-9;
#pragma unroll
    for (int c = 0; c < kChains; ++c) x[c] = c;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int c = 0; c < kChains; ++c) x[c] = fma(x[c], a, b);
    }
    double s = 0;
#pragma unroll
    for (int c = 0; c < kChains; ++c) s += x[c];
    if (s == 12345.678) out[threadIdx.x] = s;
}

template <class K>
float time_kernel(K k, int grid, int block, double* out, int iters) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k<<<grid, block>>>(out, iters / 10);  // warm-up
    cudaEventRecord(a);
    k<<<grid, block>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return ms;
}

int main() {
    int sms = 0, clk = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    CK(cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0));
    double* out = nullptr;
    CK(cudaMalloc(&out, 4096 * sizeof(double)));
    const int iters = 20000;
    double best_mma = 0, best_mma16 = 0, best_fma = 0;
    int cfg_mma = 0, cfg_mma16 = 0, cfg_fma = 0;
    for (int wps : {4, 8, 16, 32}) {       // warps per SM
        for (int bpw : {1, 2, 4}) {         // CTAs per SM (warps split across them)
            if (wps % bpw) continue;
            const int block = 32 * wps / bpw, grid = sms * bpw;
            float ms = time_kernel(dmma_m8n8k4, grid, block, out, iters);
            double tf = 512.0 * kChains * iters * (double)grid * (block / 32) / (ms * 1e-3) / 1e12;
            std::fprintf(stderr, "dmma m8n8k4: %2d warps/SM in %d CTA(s): %.2f TF/s\n", wps, bpw, tf);
            if (tf > best_mma) best_mma = tf, cfg_mma = wps;
            ms = time_kernel(dmma_m16n8k16, grid, block, out, iters / 8);
            tf = 4096.0 * (kChains / 2) * (iters / 8) * (double)grid * (block / 32) / (ms * 1e-3) / 1e12;
            if (tf > best_mma16) best_mma16 = tf, cfg_mma16 = wps;
            ms = time_kernel(dfma, grid, block, out, iters);
            tf = 2.0 * kChains * iters * (double)grid * block / (ms * 1e-3) / 1e12;
            if (tf > best_fma) best_fma = tf, cfg_fma = wps;
        }
    }
    CK(cudaGetLastError());
    std::printf(
        "{\"dmma_m8n8k4_tflops\": %.3f, \"dmma_m8n8k4_warps_per_sm\": %d, \"dmma_m16n8k16_tflops\": %.3f, "
        "\"dmma_m16n8k16_warps_per_sm\": %d, \"dfma_tflops\": %.3f, \"dfma_warps_per_sm\": %d, \"sms\": %d, "
        "\"clock_khz_attr\": %d, \"how\": \"register-resident loops, %d independent chains per warp, CUDA events, "
        "best over 4-32 warps per SM\"}\n",
        best_mma, cfg_mma, best_mma16, cfg_mma16, best_fma, cfg_fma, sms, clk, kChains);
    return 0;
}
