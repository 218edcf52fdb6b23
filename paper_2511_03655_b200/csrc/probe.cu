// FP64 FMA-pipe throughput probe (include/irk_probe.h).
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/irk_probe.h"
#include "fp64.cuh"

namespace {
__global__ void __launch_bounds__(256) dfma_probe_kernel(double *out, int iters) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    double x = 1.0 + 1e-9 * t, y = 1.0 - 1e-12 * t;
    double acc[16];
#pragma unroll
    for (int k = 0; k < 16; ++k) acc[k] = 1e-3 * (k + 1);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) acc[k] = __fma_rn(acc[k], x, y);
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < 16; ++k) s += acc[k];
    out[t] = s;
}
}  // namespace

extern "C" int64_t irk_probe_dfma(double *out, int blocks, int iters, void *stream) {
    if (!out || blocks < 1 || iters < 1) return -1;
    dfma_probe_kernel<<<blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(out, iters);
    if (cudaGetLastError() != cudaSuccess) return -1;
    return (int64_t)blocks * 256 * iters * 16 * 2;
}

namespace {
__global__ void divsqrt_probe_kernel(const double *a, const double *b, double *out, int64_t n) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= n) return;
    bool ok_d = true, ok_s = true, ok_r = true;
    const double qf = irk::ddiv_fast(a[i], b[i], ok_d);
    const double sf = irk::dsqrt_fast(b[i], ok_s);
    const double rf = irk::drcp_fast(b[i], ok_r);
    out[6 * i + 0] = ok_d ? qf : irk::ddiv(a[i], b[i]);
    out[6 * i + 1] = irk::ddiv(a[i], b[i]);
    out[6 * i + 2] = ok_s ? sf : irk::dsqrt(b[i]);
    out[6 * i + 3] = irk::dsqrt(b[i]);
    out[6 * i + 4] = ok_r ? rf : irk::ddiv(1.0, b[i]);
    out[6 * i + 5] = irk::ddiv(1.0, b[i]);
}
}  // namespace

extern "C" int irk_probe_divsqrt(const double *a, const double *b, double *out, int64_t n, void *stream) {
    if (!a || !b || !out || n < 0) return -1;
    if (n == 0) return 0;
    divsqrt_probe_kernel<<<(unsigned)((n + 255) / 256), 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(a, b, out, n);
    return cudaGetLastError() == cudaSuccess ? 0 : -1;
}
