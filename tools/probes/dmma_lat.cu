// Latency probe: dependent chains of DMMA.8x8x4 (through C), of SHFL.IDX on a
// double, and DMMA throughput per warp with 1..9 independent tiles (the shape of
// the ens_nbody8m contraction).  One warp, clock64.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_lat dmma_lat.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma(double &d0, double &d1, double a, double b, double c0, double c1) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
                 : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

template <int NT>
__global__ void dmma_chain(double *out, long long *cyc, double a, double b) {
    double d0[NT], d1[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) d0[t] = d1[t] = 1e-3 * (t + threadIdx.x);
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i) {
#pragma unroll
        for (int t = 0; t < NT; ++t) mma(d0[t], d1[t], a, b, d0[t], d1[t]);
    }
    long long t1 = clock64();
    double s = 0;
#pragma unroll
    for (int t = 0; t < NT; ++t) s += d0[t] + d1[t];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

__global__ void shfl_chain(double *out, long long *cyc, double x) {
    double v = x + threadIdx.x;
    int src = (threadIdx.x * 5 + 3) & 31;
    long long t0 = clock64();
    for (int i = 0; i < 256; ++i) v = __shfl_sync(0xffffffffu, v, src) + 1.0;
    long long t1 = clock64();
    out[threadIdx.x] = v;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
    double *o; long long *c, h;
    cudaMalloc(&o, 1024 * sizeof(double)); cudaMalloc(&c, sizeof(long long));
#define RUN(NT) dmma_chain<NT><<<1, 32>>>(o, c, 1.0000001, 0.9999999); dmma_chain<NT><<<1, 32>>>(o, c, 1.0000001, 0.9999999); \
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost); printf("DMMA %d independent chains: %.2f cyc per step (%.2f cyc/DMMA)\n", NT, h / 256.0, h / 256.0 / NT);
    RUN(1) RUN(2) RUN(4) RUN(8) RUN(9) RUN(16)
    shfl_chain<<<1, 32>>>(o, c, 1.0); shfl_chain<<<1, 32>>>(o, c, 1.0);
    cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("SHFL(double)+DADD chain: %.2f cyc/step (DADD 8.4)\n", h / 256.0);
    printf("cuda: %s\n", cudaGetErrorString(cudaGetLastError()));
}
