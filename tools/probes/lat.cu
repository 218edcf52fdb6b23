// Microbenchmark: dependent-chain latency of fp64 ops on this GPU (clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void lat(double* out, long long* cyc, double x0) {
    double x = x0, y = 1.0000001, z = 1e-300;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 128; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) x = __fma_rn(x, y, z);
    }
    long long t1 = clock64();
    double a = x;
#pragma unroll 1
    for (int i = 0; i < 128; ++i) {
#pragma unroll
        for (int u = 0; u < 8; ++u) a = __dadd_rn(a, z);
    }
    long long t2 = clock64();
    double r;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) { asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(a)); a = r; }
    long long t3 = clock64();
    double s = a;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) { s = fabs(s) > 1.0 ? s : -s; }   // DSETP + select chain
    long long t4 = clock64();
    __shared__ double sm[64];
    sm[threadIdx.x] = s; __syncthreads();
    int idx = threadIdx.x;
    long long t5 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; ++i) { idx = (int)sm[idx & 31] & 31; }
    long long t6 = clock64();
    out[threadIdx.x] = x + a + r + s + idx;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t6 - t5; }
}
// one warp, NCH independent DFMA chains: cycles per warp-instruction
template <int NCH>
__global__ void tput(double* out, long long* cyc) {
    double x[NCH];
    for (int k = 0; k < NCH; ++k) x[k] = 1.0 + k * 1e-3 + threadIdx.x * 1e-9;
    const double y = 1.0000001, z = 1e-300;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 256; ++i) {
#pragma unroll
        for (int k = 0; k < NCH; ++k) x[k] = __fma_rn(x[k], y, z);
    }
    long long t1 = clock64();
    double s = 0; for (int k = 0; k < NCH; ++k) s += x[k];
    out[threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void rsq(double* out, long long* cyc, double a) {
    long long t0 = clock64();
    double r = a;
#pragma unroll 1
    for (int i = 0; i < 256; ++i) { asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(r)); }
    long long t1 = clock64();
    out[threadIdx.x] = r;
    if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
    double* o; long long* c; cudaMalloc(&o, 64*8); cudaMallocManaged(&c, 8*8);
    lat<<<1,32>>>(o, c, 1.0); cudaDeviceSynchronize();
    lat<<<1,32>>>(o, c, 1.0); cudaDeviceSynchronize();
    printf("DFMA chain: %.2f cyc/op\nDADD chain: %.2f\nMUFU.RCP64H chain: %.2f\nfabs-cmp-select chain: %.2f\nLDS chain: %.2f\n",
           c[0]/1024.0, c[1]/1024.0, c[2]/256.0, c[3]/256.0, c[4]/256.0);
    rsq<<<1,32>>>(o, c, 2.0); cudaDeviceSynchronize(); rsq<<<1,32>>>(o, c, 2.0); cudaDeviceSynchronize();
    printf("MUFU.RSQ64H chain: %.2f\n", c[0]/256.0);
    tput<1><<<1,32>>>(o,c); cudaDeviceSynchronize(); tput<1><<<1,32>>>(o,c); cudaDeviceSynchronize(); printf("1 warp, 1 chain: %.2f cyc/DFMA\n", c[0]/256.0/1);
    tput<4><<<1,32>>>(o,c); cudaDeviceSynchronize(); tput<4><<<1,32>>>(o,c); cudaDeviceSynchronize(); printf("1 warp, 4 chains: %.2f cyc/DFMA\n", c[0]/256.0/4);
    tput<8><<<1,32>>>(o,c); cudaDeviceSynchronize(); tput<8><<<1,32>>>(o,c); cudaDeviceSynchronize(); printf("1 warp, 8 chains: %.2f cyc/DFMA\n", c[0]/256.0/8);
    tput<16><<<1,32>>>(o,c); cudaDeviceSynchronize(); tput<16><<<1,32>>>(o,c); cudaDeviceSynchronize(); printf("1 warp, 16 chains: %.2f cyc/DFMA\n", c[0]/256.0/16);
}
