// Probe (SURVEY D-3): is the FP64 tensor core (mma.m8n8k4.f64, SASS DMMA) a win
// for the 8x8 stage contraction on sm_100a?
//  (1) bitwise: which accumulation order does DMMA implement?  Compared against
//      fma chains k = 0..3 from C, the reverse chain, and (host side) the
//      exactly rounded sum.
//  (2) throughput: DMMA alone, DFMA alone, and both interleaved in one loop (do
//      they share a pipe?).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma dmma.cu
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ void mma884(double &d0, double &d1, double a, double b, double c0, double c1) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
                 : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// one warp per 8x8x4 problem: A [8][4], B [4][8], C [8][8] -> D [8][8] + chains
__global__ void order_kernel(const double *A, const double *B, const double *C, double *D, double *F, double *R,
                             int nprob) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, l = threadIdx.x & 31;
    if (w >= nprob) return;
    const double *a = A + 32 * w, *b = B + 32 * w, *c = C + 64 * w;
    const int r = l >> 2, q = l & 3;
    double d0, d1;
    mma884(d0, d1, a[r * 4 + q], b[q * 8 + r], c[r * 8 + 2 * q], c[r * 8 + 2 * q + 1]);
    D[64 * w + r * 8 + 2 * q] = d0;
    D[64 * w + r * 8 + 2 * q + 1] = d1;
    for (int e = 0; e < 2; ++e) {
        const int n = 2 * q + e;
        double acc = c[r * 8 + n];
        for (int k = 0; k < 4; ++k) acc = __fma_rn(a[r * 4 + k], b[k * 8 + n], acc);
        F[64 * w + r * 8 + n] = acc;
        acc = c[r * 8 + n];
        for (int k = 3; k >= 0; --k) acc = __fma_rn(a[r * 4 + k], b[k * 8 + n], acc);
        R[64 * w + r * 8 + n] = acc;
    }
}

template <int NACC>
__global__ void dmma_tp(double *out, int iters) {
    double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-12 * threadIdx.x;
    double c0[NACC], c1[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) c0[k] = c1[k] = 1e-3 * (k + 1);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < NACC; ++k) mma884(c0[k], c1[k], a, b, c0[k], c1[k]);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < NACC; ++k) s += c0[k] + c1[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int NACC>
__global__ void dfma_tp(double *out, int iters) {
    double x = 1.0 + 1e-9 * threadIdx.x, y = 1.0 - 1e-12 * threadIdx.x;
    double acc[NACC];
#pragma unroll
    for (int k = 0; k < NACC; ++k) acc[k] = 1e-3 * (k + 1);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < NACC; ++k) acc[k] = __fma_rn(acc[k], x, y);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < NACC; ++k) s += acc[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// per iteration: NM DMMA (each 256 FMA per warp = 8 per lane) and NF DFMA per lane
template <int NM, int NF>
__global__ void mixed_tp(double *out, int iters) {
    double a = 1.0 + 1e-9 * threadIdx.x, b = 1.0 - 1e-12 * threadIdx.x;
    double c0[NM], c1[NM], acc[NF];
#pragma unroll
    for (int k = 0; k < NM; ++k) c0[k] = c1[k] = 1e-3 * (k + 1);
#pragma unroll
    for (int k = 0; k < NF; ++k) acc[k] = 1e-3 * (k + 1);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < NM; ++k) mma884(c0[k], c1[k], a, b, c0[k], c1[k]);
#pragma unroll
        for (int k = 0; k < NF; ++k) acc[k] = __fma_rn(acc[k], a, b);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < NM; ++k) s += c0[k] + c1[k];
#pragma unroll
    for (int k = 0; k < NF; ++k) s += acc[k];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static double rnd(uint64_t &s) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    return ((s >> 11) * (1.0 / 9007199254740992.0)) * 2.0 - 1.0;
}

template <class K>
static float timeit(K kern, double *out, int blocks, int threads, int iters) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e0);
    kern<<<blocks, threads>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    return ms;
}

int main(int argc, char **argv) {
    const int nprob = 1 << 16;
    std::vector<double> A(32 * nprob), B(32 * nprob), C(64 * nprob);
    uint64_t s = 88172645463325252ull;
    for (auto &x : A) x = rnd(s);
    for (auto &x : B) x = rnd(s) * 1e3;
    for (size_t i = 0; i < C.size(); ++i) C[i] = (i % 128 < 64) ? 0.0 : rnd(s) * 10;  // half the problems C = 0
    double *dA, *dB, *dC, *dD, *dF, *dR;
    cudaMalloc(&dA, 8 * A.size()); cudaMalloc(&dB, 8 * B.size()); cudaMalloc(&dC, 8 * C.size());
    cudaMalloc(&dD, 8 * C.size()); cudaMalloc(&dF, 8 * C.size()); cudaMalloc(&dR, 8 * C.size());
    cudaMemcpy(dA, A.data(), 8 * A.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), 8 * B.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(dC, C.data(), 8 * C.size(), cudaMemcpyHostToDevice);
    order_kernel<<<nprob * 32 / 256, 256>>>(dA, dB, dC, dD, dF, dR, nprob);
    std::vector<double> D(C.size()), F(C.size()), R(C.size());
    cudaMemcpy(D.data(), dD, 8 * D.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(F.data(), dF, 8 * F.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(R.data(), dR, 8 * R.size(), cudaMemcpyDeviceToHost);
    size_t neqF = 0, neqR = 0, neqF0 = 0, n0 = 0;
    for (size_t i = 0; i < D.size(); ++i) {
        bool z = (i % 128) < 64;
        n0 += z;
        if (memcmp(&D[i], &F[i], 8)) { ++neqF; neqF0 += z; }
        if (memcmp(&D[i], &R[i], 8)) ++neqR;
    }
    printf("order: %zu outputs; DMMA != fwd fma chain: %zu (%zu of %zu with C=0); != reverse chain: %zu\n", D.size(),
           neqF, neqF0, n0, neqR);
    FILE *f = fopen(argc > 1 ? argv[1] : "dmma_order.bin", "wb");
    if (f) {  // first 4096 problems for the host-side exact-rounding check
        fwrite(A.data(), 8, 32 * 4096, f); fwrite(B.data(), 8, 32 * 4096, f); fwrite(C.data(), 8, 64 * 4096, f);
        fwrite(D.data(), 8, 64 * 4096, f); fclose(f);
    }
    int sms = 0; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double *out; cudaMalloc(&out, 8 * 148 * 8 * 1024);
    const int iters = 4096;
    for (int wpb : {4, 8, 16}) {
        const int blocks = sms * 2, threads = 32 * wpb;
        float ms = timeit(dmma_tp<8>, out, blocks, threads, iters);
        double fl = 2.0 * 256 * 8 * iters * (double)blocks * wpb;
        printf("DMMA  %2d warps/blk x %d blk: %.3f ms  %.2f TFLOP/s\n", wpb, blocks, ms, fl / ms * 1e-9);
        ms = timeit(dfma_tp<16>, out, blocks, threads, iters);
        fl = 2.0 * 16 * iters * (double)blocks * threads;
        printf("DFMA  %2d warps/blk x %d blk: %.3f ms  %.2f TFLOP/s\n", wpb, blocks, ms, fl / ms * 1e-9);
    }
    {
        const int blocks = sms * 2, wpb = 8, threads = 256;
        float ms_m = timeit(dmma_tp<4>, out, blocks, threads, iters);
        float ms_f = timeit(dfma_tp<32>, out, blocks, threads, iters);
        float ms_x = timeit(mixed_tp<4, 32>, out, blocks, threads, iters);
        double flm = 2.0 * 256 * 4 * iters * (double)blocks * wpb, flf = 2.0 * 32 * iters * (double)blocks * threads;
        printf("mixed: DMMA-only(4) %.3f ms, DFMA-only(32) %.3f ms, both in one loop %.3f ms -> %.2f TFLOP/s "
               "(sum-of-parts %.3f ms => %s)\n",
               ms_m, ms_f, ms_x, (flm + flf) / ms_x * 1e-9, ms_m + ms_f,
               ms_x < 0.75 * (ms_m + ms_f) ? "OVERLAP (separate pipes)" : "serialised (shared pipe)");
    }
    cudaError_t e = cudaDeviceSynchronize();
    printf("cuda: %s\n", cudaGetErrorString(e));
    return 0;
}
