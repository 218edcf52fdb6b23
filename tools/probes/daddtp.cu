// Probe: FP64 issue throughput of DADD vs DMUL vs DFMA on this GPU (8 independent
// chains per thread, 148 x 8 blocks of 256 threads); prints TFLOP-equivalent
// instruction rates.  fma(1, a, b) == a + b bitwise, so if DADD issues slower than
// DFMA the additions can be spelled as DFMA for free.
#include <cuda_runtime.h>
#include <cstdio>
template <int OP>
__global__ void k(double *out, int iters, double s) {
    double x[8];
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 1e-3 + j;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (OP == 0) x[j] = __dadd_rn(x[j], s);
            if (OP == 1) x[j] = __dmul_rn(x[j], s);
            if (OP == 2) x[j] = __fma_rn(x[j], s, s);
            if (OP == 3) x[j] = __fma_rn(1.0, x[j], s);
        }
    }
    double t = 0;
    for (int j = 0; j < 8; ++j) t += x[j];
    if (t == 1.2345) out[0] = t;
}
int main() {
    double *o; cudaMalloc(&o, 8);
    const int iters = 20000, blocks = 148 * 8, th = 256;
    const char *names[] = {"DADD", "DMUL", "DFMA", "DFMA(1,a,b)"};
    for (int op = 0; op < 4; ++op) {
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            if (op == 0) k<0><<<blocks, th>>>(o, iters, 1.0000001);
            if (op == 1) k<1><<<blocks, th>>>(o, iters, 1.0000001);
            if (op == 2) k<2><<<blocks, th>>>(o, iters, 1.0000001);
            if (op == 3) k<3><<<blocks, th>>>(o, iters, 1.0000001);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            double inst = (double)blocks * th * iters * 8;
            if (rep) printf("%-12s %.2f T lane-instr/s\n", names[op], inst / ms / 1e9);
        }
    }
    return 0;
}
