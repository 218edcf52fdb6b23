/*
 * include/irk_probe.h -- measurement probes shipped in libirk.so (not part of
 * the integrator API).  Used by bench.py to measure the FP64 roofline
 * denominator on the box it runs on ("the builder measures a
 * DFMA microbenchmark").
 */
#ifndef IRK_PROBE_H
#define IRK_PROBE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

/* Launch a DFMA-throughput kernel: `blocks` x 256 threads, each running `iters`
 * iterations of 16 independent fused multiply-adds (2 flops each) on registers,
 * writing one double per thread to out (device, blocks*256 doubles) so nothing
 * is dead code.  Returns the flop count the launch performs (>0), or -1 on a
 * launch error.  Asynchronous on `stream`; time it with events. */
int64_t irk_probe_dfma(double *out, int blocks, int iters, void *stream);

/* Bitwise self-check of the branch-free IEEE division / square root used on the
 * hot path (paper_2511_03655_b200/csrc/fp64.cuh): for i < n writes
 * out[6i..6i+5] = {fast a/b (exact fallback applied), __ddiv_rn(a,b),
 * fast sqrt(b) (fallback applied), __dsqrt_rn(b), fast 1/b (the G = 1 form,
 * fallback applied), __ddiv_rn(1,b)}; device pointers.
 * Returns 0, or -1 on bad arguments / launch error. */
int irk_probe_divsqrt(const double *a, const double *b, double *out, int64_t n, void *stream);

#ifdef __cplusplus
}
#endif
#endif
