/*
 * include/irk.h -- C ABI of the B200-native IRKGL16 integrator.
 *
 * The library integrates y' = f(t, y), y(t0) = y0 with constant step h
 * ("t_n = t_0 + n h", "constant step-size
 * mode") by the 8-stage, order-16 Gauss-Legendre collocation method (IRKGL16,
 * P:L109-116) in the symplectic mu-form (Eqs. Yi2/yn2), solving the
 * stage equations by the partitioned fixed-point iteration (Eqs. IRK_init2,
 * IRK_FP2) or the first-order one (Eqs. IRK_init, IRK_FP,
 * P:L218-232) with the stagnation stopping test (Eq. stopping, P:L239-244,
 * reading R2 in DESIGN.md).  All arithmetic is IEEE binary64.
 *
 * Conventions
 *  - Bulk-data pointers are CUDA DEVICE pointers owned by the caller, except in
 *    irk_integrate_host (HOST pointers).  Nothing is retained after a call
 *    returns except inside the ctx.
 *  - y is structure-of-arrays, shape [dim][batch] (row l contiguous over
 *    trajectories); component order (q_1..q_d, v_1..v_d), d = dim/2, v = M^-1 p
 *    (P:L255-264).  N-body positions are body-major xyz (P:L394's (3,N) array).
 *  - All device work is enqueued on `stream` (a cudaStream_t; NULL = legacy
 *    default stream) and is asynchronous: buffers must stay alive until the
 *    stream is synchronised.  Functions that must read device results
 *    (irk_stats) synchronise the stream themselves.  Exception: irk_integrate
 *    on IRK_NBODY_DIRECT synchronises `stream` at its start (to see whether the
 *    system diverged in an earlier call), after every energy-sample segment of
 *    its device-side sweep loop, after every sweep when IRK_OPT_DEVICE_LOOP = 0,
 *    and at the end of an IRK_OPT_EXCHANGE = 1 call (DESIGN.md section 6,
 *    nbody_direct, "Synchronisation").
 *  - Errors: functions return an irk_status; argument errors are detected
 *    synchronously and leave every buffer untouched.  irk_last_error() gives a
 *    message.  A ctx is not thread-safe; distinct ctxs are independent.
 */
#ifndef IRK_H
#define IRK_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct irk_ctx irk_ctx; /* opaque, owned by the library */

/* Problems (right-hand sides g(q,t) of q' = v, v' = g(q,t), Eq. ivp2). */
enum irk_problem {
    IRK_KEPLER = 1,        /* planar Kepler, dim = 4; params {GM}                           */
    IRK_NBODY = 2,         /* N-body Eq. Ham2, cyclic pair order, dim = 6N, 2 <= N <= 8;
                              params {G, eps, m_1..m_N}                                   */
    IRK_FPU_BETA = 3,      /* FPU-beta chain, fixed ends, dim = 2N, N in {32, 64, 96, 128}; params {beta} */
    IRK_HENON_HEILES = 4,  /* Listing 2, dim = 4; params {lambda, xi}          */
    IRK_NBODY_DIRECT = 5,  /* large-N direct sum, canonical blocked j-order, dim = 6N;
                              params {G, eps > 0, m_1..m_N}; batch must be 1                */
    IRK_SCHWARZSCHILD = 6  /* charged particle near a magnetised Schwarzschild black hole,
                              Eq. Ham_SBH, y = (r, theta, p_r, p_theta),
                              dim = 4; params {E, L, beta}; not separable: first-order mode
                              (set by irk_create, MODE = 0 rejected)                       */
};

enum irk_status {
    IRK_OK = 0,
    IRK_W_MAXITER = 1,    /* warning (irk_stats): some steps hit MAX_ITERS; results valid   */
    IRK_E_ARG = -1,       /* invalid argument (returned synchronously)                      */
    IRK_E_CUDA = -2,      /* a CUDA call failed                                             */
    IRK_E_DIVERGED = -3,  /* (irk_stats) a trajectory became non-finite and was frozen      */
    IRK_E_COMM = -4,      /* NCCL error                                                     */
    IRK_E_STATE = -5      /* call out of order (e.g. integrate before set_params)           */
};

enum irk_option {
    IRK_OPT_MODE = 1,         /* 0 = partitioned (default, Eq. IRK_FP2), 1 = first-order (Eq. IRK_FP) */
    IRK_OPT_MAX_ITERS = 2,    /* sweeps cap per step, default 100 (flagged, step accepted)   */
    IRK_OPT_ENERGY_EVERY = 3, /* E > 0: sample H(y_n) at local steps 0, E, 2E, ... (default 0) */
    IRK_OPT_MAPPING = 4,      /* Kepler / Henon-Heiles (partitioned mode): IRK_MAP_AUTO (default),
                                 IRK_MAP_G1 = one trajectory per thread, IRK_MAP_G2 / IRK_MAP_G4 =
                                 2 / 4 lanes per trajectory (4 / 2 stages per lane), IRK_MAP_G8 = 8 lanes per
                                 trajectory, one stage per lane (shared-memory all-gather, shuffle
                                 convergence reduction), IRK_MAP_G8M = one stage per lane with both
                                 stage contractions on the FP64 tensor core (DMMA m8n8k4 on shuffled
                                 fragments; ensemble_g8m.cuh; auto for small batches).  In
                                 first-order mode G8M falls back to G1.  IRK_NBODY: IRK_MAP_G1 = body per lane,
                                 IRK_MAP_G8 = stage per lane (shared-memory all-gather),
                                 IRK_MAP_G8M = stage per lane with the two stage contractions on
                                 the FP64 tensor core (DMMA m8n8k4; ensemble_nbody8m.cuh).  Auto
                                 picks by problem, N and batch size from measured crossovers
                                 ("ens_gs", "ens_gsm", "ens_nbody8", "ens_nbody8m"; the chunked IRK_OPT_SCHEDULE = 1 keeps
                                 body per lane).  Bitwise-neutral.  */
    IRK_OPT_BALANCE = 5,      /* ensemble scheduling: -1 = auto (default), 0 = off, C > 0 = run the
                                 call in chunks of C steps, re-sorting trajectories by the cost of
                                 the previous chunk (bitwise-neutral, "ens_g1q") */
    IRK_OPT_VSHARDS = 6,      /* IRK_NBODY_DIRECT only: drive P body shards from this process on one
                                 GPU through the sharded code path (testing the exchange layout)   */
    IRK_OPT_SCHEDULE = 8,     /* ensemble launch: 0 = auto (default), 1 = chunked launches with the
                                 cost sort of BALANCE, 2 = one persistent launch whose lanes pull
                                 (trajectory, step-chunk) units from a work queue (per-thread
                                 problems, partitioned mode; BALANCE = C > 0 sets the unit length).
                                 Bitwise-neutral ("ens_g1q")                   */
    IRK_OPT_DEVICE_LOOP = 9,  /* IRK_NBODY_DIRECT: 1 (default) = the fixed-point sweeps run as a CUDA-graph
                                 conditional WHILE loop on the device (one host sync per energy
                                 sample / call); 0 = host loop, one sync per sweep               */
    IRK_OPT_EXCHANGE = 10,    /* IRK_NBODY_DIRECT under irk_set_comm: how the stage positions reach the
                                 other ranks each fixed-point iteration.  0 (default) = in-place
                                 ncclAllGather after the position kernel; 1 = fused: the position
                                 kernel stores every Q value straight into each rank's copy of its
                                 slot (a symmetric NCCL window, NVLink load/store, NCCL >= 2.27, all
                                 ranks in one NVLink domain) and its last CTA signals arrival; the
                                 next kernel waits for all ranks (IRK_E_COMM after 60 s).  The window
                                 is created collectively on the first fused irk_integrate and freed
                                 by irk_destroy.  Bitwise-neutral.  With more
                                 than one rank this mode has not run across GPUs yet: irk_integrate
                                 returns IRK_E_STATE unless the environment sets
                                 IRK_EXPERIMENTAL_FUSED_EXCHANGE=1                                  */
    IRK_OPT_LOCAL_ENERGY = 7  /* 1: track Delta H^loc_max = max_n |(H(y_n)-H(y_{n-1}))/H(y_{n-1})|
                                 (Eq. DHlocmax) over each call, in-kernel; read it with
                                 irk_local_energy_error (ensemble problems only)                   */
};

enum irk_mapping { IRK_MAP_AUTO = 0, IRK_MAP_G1 = 1, IRK_MAP_G2 = 2, IRK_MAP_G4 = 4, IRK_MAP_G8 = 8, IRK_MAP_G8M = 9 };

/* Create a context for `batch` independent trajectories of `problem` in
 * dimension `dim`, step h (finite, != 0; negative allowed), nsteps >= 0 steps per
 * irk_integrate call.  Builds the tableau in __float128 (Newton on P_8,
 * Bjorck-Pereyra Vandermonde solves), checks B(16), C(8), the symplectic
 * condition and the mu~ identity, and rounds it (R-1).  Returns NULL
 * on error (message via irk_last_error(NULL)); 1 <= batch <= 2^31 - 1. */
irk_ctx *irk_create(int problem, int dim, double h, int64_t nsteps, int64_t batch);

/* Copy n host doubles of problem parameters (see enum irk_problem). */
int irk_set_params(irk_ctx *ctx, const double *host_params, int n);

int irk_set_option(irk_ctx *ctx, int key, int64_t val);

/* Read an option (any IRK_OPT_*) or a read-only fact about the last call:
 * IRK_INFO_DEVICE_LOOP_USED = 1 if the last IRK_NBODY_DIRECT call ran its sweeps as
 * the device-side graph loop (0: host loop); IRK_INFO_MAPPING_USED = the IRK_MAP_*
 * value IRK_OPT_MAPPING (auto included) resolved to in the last irk_integrate
 * (IRK_MAP_G1/G2/G4/G8 for Kepler, Henon-Heiles, Schwarzschild; G1 = body per lane,
 * G8 = stage per lane for IRK_NBODY; 0 for IRK_FPU_BETA and IRK_NBODY_DIRECT, which
 * have one mapping).  IRK_E_ARG for an unknown key. */
enum irk_info { IRK_INFO_DEVICE_LOOP_USED = 100, IRK_INFO_MAPPING_USED = 101 };
int irk_get_option(const irk_ctx *ctx, int key, int64_t *val);

/* Bytes of caller-owned DEVICE workspace irk_integrate needs.  Layout: a
 * 64-byte header {int64 n_done, ...}, then the history L_{n-1} [8][dim][batch]
 * fp64, then per-trajectory stats [4][batch] int64 {maxiter_hits, diverged_step
 * (1-based absolute step, 0 = none), sweeps_total, Delta H^loc_max of the last call
 * (fp64 bits, IRK_OPT_LOCAL_ENERGY)}, then scheduler scratch
 * (int32 permutation and cost-sort buffers).  A zero-filled workspace means "first
 * step" (zero history, n_done = 0); reusing it continues the integration bitwise
 * as if uninterrupted (t_{n-1} = t0 + (n-1) h with the absolute n). */
size_t irk_workspace_bytes(const irk_ctx *ctx);

/* Advance y (device, [dim][batch]) by nsteps steps.  t0 is the initial time of
 * the whole run.  energy (device, [(nsteps/E)+1][batch]) receives H(y) at local
 * steps 0, E, 2E, ... when ENERGY_EVERY = E > 0, else may be NULL.  iters
 * (device, [batch]) receives the number of fixed-point sweeps of this call per
 * trajectory, or NULL. */
int irk_integrate(irk_ctx *ctx, double *y, double t0, void *workspace, double *energy,
                  int64_t *iters, void *stream);

/* Same, end to end from HOST memory: copies y_host (pinned or pageable) to an
 * internal device buffer, integrates from a fresh (zero) internal workspace,
 * copies the result back into y_host and, if non-NULL, energy_host / iters_host;
 * synchronises `stream` before returning. */
int irk_integrate_host(irk_ctx *ctx, double *y_host, double t0, double *energy_host,
                       int64_t *iters_host, void *stream);

/* H(y) per trajectory (device in, device out [batch]); Neumaier-compensated,
 * canonical term order (oracle/CANON.md "Energies"). */
int irk_energy(irk_ctx *ctx, const double *y, double *H, void *stream);

/* Synchronises `stream`, reduces the workspace stats: out = {trajectories with
 * MAX_ITERS hits, diverged trajectories, first diverged step (-1), total sweeps}.
 * Returns IRK_E_DIVERGED, IRK_W_MAXITER or IRK_OK accordingly. */
int irk_stats(irk_ctx *ctx, const void *workspace, void *stream, int64_t out[4]);

/* After irk_integrate with IRK_OPT_LOCAL_ENERGY = 1: copy the per-trajectory
 * Delta H^loc_max of that call (device, [batch] fp64) from the workspace to `out`
 * (device).  Asynchronous on `stream`.  IRK_E_STATE if the option is not set. */
int irk_local_energy_error(irk_ctx *ctx, const void *workspace, double *out, void *stream);

/* Host copy of the fp64 tableau the kernels use: c~[8], b~[8], mu~[8*8], nu~[8*8]
 * (row-major [i*8+j]).  Returns IRK_OK. */
int irk_tableau(double *c, double *b, double *mu, double *nu);

/* NCCL communicator for a body-sharded IRK_NBODY_DIRECT system (one process per
 * GPU): rank r of nranks owns bodies [r*N/nranks, (r+1)*N/nranks)
 * and from then on passes only its bodies' rows to irk_integrate: y is
 * [q_local (3N/P) | v_local (3N/P)], the history [8][6N/P] (call
 * irk_workspace_bytes after this).  Each fixed-point iteration all-gathers the
 * stage positions (8 x 3N/P doubles + 2 flags per rank) in place over NCCL; the
 * stop decision is the same on every rank, and results equal the 1-GPU run bit
 * for bit.  nccl_unique_id points to 128 bytes from irk_nccl_unique_id on rank 0,
 * broadcast by the caller.  NCCL is loaded at run time (libnccl.so.2, or the path
 * in $IRK_NCCL_LIB).  Returns IRK_E_COMM on NCCL failure. */
int irk_set_comm(irk_ctx *ctx, const void *nccl_unique_id, int rank, int nranks);

/* Write a fresh 128-byte ncclUniqueId to `out` (rank 0 of irk_set_comm). */
int irk_nccl_unique_id(void *out);

/* NULL ctx: the thread-local message of the last failed irk_create. */
const char *irk_last_error(const irk_ctx *ctx);

void irk_destroy(irk_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif
