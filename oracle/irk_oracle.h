/*
 * oracle/irk_oracle.h -- TEST INFRASTRUCTURE ONLY.
 *
 * Plain, slow, scalar-C oracle of the IRKGL16 constant-step fixed-point
 * integrator of arXiv 2511.03655 ("SIMD-vectorized implicit symplectic
 * integrators can outperform explicit symplectic ones").  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
 * legs may load it.  It shares no code with the CUDA path
 * (paper_2511_03655_b200/csrc); neither includes the other.
 *
 * Citations: P:Lnnn = /root/reference/PAPER.md line nnn (section / equation).
 */
#ifndef IRK_ORACLE_H
#define IRK_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Problem ids (same numbering as include/irk.h; the numbers are the only
 * thing the two sides agree on, by documentation, not by a shared header). */
#define ORC_KEPLER 1        /* planar Kepler, d=2, params {GM}                      */
#define ORC_NBODY 2         /* N-body, cyclic pair order, params {G, eps, m_1..m_N} */
#define ORC_FPU_BETA 3      /* FPU-beta chain, fixed ends, params {beta}           */
#define ORC_HENON_HEILES 4  /* Listing 2, params {lambda, xi}         */
#define ORC_NBODY_DIRECT 5  /* large-N direct sum, blocked j-order, {G, eps>0, m}  */
#define ORC_SCHWARZSCHILD 6 /* Eq. Ham_SBH, y = (r, theta, p_r, p_theta),
                               params {E, L, beta}; first-order mode only             */

#define ORC_MODE_PARTITIONED 0 /* Eqs. IRK_init2 / IRK_FP2, P:L267-283 (default)   */
#define ORC_MODE_FIRST_ORDER 1 /* Eqs. IRK_init / IRK_FP               */

typedef struct {
    int problem, dim, mode, max_iters;
    double h, t0;
    int64_t nsteps, batch;
    int64_t n0;            /* absolute index of the first step of this call (0 = fresh run) */
    int64_t energy_every;  /* 0 = no energy samples                                 */
    const double *params;
    int nparams;
    int nthreads;          /* OpenMP threads (<=0: runtime default)                */
    double *dhloc;         /* [batch] or NULL: max_n |(H(y_n)-H(y_{n-1}))/H(y_{n-1})| over the
                              call's steps, Eq. DHlocmax                   */
} orc_cfg;

/* Tableau for s stages (1 <= s <= 16), rounded to fp64 exactly as DESIGN.md R-1:
 *   c~_i = RN(c_i), b~_i = RN(b_i), mu~_ij = RN(a_ij/b_j) (i>j), mu~_ij = 1 - mu~_ji (i<j),
 *   mu~_ii = 1/2, nu~_ij = RN(nu_ij).  mu, nu row-major [i*s+j].  Returns 0 on success. */
int orc_tableau(int s, double *c, double *b, double *mu, double *nu);

/* The same quantities before rounding, as double-double pairs (hi, lo) of the
 * __float128 values: c, b, a (s*s), nu (s*s).  For the high-precision pins. */
int orc_tableau_dd(int s, double *c_hi, double *c_lo, double *b_hi, double *b_lo,
                   double *a_hi, double *a_lo, double *nu_hi, double *nu_lo);

/* Stopping criterion, Eq. (stopping), reading R2: given a
 * per-component Delta sequence delta[0..k-1] (the Deltas of iterations that
 * have one, oldest first), return 1 iff the test fires after the last one. */
int orc_stop_test(const double *delta, int k);

/* Right-hand side (accelerations g(q,t), or the full f for first-order use is
 * built from it) for one state.  q: d positions; out: d accelerations. */
int orc_accel(int problem, int dim, const double *params, int nparams, double t,
              const double *q, double *a);

/* Full first-order right-hand side f(t, y) of one state (dim components):
 * (v, g(q,t)) for the second-order problems, Hamilton's equations for
 * ORC_SCHWARZSCHILD. */
int orc_rhs(int problem, int dim, const double *params, int nparams, double t, const double *y,
            double *f);

/* Canonical sine and cosine (CANON.md "Canonical sin/cos"): Cody-Waite reduction
 * by pi/2 in three parts, Taylor polynomials of degree 19 / 20 on |t| <= pi/4. */
void orc_sincos(double x, double *s, double *c);

/* Hamiltonian of one state y (dim), Neumaier-compensated, canonical order. */
double orc_energy(int problem, int dim, const double *params, int nparams, const double *y);

/* Integrate `batch` independent trajectories for nsteps constant steps.
 *   y      : SoA [dim][batch], in/out.
 *   hist   : [batch][8][dim], in/out; L_{n-1} of the previous step (zeros = first step).
 *   energy : [(nsteps/energy_every)+1][batch] or NULL.
 *   iters  : [batch] total fixed-point sweeps, or NULL.
 *   status : [batch][3] {maxiter_hits, diverged_step(-1 none), last_step_sweeps}, or NULL.
 * Returns 0, or -1 on argument error. */
int orc_integrate(const orc_cfg *cfg, double *y, double *hist, double *energy,
                  int64_t *iters, int64_t *status);

#ifdef __cplusplus
}
#endif
#endif
