/*
 * oracle/irk_oracle.c -- TEST INFRASTRUCTURE ONLY (see irk_oracle.h).
 *
 * A plain, slow, obviously-correct scalar C implementation of the IRKGL16
 * constant-step fixed-point integrator of arXiv 2511.03655, written from the
 * paper.  Every arithmetic operation is an explicit IEEE round-to-nearest
 * double operation in the order written here (build flags: -O2
 * -fno-tree-vectorize -ffp-contract=off, never -ffast-math); `fma` is the C99
 * correctly-rounded fused multiply-add.  The canonical operation sequence is
 * documented in oracle/CANON.md and in DESIGN.md.
 *
 * Paper map (P:Lnnn = /root/reference/PAPER.md line nnn):
 *   tableau  : collocation conditions P:L109-116 (Sec. 2.2), Gauss nodes P:L116,
 *              mu = a/b with symplectic rounding P:L146-155 (Sec. 2.3, Eq. Yi2),
 *              nu extrapolation P:L165-178 (Sec. 2.4, Eqs. Yni0/Pol0; the printed
 *              nu condition is garbled -- reading R-3 in DESIGN.md).
 *   step     : partitioned P:L267-283 (Eqs. IRK_init2, IRK_FP2), first-order
 *              P:L218-232 (Eqs. IRK_init, IRK_FP), update P:L210-214 (Eq. yn3).
 *   stop test: P:L239-244 (Eq. stopping), reading R2.
 *   RHS      : Henon-Heiles Listing 2; N-body Eq. Ham2 P:L542-547.
 *   energy   : Eq. DHglobmax P:L597-603 uses H(y_n).
 *
 * Independence: the tableau is computed here by bisection on the Legendre
 * polynomial and exact integration of the expanded Lagrange basis in
 * __float128 -- a different algorithm from the library's (Newton + Bjorck-
 * Pereyra Vandermonde solves).
 */
#include "irk_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef __float128 q128;

#define S8 8
#define NB_BLOCK 1024 /* canonical j-block of the direct N-body sum (R-8) */

/* ------------------------------------------------------------------ */
/* Tableau                        */
/* ------------------------------------------------------------------ */

/* Legendre P_s(x) by the three-term recurrence (k+1)P_{k+1} = (2k+1)xP_k - kP_{k-1}. */
static q128 legendre_q(int s, q128 x) {
    q128 p0 = 1, p1 = x;
    if (s == 0) return p0;
    for (int k = 1; k < s; ++k) {
        q128 p2 = ((2 * k + 1) * x * p1 - k * p0) / (k + 1);
        p0 = p1;
        p1 = p2;
    }
    return p1;
}

/* Zeros of P_s on (-1,1), ascending: grid scan for sign changes, then bisection
 * until the bracket stops shrinking. */
static int legendre_roots_q(int s, q128 *x) {
    const int grid = 4000;
    int found = 0;
    q128 xa = -1, fa = legendre_q(s, xa);
    for (int g = 1; g <= grid && found < s; ++g) {
        q128 xb = -1 + (q128)2 * g / grid;
        q128 fb = legendre_q(s, xb);
        if (fb == 0) {
            x[found++] = xb;
        } else if ((fa < 0 && fb > 0) || (fa > 0 && fb < 0)) {
            q128 lo = xa, hi = xb, flo = fa;
            for (int it = 0; it < 400; ++it) {
                q128 mid = (lo + hi) / 2;
                if (mid == lo || mid == hi) break;
                q128 fm = legendre_q(s, mid);
                if (fm == 0) { lo = hi = mid; break; }
                if ((fm < 0) == (flo < 0)) { lo = mid; flo = fm; } else { hi = mid; }
            }
            x[found++] = (lo + hi) / 2;
        }
        xa = xb;
        fa = fb;
    }
    return found == s ? 0 : -1;
}

/* Coefficients of the Lagrange basis polynomial l_j(t) = prod_{m!=j} (t-c_m)/(c_j-c_m),
 * coef[k] multiplies t^k, k = 0..s-1. */
static void lagrange_coef_q(int s, const q128 *c, int j, q128 *coef) {
    q128 poly[17];
    for (int k = 0; k <= s; ++k) poly[k] = 0;
    poly[0] = 1;
    int deg = 0;
    q128 den = 1;
    for (int m = 0; m < s; ++m) {
        if (m == j) continue;
        /* poly *= (t - c_m) */
        for (int k = deg + 1; k >= 1; --k) poly[k] = poly[k - 1] - c[m] * poly[k];
        poly[0] = -c[m] * poly[0];
        ++deg;
        den *= (c[j] - c[m]);
    }
    for (int k = 0; k < s; ++k) coef[k] = poly[k] / den;
}

/* integral_{alpha}^{beta} of sum_k coef[k] t^k dt, exactly term by term */
static q128 poly_integral_q(int s, const q128 *coef, q128 alpha, q128 beta) {
    q128 acc = 0, pa = alpha, pb = beta;
    for (int k = 0; k < s; ++k) {
        acc += coef[k] * (pb - pa) / (k + 1);
        pa *= alpha;
        pb *= beta;
    }
    return acc;
}

static int tableau_q(int s, q128 *c, q128 *b, q128 *a, q128 *nu) {
    if (s < 1 || s > 16) return -1;
    q128 x[16];
    if (legendre_roots_q(s, x)) return -1;
    for (int i = 0; i < s; ++i) c[i] = (1 + x[i]) / 2; /* c_i = (1+x_i)/2 */
    for (int j = 0; j < s; ++j) {
        q128 coef[16];
        lagrange_coef_q(s, c, j, coef);
        b[j] = poly_integral_q(s, coef, 0, 1);                           /* b_j = int_0^1 l_j */
        for (int i = 0; i < s; ++i) a[i * s + j] = poly_integral_q(s, coef, 0, c[i]); /* a_ij */
    }
    /* nu_ij: P_{n-1}(t_{n-1}+c_i h) - y_{n-1} = sum_j [int_1^{1+c_i} l_j] h f_j,
     * and L_{n-1,j} = h b_j f_j (Eq. Yi2), hence nu_ij = int_1^{1+c_i} l_j / b_j. */
    for (int j = 0; j < s; ++j) {
        q128 coef[16];
        lagrange_coef_q(s, c, j, coef);
        for (int i = 0; i < s; ++i) nu[i * s + j] = poly_integral_q(s, coef, 1, 1 + c[i]) / b[j];
    }
    return 0;
}

int orc_tableau(int s, double *c, double *b, double *mu, double *nu) {
    q128 cq[16], bq[16], aq[256], nuq[256];
    if (tableau_q(s, cq, bq, aq, nuq)) return -1;
    for (int i = 0; i < s; ++i) {
        c[i] = (double)cq[i];
        b[i] = (double)bq[i];
    }
    /* mu~: lower triangle rounded from a_ij/b_j, upper derived as 1 - mu~_ji */
    for (int i = 0; i < s; ++i)
        for (int j = 0; j < i; ++j) mu[i * s + j] = (double)(aq[i * s + j] / bq[j]);
    for (int i = 0; i < s; ++i) {
        mu[i * s + i] = 0.5;
        for (int j = i + 1; j < s; ++j) mu[i * s + j] = 1.0 - mu[j * s + i];
    }
    for (int i = 0; i < s * s; ++i) nu[i] = (double)nuq[i];
    return 0;
}

static void split_dd(q128 v, double *hi, double *lo) {
    *hi = (double)v;
    *lo = (double)(v - (q128)(*hi));
}

int orc_tableau_dd(int s, double *c_hi, double *c_lo, double *b_hi, double *b_lo,
                   double *a_hi, double *a_lo, double *nu_hi, double *nu_lo) {
    q128 cq[16], bq[16], aq[256], nuq[256];
    if (tableau_q(s, cq, bq, aq, nuq)) return -1;
    for (int i = 0; i < s; ++i) {
        split_dd(cq[i], &c_hi[i], &c_lo[i]);
        split_dd(bq[i], &b_hi[i], &b_lo[i]);
    }
    for (int i = 0; i < s * s; ++i) {
        split_dd(aq[i], &a_hi[i], &a_lo[i]);
        split_dd(nuq[i], &nu_hi[i], &nu_lo[i]);
    }
    return 0;
}

/* ------------------------------------------------------------------ */
/* Small canonical helpers (CANON.md)                                  */
/* ------------------------------------------------------------------ */

/* D(w, L) = w_1 L_1 (+) ... : acc = w_1*L_1; acc = fma(w_j, L_j, acc), j = 2..8 */
static double dot8(const double *w, const double *L, int stride) {
    double acc = w[0] * L[0];
    for (int j = 1; j < S8; ++j) acc = fma(w[j], L[j * stride], acc);
    return acc;
}

/* S(L) = ((L_1 + L_2) + L_3) + ... + L_8, left to right (Eq. yn3) */
static double sum8(const double *L, int stride) {
    double acc = L[0];
    for (int j = 1; j < S8; ++j) acc = acc + L[j * stride];
    return acc;
}

typedef struct { double s, c; } neum_t;

/* Neumaier compensated summation step. */
static void neum_add(neum_t *n, double x) {
    double t = n->s + x;
    if (fabs(n->s) >= fabs(x))
        n->c = n->c + ((n->s - t) + x);
    else
        n->c = n->c + ((x - t) + n->s);
    n->s = t;
}
static double neum_result(const neum_t *n) { return n->s + n->c; }

/* ------------------------------------------------------------------ */
/* Stopping criterion, Eq. (stopping), reading R2            */
/* ------------------------------------------------------------------ */

/* One component: state (m = min of the history Delta[first..k-2], p = Delta[k-1]),
 * both starting at +inf; returns the component's verdict for the new Delta and
 * advances the state.  Explicit comparisons, never fmin/fmax. */
static int stop_component(double *m, double *p, double delta) {
    double mn = (delta < *p) ? delta : *p; /* min(Delta[k-1], Delta[k]) */
    int ok = (delta == 0.0) || (*m <= mn);
    *m = (*p < *m) ? *p : *m;
    *p = delta;
    return ok;
}

int orc_stop_test(const double *delta, int k) {
    double m = INFINITY, p = INFINITY;
    int ok = 0;
    for (int i = 0; i < k; ++i) ok = stop_component(&m, &p, delta[i]);
    return ok;
}

/* ------------------------------------------------------------------ */
/* Right-hand sides g(q, t) (CANON.md C-8)                              */
/* ------------------------------------------------------------------ */

static int problem_check(int problem, int dim, int nparams, const double *params) {
    switch (problem) {
    case ORC_KEPLER: return (dim == 4 && nparams >= 1) ? 0 : -1;
    case ORC_HENON_HEILES: return (dim == 4 && nparams >= 2) ? 0 : -1;
    case ORC_FPU_BETA: return (dim >= 2 && dim % 2 == 0 && nparams >= 1) ? 0 : -1;
    case ORC_SCHWARZSCHILD: return (dim == 4 && nparams >= 3) ? 0 : -1;
    case ORC_NBODY:
    case ORC_NBODY_DIRECT: {
        if (dim % 6 != 0 || dim < 12) return -1;
        int N = dim / 6;
        if (nparams != 2 + N) return -1;
        if (problem == ORC_NBODY_DIRECT && !(params[1] > 0.0)) return -1;
        return 0;
    }
    default: return -1;
    }
}

/* Kepler: r2 = fma(q1,q1,q2*q2); r3 = r2*sqrt(r2); w = GM/r3; a = -(w*q) */
static void accel_kepler(const double *P, const double *q, double *a) {
    double r2 = fma(q[0], q[0], q[1] * q[1]);
    double r3 = r2 * sqrt(r2);
    double w = P[0] / r3;
    a[0] = -(w * q[0]);
    a[1] = -(w * q[1]);
}

/* Henon-Heiles, Listing 2 literally:
 *   aux = lambda + xi*sin(t) (canonical sin); a1 = -q1 - 2*aux*q1*q2; a2 = -q2 - aux*(q1^2 - q2^2) */
static void accel_hh(const double *P, double t, const double *q, double *a) {
    double aux = P[0];
    if (P[1] != 0.0) {  /* canonical sin (CANON.md, R-12): bitwise the GPU's */
        double sn, cs;
        orc_sincos(t, &sn, &cs);
        aux = P[0] + P[1] * sn;
    }
    a[0] = -q[0] - ((2.0 * aux) * q[0]) * q[1];
    a[1] = -q[1] - aux * (q[0] * q[0] - q[1] * q[1]);
}

/* FPU-beta, fixed ends q_0 = q_{N+1} = 0; bond b (b=0..N) has Delta_b = q_{b+1} - q_b,
 * force f_b = V'(Delta_b) = fma(beta*(Delta*Delta), Delta, Delta); a_i = f_i - f_{i-1}. */
static void accel_fpu(int N, const double *P, const double *q, double *a) {
    double beta = P[0];
    double fprev = 0.0;
    for (int bnd = 0; bnd <= N; ++bnd) {
        double ql = (bnd == 0) ? 0.0 : q[bnd - 1];
        double qr = (bnd == N) ? 0.0 : q[bnd];
        double dl = qr - ql;
        double t = beta * (dl * dl);
        double f = fma(t, dl, dl);
        if (bnd >= 1) a[bnd - 1] = f - fprev;
        fprev = f;
    }
}

/* N-body ensembles (Eq. Ham2), cyclic partner order (CANON.md):
 *   d = q_j - q_i; r2 = fma(dz,dz,fma(dy,dy,fma(dx,dx,eps^2))); w = G/(r2*sqrt(r2));
 *   a_i = fma(m_j*w, d, a_i) for j = (i+1)%N, (i+2)%N, ..., (i+N-1)%N. */
static void accel_nbody_pairs(int N, const double *P, const double *q, double *a) {
    /* Eq. Ham2 force on each body i: the sum over the other bodies j
     * taken in cyclic order j = (i + delta) mod N, delta = 1..N-1 (R-8;
     * the paper does not fix a summation order). */
    double G = P[0], eps2 = P[1] * P[1];
    const double *m = P + 2;
    for (int i = 0; i < N; ++i) {
        double ax = 0.0, ay = 0.0, az = 0.0;
        for (int delta = 1; delta < N; ++delta) {
            int j = (i + delta) % N;
            double dx = q[3 * j] - q[3 * i];
            double dy = q[3 * j + 1] - q[3 * i + 1];
            double dz = q[3 * j + 2] - q[3 * i + 2];
            double r2 = fma(dz, dz, fma(dy, dy, fma(dx, dx, eps2)));
            double w = G / (r2 * sqrt(r2));
            double s = m[j] * w;
            ax = fma(s, dx, ax);
            ay = fma(s, dy, ay);
            az = fma(s, dz, az);
        }
        a[3 * i] = ax;
        a[3 * i + 1] = ay;
        a[3 * i + 2] = az;
    }
}

/* N-body direct sum for one body i, canonical blocked j-order (R-8):
 * j ascending in blocks of NB_BLOCK; part = fma(m_j*w, d, part) within a block
 * (starting from +0); acc = acc + part across blocks, left to right.  j = i is
 * included (d = +0, eps > 0). */
static void accel_direct_body(int N, const double *P, const double *q, int i, double *ai) {
    double G = P[0], eps2 = P[1] * P[1];
    const double *m = P + 2;
    double ax = 0.0, ay = 0.0, az = 0.0;
    for (int j0 = 0; j0 < N; j0 += NB_BLOCK) {
        int j1 = j0 + NB_BLOCK < N ? j0 + NB_BLOCK : N;
        double px = 0.0, py = 0.0, pz = 0.0;
        for (int j = j0; j < j1; ++j) {
            double dx = q[3 * j] - q[3 * i];
            double dy = q[3 * j + 1] - q[3 * i + 1];
            double dz = q[3 * j + 2] - q[3 * i + 2];
            double r2 = fma(dz, dz, fma(dy, dy, fma(dx, dx, eps2)));
            double w = G / (r2 * sqrt(r2));
            double s = m[j] * w;
            px = fma(s, dx, px);
            py = fma(s, dy, py);
            pz = fma(s, dz, pz);
        }
        ax = ax + px;
        ay = ay + py;
        az = az + pz;
    }
    ai[0] = ax;
    ai[1] = ay;
    ai[2] = az;
}

static void accel_direct(int N, const double *P, const double *q, double *a, int par) {
#pragma omp parallel for schedule(static) num_threads(par > 1 ? par : 1) if (par > 1)
    for (int i = 0; i < N; ++i) accel_direct_body(N, P, q, i, a + 3 * i);
}

static void accel_any(int problem, int dim, const double *P, double t, const double *q,
                      double *a, int par) {
    switch (problem) {
    case ORC_KEPLER: accel_kepler(P, q, a); break;
    case ORC_HENON_HEILES: accel_hh(P, t, q, a); break;
    case ORC_FPU_BETA: accel_fpu(dim / 2, P, q, a); break;
    case ORC_NBODY: accel_nbody_pairs(dim / 6, P, q, a); break;
    case ORC_NBODY_DIRECT: accel_direct(dim / 6, P, q, a, par); break;
    }
}

int orc_accel(int problem, int dim, const double *params, int nparams, double t,
              const double *q, double *a) {
    if (problem_check(problem, dim, nparams, params)) return -1;
    accel_any(problem, dim, params, t, q, a, 0);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Canonical sin / cos and the Schwarzschild black-hole problem          */
/* ------------------------------------------------------------------ */

/* Taylor coefficients RN((-1)^k / (2k+1)!) (sin) and RN((-1)^k / (2k)!) (cos),
 * computed once from the exact factorials in __float128. */
static double SIN_C[9], COS_C[10];
static int have_sc = 0;

static void sincos_init(void) {
#pragma omp critical(orc_sincos_init)
    {
        if (!have_sc) {
            q128 fact = 1;
            for (int n = 1; n <= 20; ++n) {
                fact *= n;
                if (n >= 3 && n % 2 == 1) SIN_C[(n - 3) / 2] = (double)((((n - 1) / 2) % 2 ? -1 : 1) / fact);
                if (n >= 2 && n % 2 == 0) COS_C[(n - 2) / 2] = (double)(((n / 2) % 2 ? -1 : 1) / fact);
            }
            have_sc = 1;
        }
    }
}

void orc_sincos(double x, double *sn, double *cs) {
    if (!have_sc) sincos_init();
    /* x = k pi/2 + t, |t| <= pi/4: pi/2 = P1 + P2 + P3 (each RN of the remainder) */
    const double TWO_OVER_PI = 0x1.45f306dc9c883p-1;
    const double P1 = 0x1.921fb54442d18p+0, P2 = 0x1.1a62633145c07p-54, P3 = -0x1.f1976b7ed8fbcp-110;
    double k = rint(x * TWO_OVER_PI);
    double t = fma(-k, P1, x);
    t = fma(-k, P2, t);
    t = fma(-k, P3, t);
    double z = t * t;
    double ps = SIN_C[8];
    for (int i = 7; i >= 0; --i) ps = fma(ps, z, SIN_C[i]);
    double st = fma(t * z, ps, t);           /* t + t^3 (S3 + z (S5 + ...)) */
    double pc = COS_C[9];
    for (int i = 8; i >= 0; --i) pc = fma(pc, z, COS_C[i]);
    double ct = fma(z, pc, 1.0);             /* 1 + z (C2 + z (C4 + ...)) */
    int q = (int)((long long)k & 3);
    switch (q) {
    case 0: *sn = st; *cs = ct; break;
    case 1: *sn = ct; *cs = -st; break;
    case 2: *sn = -st; *cs = -ct; break;
    default: *sn = -ct; *cs = st; break;
    }
}

/* Hamilton's equations of Eq. Ham_SBH, y = (r, theta, p_r, p_theta),
 * P = {E, L, beta}; f = 1 - 2/r, s = sin theta, A = L - (beta/2) r^2 s^2:
 *   r'       =  dH/dp_r     = f p_r
 *   theta'   =  dH/dp_theta = p_theta / r^2
 *   p_r'     = -dH/dr       = -(p_r^2/r^2 + E^2/(r^2 f^2) - p_theta^2/r^3 - beta A/r - A^2/(r^3 s^2))
 *   p_theta' = -dH/dtheta   = beta A cos/s + A^2 cos/(r^2 s^3)
 * in the canonical operation order of CANON.md. */
static void rhs_schwarzschild(const double *P, const double *y, double *f) {
    const double E = P[0], L = P[1], beta = P[2];
    const double r = y[0], th = y[1], pr = y[2], pth = y[3];
    double s, c;
    orc_sincos(th, &s, &c);
    const double fr = 1.0 - 2.0 / r;
    const double r2 = r * r, s2 = s * s;
    const double A = L - (0.5 * beta) * (r2 * s2);
    const double r3 = r2 * r;
    const double t1 = (pr * pr) / r2;
    const double t2 = (E * E) / (r2 * (fr * fr));
    const double t3 = (pth * pth) / r3;
    const double t4 = (beta * A) / r;
    const double t5 = (A * A) / (r3 * s2);
    f[0] = fr * pr;
    f[1] = pth / r2;
    f[2] = -((((t1 + t2) - t3) - t4) - t5);
    f[3] = ((beta * A) * c) / s + ((A * A) * c) / (r2 * (s2 * s));
}

static double energy_schwarzschild(const double *P, const double *y) {
    const double E = P[0], L = P[1], beta = P[2];
    const double r = y[0], th = y[1], pr = y[2], pth = y[3];
    double s, c;
    orc_sincos(th, &s, &c);
    const double fr = 1.0 - 2.0 / r;
    const double r2 = r * r, s2 = s * s;
    const double A = L - (0.5 * beta) * (r2 * s2);
    neum_t n = {0.0, 0.0};
    neum_add(&n, 0.5 * (fr * (pr * pr)));
    neum_add(&n, -(0.5 * ((E * E) / fr)));
    neum_add(&n, (pth * pth) / (2.0 * r2));
    neum_add(&n, (A * A) / (2.0 * (r2 * s2)));
    return neum_result(&n);
}

int orc_rhs(int problem, int dim, const double *params, int nparams, double t, const double *y, double *f) {
    if (problem_check(problem, dim, nparams, params)) return -1;
    if (problem == ORC_SCHWARZSCHILD) {
        rhs_schwarzschild(params, y, f);
        return 0;
    }
    const int d = dim / 2;
    for (int l = 0; l < d; ++l) f[l] = y[d + l];
    accel_any(problem, dim, params, t, y, f + d, 0);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Energies (canonical term order, Neumaier sums; CANON.md)             */
/* ------------------------------------------------------------------ */

static double energy_nbody(int N, const double *P, const double *y) {
    double G = P[0], eps2 = P[1] * P[1];
    const double *m = P + 2;
    const double *q = y, *v = y + 3 * N;
    neum_t tot = {0.0, 0.0};
    for (int i = 0; i < N; ++i) {
        double k = fma(v[3 * i + 2], v[3 * i + 2], fma(v[3 * i + 1], v[3 * i + 1], v[3 * i] * v[3 * i]));
        neum_add(&tot, (0.5 * m[i]) * k);
    }
    for (int i = 0; i < N; ++i) { /* row i: pairs (i, j>i), its own Neumaier sum */
        neum_t row = {0.0, 0.0};
        for (int j = i + 1; j < N; ++j) {
            double dx = q[3 * j] - q[3 * i];
            double dy = q[3 * j + 1] - q[3 * i + 1];
            double dz = q[3 * j + 2] - q[3 * i + 2];
            double r2 = fma(dz, dz, fma(dy, dy, fma(dx, dx, eps2)));
            neum_add(&row, -((G * (m[i] * m[j])) / sqrt(r2)));
        }
        neum_add(&tot, neum_result(&row));
    }
    return neum_result(&tot);
}

double orc_energy(int problem, int dim, const double *P, int nparams, const double *y) {
    if (problem_check(problem, dim, nparams, P)) return NAN;
    int d = dim / 2;
    const double *q = y, *v = y + d;
    neum_t n = {0.0, 0.0};
    switch (problem) {
    case ORC_KEPLER: /* H = |v|^2/2 - GM/|q| */
        neum_add(&n, 0.5 * (v[0] * v[0]));
        neum_add(&n, 0.5 * (v[1] * v[1]));
        neum_add(&n, -(P[0] / sqrt(fma(q[0], q[0], q[1] * q[1]))));
        return neum_result(&n);
    case ORC_HENON_HEILES: /* H = |p|^2/2 + |q|^2/2 + lambda (q1^2 q2 - q2^3/3) (autonomous part) */
        neum_add(&n, 0.5 * (v[0] * v[0]));
        neum_add(&n, 0.5 * (v[1] * v[1]));
        neum_add(&n, 0.5 * (q[0] * q[0]));
        neum_add(&n, 0.5 * (q[1] * q[1]));
        neum_add(&n, P[0] * ((q[0] * q[0]) * q[1]));
        neum_add(&n, -(P[0] * (((q[1] * q[1]) * q[1]) / 3.0)));
        return neum_result(&n);
    case ORC_FPU_BETA: { /* H = sum p^2/2 + sum_b (D^2/2 + beta D^4/4) */
        double beta = P[0];
        for (int i = 0; i < d; ++i) neum_add(&n, 0.5 * (v[i] * v[i]));
        for (int bnd = 0; bnd <= d; ++bnd) {
            double ql = (bnd == 0) ? 0.0 : q[bnd - 1];
            double qr = (bnd == d) ? 0.0 : q[bnd];
            double dl = qr - ql;
            double d2 = dl * dl;
            neum_add(&n, 0.5 * d2 + (0.25 * beta) * (d2 * d2));
        }
        return neum_result(&n);
    }
    case ORC_NBODY:
    case ORC_NBODY_DIRECT: return energy_nbody(dim / 6, P, y);
    case ORC_SCHWARZSCHILD: return energy_schwarzschild(P, y);
    }
    return NAN;
}

/* ------------------------------------------------------------------ */
/* Integrator                                                           */
/* ------------------------------------------------------------------ */

typedef struct {
    double c[S8], b[S8], mu[S8 * S8], nu[S8 * S8], hb[S8];
} coef_t;

typedef struct {
    double *Q, *Qn, *V, *Lq, *Lv, *F, *Y, *Yn, *L; /* [8][n] each, stage-major */
    double *m, *p;
} work_t;

static int work_alloc(work_t *w, int D) {
    size_t n = (size_t)S8 * D;
    double *buf = (double *)calloc(9 * n + 2 * (size_t)D, sizeof(double));
    if (!buf) return -1;
    w->Q = buf; w->Qn = buf + n; w->V = buf + 2 * n; w->Lq = buf + 3 * n; w->Lv = buf + 4 * n;
    w->F = buf + 5 * n; w->Y = buf + 6 * n; w->Yn = buf + 7 * n; w->L = buf + 8 * n;
    w->m = buf + 9 * n; w->p = w->m + D;
    return 0;
}

/* One partitioned step (Eqs. IRK_init2, IRK_FP2, yn3).
 * y = (q, v) of one trajectory (dim), hist = [8][dim] (only the v block is used).
 * Returns the number of sweeps; *capped = 1 when MAX_ITERS stopped it. */
static int step_partitioned(const orc_cfg *cfg, const coef_t *K, double tn1, double *y,
                            double *hist, work_t *w, int par, int *capped) {
    const int D = cfg->dim, d = D / 2;
    double *q = y, *v = y + d;
    /* a1: V_i^[0] = v + sum_j nu_ij Lv_{n-1,j}   (Eq. IRK_init2, velocities only) */
    for (int i = 0; i < S8; ++i)
        for (int l = 0; l < d; ++l) w->V[i * d + l] = v[l] + dot8(&K->nu[i * S8], &hist[d + l], D);
    for (int l = 0; l < d; ++l) w->m[l] = w->p[l] = INFINITY;
    int k = 0, stop = 0;
    *capped = 0;
    for (;;) {
        ++k;
        /* a2: Lq_j = hb_j * V_j ; Q_i^[k] = q + sum_j mu_ij Lq_j */
        for (int j = 0; j < S8; ++j)
            for (int l = 0; l < d; ++l) w->Lq[j * d + l] = K->hb[j] * w->V[j * d + l];
        for (int i = 0; i < S8; ++i)
            for (int l = 0; l < d; ++l) w->Qn[i * d + l] = q[l] + dot8(&K->mu[i * S8], &w->Lq[l], d);
        /* a5: stop test over positions, Delta^[k] defined from k = 2 (reading R2) */
        if (k >= 2) {
            stop = 1;
            for (int l = 0; l < d; ++l) {
                double delta = 0.0;
                for (int i = 0; i < S8; ++i) {
                    double e = fabs(w->Qn[i * d + l] - w->Q[i * d + l]);
                    delta = (e > delta) ? e : delta;
                }
                if (!stop_component(&w->m[l], &w->p[l], delta)) stop = 0;
            }
        }
        memcpy(w->Q, w->Qn, sizeof(double) * S8 * d);
        /* a3: F_i = g(Q_i, t_{n-1} + c_i h) */
        for (int i = 0; i < S8; ++i) {
            double ti = tn1 + K->c[i] * cfg->h;
            accel_any(cfg->problem, D, cfg->params, ti, &w->Q[i * d], &w->F[i * d], par);
        }
        /* a4: Lv_j = hb_j * F_j ; V_i^[k] = v + sum_j mu_ij Lv_j */
        for (int j = 0; j < S8; ++j)
            for (int l = 0; l < d; ++l) w->Lv[j * d + l] = K->hb[j] * w->F[j * d + l];
        for (int i = 0; i < S8; ++i)
            for (int l = 0; l < d; ++l) w->V[i * d + l] = v[l] + dot8(&K->mu[i * S8], &w->Lv[l], d);
        if (stop) break;
        if (k >= cfg->max_iters) { *capped = 1; break; }
    }
    /* a6: q += S(Lq), v += S(Lv) with the last iteration's L (Eq. yn3); history <- Lv */
    for (int l = 0; l < d; ++l) {
        q[l] = q[l] + sum8(&w->Lq[l], d);
        v[l] = v[l] + sum8(&w->Lv[l], d);
    }
    /* the partitioned history is L^v only (Eq. IRK_init2 extrapolates velocities);
     * the q block is zeroed (R-4) */
    for (int j = 0; j < S8; ++j)
        for (int l = 0; l < d; ++l) {
            hist[j * D + l] = 0.0;
            hist[j * D + d + l] = w->Lv[j * d + l];
        }
    return k;
}

/* One first-order step (Eqs. IRK_init, IRK_FP, yn3) for f(t,y) = (v, g(q,t)).
 * The stop test runs over all D components; Delta^[1] = ||Y^[1]-Y^[0]|| exists here. */
static int step_first_order(const orc_cfg *cfg, const coef_t *K, double tn1, double *y,
                            double *hist, work_t *w, int par, int *capped) {
    const int D = cfg->dim, d = D / 2;
    for (int i = 0; i < S8; ++i)
        for (int l = 0; l < D; ++l) w->Y[i * D + l] = y[l] + dot8(&K->nu[i * S8], &hist[l], D);
    for (int l = 0; l < D; ++l) w->m[l] = w->p[l] = INFINITY;
    int k = 0, stop = 0;
    *capped = 0;
    for (;;) {
        ++k;
        /* F_i = f(t_{n-1} + c_i h, Y_i^[k-1]): (V_i, g(Q_i)) for the second-order
         * problems, Hamilton's equations for Eq. Ham_SBH */
        for (int i = 0; i < S8; ++i) {
            double ti = tn1 + K->c[i] * cfg->h;
            if (cfg->problem == ORC_SCHWARZSCHILD) {
                rhs_schwarzschild(cfg->params, &w->Y[i * D], &w->F[i * D]);
                continue;
            }
            for (int l = 0; l < d; ++l) w->F[i * D + l] = w->Y[i * D + d + l];
            accel_any(cfg->problem, D, cfg->params, ti, &w->Y[i * D], &w->F[i * D + d], par);
        }
        for (int j = 0; j < S8; ++j)
            for (int l = 0; l < D; ++l) w->L[j * D + l] = K->hb[j] * w->F[j * D + l];
        for (int i = 0; i < S8; ++i)
            for (int l = 0; l < D; ++l) w->Yn[i * D + l] = y[l] + dot8(&K->mu[i * S8], &w->L[l], D);
        stop = 1;
        for (int l = 0; l < D; ++l) {
            double delta = 0.0;
            for (int i = 0; i < S8; ++i) {
                double e = fabs(w->Yn[i * D + l] - w->Y[i * D + l]);
                delta = (e > delta) ? e : delta;
            }
            if (!stop_component(&w->m[l], &w->p[l], delta)) stop = 0;
        }
        memcpy(w->Y, w->Yn, sizeof(double) * S8 * D);
        if (stop) break;
        if (k >= cfg->max_iters) { *capped = 1; break; }
    }
    for (int l = 0; l < D; ++l) y[l] = y[l] + sum8(&w->L[l], D);
    memcpy(hist, w->L, sizeof(double) * S8 * D);
    return k;
}

static int all_finite(const double *y, int D) {
    for (int l = 0; l < D; ++l)
        if (!isfinite(y[l])) return 0;
    return 1;
}

int orc_integrate(const orc_cfg *cfg, double *y, double *hist, double *energy, int64_t *iters,
                  int64_t *status) {
    if (!cfg || problem_check(cfg->problem, cfg->dim, cfg->nparams, cfg->params)) return -1;
    if (!(cfg->h == cfg->h) || cfg->h == 0.0 || isinf(cfg->h) || cfg->nsteps < 0 || cfg->batch < 1)
        return -1;
    if (cfg->max_iters < 1 || (cfg->mode != ORC_MODE_PARTITIONED && cfg->mode != ORC_MODE_FIRST_ORDER))
        return -1;
    /* Eq. Ham_SBH is not separable: only the first-order iteration applies */
    if (cfg->problem == ORC_SCHWARZSCHILD && cfg->mode != ORC_MODE_FIRST_ORDER) return -1;
    sincos_init();
    /* the s = 8 tableau is computed once per process (pure function of s) */
    static coef_t K8;
    static int have_K8 = 0;
    coef_t K;
#pragma omp critical(orc_tableau_cache)
    {
        if (!have_K8 && orc_tableau(S8, K8.c, K8.b, K8.mu, K8.nu) == 0) have_K8 = 1;
        K = K8;
    }
    if (!have_K8) return -1;
    for (int j = 0; j < S8; ++j) K.hb[j] = cfg->h * K.b[j]; /* hb~_j = fl(h * b~_j) */

    const int D = cfg->dim;
    const int64_t B = cfg->batch;
    const int64_t E = cfg->energy_every;
    int nt = cfg->nthreads;
#ifdef _OPENMP
    if (nt <= 0) nt = omp_get_max_threads();
#else
    nt = 1;
#endif
    const int inner_par = (B == 1 && nt > 1) ? nt : 0; /* single large system: parallel force loop */
    int err = 0;

#pragma omp parallel for schedule(dynamic, 1) num_threads(nt) if (B > 1)
    for (int64_t bi = 0; bi < B; ++bi) {
        work_t w;
        double *yb = (double *)malloc(sizeof(double) * D);
        if (!yb || work_alloc(&w, D)) {
#pragma omp atomic write
            err = 1;
            free(yb);
            continue;
        }
        for (int l = 0; l < D; ++l) yb[l] = y[(int64_t)l * B + bi];
        double *hb_hist = hist + bi * (int64_t)S8 * D;
        int64_t total = 0, hits = 0, bad = -1, last = 0;
        if (energy && E > 0) energy[bi] = orc_energy(cfg->problem, D, cfg->params, cfg->nparams, yb);
        /* Eq. DHlocmax: local relative energy error, max over this call's steps */
        double hprev = cfg->dhloc ? orc_energy(cfg->problem, D, cfg->params, cfg->nparams, yb) : 0.0;
        double dhmax = 0.0;
        for (int64_t n = 1; n <= cfg->nsteps; ++n) {
            if (bad >= 0) break; /* diverged trajectories are frozen */
            double tn1 = cfg->t0 + (double)(cfg->n0 + n - 1) * cfg->h; /* t_{n-1} = t0 + (n-1) h */
            int capped = 0;
            int k = (cfg->mode == ORC_MODE_PARTITIONED)
                        ? step_partitioned(cfg, &K, tn1, yb, hb_hist, &w, inner_par, &capped)
                        : step_first_order(cfg, &K, tn1, yb, hb_hist, &w, inner_par, &capped);
            total += k;
            hits += capped;
            last = k;
            if (!all_finite(yb, D)) bad = cfg->n0 + n;
            if (energy && E > 0 && n % E == 0)
                energy[(n / E) * B + bi] = orc_energy(cfg->problem, D, cfg->params, cfg->nparams, yb);
            if (cfg->dhloc) {
                double hn = orc_energy(cfg->problem, D, cfg->params, cfg->nparams, yb);
                double loc = fabs((hn - hprev) / hprev);
                dhmax = (loc > dhmax) ? loc : dhmax;
                hprev = hn;
            }
        }
        for (int l = 0; l < D; ++l) y[(int64_t)l * B + bi] = yb[l];
        if (iters) iters[bi] = total;
        if (cfg->dhloc) cfg->dhloc[bi] = dhmax;
        if (status) {
            status[3 * bi] = hits;
            status[3 * bi + 1] = bad;
            status[3 * bi + 2] = last;
        }
        free(w.Q);
        free(yb);
    }
    return err ? -1 : 0;
}
