/* tests/oracle_sanitize_main.c -- TEST INFRASTRUCTURE ONLY.
 *
 * Drives every entry point of the scalar-C oracle (oracle/irk_oracle.c) on small
 * seeded inputs of every problem, in both modes, with energy samples, local
 * energy errors, chained calls and a diverging trajectory, so that a build with
 * -fsanitize=address,undefined (tests/test_oracle_sanitize.py) checks the
 * oracle's memory accesses and arithmetic for undefined behaviour.  Exit code 0
 * and no sanitizer report = pass.
 */
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "../oracle/irk_oracle.h"

static unsigned long long rng = 88172645463325252ull;
static double urand(void) { /* xorshift64, uniform in [-1, 1) */
    rng ^= rng << 13; rng ^= rng >> 7; rng ^= rng << 17;
    return (double)(rng >> 11) * (2.0 / 9007199254740992.0) - 1.0;
}

static int run(int problem, int dim, int mode, const double *params, int np, double h, int nsteps,
               int batch, const double *y0, int energy_every) {
    const int D = dim;
    double *y = malloc(sizeof(double) * D * batch), *hist = calloc((size_t)batch * 8 * D, sizeof(double));
    const int ne = energy_every ? nsteps / energy_every + 1 : 0;
    double *E = ne ? malloc(sizeof(double) * ne * batch) : NULL, *dh = malloc(sizeof(double) * batch);
    int64_t *it = malloc(sizeof(int64_t) * batch), *st = malloc(sizeof(int64_t) * 3 * batch);
    memcpy(y, y0, sizeof(double) * D * batch);
    orc_cfg c = {problem, dim, mode, 100, h, 0.25, nsteps / 2, batch, 0, energy_every, params, np, 2, dh};
    int rc = orc_integrate(&c, y, hist, E, it, st);              /* first half */
    c.n0 = nsteps / 2;
    c.nsteps = nsteps - nsteps / 2;
    rc |= orc_integrate(&c, y, hist, E, it, st);                 /* chained second half */
    double y1[256], f[256], a[256];  /* trajectory 0 as one state */
    for (int l = 0; l < D; ++l) y1[l] = y[(size_t)l * batch];
    rc |= orc_rhs(problem, dim, params, np, 0.5, y1, f);
    if (mode == ORC_MODE_PARTITIONED) rc |= orc_accel(problem, dim, params, np, 0.5, y1, a);
    double acc = orc_energy(problem, dim, params, np, y1) + (E ? E[0] : 0.0);
    for (int b = 0; b < batch; ++b) acc += y[b] + (double)it[b] + dh[b];
    free(y); free(hist); free(E); free(dh); free(it); free(st);
    printf("problem %d mode %d rc %d check %.3e\n", problem, mode, rc, acc);
    return rc;
}

int main(void) {
    int rc = 0;
    double c[16], b[16], mu[256], nu[256];
    double ch[16], cl[16], bh[16], bl[16], ah[256], al[256], nh[256], nl[256];
    for (int s = 1; s <= 16; ++s) {
        rc |= orc_tableau(s, c, b, mu, nu);
        rc |= orc_tableau_dd(s, ch, cl, bh, bl, ah, al, nh, nl);
    }
    const double delta[6] = {1e-3, 1e-6, 1e-9, 0.0, 1e-12, NAN};
    for (int k = 1; k <= 6; ++k) rc |= orc_stop_test(delta, k) < 0;
    double s1, c1;
    for (int i = -50; i <= 50; ++i) orc_sincos(i * 0.7, &s1, &c1);

    enum { B = 3 };
    double y[600];
    /* Kepler, e = 0.5 at pericentre; the last trajectory diverges (q = 0) */
    const double gm[1] = {1.0};
    for (int bb = 0; bb < B; ++bb) { y[bb] = 0.5; y[B + bb] = 0.0; y[2 * B + bb] = 0.0; y[3 * B + bb] = sqrt(3.0); }
    y[B - 1] = 0.0; y[3 * B - 1] = 0.0;
    rc |= run(ORC_KEPLER, 4, ORC_MODE_PARTITIONED, gm, 1, 0.05, 40, B, y, 10);
    /* N-body, N = 4, softened */
    const double nb[6] = {1.0, 0.05, 1.0, 0.5, 0.3, 0.2};
    for (int i = 0; i < 24 * B; ++i) y[i] = urand();
    rc |= run(ORC_NBODY, 24, ORC_MODE_PARTITIONED, nb, 6, 0.01, 20, B, y, 5);
    /* FPU-beta, N = 8 */
    const double beta[1] = {1.0};
    for (int i = 0; i < 16 * B; ++i) y[i] = 0.3 * urand();
    rc |= run(ORC_FPU_BETA, 16, ORC_MODE_PARTITIONED, beta, 1, 0.1, 20, B, y, 5);
    /* Henon-Heiles with xi != 0, both modes */
    const double hh[2] = {1.0, 0.1};
    for (int i = 0; i < 4 * B; ++i) y[i] = 0.2 * urand();
    rc |= run(ORC_HENON_HEILES, 4, ORC_MODE_PARTITIONED, hh, 2, 0.05, 20, B, y, 5);
    rc |= run(ORC_HENON_HEILES, 4, ORC_MODE_FIRST_ORDER, hh, 2, 0.05, 20, B, y, 5);
    /* large-N direct sum, N = 40 (one system) */
    double dp[42];
    dp[0] = 1.0; dp[1] = 0.05;
    for (int i = 0; i < 40; ++i) dp[2 + i] = 1.0 / 40;
    for (int i = 0; i < 240; ++i) y[i] = urand();
    rc |= run(ORC_NBODY_DIRECT, 240, ORC_MODE_PARTITIONED, dp, 42, 1e-3, 6, 1, y, 3);
    /* Schwarzschild, first-order mode: r = 10, theta = pi/2 + 0.1 */
    const double sbh[3] = {0.97, 4.0, 1.0};
    for (int bb = 0; bb < B; ++bb) { y[bb] = 10.0 + bb; y[B + bb] = 1.6707963; y[2 * B + bb] = 0.0; y[3 * B + bb] = 0.1; }
    rc |= run(ORC_SCHWARZSCHILD, 4, ORC_MODE_FIRST_ORDER, sbh, 3, 0.5, 20, B, y, 5);
    printf("rc %d\n", rc);
    return rc != 0;
}
