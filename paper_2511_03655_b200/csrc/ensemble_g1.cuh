// Ensemble kernel, mapping "g1": one trajectory per thread, the whole 8-stage
// tile (Q, V, Lq, Lv: 32*d doubles) in registers, persistent over all nsteps
// steps of the call (state and history touch HBM once per call).
//
// Hot path rows (DESIGN.md / SURVEY.md 8(a)):
//   a1  nu-init          V_i = v + sum_j nu_ij Lv_{n-1,j}        Eq. IRK_init2
//   a2  position sweep   Lq = hb o V ; Q_i = q + sum_j mu_ij Lq_j Eq. IRK_FP2 l.1-2
//   a5  stop test        Delta_l = max_i |Q_i - Q_i^old|, R2     Eq. stopping
//   a3  8 RHS            F_i = g(Q_i, t_{n-1} + c_i h)           Eq. IRK_FP2 l.3
//   a4  velocity sweep   Lv = hb o F ; V_i = v + sum_j mu_ij Lv_j Eq. IRK_FP2 l.4-5
//   a6  update           q += S(Lq), v += S(Lv), H = Lv           Eq. yn3
//   a7  energy sample    H(y_n) every E steps                    Eq. DHglobmax
//
// Sweep-granular loop: one loop trip is one sweep of one trajectory; a lane
// whose step converged does the update and the next step's nu-init inside the
// same trip (the contraction a4 then uses nu instead of mu: the V computed with
// mu on a converged sweep is discarded in the canonical sequence, so selecting
// the coefficient per lane is bitwise-neutral).  Warps therefore stay in lock
// step on the sweep body instead of waiting for their slowest lane every step.
#pragma once
#include <cstdint>

#include "fp64.cuh"
#include "tableau.h"

namespace irk {

struct EnsArgs {
    Tableau T;
    double *y;            // [dim][batch]
    double *hist;         // [8][dim][batch]
    int64_t *stats;       // [4][batch]
    const int64_t *n_done;
    double *energy;       // [(nsteps/E)+1][batch] or null
    int64_t *iters;       // [batch] or null
    int64_t batch, nsteps, energy_every;
    double h, t0;
    int max_iters;
};

template <class P>
__global__ void __launch_bounds__(64, 8) ens_g1_kernel(const __grid_constant__ EnsArgs a,
                                                    const __grid_constant__ P prob) {
    constexpr int d = P::d, D = 2 * d;
    const int64_t B = a.batch;
    const int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= B) return;

    int64_t bad = a.stats[1 * B + b];
    int64_t hits = 0, sweeps = 0;
    double q[d], v[d], V[8][d], Q[8][d], Lq[8][d], m[d], p[d];
#pragma unroll
    for (int l = 0; l < d; ++l) {
        q[l] = a.y[l * B + b];
        v[l] = a.y[(d + l) * B + b];
    }
    const int64_t n0 = *a.n_done;
    const bool sample = (a.energy != nullptr) && (a.energy_every > 0);
    if (sample) a.energy[b] = prob.energy(q, v);
    if (bad > 0 || a.nsteps == 0) {  // frozen (diverged at step `bad`, 1-based) or nothing to do
        if (a.iters) a.iters[b] = 0;
        return;
    }
    {   // a1: nu-init from the history (zeros = first step)
        double H[8][d];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int l = 0; l < d; ++l) H[j][l] = a.hist[((int64_t)j * D + d + l) * B + b];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int l = 0; l < d; ++l) {
                double acc = dmul(a.T.nu[i][0], H[0][l]);
#pragma unroll
                for (int j = 1; j < 8; ++j) acc = dfma(a.T.nu[i][j], H[j][l], acc);
                V[i][l] = dadd(v[l], acc);
            }
    }
#pragma unroll
    for (int l = 0; l < d; ++l) {
        m[l] = p[l] = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
        for (int i = 0; i < 8; ++i) Q[i][l] = 0.0;  // Q^[0] is never compared (R2)
    }

    int64_t n = 0;
    int k = 0;
    while (n < a.nsteps) {
        ++k;
        // a2: Lq_j = hb_j V_j ; Q_i^[k] = q + D(mu_i., Lq)   (+ a5 on the fly)
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int l = 0; l < d; ++l) Lq[j][l] = dmul(a.T.hb[j], V[j][l]);
        bool stop = (k >= 2);
#pragma unroll
        for (int l = 0; l < d; ++l) {
            double delta = 0.0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double acc = dmul(a.T.mu[i][0], Lq[0][l]);
#pragma unroll
                for (int j = 1; j < 8; ++j) acc = dfma(a.T.mu[i][j], Lq[j][l], acc);
                double qn = dadd(q[l], acc);
                double e = dabs(dsub(qn, Q[i][l]));
                delta = (e > delta) ? e : delta;
                Q[i][l] = qn;
            }
            if (k >= 2) {  // a5, reading R2: Delta^[k] exists from k = 2
                double mn = (delta < p[l]) ? delta : p[l];
                bool ok = (delta == 0.0) || (m[l] <= mn);
                m[l] = (p[l] < m[l]) ? p[l] : m[l];
                p[l] = delta;
                stop = stop && ok;
            }
        }
        // a3 + a4 (first half): F_i = g(Q_i, t_i) ; Lv_i = hb_i F_i
        const double tn1 = dadd(a.t0, dmul((double)(n0 + n), a.h));
        double Lv[8][d];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            double F[d];
            prob.accel(Q[i], F, dadd(tn1, dmul(a.T.c[i], a.h)));
#pragma unroll
            for (int l = 0; l < d; ++l) Lv[i][l] = dmul(a.T.hb[i], F[l]);
        }
        const bool fin = stop || (k >= a.max_iters);
        if (fin) {  // a6: update with the last iteration's L, history <- Lv
            bool finite = true;
#pragma unroll
            for (int l = 0; l < d; ++l) {
                double sq = Lq[0][l], sv = Lv[0][l];
#pragma unroll
                for (int j = 1; j < 8; ++j) {
                    sq = dadd(sq, Lq[j][l]);
                    sv = dadd(sv, Lv[j][l]);
                }
                q[l] = dadd(q[l], sq);
                v[l] = dadd(v[l], sv);
                finite = finite && isfinite(q[l]) && isfinite(v[l]);
            }
            ++n;
            sweeps += k;
            hits += stop ? 0 : 1;
            k = 0;
#pragma unroll
            for (int l = 0; l < d; ++l) m[l] = p[l] = __longlong_as_double(0x7ff0000000000000LL);
            if (sample && (n % a.energy_every) == 0)
                a.energy[(n / a.energy_every) * B + b] = prob.energy(q, v);
            if (n == a.nsteps || !finite) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
#pragma unroll
                    for (int l = 0; l < d; ++l) {
                        a.hist[((int64_t)j * D + l) * B + b] = Lq[j][l];
                        a.hist[((int64_t)j * D + d + l) * B + b] = Lv[j][l];
                    }
                if (!finite) bad = n0 + n;
                break;
            }
        }
        // a4 (second half) / next step's a1: V_i = v + D(W_i., Lv), W = fin ? nu : mu
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int l = 0; l < d; ++l) {
                double acc = dmul(fin ? a.T.nu[i][0] : a.T.mu[i][0], Lv[0][l]);
#pragma unroll
                for (int j = 1; j < 8; ++j) acc = dfma(fin ? a.T.nu[i][j] : a.T.mu[i][j], Lv[j][l], acc);
                V[i][l] = dadd(v[l], acc);
            }
    }
#pragma unroll
    for (int l = 0; l < d; ++l) {
        a.y[l * B + b] = q[l];
        a.y[(d + l) * B + b] = v[l];
    }
    a.stats[0 * B + b] += hits;
    a.stats[1 * B + b] = bad;
    a.stats[2 * B + b] += sweeps;
    if (a.iters) a.iters[b] = sweeps;
}

}  // namespace irk
