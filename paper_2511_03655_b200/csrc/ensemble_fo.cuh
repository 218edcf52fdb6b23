// First-order mode (Eqs. IRK_init / IRK_FP) as a sweep-granular
// persistent work-queue kernel, one trajectory per thread: the paper's
// first-order test problem (the Schwarzschild black hole, Eq. Ham_SBH, not
// separable) and the second-order problems run with IRK_OPT_MODE = 1.
//
//   init   Y_i = y + D(nu_i., L_{n-1})           all D components   Eq. IRK_init
//   sweep  F_i = f(Y_i, t_{n-1} + c_i h); L_j = hb_j F_j              Eq. IRK_FP
//          Yn_i = y + D(mu_i., L); Delta_l = max_i |Yn_i - Y_i| over all D
//          components, stop test from k = 1 (Delta^[1] exists here)  Eq. stopping
//   update y += S(L), history <- L (all of it, R-4)          Eq. yn3
//
// Sweep-granular as ens_g1q: a lane whose step converged updates and overwrites
// its (discarded) Yn with the next step's nu-init in the same trip, so lanes with
// different sweep counts stay busy.  Y^[k] lives in shared memory
// [element][thread] (read by the RHS, compared and overwritten by the
// contraction); L in registers.  Division / square root use the branch-free
// bitwise fast paths with an exact re-evaluation of the sweep's RHS when any
// operand leaves the fast range.  Same arithmetic per step as the oracle's
// step_first_order, so bitwise for any schedule.
#pragma once
#include <cstdint>

#include "ens_common.cuh"
#include "ensemble_g1.cuh"
#include "fp64.cuh"

namespace irk {

constexpr int FO_THREADS = 64;
#ifndef FO8_MAXREG
#define FO8_MAXREG 168  // ens_fo8: 162 registers, no spills (Schwarzschild, 1,000 steps, B = 1 / 4,096 / 65,536: 2.13 / 3.30 / 38.5 ms; at 128: spills, 2.8 / 3.87 / 39.4)
#endif
#ifndef FO_MAXREG
#define FO_MAXREG 168
#endif

// f(Y_i): Hamilton's equations of a first-order problem, or (v, g(q, t)).
template <class P, bool EXACT>
__device__ __forceinline__ void fo_rhs(const P &prob, const double *Y, double *F, double t, bool &ok) {
    constexpr int d = P::d;
    if constexpr (P::first_order) {
        prob.template rhs<EXACT>(Y, F, t, ok);
    } else {
#pragma unroll
        for (int l = 0; l < d; ++l) F[l] = Y[d + l];
        prob.template accel<EXACT>(Y, F + d, t, ok);
    }
}

template <class P>
__global__ void __maxnreg__(FO_MAXREG) ens_fo_q_kernel(const __grid_constant__ EnsArgs a,
                                                      const __grid_constant__ QueueArgs qa,
                                                      const __grid_constant__ P prob) {
    constexpr int d = P::d, D = 2 * d;
    const int64_t B = a.batch;
    constexpr int kNuOff = 66;  // mu~ at [0, 64), nu~ at [66, 130): different banks
    __shared__ __align__(16) double sW[kNuOff + 64];
    for (int e = threadIdx.x; e < 128; e += blockDim.x)
        sW[(e < 64) ? e : kNuOff + e - 64] = (e < 64) ? (&c_mu[0][0])[e] : (&c_nu[0][0])[e - 64];
    __syncthreads();
    __shared__ double sY[8 * D][FO_THREADS];
    __shared__ int64_t sM[D][FO_THREADS], sP[D][FO_THREADS];
    const int tx = threadIdx.x;
    const int64_t n0 = *a.n_done;
    const bool sample = (a.energy != nullptr) && (a.energy_every > 0);
    const int64_t total = B * qa.nchunks;

    double y[D];
    int32_t b = -1, bb = 0;
    int64_t c = 0, len = 0, n = 0, hits = 0, sweeps = 0, u = -1;
    double hprev = 0.0, dhmax = 0.0;
    int k = 0;
    for (;;) {
        if (b < 0) {  // ---- acquire the next unit (see ens_g1q) ----
            if (u < 0) {
                u = (int64_t)atomicAdd(qa.counter, 1ull);
                if (u >= total) break;
                c = u / B;
                bb = (int32_t)(u - c * B);
            }
            if (c > 0 && ld_acquire(&qa.progress[bb]) < c) {
                __nanosleep(1024);
                continue;
            }
            u = -1;
            b = bb;
            const int64_t c0 = c * qa.qchunk;
            len = (a.nsteps - c0 < qa.qchunk) ? a.nsteps - c0 : qa.qchunk;
#pragma unroll
            for (int l = 0; l < D; ++l) y[l] = __ldcg(&a.y[l * B + b]);
            if (sample && c == 0) a.energy[b] = prob.energy(y, y + d);
            hprev = a.local_energy ? prob.energy(y, y + d) : 0.0;
            dhmax = 0.0;
            if (__ldcg(&a.stats[1 * B + b]) > 0 || len <= 0) {  // frozen or nothing to do
                if (c == 0) {
                    if (a.local_energy) a.stats[3 * B + b] = 0;
                    if (a.iters) a.iters[b] = 0;
                }
                st_release(&qa.progress[b], (int32_t)(c + 1));
                b = -1;
                continue;
            }
            {   // Y_i^[0] = y + D(nu_i., L_{n-1}) over all D components (zeros: first step)
                double H[8][D];
#pragma unroll
                for (int j = 0; j < 8; ++j)
#pragma unroll
                    for (int l = 0; l < D; ++l) H[j][l] = __ldcg(&a.hist[((int64_t)j * D + l) * B + b]);
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int l = 0; l < D; ++l) {
                        double acc = dmul(c_nu[i][0], H[0][l]);
#pragma unroll
                        for (int j = 1; j < 8; ++j) acc = dfma(c_nu[i][j], H[j][l], acc);
                        sY[i * D + l][tx] = dadd(y[l], acc);
                    }
            }
#pragma unroll
            for (int l = 0; l < D; ++l) sM[l][tx] = sP[l][tx] = kInfBits;
            n = hits = sweeps = 0;
            k = 0;
        }
        ++k;
        // F_i = f(Y_i^[k-1], t_i) ; L_j = hb_j F_j (all eight stages in flight)
        const int64_t nabs = n0 + c * qa.qchunk + n;
        const double tn1 = dadd(a.t0, dmul((double)nabs, a.h));
        double L[8][D];
        {
            bool ok = true;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double Yi[D];
#pragma unroll
                for (int l = 0; l < D; ++l) Yi[l] = sY[i * D + l][tx];
                fo_rhs<P, false>(prob, Yi, L[i], dadd(tn1, dmul(c_c[i], a.h)), ok);
            }
            if (!ok) {  // some operand outside the fast-path range: exact intrinsics, same bits
                double Fx[8][D];  // rare path: a local-memory array, copied back with static indices
#pragma unroll 1
                for (int i = 0; i < 8; ++i) {
                    double Yi[D];
#pragma unroll
                    for (int l = 0; l < D; ++l) Yi[l] = sY[i * D + l][tx];
                    fo_rhs<P, true>(prob, Yi, Fx[i], dadd(tn1, dmul(c_c[i], a.h)), ok);
                }
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int l = 0; l < D; ++l) L[i][l] = Fx[i][l];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int l = 0; l < D; ++l) L[i][l] = dmul(a.hb[i], L[i][l]);
        }
        // Yn_i = y + D(mu_i., L) ; Delta vs Y^[k-1] ; Y <- Yn
        bool stop = true;
        {
            const double2 *M = reinterpret_cast<const double2 *>(&c_mu[0][0]);
#pragma unroll
            for (int l = 0; l < D; ++l) {
                int64_t ev[8];
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    double acc = dmul(M[i * 4].x, L[0][l]);
                    acc = dfma(M[i * 4].y, L[1][l], acc);
#pragma unroll
                    for (int jj = 1; jj < 4; ++jj) {
                        acc = dfma(M[i * 4 + jj].x, L[2 * jj][l], acc);
                        acc = dfma(M[i * 4 + jj].y, L[2 * jj + 1][l], acc);
                    }
                    const double yn = dadd(y[l], acc);
                    ev[i] = absdiff_bits(yn, sY[i * D + l][tx]);
                    sY[i * D + l][tx] = yn;
                }
                const int64_t delta = delta_bits8(ev);  // stop test from k = 1 (Delta^[1] exists)
                const int64_t pl = sP[l][tx], ml = sM[l][tx];
                const bool okc = (delta == 0) || (ml <= imin64(delta, pl));
                sM[l][tx] = imin64(pl, ml);
                sP[l][tx] = delta;
                stop = stop && okc;
            }
        }
        if (!(stop || k >= a.max_iters)) continue;
        // ---- step finished: update with this sweep's L, history, samples ----
        bool finite = true;
#pragma unroll
        for (int l = 0; l < D; ++l) {
            double s = L[0][l];
#pragma unroll
            for (int j = 1; j < 8; ++j) s = dadd(s, L[j][l]);
            y[l] = dadd(y[l], s);
            finite = finite && isfinite(y[l]);
        }
        ++n;
        sweeps += k;
        hits += stop ? 0 : 1;
        k = 0;
#pragma unroll
        for (int l = 0; l < D; ++l) sM[l][tx] = sP[l][tx] = kInfBits;
        const int64_t nloc = c * qa.qchunk + n;
        if (sample && (nloc % a.energy_every) == 0) a.energy[(nloc / a.energy_every) * B + b] = prob.energy(y, y + d);
        if (a.local_energy) dhloc_update(prob.energy(y, y + d), hprev, dhmax);
        if (n == len || !finite) {  // ---- release the unit ----
#pragma unroll
            for (int j = 0; j < 8; ++j)
#pragma unroll
                for (int l = 0; l < D; ++l) a.hist[((int64_t)j * D + l) * B + b] = L[j][l];
#pragma unroll
            for (int l = 0; l < D; ++l) a.y[l * B + b] = y[l];
            a.stats[0 * B + b] = __ldcg(&a.stats[0 * B + b]) + hits;
            if (!finite) a.stats[1 * B + b] = n0 + nloc;
            a.stats[2 * B + b] = __ldcg(&a.stats[2 * B + b]) + sweeps;
            if (a.iters) a.iters[b] = (c == 0) ? sweeps : __ldcg(&a.iters[b]) + sweeps;
            if (a.local_energy) dhloc_store(&a.stats[3 * B + b], c == 0, dhmax);
            st_release(&qa.progress[b], (int32_t)(c + 1));
            b = -1;
            continue;
        }
        // next step's init: Y_i = y + D(nu_i., L) (overwrites the discarded Yn)
        {
            const double2 *W = reinterpret_cast<const double2 *>(&sW[kNuOff]);
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int l = 0; l < D; ++l) {
                    double acc = dmul(W[i * 4].x, L[0][l]);
                    acc = dfma(W[i * 4].y, L[1][l], acc);
#pragma unroll
                    for (int jj = 1; jj < 4; ++jj) {
                        acc = dfma(W[i * 4 + jj].x, L[2 * jj][l], acc);
                        acc = dfma(W[i * 4 + jj].y, L[2 * jj + 1][l], acc);
                    }
                    sY[i * D + l][tx] = dadd(y[l], acc);
                }
        }
    }
}

}  // namespace irk

namespace irk {

// First-order mode, stage per lane ("g8", small batches and single trajectories,
// e.g. the paper's one-orbit Schwarzschild runs): a group of 8 lanes per
// trajectory, lane s owns stage s -- Y_s (all D components) and its right-hand
// side f(Y_s); L is all-gathered through a per-group shared-memory tile, every
// lane forms Yn_s = y + D(mu_s., L), Delta_l = max over the 8 stages by an
// xor-shuffle max, the stop test and y are replicated in the group.  On a
// finished step the lane overwrites its discarded Yn_s with the next step's
// nu-init.  Same canonical sequence as the oracle's step_first_order.
constexpr int FO8_THREADS = 64;

template <class P>
__global__ void __maxnreg__(FO8_MAXREG) ens_fo8_kernel(const __grid_constant__ EnsArgs a, const __grid_constant__ P prob) {
    constexpr int d = P::d, D = 2 * d;
    const unsigned FULL = 0xffffffffu;
    const int64_t B = a.batch;
    const int lane = threadIdx.x & 31, s = lane & 7, gib = threadIdx.x >> 3;
    const int64_t b = ((int64_t)blockIdx.x * FO8_THREADS + threadIdx.x) >> 3;
    const bool valid = b < B;
    const int64_t bb = valid ? b : 0;
    __shared__ double sW[72 + 64], sHB[8], sC[8];
    __shared__ __align__(16) double sG[FO8_THREADS / 8][8 * D + 2];  // L rows, groups in different banks
    for (int e = threadIdx.x; e < 64; e += blockDim.x) {
        sW[(e & 7) * 8 + (e >> 3)] = (&c_mu[0][0])[e];
        sW[72 + (e & 7) * 8 + (e >> 3)] = (&c_nu[0][0])[e];
    }
    if (threadIdx.x < 8) {
        sHB[threadIdx.x] = a.hb[threadIdx.x];
        sC[threadIdx.x] = c_c[threadIdx.x];
    }
    __syncthreads();
    const double *Mu = sW + s, *Nu = sW + 72 + s;
    double *G = sG[gib];

    double y[D];
#pragma unroll
    for (int l = 0; l < D; ++l) y[l] = a.y[l * B + bb];
    int64_t bad = a.stats[1 * B + bb];
    const int64_t n0 = *a.n_done;
    const bool sample = (a.energy != nullptr) && (a.energy_every > 0);
    double hprev = 0.0, dhmax = 0.0;
    if (valid && s == 0) {
        if (sample && a.c0 == 0) a.energy[b] = prob.energy(y, y + d);
        if (a.local_energy) hprev = prob.energy(y, y + d);
    }
    bool live = valid && bad == 0 && a.nsteps > 0;
    if (valid && !live && s == 0) {
        if (a.iters && a.c0 == 0) a.iters[b] = 0;
        if (a.csweeps) a.csweeps[b] = 0;
        if (a.local_energy && a.c0 == 0) a.stats[3 * B + b] = 0;
    }
    // Y_s^[0] = y + D(nu_s., L_{n-1}) over all D components (history row s -> tile)
    double Ys[D];
#pragma unroll
    for (int l = 0; l < D; ++l) G[s * D + l] = live ? a.hist[((int64_t)s * D + l) * B + b] : 0.0;
    __syncwarp();
#pragma unroll
    for (int l = 0; l < D; ++l) {
        double acc = dmul(Nu[0], G[l]);
#pragma unroll
        for (int j = 1; j < 8; ++j) acc = dfma(Nu[8 * j], G[j * D + l], acc);
        Ys[l] = dadd(y[l], acc);
    }
    __syncwarp();
    constexpr int64_t kInf = 0x7ff0000000000000LL;
    int64_t m[D], p[D];
#pragma unroll
    for (int l = 0; l < D; ++l) m[l] = p[l] = kInf;
    int64_t n = 0, hits = 0, sweeps = 0;
    int k = 0;
    while (__any_sync(FULL, live)) {  // warp-uniform: the group tiles and votes need every lane
        ++k;
        // F_s = f(Y_s, t_s) ; L_s = hb_s F_s -> tile row s
        const double tn1 = dadd(a.t0, dmul((double)(n0 + n), a.h));
        const double ts = dadd(tn1, dmul(sC[s], a.h));
        double Ls[D];
        {
            bool ok = true;
            fo_rhs<P, false>(prob, Ys, Ls, ts, ok);
            if (!ok && live) fo_rhs<P, true>(prob, Ys, Ls, ts, ok);  // exact intrinsics, same bits (live groups)
        }
#pragma unroll
        for (int l = 0; l < D; ++l) G[s * D + l] = Ls[l] = dmul(sHB[s], Ls[l]);
        __syncwarp();
        // Yn_s = y + D(mu_s., L) ; Delta over the group ; stop test (from k = 1)
        bool stop = true;
        double Yn[D];
#pragma unroll
        for (int l = 0; l < D; ++l) {
            double acc = dmul(Mu[0], G[l]);
#pragma unroll
            for (int j = 1; j < 8; ++j) acc = dfma(Mu[8 * j], G[j * D + l], acc);
            Yn[l] = dadd(y[l], acc);
            int64_t e = dabs_bits(dsub(Yn[l], Ys[l]));
            e = (e > kInf) ? 0 : e;  // NaN-ignoring max
#pragma unroll
            for (int off = 1; off < 8; off <<= 1) {
                const int64_t o = __shfl_xor_sync(FULL, e, off);
                e = (o > e) ? o : e;
            }
            const bool okc = (e == 0) || (m[l] <= ((e < p[l]) ? e : p[l]));
            m[l] = (p[l] < m[l]) ? p[l] : m[l];
            p[l] = e;
            stop = stop && okc;
        }
        const bool fin = live && (stop || k >= a.max_iters);
        if (fin) {  // update with this sweep's L (replicated), samples, history row s
            bool finite = true;
#pragma unroll
            for (int l = 0; l < D; ++l) {
                double sl = G[l];
#pragma unroll
                for (int j = 1; j < 8; ++j) sl = dadd(sl, G[j * D + l]);
                y[l] = dadd(y[l], sl);
                finite = finite && isfinite(y[l]);
            }
            ++n;
            sweeps += k;
            hits += stop ? 0 : 1;
            k = 0;
#pragma unroll
            for (int l = 0; l < D; ++l) m[l] = p[l] = kInf;
            if ((sample || a.local_energy) && s == 0) {  // (sample test first: no divergent branch per step)
                if (sample && ((a.c0 + n) % a.energy_every) == 0)
                    a.energy[((a.c0 + n) / a.energy_every) * B + b] = prob.energy(y, y + d);
                if (a.local_energy) dhloc_update(prob.energy(y, y + d), hprev, dhmax);
            }
            if (n == a.nsteps || !finite) {
#pragma unroll
                for (int l = 0; l < D; ++l) a.hist[((int64_t)s * D + l) * B + b] = Ls[l];
                if (!finite) bad = n0 + n;
                live = false;
            }
            // next step's init: Y_s = y + D(nu_s., L)
#pragma unroll
            for (int l = 0; l < D; ++l) {
                double acc = dmul(Nu[0], G[l]);
#pragma unroll
                for (int j = 1; j < 8; ++j) acc = dfma(Nu[8 * j], G[j * D + l], acc);
                Yn[l] = dadd(y[l], acc);
            }
        }
#pragma unroll
        for (int l = 0; l < D; ++l) Ys[l] = Yn[l];
        __syncwarp();  // tile reads done before the next sweep's writes
    }
    if (valid && s == 0) {
#pragma unroll
        for (int l = 0; l < D; ++l) a.y[l * B + b] = y[l];
        if (a.nsteps > 0 && a.stats[1 * B + b] == 0) {
            a.stats[0 * B + b] += hits;
            a.stats[1 * B + b] = bad;
            a.stats[2 * B + b] += sweeps;
            if (a.iters) a.iters[b] = (a.c0 == 0) ? sweeps : a.iters[b] + sweeps;
            if (a.csweeps) a.csweeps[b] = (int32_t)sweeps;
            if (a.local_energy) dhloc_store(&a.stats[3 * B + b], a.c0 == 0, dhmax);
        }
    }
}

}  // namespace irk
