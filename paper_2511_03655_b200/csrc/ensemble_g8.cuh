// Ensemble kernel, mapping "g8" (stage-per-lane): one group of 8 lanes per
// trajectory, lane s of a group owns stage s (4 trajectories per warp).  The
// north star's alternative to one trajectory per thread (the paper's own SIMD
// mapping puts the 8 stages in the 8 lanes of an AVX-512 register):
//
//   a2  Lq_s = hb_s V_s; the group all-gathers Lq_0..7 by warp shuffles and lane s
//       forms its row Q_s = q + D(mu_s., Lq)                    Eq. IRK_FP2 l.1-2
//   a5  Delta_l = max_s |Q_s - Q_s^old|: a 3-step xor-shuffle max over the group
//       (on the int64 bit patterns, NaN dropped), stop test replicated in the
//       8 lanes                                                  Eq. stopping
//   a3  F_s = g(Q_s, t + c_s h): ONE right-hand side per lane       Eq. IRK_FP2 l.3
//   a4  Lv_s = hb_s F_s, all-gathered; V_s = v + D(W_s., Lv), W = nu on the sweep
//       that finishes a step (next step's nu-init), else mu      Eq. IRK_FP2 l.4-5
//   a6  q += S(Lq), v += S(Lv) from the gathered stages (every lane keeps the
//       replicated q, v), history row s <- Lv_s                   Eq. yn3
//
// The coefficient rows mu_s., nu_s. are read from shared memory.  Every lane
// executes the canonical operation sequence of its stage, so results are
// bitwise those of the oracle and of the g1 mapping.  Trade-off (DESIGN.md
// "Mappings"): 8x the lanes per trajectory (latency hiding at small batch) for
// 2 x 8d shuffled doubles per sweep and the replicated update; g1 wins when the
// batch fills the GPU, g8 when it does not (IRK_OPT_MAPPING auto).
#pragma once
#include <cstdint>

#include "ens_common.cuh"
#include "fp64.cuh"

namespace irk {

constexpr int G8_THREADS = 64;  // 8 trajectories per block

#ifndef G8_SMEM
#define G8_SMEM 1  // all-gathers through a shared-memory tile (0: shuffles; 2,000 steps at B = 512: 3.65 vs 4.65 ms)
#endif
#ifndef GS_UNIFORM_EXACT
#define GS_UNIFORM_EXACT 1  // exact-RHS re-evaluation as a warp-uniform branch (g4 at 8,192: 23.2 -> 22.5 ms)
#endif
#ifndef G8_MAXREG
#define G8_MAXREG 168  // g8 uses 119 (B = 2048: 80 regs 5.8 ms, 96: 5.2, 119: 3.7); g4 / g2 use 124 / 156 (at 128 g2 spilled: 7.35 vs 6.88 ms at 8,192)
#endif

// G lanes per trajectory (G = 8: "g8", one stage per lane; G = 4: "g4", two
// stages per lane -- half the lanes and half the replicated work per trajectory,
// for batches too large for g8 and too small for g1).  Lane s of a group owns
// stages s*SPL .. s*SPL + SPL - 1.
template <class P, int G>
__global__ void __maxnreg__(G8_MAXREG) ens_gs_kernel(const __grid_constant__ EnsArgs a,
                                                     const __grid_constant__ P prob) {
    static_assert(G == 8 || G == 4 || G == 2, "G lanes per trajectory: 8, 4 or 2");
    constexpr int d = P::d, D = 2 * d, SPL = 8 / G, GPB = G8_THREADS / G;
    const unsigned FULL = 0xffffffffu;
    const int64_t B = a.batch;
    const int lane = threadIdx.x & 31, s = lane & (G - 1), base = lane & ~(G - 1);
    const int64_t b = ((int64_t)blockIdx.x * G8_THREADS + threadIdx.x) / G;  // trajectory of the group
    const bool valid = b < B;
    const int64_t bb = valid ? b : 0;

    // Lane-dependent coefficients from shared memory, column-major [j][i] so that
    // the lanes of a group read consecutive doubles (all groups of the warp the
    // same ones); nu~ offset by 72 doubles to sit in other banks than mu~.
    // (Kept in registers they were rematerialised from the constant bank with
    // lane-divergent addresses: serialised LDC, ncu mio_throttle.)
    __shared__ double sW[72 + 64], sHB[8], sC[8];
    // per-group all-gather tile [stage][component], groups padded into different banks
    // (G8_SMEM = 0: shuffles instead, one stage per lane only)
    constexpr bool SMEM = G8_SMEM || G != 8;
    __shared__ __align__(16) double sG[GPB][SMEM ? 8 * d + 2 : 2];
    const int gib = threadIdx.x / G;
    for (int e = threadIdx.x; e < 64; e += blockDim.x) {
        sW[(e & 7) * 8 + (e >> 3)] = (&c_mu[0][0])[e];       // mu~[i][j] at [j][i]
        sW[72 + (e & 7) * 8 + (e >> 3)] = (&c_nu[0][0])[e];
    }
    if (threadIdx.x < 8) {
        sHB[threadIdx.x] = a.hb[threadIdx.x];
        sC[threadIdx.x] = c_c[threadIdx.x];
    }
    __syncthreads();
    const int st0 = s * SPL;                           // first owned stage
    const double *Mu = sW + st0, *Nu = sW + 72 + st0;  // coefficient (st0 + t, j) at [8 j + t]
    // g8 keeps its lane's coefficient rows mu~_s., nu~_s. and hb_s in registers (16 + 1
    // doubles): 18 fewer shared loads per sweep on the single-trajectory critical
    // path.  The values pass through an empty asm so that the compiler cannot
    // re-load them from shared memory inside the loop.
    constexpr bool CREG = (G == 8);
    double rMu[8], rNu[8], rHB[SPL];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        rMu[j] = CREG ? Mu[8 * j] : 0.0;
        rNu[j] = CREG ? Nu[8 * j] : 0.0;
        asm("" : "+d"(rMu[j]), "+d"(rNu[j]));
    }
#pragma unroll
    for (int t = 0; t < SPL; ++t) {
        rHB[t] = sHB[st0 + t];
        asm("" : "+d"(rHB[t]));
    }
    auto MU = [&](int j, int t) -> double { return CREG ? rMu[j] : Mu[8 * j + t]; };

    double q[d], v[d];
#pragma unroll
    for (int l = 0; l < d; ++l) {
        q[l] = a.y[l * B + bb];
        v[l] = a.y[(d + l) * B + bb];
    }
    int64_t bad = a.stats[1 * B + bb];
    const int64_t n0 = *a.n_done;
    const bool sample = (a.energy != nullptr) && (a.energy_every > 0);
    double hprev = 0.0, dhmax = 0.0;
    if (valid && s == 0) {
        if (sample && a.c0 == 0) a.energy[b] = prob.energy(q, v);
        if (a.local_energy) hprev = prob.energy(q, v);
    }
    bool live = valid && bad == 0 && a.nsteps > 0;
    if (valid && !live && s == 0) {
        if (a.iters && a.c0 == 0) a.iters[b] = 0;
        if (a.csweeps) a.csweeps[b] = 0;
        if (a.local_energy && a.c0 == 0) a.stats[3 * B + b] = 0;
    }

    // a1: V_i = v + D(nu_i., H) for the owned stages, H = the history rows of all 8 stages
    double Vs[SPL][d];
    {
        double Hs[SPL][d];
#pragma unroll
        for (int t = 0; t < SPL; ++t)
#pragma unroll
            for (int l = 0; l < d; ++l) Hs[t][l] = live ? a.hist[((int64_t)(st0 + t) * D + d + l) * B + b] : 0.0;
#pragma unroll
        for (int l = 0; l < d; ++l) {
            double H[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) H[j] = __shfl_sync(FULL, Hs[j % SPL][l], base + j / SPL);
#pragma unroll
            for (int t = 0; t < SPL; ++t) {
                double acc = dmul(Nu[t], H[0]);
#pragma unroll
                for (int j = 1; j < 8; ++j) acc = dfma(Nu[8 * j + t], H[j], acc);
                Vs[t][l] = dadd(v[l], acc);
            }
        }
    }
    constexpr int64_t kInfBits = 0x7ff0000000000000LL;
    int64_t m[d], p[d];
    double Qold[SPL][d];
#pragma unroll
    for (int l = 0; l < d; ++l) {
        m[l] = p[l] = kInfBits;
#pragma unroll
        for (int t = 0; t < SPL; ++t) Qold[t][l] = 0.0;
    }
    int64_t n = 0, hits = 0, sweeps = 0;
    int k = 0;
    while (__any_sync(FULL, live)) {  // warp-uniform: every lane takes part in the shuffles
        ++k;
        // ---- a2 + a5 ----
        double sLq[d], Qs[SPL][d];  // S(Lq) is formed on the fly (the gathered Lq die here)
        int64_t delta[d];
        bool stop = (k >= 2);
        double lq[d];
        if constexpr (SMEM) {
#pragma unroll
            for (int t = 0; t < SPL; ++t)
#pragma unroll
                for (int l = 0; l < d; ++l) sG[gib][(st0 + t) * d + l] = dmul(rHB[t], Vs[t][l]);
            __syncwarp();
        } else {
#pragma unroll
            for (int l = 0; l < d; ++l) lq[l] = dmul(rHB[0], Vs[0][l]);
        }
#pragma unroll
        for (int l = 0; l < d; ++l) {
            double g = SMEM ? sG[gib][l] : __shfl_sync(FULL, lq[l], base);
            double acc[SPL];
#pragma unroll
            for (int t = 0; t < SPL; ++t) acc[t] = dmul(MU(0, t), g);
            sLq[l] = g;
#pragma unroll
            for (int j = 1; j < 8; ++j) {
                g = SMEM ? sG[gib][j * d + l] : __shfl_sync(FULL, lq[l], base + j);
#pragma unroll
                for (int t = 0; t < SPL; ++t) acc[t] = dfma(MU(j, t), g, acc[t]);
                sLq[l] = dadd(sLq[l], g);
            }
            int64_t e = 0;
#pragma unroll
            for (int t = 0; t < SPL; ++t) {
                Qs[t][l] = dadd(q[l], acc[t]);
                int64_t et = dabs_bits(dsub(Qs[t][l], Qold[t][l]));
                et = (et > kInfBits) ? 0 : et;  // NaN-ignoring max (canonical left-to-right form)
                e = (et > e) ? et : e;
                Qold[t][l] = Qs[t][l];
            }
#pragma unroll
            for (int off = 1; off < G; off <<= 1) {
                const int64_t o = __shfl_xor_sync(FULL, e, off);
                e = (o > e) ? o : e;
            }
            delta[l] = e;
        }
        // ---- a3: SPL right-hand sides per lane ----
        const double tn1 = dadd(a.t0, dmul((double)(n0 + n), a.h));
        double Fs[SPL][d];
        {
            bool ok = true;
#pragma unroll
            for (int t = 0; t < SPL; ++t)
                prob.template accel<false>(Qs[t], Fs[t], dadd(tn1, dmul(sC[st0 + t], a.h)), ok);
#if GS_UNIFORM_EXACT
            if (__any_sync(FULL, !ok && live))  // exact slow path, same bits (warp-uniform)
#else
            if (!ok && live)  // exact slow path, same bits (live groups only)
#endif
#pragma unroll
                for (int t = 0; t < SPL; ++t)
                    prob.template accel<true>(Qs[t], Fs[t], dadd(tn1, dmul(sC[st0 + t], a.h)), ok);
        }
        // ---- a4 (first half): Lv, all-gather ----
        double Lvg[8][d], Lvs[SPL][d];
        if constexpr (SMEM) {
            __syncwarp();  // the Lq reads of this sweep are done
#pragma unroll
            for (int t = 0; t < SPL; ++t)
#pragma unroll
                for (int l = 0; l < d; ++l) sG[gib][(st0 + t) * d + l] = Lvs[t][l] = dmul(rHB[t], Fs[t][l]);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j)
#pragma unroll
                for (int l = 0; l < d; ++l) Lvg[j][l] = sG[gib][j * d + l];
            __syncwarp();  // before the next sweep's writes
        } else {
#pragma unroll
            for (int l = 0; l < d; ++l) {
                Lvs[0][l] = dmul(rHB[0], Fs[0][l]);
#pragma unroll
                for (int j = 0; j < 8; ++j) Lvg[j][l] = __shfl_sync(FULL, Lvs[0][l], base + j);
            }
        }
        // the stop test after the right-hand sides: the RHS does not need it, so the
        // Delta shuffles and the RHS chains share one basic block and overlap
        {   // reading R2, on the bit patterns as in ens_g1q; branch-free so
            // that groups at k = 1 and k >= 2 do not diverge
            const bool k2 = k >= 2;
#pragma unroll
            for (int l = 0; l < d; ++l) {
                const int64_t e = delta[l];
                const int64_t mn = (e < p[l]) ? e : p[l];
                const bool ok = (e == 0) || (m[l] <= mn);
                m[l] = k2 ? ((p[l] < m[l]) ? p[l] : m[l]) : m[l];
                p[l] = k2 ? e : p[l];
                stop = stop && ok;  // (stop starts as k >= 2)
            }
        }
        const bool fin = live && (stop || k >= a.max_iters);
        // ---- a4 (second half) / next step's a1, contraction part: D(W_i., Lv), W = nu
        // when the step finishes.  Formed before the update so that its chain runs
        // beside the S(Lv) chain of a6 (only the final v + D depends on the update).
        double accV[SPL][d];
        {
            const double *W = fin ? Nu : Mu;
            double rW[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) rW[j] = fin ? rNu[j] : rMu[j];
#pragma unroll
            for (int l = 0; l < d; ++l)
#pragma unroll
                for (int t = 0; t < SPL; ++t) {
                    double acc = dmul(CREG ? rW[0] : W[t], Lvg[0][l]);
#pragma unroll
                    for (int j = 1; j < 8; ++j) acc = dfma(CREG ? rW[j] : W[8 * j + t], Lvg[j][l], acc);
                    accV[t][l] = acc;
                }
        }
        // S(Lv) of a6, formed every sweep beside the chain above (off the update's path)
        double sv[d];
#pragma unroll
        for (int l = 0; l < d; ++l) {
            sv[l] = Lvg[0][l];
#pragma unroll
            for (int j = 1; j < 8; ++j) sv[l] = dadd(sv[l], Lvg[j][l]);
        }
        if (fin) {  // ---- a6: update (replicated in the group), history, samples ----
            bool finite = true;
#pragma unroll
            for (int l = 0; l < d; ++l) {
                q[l] = dadd(q[l], sLq[l]);
                v[l] = dadd(v[l], sv[l]);
                finite = finite && isfinite(q[l]) && isfinite(v[l]);
            }
            ++n;
            sweeps += k;
            hits += stop ? 0 : 1;
            k = 0;
#pragma unroll
            for (int l = 0; l < d; ++l) m[l] = p[l] = kInfBits;
            if ((sample || a.local_energy) && s == 0) {  // (sample test first: no divergent branch per step)
                if (sample && ((a.c0 + n) % a.energy_every) == 0)
                    a.energy[((a.c0 + n) / a.energy_every) * B + b] = prob.energy(q, v);
                if (a.local_energy) dhloc_update(prob.energy(q, v), hprev, dhmax);
            }
            if (n == a.nsteps || !finite) {  // leave: history rows = Lv of the owned stages, q block zeroed (R-4)
#pragma unroll
                for (int t = 0; t < SPL; ++t)
#pragma unroll
                    for (int l = 0; l < d; ++l) {
                        a.hist[((int64_t)(st0 + t) * D + l) * B + b] = 0.0;
                        a.hist[((int64_t)(st0 + t) * D + d + l) * B + b] = Lvs[t][l];
                    }
                if (!finite) bad = n0 + n;
                live = false;
            }
        }
        // ---- a4 (second half) / next step's a1: V_i = v + D(W_i., Lv) ----
#pragma unroll
        for (int l = 0; l < d; ++l)
#pragma unroll
            for (int t = 0; t < SPL; ++t) Vs[t][l] = dadd(v[l], accV[t][l]);
    }
    if (valid && s == 0) {
#pragma unroll
        for (int l = 0; l < d; ++l) {
            a.y[l * B + b] = q[l];
            a.y[(d + l) * B + b] = v[l];
        }
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
