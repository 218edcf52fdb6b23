// Ensemble kernel, mapping "g8m" (IRK_MAP_G8M for Kepler / Henon-Heiles):
// stage per lane with both stage contractions of a sweep on the FP64 tensor core.
// The small-batch / single-trajectory path (config 1), where a sweep is one
// serial chain and its length is the whole cost.
//
// A warp holds a slot of 4 trajectories; lane L = 4 s + g owns stage s of
// trajectory g (the layout of ens_nbody8m, ensemble_nbody8m.cuh, whose comment
// derives the fragment algebra).  Per half-sweep the 8 x 8 stage contraction
// D[s][(g, l)] = sum_j W[s][j] X_j[(g, l)] (X = Lq or Lv) is tile t = components
// 2t, 2t+1 of the 4 trajectories; two chained mma.m8n8k4.f64 (k halves j = 0..3,
// 4..7; C = -0 for the first, which reproduces the leading dmul including signed
// zeros) are the canonical fma chain over j bit for bit (profiles/r1/
// dmma_probe.txt), and D lands in the lane that owns (g, s).  The B fragments
// come from the owners by two shuffles per tile (no shared memory, no
// __syncwarp round trip): the critical path of a half-sweep is DMUL -> 2 SHFL ->
// 2 DMMA -> DADD instead of DMUL -> STS -> LDS -> 8 DFMA -> DADD (ens_gs<8>).
//
//   a2  Q_s = q + D(mu~, Lq)                                    Eq. IRK_FP2 l.1-2
//   a5  reading R2 from two ballots per component over the trajectory's 8 stage
//       lanes (Delta == 0, some stage difference >= m); the exact Delta_l =
//       max_s |Q_s,l - Q_s,l^old| for the next sweep's (m, p) by xor-shuffles
//       4, 8, 16 off the critical path (int64 bit patterns, NaN dropped)  Eq. stopping
//   a3  F_s = g(Q_s, t + c_s h): one right-hand side per lane    Eq. IRK_FP2 l.3
//   a4  V_s = v + D(W, Lv), W = nu~ on the sweep that ends a step (next step's
//       nu-init), mu~ otherwise; the W fragment is shared by the slot, so a slot
//       whose live trajectories disagree runs a second (nu~) pass  Eq. IRK_FP2 l.4-5
//   a6  q += S(Lq), v += S(Lv): S = the dadd chain over stages 0..7 (oracle
//       update order) as a ones x X DMMA pair -- fma(1, x0, -0) = x0, then
//       fma(1, x_j, acc) = RN(acc + x_j) -- on sweeps where a trajectory of the
//       slot finishes its step; history row s <- Lv_s              Eq. yn3
//
// One launch for the whole call (every trajectory integrates all nsteps); same
// canonical operation sequence as the oracle and the other mappings: bitwise.
#pragma once
#include <cstdint>

#include "ens_common.cuh"
#include "ensemble_g1.cuh"
#include "ensemble_nbody8m.cuh"
#include "fp64.cuh"

namespace irk {

constexpr int G8M_THREADS = 64;  // two slots (8 trajectories) per block
#ifndef G8M_SKIPK1
#define G8M_SKIPK1 0  // 1: skip the stop-test work on sweeps where no trajectory tests (config 1 16.5 vs 11.9 ms)
#endif
#ifndef G8M_SHADOW
#define G8M_SHADOW 1
#endif
#ifndef G8M_UNIFORM_EXACT
#define G8M_UNIFORM_EXACT 1  // exact-RHS re-evaluation as a warp-uniform branch (config 1 12.35 -> 12.24 ms)
#endif
#ifndef G8M_MAXREG
#define G8M_MAXREG 128
#endif

// B fragments of tile t (both k halves) from the owners' pair (x0, x1) =
// components (2t, 2t+1) of X_s for trajectory g.  Destination L needs X_j, j =
// 4 kk + L % 4, of trajectory L / 8, component e = (L / 4) % 2, held by lane
// 4 j + L / 8.  Shuffle A reads stage L % 4 + 4 e, whose owner offers component
// (s < 4 ? 0 : 1); shuffle B reads stage L % 4 + 4 (1 - e), offering the other
// one: destination e = 0 finds its k-half-0 value in A and k-half-1 value in B,
// e = 1 the reverse.
struct G8MFrag {
    int srcA, srcB;
    bool lo, e1;  // owner stage < 4; destination column parity
    __device__ __forceinline__ G8MFrag(int L) {
        const int s = L >> 2, e = (L >> 2) & 1, kq = L & 3, gp = L >> 3;
        srcA = 4 * (kq + 4 * e) + gp;
        srcB = 4 * (kq + 4 * (1 - e)) + gp;
        lo = s < 4;
        e1 = e != 0;
    }
    __device__ __forceinline__ void get(double x0, double x1, double &b0, double &b1) const {
        const unsigned FULL = 0xffffffffu;
        const double shA = __shfl_sync(FULL, lo ? x0 : x1, srcA);
        const double shB = __shfl_sync(FULL, lo ? x1 : x0, srcB);
        b0 = e1 ? shB : shA;
        b1 = e1 ? shA : shB;
    }
};

// Two launch-time variants (measured, tools/mapping_ab.py, profiles/r2/ab_g8m_variants.json):
//   BALLOT: this sweep's R2 decision from ballots (Delta == 0 <=> no e_s != 0;
//     m <= min(Delta, p) <=> m <= p and some e_s >= m), the exact Delta only feeding
//     the next sweep's (m, p): the stop decision no longer waits for the 3-round
//     xor-shuffle max (one slot, config 1: 13.9 -> 13.1 ms);
//   SPEC: mu~ and nu~ velocity passes every sweep, selected per lane, so the DMMAs
//     do not wait for the slot's stop decision (many slots: 2,048 trajectories
//     14.3 -> 13.0 ms, 6,144: 22.2 -> 20.9 ms).
template <class P, bool BALLOT, bool SPEC>
__global__ void __maxnreg__(G8M_MAXREG) ens_gsm_kernel(const __grid_constant__ EnsArgs a,
                                                      const __grid_constant__ P prob) {
    constexpr int d = P::d, D = 2 * d, T = d / 2;
    static_assert(d % 2 == 0, "g8m: even d (tiles of two components)");
    const unsigned FULL = 0xffffffffu;
    const int64_t B = a.batch;
    const int L = threadIdx.x & 31, s = L >> 2, g = L & 3;
    const unsigned gmask = 0x11111111u << g;  // the 8 stage lanes of trajectory g
    const int64_t b = ((int64_t)blockIdx.x * G8M_THREADS + threadIdx.x) / 32 * 4 + g;  // trajectory of the lane
    const bool valid = b < B;
    // lanes of a ragged slot's missing trajectories shadow the slot's first one (same
    // loads, same control flow, no stores): with one trajectory (config 1) the warp
    // stays converged through the step-end branches (G8M_SHADOW; config 1 -x %)
    const int64_t bslot = b - g;
    const bool shadow = G8M_SHADOW && !valid && bslot < B;
    const int64_t bb = valid ? b : (shadow ? bslot : 0);
    const G8MFrag fr(L);
    // coefficient fragments A[m = s][k = L % 4] of mu~, nu~ for the two k halves
    const double aM0 = c_mu[s][L & 3], aM1 = c_mu[s][4 + (L & 3)];
    const double aN0 = c_nu[s][L & 3], aN1 = c_nu[s][4 + (L & 3)];
    const double hb_s = a.hb[s], cs_h = dmul(c_c[s], a.h);

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
    bool live = (valid || shadow) && bad == 0 && a.nsteps > 0;
    if (valid && !live && s == 0) {
        if (a.iters && a.c0 == 0) a.iters[b] = 0;
        if (a.csweeps) a.csweeps[b] = 0;
        if (a.local_energy && a.c0 == 0) a.stats[3 * B + b] = 0;
    }
    // a1: V_s = v + D(nu~_s., H), H = the history rows (own row s = Lv_s of the last step)
    double V[d];
    {
        double H[d];
#pragma unroll
        for (int l = 0; l < d; ++l) H[l] = live ? a.hist[((int64_t)s * D + d + l) * B + bb] : 0.0;
#pragma unroll
        for (int t = 0; t < T; ++t) {
            double b0, b1, D0, D1;
            fr.get(H[2 * t], H[2 * t + 1], b0, b1);
            dmma884(D0, D1, aN0, b0, -0.0, -0.0);
            dmma884(D0, D1, aN1, b1, D0, D1);
            V[2 * t] = dadd(v[2 * t], D0);
            V[2 * t + 1] = dadd(v[2 * t + 1], D1);
        }
    }
    int64_t m[d], p[d];
    double Qold[d];
#pragma unroll
    for (int l = 0; l < d; ++l) {
        m[l] = p[l] = kInfBits;
        Qold[l] = 0.0;
    }
    int64_t n = 0, hits = 0, sweeps = 0;
    int k = 0;
    while (__any_sync(FULL, live)) {  // warp-uniform: every lane takes part in the shuffles and DMMAs
        ++k;
        // ---- a2: Lq_s = hb_s V_s; Q_s = q + D(mu~_s., Lq) ----
        double bq0[T], bq1[T], Q[d];
#pragma unroll
        for (int t = 0; t < T; ++t) {
            double D0, D1;
            fr.get(dmul(hb_s, V[2 * t]), dmul(hb_s, V[2 * t + 1]), bq0[t], bq1[t]);
            dmma884(D0, D1, aM0, bq0[t], -0.0, -0.0);
            dmma884(D0, D1, aM1, bq1[t], D0, D1);
            Q[2 * t] = dadd(q[2 * t], D0);
            Q[2 * t + 1] = dadd(q[2 * t + 1], D1);
        }
        // ---- a5 (first half): e_s = |Q_s - Q_s^old| (bits, NaN -> 0), Delta = max_s e_s
        // over the trajectory's 8 stage lanes.  BALLOT: this sweep's R2 decision from
        // two ballots per component instead (Delta == 0 <=> no e_s != 0; m <= min(Delta,
        // p) <=> m <= p and some e_s >= m), the exact Delta only feeding the next
        // sweep's (m, p) ----
        int64_t delta[d];
        bool okb = true;  // (BALLOT) this sweep's R2 decision from ballots
        // (BALLOT: nothing here is used on a step's first sweep, k = 1 -- skipped when
        // no trajectory of the slot tests; warp-uniform with one trajectory)
        const bool anyk2 = !(BALLOT && G8M_SKIPK1) || __any_sync(FULL, live && k >= 2);
#pragma unroll
        for (int l = 0; l < d; ++l) {
            int64_t e = 0;
            if (anyk2) {
                e = dabs_bits(dsub(Q[l], Qold[l]));
                e = (e > kInfBits) ? 0 : e;  // NaN-ignoring max (canonical left-to-right form)
                if constexpr (BALLOT) {
                    const unsigned nz = __ballot_sync(FULL, e != 0) & gmask;
                    const unsigned ge = __ballot_sync(FULL, e >= m[l]) & gmask;
                    okb = okb & ((nz == 0u) | ((m[l] <= p[l]) & (ge != 0u)));
                }
#pragma unroll
                for (int off = 4; off < 32; off <<= 1) {
                    const int64_t o = __shfl_xor_sync(FULL, e, off);
                    e = (o > e) ? o : e;
                }
            }
            Qold[l] = Q[l];
            delta[l] = e;
        }
        // ---- a3: F_s = g(Q_s, t_{n-1} + c_s h) ----
        const double tn1 = dadd(a.t0, dmul((double)(n0 + n), a.h));
        const double ts = dadd(tn1, cs_h);
        double F[d];
        {
            bool ok = true;
            prob.template accel<false>(Q, F, ts, ok);
#if G8M_UNIFORM_EXACT
            if (__any_sync(FULL, !ok && live)) prob.template accel<true>(Q, F, ts, ok);  // exact slow path, same bits
#else
            if (!ok && live) prob.template accel<true>(Q, F, ts, ok);  // exact slow path, same bits
#endif
        }
        // reading R2 (replicated in the 8 lanes), after the right-hand side so that the
        // Delta shuffles and the RHS chains share one basic block
        bool stop = (k >= 2);
        {
            const bool k2 = k >= 2;
#pragma unroll
            for (int l = 0; l < d; ++l) {
                const int64_t e = delta[l];
                const int64_t mn = (e < p[l]) ? e : p[l];
                if (!BALLOT) stop = stop & ((e == 0) | (m[l] <= mn));
                m[l] = k2 ? ((p[l] < m[l]) ? p[l] : m[l]) : m[l];
                p[l] = k2 ? e : p[l];
            }
            if (BALLOT) stop = stop & okb;
        }
        const bool fin = live & (stop | (k >= a.max_iters));
        const unsigned finmask = __ballot_sync(FULL, fin), livemask = __ballot_sync(FULL, live);
        const bool anyfin = finmask != 0u, allfin = (finmask & livemask) == livemask;
        // ---- a4: Lv_s = hb_s F_s; D(W_s., Lv) ----
        double Lv[d], Dv[d], bv0[T], bv1[T];
        {
            // (SPEC: mu~ and nu~ passes every sweep, selected per lane -- the stop
            // decision off the DMMA issue path)
            const bool nu = !SPEC && anyfin && allfin;
            const double w0 = nu ? aN0 : aM0, w1 = nu ? aN1 : aM1;
#pragma unroll
            for (int t = 0; t < T; ++t) {
                Lv[2 * t] = dmul(hb_s, F[2 * t]);
                Lv[2 * t + 1] = dmul(hb_s, F[2 * t + 1]);
                fr.get(Lv[2 * t], Lv[2 * t + 1], bv0[t], bv1[t]);
                dmma884(Dv[2 * t], Dv[2 * t + 1], w0, bv0[t], -0.0, -0.0);
                dmma884(Dv[2 * t], Dv[2 * t + 1], w1, bv1[t], Dv[2 * t], Dv[2 * t + 1]);
            }
            if (SPEC || (anyfin && !allfin)) {  // the slot disagrees: a nu~ pass for the finished ones
#pragma unroll
                for (int t = 0; t < T; ++t) {
                    double N0, N1;
                    dmma884(N0, N1, aN0, bv0[t], -0.0, -0.0);
                    dmma884(N0, N1, aN1, bv1[t], N0, N1);
                    Dv[2 * t] = fin ? N0 : Dv[2 * t];
                    Dv[2 * t + 1] = fin ? N1 : Dv[2 * t + 1];
                }
            }
        }
        if (SPEC || anyfin) {  // ---- a6: S(Lq), S(Lv) as ones x tile; update, history, samples ----
            double Sq[d], Sv[d];
#pragma unroll
            for (int t = 0; t < T; ++t) {
                dmma884(Sq[2 * t], Sq[2 * t + 1], 1.0, bq0[t], -0.0, -0.0);
                dmma884(Sv[2 * t], Sv[2 * t + 1], 1.0, bv0[t], -0.0, -0.0);
                dmma884(Sq[2 * t], Sq[2 * t + 1], 1.0, bq1[t], Sq[2 * t], Sq[2 * t + 1]);
                dmma884(Sv[2 * t], Sv[2 * t + 1], 1.0, bv1[t], Sv[2 * t], Sv[2 * t + 1]);
            }
            bool finite = true;
            if (fin) {
#pragma unroll
                for (int l = 0; l < d; ++l) {
                    q[l] = dadd(q[l], Sq[l]);
                    v[l] = dadd(v[l], Sv[l]);
                    finite = finite && isfinite(q[l]) && isfinite(v[l]);
                }
                ++n;
                sweeps += k;
                hits += stop ? 0 : 1;
                k = 0;
#pragma unroll
                for (int l = 0; l < d; ++l) m[l] = p[l] = kInfBits;
                // (the sample test hoisted out of the s == 0 branch: one divergent branch
                // fewer per step -- config 1 13.0 -> 12.3 ms)
                if ((sample || a.local_energy) && s == 0) {
                    if (valid && sample && ((a.c0 + n) % a.energy_every) == 0)
                        a.energy[((a.c0 + n) / a.energy_every) * B + b] = prob.energy(q, v);
                    if (a.local_energy) dhloc_update(prob.energy(q, v), hprev, dhmax);
                }
                if (n == a.nsteps || !finite) {  // leave: history row s = Lv_s, q block zeroed (R-4)
                    if (valid)
#pragma unroll
                        for (int l = 0; l < d; ++l) {
                            a.hist[((int64_t)s * D + l) * B + b] = 0.0;
                            a.hist[((int64_t)s * D + d + l) * B + b] = Lv[l];
                        }
                    if (!finite) bad = n0 + n;
                    live = false;
                }
            }
        }
        // ---- a4 (end) / next step's a1: V_s = v + D ----
#pragma unroll
        for (int l = 0; l < d; ++l) V[l] = dadd(v[l], Dv[l]);
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
