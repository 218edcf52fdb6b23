// Ensemble kernel for small N-body systems, mapping "stage-per-lane" (g8): a
// group of 8 lanes per trajectory, lane s owns stage s -- its 3N stage
// positions Q_s (registers), V_s (registers) and its right-hand side: all
// N(N-1)/2 pair weights of the stage in ONE lane (15 independent sqrt/div
// chains for N = 6: the ILP the body-per-lane mapping lacks), each weight
// evaluated once.  The stage contractions need every stage's L, which the group
// all-gathers through a shared-memory tile T[8][3N] (one row per lane, read back
// with 16-byte broadcast loads); the Delta reduction over stages goes through a
// second tile; q, v and the stop-test state (m, p) live in shared memory, each
// component owned by lane l mod 8 for its update.
//
//   a2  Lq_s = hb_s V_s -> T[s];  Q_s = q + D(mu_s., T)            Eq. IRK_FP2 l.1-2
//   a5  Delta_l = max_s |Q_s,l - Q_s,l^old| (tile E), R2 test by the owner lane
//   a6  fin: q_l += S(T[.][l]) by the owner lane                    Eq. yn3
//   a3  F_s = accelerations of all bodies at stage s (cyclic partner order of
//       DESIGN.md R-8, weights shared by the two bodies of a pair)    Eq. IRK_FP2 l.3
//   a4  Lv_s = hb_s F_s -> T[s]; fin: v_l += S(T[.][l]);
//       V_s = v + D(W_s., T), W = fin ? nu : mu                     Eq. IRK_FP2 l.4-5
//
// Sweep-granular, one persistent launch: each group pulls (trajectory, step-chunk)
// units from the work queue and the loop is warp-uniform (4 groups per warp at
// their own steps).  Same canonical operation sequence as the oracle: bitwise.
#pragma once
#include <cstdint>

#include "ens_common.cuh"
#include "ensemble_g1.cuh"
#include "ensemble_nbody.cuh"
#include "fp64.cuh"

namespace irk {

constexpr int N8_THREADS = 64;  // 8 groups (trajectories) per block
#ifndef N8_MAXREG
#define N8_MAXREG 168
#endif

// Accelerations of all NB bodies at one stage from its positions Q (registers):
// pair weights w_ij (i < j) once, then per body i the partners j = (i + delta) mod
// NB in cyclic order, d = Q_j - Q_i, a_i = fma(m_j w_ij, d, a_i)  (oracle
// accel_nbody_pairs; w_ij = w_ji bit for bit since the squared differences are
// the same).
template <int NB, bool EXACT, bool G1 = false>
__device__ __forceinline__ void n8_accel(const double *Q, double *A, const NBodyParams &P, const double *sm,
                                         bool &ok) {
    constexpr int NP = NB * (NB - 1) / 2;
    double w[NP];
    // constant trip counts and a closed-form pair index: fully unrolled, so Q and w
    // stay in registers (a triangular loop with a running index was not unrolled and
    // put Q in local memory)
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            if (j <= i) continue;
            const int p = i * NB - i * (i + 1) / 2 + (j - i - 1);
            const double dx = dsub(Q[3 * j], Q[3 * i]), dy = dsub(Q[3 * j + 1], Q[3 * i + 1]),
                         dz = dsub(Q[3 * j + 2], Q[3 * i + 2]);
            const double r2 = dfma(dz, dz, dfma(dy, dy, dfma(dx, dx, P.eps2)));
            if (!EXACT && G1) {  // G == 1: reciprocal form, one range predicate per pair (fp64.cuh)
                bool unused = true;
                ok = ok && weight_range_ok(r2);
                w[p] = drcp_fast(dmul(r2, dsqrt_fast(r2, unused)), unused);
            } else {
                w[p] = EXACT ? ddiv(P.G, dmul(r2, dsqrt(r2))) : ddiv_fast(P.G, dmul(r2, dsqrt_fast(r2, ok)), ok);
            }
        }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        double ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll
        for (int delta = 1; delta < NB; ++delta) {
            const int j = (i + delta) % NB;
            const int lo = i < j ? i : j, hi = i < j ? j : i;
            const int p = lo * NB - lo * (lo + 1) / 2 + (hi - lo - 1);  // index of pair (lo, hi)
            const double dx = dsub(Q[3 * j], Q[3 * i]), dy = dsub(Q[3 * j + 1], Q[3 * i + 1]),
                         dz = dsub(Q[3 * j + 2], Q[3 * i + 2]);
            const double s = dmul(sm[j], w[p]);
            ax = dfma(s, dx, ax);
            ay = dfma(s, dy, ay);
            az = dfma(s, dz, az);
        }
        A[3 * i] = ax;
        A[3 * i + 1] = ay;
        A[3 * i + 2] = az;
    }
}

// The exact-intrinsic re-evaluation (rare: an operand outside the div/sqrt fast
// path) through the lane's own tile row, out of line: called on the registers Q,
// F directly it made ptxas keep both arrays addressable in local memory on the
// hot path too.
template <int NB>
__device__ __noinline__ void n8_accel_exact_row(double *row, const NBodyParams &P, const double *sm) {
    constexpr int d = 3 * NB;
    double Q[d], F[d];
    bool ok = true;
    for (int l = 0; l < d; ++l) Q[l] = row[l];
    n8_accel<NB, true>(Q, F, P, sm, ok);
    for (int l = 0; l < d; ++l) row[l] = F[l];
}

template <int NB, bool G1>
__global__ void __maxnreg__(N8_MAXREG) ens_nbody8_kernel(const __grid_constant__ EnsArgs a,
                                                        const __grid_constant__ QueueArgs qa,
                                                        const __grid_constant__ NBodyParams P) {
    constexpr int d = 3 * NB, D = 6 * NB, GPB = N8_THREADS / 8;
    constexpr int DP = d + (d & 1);  // tile row stride (even: 16-byte aligned rows)
    const unsigned FULL = 0xffffffffu;
    const int64_t B = a.batch;
    const int tx = threadIdx.x, lane = tx & 31, s = tx & 7, gib = tx >> 3, gbase = lane & ~7;
    const unsigned gmask = 0xffu << gbase;

    // coefficients column-major [j][i] (lane s reads 8 consecutive doubles), nu~ in other banks
    __shared__ __align__(16) double sW[72 + 64];
    // Per-group tiles padded so that the 4 groups of a warp start in different banks
    // (unpadded, the 1,152-byte group stride is 0 mod 128: ncu counted 4.2e9 shared
    // bank conflicts on the broadcast loads)
    constexpr int TS = 8 * DP + 2, ES = 8 * d + 1;
    __shared__ __align__(16) double sT[GPB][TS];           // Lq or Lv rows of the 8 stages
    __shared__ int64_t sE[GPB][ES];                        // |Q_s - Q_s^old| bits for Delta
    __shared__ __align__(16) double sQV[GPB][D];           // q, v
    __shared__ int64_t sMP[GPB][2][d];                     // stop-test state m, p
    __shared__ double sm[NB];
    for (int e = tx; e < 64; e += N8_THREADS) {
        sW[(e & 7) * 8 + (e >> 3)] = (&c_mu[0][0])[e];
        sW[72 + (e & 7) * 8 + (e >> 3)] = (&c_nu[0][0])[e];
    }
    for (int e = tx; e < NB; e += N8_THREADS) sm[e] = P.m[e];
    __syncthreads();
    const double *Mu = sW + s, *Nu = sW + 72 + s;  // (s, j) at [8 j]
    const double hb_s = a.hb[s];
    double *T = &sT[gib][0];
    double *qv = sQV[gib];

    const int64_t n0 = *a.n_done;
    const bool sample = (a.energy != nullptr) && (a.energy_every > 0);
    const int64_t total = B * qa.nchunks;
    const int64_t kInfBits = 0x7ff0000000000000LL;

    double Q[d], V[d];
#pragma unroll
    for (int l = 0; l < d; ++l) Q[l] = V[l] = 0.0;
    int64_t b = -1, c = 0, len = 0, n = 0, hits = 0, sweeps = 0, u = -1;
    double hprev = 0.0, dhmax = 0.0;
    int k = 0;
    bool done = false;  // the queue is drained for this group
    for (;;) {
        // ---- acquire (warp-uniform control flow; per-group decisions) ----
        bool need = !done && b < 0;
        if (__all_sync(FULL, done)) break;
        if (__any_sync(FULL, need)) {
            unsigned long long uu = 0;
            if (need && s == 0 && u < 0) uu = atomicAdd(qa.counter, 1ull);
            uu = __shfl_sync(FULL, uu, gbase);
            if (need && u < 0) u = (int64_t)uu;
            bool ready = false;
            if (need) {
                if (u >= total) {
                    done = true;
                    need = false;
                } else {
                    c = u / B;
                    const int64_t bb = u - c * B;
                    ready = !(c > 0 && ld_acquire(&qa.progress[bb]) < c);
                    if (ready) {
                        b = bb;
                        u = -1;
                    }
                }
            }
            const bool load = need && ready;
            // state of the unit: q, v (component l by lane l mod 8), history rows -> T
            if (load) {
                const int64_t c0 = c * qa.qchunk;
                len = (a.nsteps - c0 < qa.qchunk) ? a.nsteps - c0 : qa.qchunk;
                for (int l = s; l < D; l += 8) qv[l] = __ldcg(&a.y[(int64_t)l * B + b]);
#pragma unroll
                for (int l = 0; l < d; ++l) T[s * DP + l] = __ldcg(&a.hist[((int64_t)s * D + d + l) * B + b]);
            }
            __syncwarp();
            bool frozen = false;
            if (load) {
                frozen = __ldcg(&a.stats[1 * B + b]) > 0 || len <= 0;
                if (s == 0 && ((sample && c == 0) || a.local_energy)) {
                    const double h0 = nbody_energy<NB>(qv, P);
                    if (sample && c == 0) a.energy[b] = h0;
                    hprev = h0;
                }
                dhmax = 0.0;
                if (frozen) {
                    if (s == 0 && c == 0) {
                        if (a.local_energy) a.stats[3 * B + b] = 0;
                        if (a.iters) a.iters[b] = 0;
                    }
                } else {  // a1: V_s = v + D(nu_s., H) ; stop-test state reset
#pragma unroll
                    for (int l = 0; l < d; ++l) {
                        double acc = dmul(Nu[0], T[l]);
#pragma unroll
                        for (int j = 1; j < 8; ++j) acc = dfma(Nu[8 * j], T[j * DP + l], acc);
                        V[l] = dadd(qv[d + l], acc);
                    }
                    for (int l = s; l < d; l += 8) sMP[gib][0][l] = sMP[gib][1][l] = kInfBits;
                    n = hits = sweeps = 0;
                    k = 0;
                }
            }
            __syncwarp();
            if (load && frozen) {
                if (s == 0) st_release(&qa.progress[b], (int32_t)(c + 1));
                b = -1;
            }
        }
        const bool live = !done && b >= 0;
        if (!__any_sync(FULL, live)) {  // nobody in the warp has work this trip (vote by every lane)
            __nanosleep(512);
            continue;
        }
        if (live) ++k;
        // ---- a2: Lq_s -> T[s] ; Q_s = q + D(mu_s., T) ; |Q_s - Q_s^old| -> E ----
#pragma unroll
        for (int l = 0; l < d; ++l) T[s * DP + l] = dmul(hb_s, V[l]);
        __syncwarp();
#pragma unroll
        for (int l = 0; l < d; l += 2) {
            double2 t0 = *reinterpret_cast<const double2 *>(&T[l]);
            double acc0 = dmul(Mu[0], t0.x), acc1 = dmul(Mu[0], t0.y);
#pragma unroll
            for (int j = 1; j < 8; ++j) {
                const double2 tj = *reinterpret_cast<const double2 *>(&T[j * DP + l]);
                acc0 = dfma(Mu[8 * j], tj.x, acc0);
                acc1 = dfma(Mu[8 * j], tj.y, acc1);
            }
            const double qn0 = dadd(qv[l], acc0);
            sE[gib][s * d + l] = absdiff_bits(qn0, Q[l]);
            Q[l] = qn0;
            if (l + 1 < d) {
                const double qn1 = dadd(qv[l + 1], acc1);
                sE[gib][s * d + l + 1] = absdiff_bits(qn1, Q[l + 1]);
                Q[l + 1] = qn1;
            }
        }
        __syncwarp();
        // ---- a5: Delta and the stop test for the lane's components (l = s mod 8) ----
        bool ok_lane = true;
        if (live && k >= 2) {
            for (int l = s; l < d; l += 8) {
                int64_t ev[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) ev[j] = sE[gib][j * d + l];
                const int64_t delta = delta_bits8(ev);
                const int64_t pl = sMP[gib][1][l], ml = sMP[gib][0][l];
                ok_lane = ok_lane && ((delta == 0) || (ml <= imin64(delta, pl)));
                sMP[gib][0][l] = imin64(pl, ml);
                sMP[gib][1][l] = delta;
            }
        }
        const unsigned notok = __ballot_sync(FULL, !ok_lane);
        const bool stop = live && (k >= 2) && ((notok & gmask) == 0u);
        const bool fin = live && (stop || k >= a.max_iters);
        if (fin)  // a6 (positions): q_l += S(Lq) by the owner lane
            for (int l = s; l < d; l += 8) {
                double sq = T[l];
#pragma unroll
                for (int j = 1; j < 8; ++j) sq = dadd(sq, T[j * DP + l]);
                qv[l] = dadd(qv[l], sq);
            }
        __syncwarp();  // T (Lq) fully read; q updated
        // ---- a3: F_s (all bodies at stage s) ; Lv_s -> T[s] ----
        {
            double F[d];
            bool ok = true;
            n8_accel<NB, false, G1>(Q, F, P, sm, ok);
            // exact intrinsics, same bits (row s of T is free until the Lv store below);
            // not for idle groups: their zero tiles fail the fast-path range every sweep
            // (a lone trajectory ran 3x slower for that)
            if (!ok && live) {
#pragma unroll
                for (int l = 0; l < d; ++l) T[s * DP + l] = Q[l];
                n8_accel_exact_row<NB>(&T[s * DP], P, sm);
#pragma unroll
                for (int l = 0; l < d; ++l) F[l] = T[s * DP + l];
            }
#pragma unroll
            for (int l = 0; l < d; ++l) T[s * DP + l] = dmul(hb_s, F[l]);
        }
        __syncwarp();
        // ---- a6 (velocities), history, samples; a4 / next nu-init ----
        bool finite = true;
        if (fin) {
            for (int l = s; l < d; l += 8) {
                double sv = T[l];
#pragma unroll
                for (int j = 1; j < 8; ++j) sv = dadd(sv, T[j * DP + l]);
                qv[d + l] = dadd(qv[d + l], sv);
                finite = finite && isfinite(qv[l]) && isfinite(qv[d + l]);
                sMP[gib][0][l] = sMP[gib][1][l] = kInfBits;
            }
        }
        const unsigned nonfinite = __ballot_sync(FULL, fin && !finite);
        const bool grp_bad = fin && ((nonfinite & gmask) != 0u);
        __syncwarp();  // v updated
        if (fin) {
            ++n;
            sweeps += k;
            hits += stop ? 0 : 1;
            k = 0;
        }
        const int64_t nloc = c * qa.qchunk + n;
        if (fin && s == 0) {
            const bool due = sample && (nloc % a.energy_every) == 0;
            if (due || a.local_energy) {
                const double hn = nbody_energy<NB>(qv, P);
                if (due) a.energy[(nloc / a.energy_every) * B + b] = hn;
                if (a.local_energy) dhloc_update(hn, hprev, dhmax);
            }
        }
        const bool release = fin && (n == len || grp_bad);
        if (release) {  // history row s = Lv_s (q block zeroed, R-4); state, stats
#pragma unroll
            for (int l = 0; l < d; ++l) {
                a.hist[((int64_t)s * D + l) * B + b] = 0.0;
                a.hist[((int64_t)s * D + d + l) * B + b] = T[s * DP + l];
            }
            for (int l = s; l < D; l += 8) a.y[(int64_t)l * B + b] = qv[l];
            if (s == 0) {
                a.stats[0 * B + b] = __ldcg(&a.stats[0 * B + b]) + hits;
                if (grp_bad) a.stats[1 * B + b] = n0 + nloc;
                a.stats[2 * B + b] = __ldcg(&a.stats[2 * B + b]) + sweeps;
                if (a.iters) a.iters[b] = (c == 0) ? sweeps : __ldcg(&a.iters[b]) + sweeps;
                if (a.local_energy) dhloc_store(&a.stats[3 * B + b], c == 0, dhmax);
            }
            __threadfence();
        }
        __syncwarp();
        if (release) {
            if (s == 0) st_release(&qa.progress[b], (int32_t)(c + 1));
            b = -1;
        }
        {   // V_s = v + D(W_s., Lv), W = nu after a finished step (the next step's a1)
            const double *W = fin ? Nu : Mu;
#pragma unroll
            for (int l = 0; l < d; l += 2) {
                const double2 t0 = *reinterpret_cast<const double2 *>(&T[l]);
                double acc0 = dmul(W[0], t0.x), acc1 = dmul(W[0], t0.y);
#pragma unroll
                for (int j = 1; j < 8; ++j) {
                    const double2 tj = *reinterpret_cast<const double2 *>(&T[j * DP + l]);
                    acc0 = dfma(W[8 * j], tj.x, acc0);
                    acc1 = dfma(W[8 * j], tj.y, acc1);
                }
                V[l] = dadd(qv[d + l], acc0);
                if (l + 1 < d) V[l + 1] = dadd(qv[d + l + 1], acc1);
            }
        }
        __syncwarp();  // T reads done before the next sweep's writes
    }
}

}  // namespace irk
