// Ensemble kernel, mapping "body-per-lane": one group of NB lanes per
// trajectory of a small gravitational N-body system (config 3: NB = 6, d = 18);
// lane k of a group owns body k -- its 3 position and 3 velocity components for
// all 8 stages.  32/NB groups share a warp (5 for NB = 6).
//
// Why this mapping: a 6-body stage tile is 3 x 144
// doubles, too large for one thread's registers or for one thread per
// trajectory in shared memory at 111 trajectories per SM; splitting by body makes
// both 8x8 contractions (a1, a2, a4) thread-local (components are independent)
// and leaves only the RHS (a3) needing other bodies' stage positions, which the
// group exchanges through a shared-memory tile that doubles as Q^[k-1] for the
// stop test.
//
// Canonical RHS (R-8, oracle accel_nbody_pairs): body k sums over its
// partners j = (k + delta) mod NB in the cyclic order delta = 1..NB-1, with
// d = q_j - q_k, r2 = fma(dz,dz,fma(dy,dy,fma(dx,dx,eps^2))),
// w = G / (r2 sqrt(r2)), a_k = fma(m_j w, d, a_k).  The pair weight w is
// symmetric in (k, j) bit for bit (the two differences are exact negatives), so
// each lane evaluates it only for delta = 1..NB/2 and takes delta > NB/2 -- the
// pair (k - o, k), o = NB - delta -- from lane k - o by a warp shuffle: 3 weight
// evaluations per lane and stage for NB = 6 instead of 5, every lane running the
// same delta sequence (no per-lane selects).
//
// The loop is warp-uniform (it runs until every group of the warp is done;
// finished groups idle) so that __syncwarp / __ballot_sync always see the full
// warp.  Sweep-granular as in ens_g1: a group whose step converged updates and
// re-initialises in the same trip.
#pragma once
#include <cstdint>

#include "ens_common.cuh"
#include "fp64.cuh"

namespace irk {

struct NBodyParams {
    double G, eps2;
    double m[16];
};

constexpr int NB_THREADS = 64;

// Hamiltonian of one system from shared memory (canonical term order, Neumaier;
// oracle energy_nbody): kinetic terms i = 0..N-1, then row sums over j > i.
template <int NB>
__device__ double nbody_energy(const double *q, const double *v, const NBodyParams &P) {
    Neumaier tot;
    for (int i = 0; i < NB; ++i) {
        double k = dfma(v[3 * i + 2], v[3 * i + 2], dfma(v[3 * i + 1], v[3 * i + 1], dmul(v[3 * i], v[3 * i])));
        tot.add(dmul(dmul(0.5, P.m[i]), k));
    }
    for (int i = 0; i < NB; ++i) {
        Neumaier row;
        for (int j = i + 1; j < NB; ++j) {
            double dx = dsub(q[3 * j], q[3 * i]);
            double dy = dsub(q[3 * j + 1], q[3 * i + 1]);
            double dz = dsub(q[3 * j + 2], q[3 * i + 2]);
            double r2 = dfma(dz, dz, dfma(dy, dy, dfma(dx, dx, P.eps2)));
            row.add(-ddiv(dmul(P.G, dmul(P.m[i], P.m[j])), dsqrt(r2)));
        }
        tot.add(row.result());
    }
    return tot.result();
}
template <int NB>
__device__ double nbody_energy(const double *qv, const NBodyParams &P) {
    return nbody_energy<NB>(qv, qv + 3 * NB, P);
}

// Acceleration of body `body` at one stage (canonical RHS, see the header).
template <int NB, bool EXACT>
__device__ __forceinline__ void nb_stage_accel(const double *Qi, int body, int lane, const NBodyParams &P,
                                               const double *sm, bool &ok, double &ax, double &ay, double &az) {
    const double qx = Qi[3 * body], qy = Qi[3 * body + 1], qz = Qi[3 * body + 2];
    ax = 0.0, ay = 0.0, az = 0.0;
    // partners j = (k + delta) mod NB, delta = 1..NB-1.  Offsets delta <= NB/2 are
    // evaluated here; delta > NB/2 is the pair (k - o, k), o = NB - delta, whose
    // weight lane k - o evaluated as its offset o: fetched by shuffle.
    constexpr int HF = NB / 2, HB = (NB - 1) / 2;
    double wf[HF + 1], dfx[HF + 1], dfy[HF + 1], dfz[HF + 1];
#pragma unroll
    for (int o = 1; o <= HF; ++o) {
        const int j = (body + o < NB) ? body + o : body + o - NB;
        dfx[o] = dsub(Qi[3 * j], qx), dfy[o] = dsub(Qi[3 * j + 1], qy), dfz[o] = dsub(Qi[3 * j + 2], qz);
        const double r2 = dfma(dfz[o], dfz[o], dfma(dfy[o], dfy[o], dfma(dfx[o], dfx[o], P.eps2)));
        wf[o] = EXACT ? ddiv(P.G, dmul(r2, dsqrt(r2))) : ddiv_fast(P.G, dmul(r2, dsqrt_fast(r2, ok)), ok);
    }
    double wb[HB + 1];
#pragma unroll
    for (int o = 1; o <= HB; ++o) {
        const int src = lane - body + ((body - o >= 0) ? body - o : body - o + NB);
        wb[o] = __shfl_sync(0xffffffffu, wf[o], src & 31);
    }
#pragma unroll
    for (int delta = 1; delta < NB; ++delta) {
        const int j = (body + delta < NB) ? body + delta : body + delta - NB;
        double dx, dy, dz, w;
        if (delta <= HF) {
            dx = dfx[delta], dy = dfy[delta], dz = dfz[delta], w = wf[delta];
        } else {
            dx = dsub(Qi[3 * j], qx), dy = dsub(Qi[3 * j + 1], qy), dz = dsub(Qi[3 * j + 2], qz);
            w = wb[NB - delta];
        }
        const double s = dmul(sm[j], w);
        ax = dfma(s, dx, ax);
        ay = dfma(s, dy, ay);
        az = dfma(s, dz, az);
    }
}

#ifndef NB_PHASED
#define NB_PHASED 4  // RHS in groups of 8/NB_PHASED stages: weights, then shuffles, then sums (config 3, 5,000 steps: per-stage 219 ms, 4 groups 206)
#endif
#ifndef NB_MAXREG
#define NB_MAXREG 168  // config 3, 5,000 steps: 168 -> 306 ms, 255 -> 309, 128 -> 342 (tools/variants.py)
#endif
#ifndef NB_RHS_UNROLL
#define NB_RHS_UNROLL 4  // stages of the RHS loop in flight (config 3, 5,000 steps: 2 -> 235 ms, 4 -> 230)
#endif
constexpr int kNbRhsUnroll = NB_RHS_UNROLL;

// One warp integrates its GPW trajectories (b = -1: idle group) over the
// call-local steps [c0, c0 + nsteps).  Shared tiles belong to the calling block.
template <int NB>
__device__ __forceinline__ void nbody_unit(const EnsArgs &a, const NBodyParams &P, const int64_t b_in,
                                           const int64_t c0, const int64_t nsteps, const double (*sW)[64],
                                           double *sQ, double (*sQV)[6 * NB], const double *sm) {
    constexpr int GPW = 32 / NB;                 // groups (trajectories) per warp
    constexpr int d = 3 * NB, D = 6 * NB;
    constexpr int GS = 8 * d + (((5 - 8 * d) % 16) + 16) % 16;
    const unsigned FULL = 0xffffffffu;
    const int64_t B = a.batch;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / NB, body = lane % NB;
    const bool lane_ok = grp < GPW;
    const int gib = warp * GPW + (lane_ok ? grp : 0);   // group index inside the block
    const int64_t b = lane_ok ? b_in : -1;
    const bool valid = b >= 0;
    const unsigned gmask = lane_ok ? (((1u << NB) - 1u) << (grp * NB)) : 0u;

    double q[3] = {0, 0, 0}, v[3] = {0, 0, 0};
    int64_t bad = 0;
    if (valid) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            q[c] = __ldcg(&a.y[(int64_t)(3 * body + c) * B + b]);  // L2: may come from another SM
            v[c] = __ldcg(&a.y[(int64_t)(d + 3 * body + c) * B + b]);
        }
        bad = __ldcg(&a.stats[1 * B + b]);
    }
    const int64_t n0 = *a.n_done;
    const bool sample = (a.energy != nullptr) && (a.energy_every > 0);
    // energy at local step 0 (first chunk only); H(y) at the chunk start for DH^loc
    double hprev = 0.0, dhmax = 0.0;
    if ((sample && c0 == 0) || a.local_energy) {
        if (lane_ok) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                sQV[gib][3 * body + c] = q[c];
                sQV[gib][d + 3 * body + c] = v[c];
            }
        }
        __syncwarp();
        if (valid && body == 0) {
            hprev = nbody_energy<NB>(sQV[gib], P);
            if (sample && c0 == 0) a.energy[b] = hprev;
        }
        __syncwarp();
    }
    bool live = valid && bad == 0 && nsteps > 0;
    if (valid && !live) {
        if (a.iters && c0 == 0 && body == 0) a.iters[b] = 0;
        if (a.csweeps && body == 0) a.csweeps[b] = 0;
    }

    // a1: nu-init of own velocity components from the history (zeros = first step)
    double V[8][3];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int c = 0; c < 3; ++c) V[i][c] = v[c];
    if (live) {
        double H[8][3];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int c = 0; c < 3; ++c) H[j][c] = __ldcg(&a.hist[((int64_t)j * D + d + 3 * body + c) * B + b]);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double acc = dmul(c_nu[i][0], H[0][c]);
#pragma unroll
                for (int j = 1; j < 8; ++j) acc = dfma(c_nu[i][j], H[j][c], acc);
                V[i][c] = dadd(v[c], acc);
            }
    }
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    double m[3] = {kInf, kInf, kInf}, p[3] = {kInf, kInf, kInf};
    int64_t n = 0, hits = 0, sweeps = 0;
    int k = 0;
    double Lv[8][3];

    while (__any_sync(FULL, live)) {
        ++k;
        // ---- a2: Lq = hb o V ; Q_i = q + D(mu_i., Lq) ; Delta vs Q^[k-1] (smem) ----
        double Lq[8][3], sLq[3], delta[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int c = 0; c < 3; ++c) Lq[j][c] = dmul(a.hb[j], V[j][c]);
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            sLq[c] = Lq[0][c];
#pragma unroll
            for (int j = 1; j < 8; ++j) sLq[c] = dadd(sLq[c], Lq[j][c]);
        }
        {
            const double2 *M = reinterpret_cast<const double2 *>(&c_mu[0][0]);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double2 w[4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) w[jj] = M[i * 4 + jj];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    double acc = dmul(w[0].x, Lq[0][c]);
                    acc = dfma(w[0].y, Lq[1][c], acc);
#pragma unroll
                    for (int jj = 1; jj < 4; ++jj) {
                        acc = dfma(w[jj].x, Lq[2 * jj][c], acc);
                        acc = dfma(w[jj].y, Lq[2 * jj + 1][c], acc);
                    }
                    const double qn = dadd(q[c], acc);
                    if (lane_ok) {
                        const double e = dabs(dsub(qn, sQ[gib * GS + i * d + 3 * body + c]));  // unused at k = 1
                        delta[c] = (e > delta[c]) ? e : delta[c];
                        sQ[gib * GS + i * d + 3 * body + c] = qn;
                    }
                }
            }
        }
        // ---- a5: stop test over the group's 3*NB position components (R2) ----
        bool ok_lane = true;
        if (k >= 2) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                const double mn = (delta[c] < p[c]) ? delta[c] : p[c];
                const bool okc = (delta[c] == 0.0) || (m[c] <= mn);
                m[c] = (p[c] < m[c]) ? p[c] : m[c];
                p[c] = delta[c];
                ok_lane = ok_lane && okc;
            }
        }
        const unsigned notok = __ballot_sync(FULL, !ok_lane);
        const bool stop = (k >= 2) && ((notok & gmask) == 0u);
        __syncwarp();  // every body's Q^[k] is in sQ
        // ---- a3: F_i(body) = sum over the other bodies, cyclic order (header) ----
        const double tn1 = dadd(a.t0, dmul((double)(n0 + n), a.h));
        (void)tn1;  // the N-body RHS is autonomous
        bool okdiv = true;
#if NB_PHASED
        {   // phase-separated: all stages' own pair weights, then the shuffles, then the sums
            constexpr int HF = NB / 2, HB = (NB - 1) / 2, SPH = 8 / NB_PHASED;  // stages per phase group
#pragma unroll
            for (int i0 = 0; i0 < 8; i0 += SPH) {
            double wf[8][HF + 1], wb[8][HB + 1];
#pragma unroll
            for (int i = i0; i < i0 + SPH; ++i) {
                const double *Qi = &sQ[gib * GS + i * d];
                const double qx = Qi[3 * body], qy = Qi[3 * body + 1], qz = Qi[3 * body + 2];
#pragma unroll
                for (int o = 1; o <= HF; ++o) {
                    const int j = (body + o < NB) ? body + o : body + o - NB;
                    const double dx = dsub(Qi[3 * j], qx), dy = dsub(Qi[3 * j + 1], qy), dz = dsub(Qi[3 * j + 2], qz);
                    const double r2 = dfma(dz, dz, dfma(dy, dy, dfma(dx, dx, P.eps2)));
                    wf[i][o] = ddiv_fast(P.G, dmul(r2, dsqrt_fast(r2, okdiv)), okdiv);
                }
            }
#pragma unroll
            for (int i = i0; i < i0 + SPH; ++i)
#pragma unroll
                for (int o = 1; o <= HB; ++o) {
                    const int src = lane - body + ((body - o >= 0) ? body - o : body - o + NB);
                    wb[i][o] = __shfl_sync(FULL, wf[i][o], src & 31);
                }
#pragma unroll
            for (int i = i0; i < i0 + SPH; ++i) {
                const double *Qi = &sQ[gib * GS + i * d];
                const double qx = Qi[3 * body], qy = Qi[3 * body + 1], qz = Qi[3 * body + 2];
                double ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll
                for (int delta = 1; delta < NB; ++delta) {
                    const int j = (body + delta < NB) ? body + delta : body + delta - NB;
                    const double dx = dsub(Qi[3 * j], qx), dy = dsub(Qi[3 * j + 1], qy), dz = dsub(Qi[3 * j + 2], qz);
                    const double s = dmul(sm[j], (delta <= HF) ? wf[i][delta] : wb[i][NB - delta]);
                    ax = dfma(s, dx, ax);
                    ay = dfma(s, dy, ay);
                    az = dfma(s, dz, az);
                }
                Lv[i][0] = dmul(a.hb[i], ax);
                Lv[i][1] = dmul(a.hb[i], ay);
                Lv[i][2] = dmul(a.hb[i], az);
            }
            }
        }
#else
#pragma unroll kNbRhsUnroll
        for (int i = 0; i < 8; ++i) {
            double ax, ay, az;
            nb_stage_accel<NB, false>(&sQ[gib * GS + i * d], body, lane, P, sm, okdiv, ax, ay, az);
            Lv[i][0] = dmul(a.hb[i], ax);
            Lv[i][1] = dmul(a.hb[i], ay);
            Lv[i][2] = dmul(a.hb[i], az);
        }
#endif
        if (__any_sync(FULL, live && !okdiv)) {  // exact-intrinsic re-evaluation (same bits)
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double ax, ay, az;
                nb_stage_accel<NB, true>(&sQ[gib * GS + i * d], body, lane, P, sm, okdiv, ax, ay, az);
                Lv[i][0] = dmul(a.hb[i], ax);
                Lv[i][1] = dmul(a.hb[i], ay);
                Lv[i][2] = dmul(a.hb[i], az);
            }
        }
        __syncwarp();  // sQ (Q^[k]) stays for the next sweep's Delta; no writer until then
        // ---- a6 (group finished its step): update, history, energy sample ----
        const bool fin = live && (stop || k >= a.max_iters);
        bool finite = true;
        if (fin) {
#pragma unroll
            for (int c = 0; c < 3; ++c) {
                double sv = Lv[0][c];
#pragma unroll
                for (int j = 1; j < 8; ++j) sv = dadd(sv, Lv[j][c]);
                q[c] = dadd(q[c], sLq[c]);
                v[c] = dadd(v[c], sv);
                finite = finite && isfinite(q[c]) && isfinite(v[c]);
            }
            ++n;
            sweeps += k;
            hits += stop ? 0 : 1;
        }
        const unsigned nonfinite = __ballot_sync(FULL, fin && !finite);
        const bool grp_bad = fin && ((nonfinite & gmask) != 0u);
        const bool due = fin && sample && ((c0 + n) % a.energy_every) == 0;
        const bool need = due || (fin && a.local_energy);
        if (__any_sync(FULL, need)) {
            if (need) {
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    sQV[gib][3 * body + c] = q[c];
                    sQV[gib][d + 3 * body + c] = v[c];
                }
            }
            __syncwarp();
            if (need && body == 0) {
                const double hn = nbody_energy<NB>(sQV[gib], P);
                if (due) a.energy[((c0 + n) / a.energy_every) * B + b] = hn;
                if (a.local_energy) dhloc_update(hn, hprev, dhmax);
            }
            __syncwarp();
        }
        if (fin && (n == nsteps || grp_bad)) {  // leave: history = Lv (R-4), q block zeroed
#pragma unroll
            for (int j = 0; j < 8; ++j)
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    a.hist[((int64_t)j * D + 3 * body + c) * B + b] = 0.0;
                    a.hist[((int64_t)j * D + d + 3 * body + c) * B + b] = Lv[j][c];
                }
            if (grp_bad) bad = n0 + n;
            live = false;
        }
        if (fin) {
            k = 0;
#pragma unroll
            for (int c = 0; c < 3; ++c) m[c] = p[c] = kInf;
        }
        // ---- a4 / next step's a1: V_i = v + D(W_i., Lv), W = fin ? nu : mu ----
        {
            const double2 *W = reinterpret_cast<const double2 *>(&sW[fin ? 1 : 0][0]);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double2 w[4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) w[jj] = W[i * 4 + jj];
#pragma unroll
                for (int c = 0; c < 3; ++c) {
                    double acc = dmul(w[0].x, Lv[0][c]);
                    acc = dfma(w[0].y, Lv[1][c], acc);
#pragma unroll
                    for (int jj = 1; jj < 4; ++jj) {
                        acc = dfma(w[jj].x, Lv[2 * jj][c], acc);
                        acc = dfma(w[jj].y, Lv[2 * jj + 1][c], acc);
                    }
                    V[i][c] = dadd(v[c], acc);
                }
            }
        }
    }
    if (valid) {
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            a.y[(int64_t)(3 * body + c) * B + b] = q[c];
            a.y[(int64_t)(d + 3 * body + c) * B + b] = v[c];
        }
        if (body == 0) {
            if (nsteps > 0 && __ldcg(&a.stats[1 * B + b]) == 0) {
                a.stats[0 * B + b] = __ldcg(&a.stats[0 * B + b]) + hits;
                a.stats[1 * B + b] = bad;
                a.stats[2 * B + b] = __ldcg(&a.stats[2 * B + b]) + sweeps;
                if (a.iters) a.iters[b] = (c0 == 0) ? sweeps : __ldcg(&a.iters[b]) + sweeps;
                if (a.csweeps) a.csweeps[b] = (int32_t)sweeps;
                if (a.local_energy) dhloc_store(&a.stats[3 * B + b], c0 == 0, dhmax);
            } else if (a.local_energy && c0 == 0) {
                a.stats[3 * B + b] = 0;
            }
        }
    }
}

#define NB_SHARED_TILES                                                                              \
    constexpr int GPW = 32 / NB, GPB = GPW * (NB_THREADS / 32), d = 3 * NB;                          \
    constexpr int GS = 8 * d + (((5 - 8 * d) % 16) + 16) % 16;                                        \
    __shared__ __align__(16) double sW[2][64];  /* mu~, nu~ for the per-group choice in a4 */          \
    __shared__ double sQ[GPB * GS];             /* Q^[k] (+ Q^[k-1] for Delta), padded stride GS */     \
    __shared__ double sQV[GPB][6 * NB];         /* (q, v) gathered for energy samples */               \
    __shared__ double sm[NB];                                                                          \
    for (int e = threadIdx.x; e < 128; e += blockDim.x)                                                \
        sW[e >> 6][e & 63] = (e < 64) ? (&c_mu[0][0])[e] : (&c_nu[0][0])[e - 64];                      \
    for (int e = threadIdx.x; e < NB; e += blockDim.x) sm[e] = P.m[e];                                 \
    __syncthreads();

// Chunked launch (IRK_OPT_SCHEDULE = 1): one warp per GPW slots of the (cost-sorted) order.
template <int NB>
__global__ void __maxnreg__(NB_MAXREG) ens_nbody_kernel(const __grid_constant__ EnsArgs a,
                                                       const __grid_constant__ NBodyParams P) {
    NB_SHARED_TILES
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int grp = lane / NB;
    const int64_t slot = (int64_t)blockIdx.x * GPB + warp * GPW + (grp < GPW ? grp : 0);
    int64_t b = -1;
    if (grp < GPW && slot < a.nslots) b = a.perm ? (int64_t)a.perm[slot] : slot;
    if (b >= a.batch) b = -1;
    nbody_unit<NB>(a, P, b, a.c0, a.nsteps, sW, sQ, sQV, sm);
}

// Persistent warp-level work queue (IRK_OPT_SCHEDULE auto / 2): a unit is (warp
// slot w = trajectories w*GPW .. w*GPW + GPW - 1, step chunk c); unit (w, c) waits
// for progress[w] = c.  Same arithmetic per unit: bitwise any schedule.
template <int NB>
__global__ void __maxnreg__(NB_MAXREG) ens_nbody_q_kernel(const __grid_constant__ EnsArgs a,
                                                         const __grid_constant__ QueueArgs qa,
                                                         const __grid_constant__ NBodyParams P) {
    NB_SHARED_TILES
    const int lane = threadIdx.x & 31;
    const int grp = lane / NB;
    const int64_t W = (a.batch + GPW - 1) / GPW, total = W * qa.nchunks;
    int64_t c = 0, w = 0;
    bool carry = false;  // continue slot w with unit c (parked for this warp by its fetcher)
    for (;;) {
        if (!carry) {
            unsigned long long u = 0;
            if (lane == 0) u = atomicAdd(qa.counter, 1ull);
            u = __shfl_sync(0xffffffffu, u, 0);
            if ((int64_t)u >= total) break;
            c = (int64_t)u / W;
            w = (int64_t)u - c * W;
            // Predecessor (w, c - 1) still running: park the unit for the warp that
            // runs it (hand-off protocol of ens_common.cuh) and fetch another one,
            // rather than idling a warp for up to a whole unit.  Without this the
            // queue fell into a convoy of waiting warps in some runs (config 3: 2.08
            // or 2.85 s at random).
            int go = 1;
            if (lane == 0 && c > 0 && ld_acquire(&qa.progress[w]) < c) {
                if (atomicCAS(&qa.orphan[w], 0, (int)c) == 0) {
                    __threadfence();
                    go = (ld_acquire(&qa.progress[w]) >= c && atomicCAS(&qa.orphan[w], (int)c, 0) == (int)c) ? 1 : 0;
                } else {  // another unit of w already parked (rare): wait
                    while (ld_acquire(&qa.progress[w]) < c) __nanosleep(1024);
                }
            }
            go = __shfl_sync(0xffffffffu, go, 0);
            if (!go) continue;
        }
        __syncwarp();
        int64_t b = (grp < GPW) ? w * GPW + grp : -1;
        if (b >= a.batch) b = -1;
        const int64_t c0 = c * qa.qchunk;
        nbody_unit<NB>(a, P, b, c0, (a.nsteps - c0 < qa.qchunk) ? a.nsteps - c0 : qa.qchunk, sW, sQ, sQV, sm);
        __threadfence();  // this warp's stores of the unit, before the hand-off
        __syncwarp();
        int claimed = 0;
        if (lane == 0) {
            st_release(&qa.progress[w], (int32_t)(c + 1));
            claimed = claim_orphan(qa, (int32_t)w, c + 1) ? 1 : 0;
        }
        carry = __shfl_sync(0xffffffffu, claimed, 0) != 0;
        if (carry) ++c;
    }
}
#undef NB_SHARED_TILES

}  // namespace irk
