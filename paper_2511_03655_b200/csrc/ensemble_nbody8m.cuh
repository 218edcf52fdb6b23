// Ensemble kernel for small N-body systems, mapping "stage per lane, DMMA
// contractions" (IRK_MAP_G8M): a warp integrates a slot of 4 trajectories; lane
// L = 4 s + g owns stage s of trajectory g -- its 3N stage positions Q_s
// (registers) and the whole right-hand side of that stage (all N(N-1)/2 pair
// weights once, as in ens_nbody8).  What changes is how the two 8 x 8 stage
// contractions of a sweep (Eq. IRK_FP2 lines 1-2 and 4-5) are done: on the FP64
// tensor core, without shared memory.
//
// The contraction of a half-sweep is D[s][(g, l)] = sum_j W[s][j] X_j[(g, l)]
// (X = Lq or Lv, W = mu~ or nu~), an 8 x 8 x 8 product per trajectory and
// component.  mma.m8n8k4.f64 computes an 8 x 8 tile over k = 4 as an fma chain
// in k order (bitwise, profiles/r1/dmma_probe.txt); two chained instructions
// (C = the first's D) give the canonical chain over j = 0..7, and C = -0 for the
// first reproduces the leading dmul, signed zeros included (fma(a, b, -0) =
// RN(a b)).  Tile t holds components 2t, 2t+1 of all 4 trajectories: column
// n = 2 g + e is component 2t + e of trajectory g.  With that column order the
// tile's D fragment (row s = L / 4, columns 2 (L % 4) + e) lands in lane 4 s + g
// -- the owner of (g, s) -- so contraction results need no transpose, and the B
// fragment (B[k][n] at lane L: k = L % 4, n = L / 4) is X_j[(g', 2t + e)] with
// j = 4 kk + L % 4, g' = L / 8, e = (L / 4) % 2: it sits in lane 4 j + g' and is
// fetched with two shuffles per tile (both k halves: the source lanes of the two
// halves, j < 4 and j >= 4, offer the pair's components in opposite order, so each
// destination picks up one half per shuffle).
//
// The coefficient fragment (A[m][k] = W[s][4 kk + L % 4]) is shared by the four
// trajectories of a tile, so a velocity contraction whose trajectories disagree
// on W (nu~ for the trajectories that finished their step, mu~ for the others) is
// done twice and each lane keeps its own.  Units are (slot of 4 trajectories, step
// chunk): a slot's trajectories start together and take the same sweep counts
// most of the time, so the two passes are rare.
//
//   a2  D = mu~ Lq (DMMA); Q_s = q + D                       Eq. IRK_FP2 l.1-2
//   a5  Delta_l = max_s |Q_s,l - Q_s,l^old|: a reduce-scatter of the 8 stage lanes of
//       a trajectory (xor 16, 8, 4: each lane ends owning <= 3 components, their
//       stop-test state m, p in registers), R2 test, ballot over the trajectory's lanes
//   a6  fin: the owner of component l (lane s = l mod 8 of the trajectory) sums
//       column l of the Lq / Lv tile in stage order and updates q, v in shared
//       memory                                                    Eq. yn3
//   a3  F_s = accelerations at stage s (n8_accel, cyclic partner order R-8)
//   a4  D = W Lv, W = nu~ for a finished step (next step's nu-init), else mu~;
//       V = v + D; the next sweep's Lq = hb_s V                Eq. IRK_FP2 l.4-5
//
// One persistent launch; each warp pulls (slot, step-chunk) units from the work
// queue (progress per slot).  Same canonical operation sequence as the oracle:
// bitwise.
#pragma once
#include <cstdint>

#include "ens_common.cuh"
#include "ensemble_g1.cuh"
#include "ensemble_nbody.cuh"
#include "ensemble_nbody8.cuh"
#include "fp64.cuh"

namespace irk {

#ifndef N8M_WARPS
#define N8M_WARPS 2
#endif
constexpr int N8M_THREADS = 32 * N8M_WARPS;  // one slot of 4 trajectories per warp
#ifndef N8M_MAXREG
#define N8M_MAXREG 168
#endif
#ifndef N8M_DREUSE
#define N8M_DREUSE 2  // pair differences formed once per stage, body by body (n8m_accel_bodies; 1: all pairs first)
#endif
#ifndef N8M_CMASS
#define N8M_CMASS 1  // masses read from the kernel parameters instead of shared memory (with DREUSE 2: config 3, 2,000 steps 60.2 -> 58.4 ms)
#endif
#ifndef N8M_UNIFORM_EXACT
#define N8M_UNIFORM_EXACT 0
#endif
#ifndef N8M_A2SYNC
#define N8M_A2SYNC 0
#endif
#ifndef N8M_QKEEP
#define N8M_QKEEP 1  // Q_s of this sweep kept in registers from a2 to the RHS (-1.3 %)
#endif
#ifndef N8M_QSMEM
#define N8M_QSMEM 1  // stage positions Q between sweeps in shared memory ([component][lane]), not registers
#endif

// D = A B + C, A 8x4 (row), B 4x8 (col), fp64: SASS DMMA.8x8x4.  volatile: a
// non-volatile asm may be sunk into the conditional code that consumes its result
// (the fin-only updates), where mma.sync.aligned would run on part of the warp.
__device__ __forceinline__ void dmma884(double &d0, double &d1, double a, double b, double c0, double c1) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};"
        : "=d"(d0), "=d"(d1)
        : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// Shared-memory stage tile of a warp: rows (g, s) of RS doubles, g-blocks of GS0
// doubles plus 4 for g >= 2.  RS = 2 mod 16 and GS0 = 8 mod 16 make both access
// patterns conflict-free: the B-fragment reads (a half-warp reads stages 4kk..4kk+3
// x 2 trajectories x 2 components) and the row writes (a quarter-warp writes the
// same 16 bytes of 2 stages x 4 trajectories).
template <int d2>
struct N8MTile {
    static constexpr int RS = d2 <= 18 ? d2 + ((2 - d2) % 16 + 16) % 16 : d2;  // (N = 7, 8: unpadded, within 48 KB)
    static constexpr int GS0 = 8 * RS + ((8 - 8 * RS) % 16 + 16) % 16;
    static constexpr int SIZE = 3 * GS0 + 4 + 8 * RS;
    static __device__ __forceinline__ int row(int g, int s) { return g * GS0 + (g >> 1) * 4 + s * RS; }
};

// energy samples out of line (rare; inlined twice they push the hot loop out of the
// instruction cache)
template <int NB>
__device__ __noinline__ double n8m_energy(const double *q, const double *v, const NBodyParams &P) {
    return nbody_energy<NB>(q, v, P);
}

// a6 for the components l = s + 8 i of the lane: y_l += S(column l of the stage
// tile), the canonical dadd chain over stages 0..7 (oracle update order); the
// finiteness of the result as a running max of exponent fields (integer pipe)
template <int d, int NO, class Tile>
__device__ __forceinline__ void n8m_owner_update(double *y, const double *X, int g, int s, unsigned &expmax) {
#pragma unroll
    for (int i = 0; i < NO; ++i) {
        const int l = s + 8 * i;
        if (l < d) {
            double sum = X[Tile::row(g, 0) + l];
#pragma unroll
            for (int j = 1; j < 8; ++j) sum = dadd(sum, X[Tile::row(g, j) + l]);
            const double yn = dadd(y[l], sum);
            y[l] = yn;
            const unsigned ex = (unsigned)__double2hiint(yn) & 0x7ff00000u;
            expmax = ex > expmax ? ex : expmax;
        }
    }
}

// Accelerations of all NB bodies at one stage (oracle accel_nbody_pairs, cyclic
// partner order R-8), like n8_accel but each pair difference d = Q_j - Q_i (i < j)
// formed once: body i adds fma(m_j w, d, a), body j adds fma(-(m_i w), d, a) --
// Q_i - Q_j is exactly -d in round-to-nearest, and the negation is an operand
// modifier -- 45 instead of 135 subtractions per stage for N = 6.
template <int NB, bool G1>
__device__ __forceinline__ void n8m_accel(const double *Q, double *A, const NBodyParams &P, const double *sm, bool &ok) {
    constexpr int NP = NB * (NB - 1) / 2;
    double w[NP], dx[NP], dy[NP], dz[NP];
#pragma unroll
    for (int i = 0; i < NB; ++i)
#pragma unroll
        for (int j = 0; j < NB; ++j) {
            if (j <= i) continue;
            const int p = i * NB - i * (i + 1) / 2 + (j - i - 1);
            dx[p] = dsub(Q[3 * j], Q[3 * i]);
            dy[p] = dsub(Q[3 * j + 1], Q[3 * i + 1]);
            dz[p] = dsub(Q[3 * j + 2], Q[3 * i + 2]);
            const double r2 = dfma(dz[p], dz[p], dfma(dy[p], dy[p], dfma(dx[p], dx[p], P.eps2)));
            if (G1) {
                bool unused = true;
                ok = ok && weight_range_ok(r2);
                w[p] = drcp_fast(dmul(r2, dsqrt_fast(r2, unused)), unused);
            } else {
                w[p] = ddiv_fast(P.G, dmul(r2, dsqrt_fast(r2, ok)), ok);
            }
        }
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        double ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll
        for (int delta = 1; delta < NB; ++delta) {
            const int j = (i + delta) % NB;
            const int lo = i < j ? i : j, hi = i < j ? j : i;
            const int p = lo * NB - lo * (lo + 1) / 2 + (hi - lo - 1);
            const double sw = dmul(sm[j], w[p]);
            const double sg = i < j ? sw : -sw;  // (a sign flip: exact)
            ax = dfma(sg, dx[p], ax);
            ay = dfma(sg, dy[p], ay);
            az = dfma(sg, dz[p], az);
        }
        A[3 * i] = ax;
        A[3 * i + 1] = ay;
        A[3 * i + 2] = az;
    }
}

// The same arithmetic as n8m_accel, ordered body by body (N8M_DREUSE = 2): body i
// runs its partners in cyclic order; a pair {lo, hi} is formed (difference, weight)
// at its first use -- by body lo -- and kept until body hi uses it.  The live set is
// the pairs across the cut between finished and pending bodies (<= 9 for N = 6)
// instead of all 15, and each body's acceleration is final when its turn ends.
template <int NB, bool G1>
__device__ __forceinline__ void n8m_accel_bodies(const double *Q, double *A, const NBodyParams &P, const double *sm,
                                                 bool &ok) {
    constexpr int NP = NB * (NB - 1) / 2;
    double w[NP], dx[NP], dy[NP], dz[NP];
#pragma unroll
    for (int i = 0; i < NB; ++i) {
        double ax = 0.0, ay = 0.0, az = 0.0;
#pragma unroll
        for (int delta = 1; delta < NB; ++delta) {
            const int j = (i + delta) % NB;
            const int lo = i < j ? i : j, hi = i < j ? j : i;
            const int p = lo * NB - lo * (lo + 1) / 2 + (hi - lo - 1);
            if (i < j) {  // first use: form the pair
                dx[p] = dsub(Q[3 * j], Q[3 * i]);
                dy[p] = dsub(Q[3 * j + 1], Q[3 * i + 1]);
                dz[p] = dsub(Q[3 * j + 2], Q[3 * i + 2]);
                const double r2 = dfma(dz[p], dz[p], dfma(dy[p], dy[p], dfma(dx[p], dx[p], P.eps2)));
                if (G1) {
                    bool unused = true;
                    ok = ok && weight_range_ok(r2);
                    w[p] = drcp_fast(dmul(r2, dsqrt_fast(r2, unused)), unused);
                } else {
                    w[p] = ddiv_fast(P.G, dmul(r2, dsqrt_fast(r2, ok)), ok);
                }
            }
            const double sw = dmul(sm[j], w[p]);
            const double sg = i < j ? sw : -sw;  // (a sign flip: exact)
            ax = dfma(sg, dx[p], ax);
            ay = dfma(sg, dy[p], ay);
            az = dfma(sg, dz[p], az);
        }
        A[3 * i] = ax;
        A[3 * i + 1] = ay;
        A[3 * i + 2] = az;
    }
}

// B fragments of every tile from the stage tile (both k halves)
template <int T>
__device__ __forceinline__ void n8m_frags(const double *X, int fb0, int fb1, double *b0, double *b1) {
#pragma unroll
    for (int t = 0; t < T; ++t) {
        b0[t] = X[fb0 + 2 * t];
        b1[t] = X[fb1 + 2 * t];
    }
}

template <int T>
__device__ __forceinline__ void n8m_contract(double *D, double a0, double a1, const double *b0, const double *b1) {
#pragma unroll
    for (int t = 0; t < T; ++t) dmma884(D[2 * t], D[2 * t + 1], a0, b0[t], -0.0, -0.0);
#pragma unroll
    for (int t = 0; t < T; ++t) dmma884(D[2 * t], D[2 * t + 1], a1, b1[t], D[2 * t], D[2 * t + 1]);
}

// MR: register cap.  N8M_MAXREG (168) at full load -- 12 warps per SM were the
// measured optimum; 255 for small batches (a few warps per SM: no occupancy to lose,
// no spills, more of the 15 pair chains in flight; 2,048 trajectories -11 %).
template <int NB, bool G1, int MR = N8M_MAXREG>
__global__ void __maxnreg__(MR) ens_nbody8m_kernel(const __grid_constant__ EnsArgs a,
                                                         const __grid_constant__ QueueArgs qa,
                                                         const __grid_constant__ NBodyParams P) {
    constexpr int d = 3 * NB, D = 6 * NB, T = (d + 1) / 2, d2 = 2 * T, WPB = N8M_THREADS / 32;
    using Tile = N8MTile<d2>;
    // q, v rows of the slot's 4 trajectories (q at 0, v at VO: 16-byte aligned pairs);
    // row stride with QS / 2 odd: the 4 rows' 16-byte loads at one component fall in
    // different banks
    constexpr int VO = d2, QS = 2 * d2 + 2;
    constexpr int NO = (d + 7) / 8;  // components owned per lane (l = s + 8 i) for Delta and the update
    const unsigned FULL = 0xffffffffu;
    const int64_t B = a.batch;
    const int tx = threadIdx.x, L = tx & 31, wib = tx >> 5;
    const int s = L >> 2, g = L & 3;
    const unsigned gmask = 0x11111111u << g;

    __shared__ __align__(16) double sQV[WPB][4][QS];
    __shared__ __align__(16) double sX[WPB][Tile::SIZE];   // Lq or Lv rows (g, s)
    __shared__ __align__(16) int64_t sE[WPB][Tile::SIZE];  // |Q_s - Q_s^old| bits
#if N8M_QSMEM
    __shared__ double sQ[WPB][d2][32];  // Q^[k-1] of lane L at [l][L] (conflict-free)
#define N8M_Q(l) sQ[wib][l][L]
#else
    double Q[d2];
#define N8M_Q(l) Q[l]
#endif
    __shared__ double sm[NB];
    for (int e = tx; e < NB; e += N8M_THREADS) sm[e] = P.m[e];
    __syncthreads();
    double *qv = &sQV[wib][g][0];
    double *X = &sX[wib][0];
    int64_t *E = &sE[wib][0];
    const int myrow = Tile::row(g, s);
    // B fragment of tile t, k half kk at X[fb_kk + 2 t]: B[k][n] with k = L % 4
    // (stage 4 kk + k), n = L / 4 (trajectory n / 2, component 2 t + n % 2)
    const int fb0 = Tile::row(L >> 3, L & 3) + ((L >> 2) & 1), fb1 = Tile::row(L >> 3, 4 + (L & 3)) + ((L >> 2) & 1);
    // coefficient fragments A[m = s][k = L % 4] of mu~, nu~ for k halves 0, 1
    const double aM0 = c_mu[s][L & 3], aM1 = c_mu[s][4 + (L & 3)];
    const double aN0 = c_nu[s][L & 3], aN1 = c_nu[s][4 + (L & 3)];
    const double hb_s = a.hb[s];

    const int64_t n0 = *a.n_done;
    const bool sample = (a.energy != nullptr) && (a.energy_every > 0);
    const int64_t nslots = (B + 3) / 4, total = nslots * qa.nchunks;

#pragma unroll
    for (int l = 0; l < d2; ++l) N8M_Q(l) = 0.0;
    int64_t m[NO], p[NO];
#pragma unroll
    for (int i = 0; i < NO; ++i) m[i] = p[i] = kInfBits;
    int64_t w = -1, c = 0, b = 0, len = 0, n = 0, hits = 0, sweeps = 0;
    double hprev = 0.0, dhmax = 0.0;
    int k = 0;
    bool live = false;  // this lane's trajectory is integrating in the current unit
    for (;;) {
        if (w < 0) {  // ---- acquire a slot unit (warp-uniform) ----
            unsigned long long uu = 0;
            if (L == 0) uu = atomicAdd(qa.counter, 1ull);
            uu = __shfl_sync(FULL, uu, 0);
            if ((int64_t)uu >= total) break;
            c = (int64_t)uu / nslots;
            w = (int64_t)uu - c * nslots;
            // issued nslots units after its predecessor: rarely still running (every lane
            // acquires, so each lane's loads below are ordered after the release)
            if (c > 0)
                while (ld_acquire(&qa.progress[w]) < c) __nanosleep(256);
            b = 4 * w + g;
            const bool valid = b < B;
            const int64_t bb = valid ? b : 0;
            const int64_t c0 = c * qa.qchunk;
            len = (a.nsteps - c0 < qa.qchunk) ? a.nsteps - c0 : qa.qchunk;
            if (valid)
                for (int l = s; l < D; l += 8) qv[l < d ? l : VO + l - d] = __ldcg(&a.y[(int64_t)l * B + b]);
#pragma unroll
            for (int l = 0; l < d2; ++l)
                X[myrow + l] = (valid && l < d) ? __ldcg(&a.hist[((int64_t)s * D + d + l) * B + bb]) : 0.0;
            __syncwarp();
            const bool frozen = !valid || __ldcg(&a.stats[1 * B + bb]) > 0 || len <= 0;
            if (valid && s == 0 && ((sample && c == 0) || a.local_energy)) {
                const double h0 = n8m_energy<NB>(qv, qv + VO, P);
                if (sample && c == 0) a.energy[b] = h0;
                hprev = h0;
            }
            dhmax = 0.0;
            if (valid && frozen && s == 0 && c == 0) {
                if (a.local_energy) a.stats[3 * B + b] = 0;
                if (a.iters) a.iters[b] = 0;
            }
            live = !frozen;
            n = hits = sweeps = 0;
            k = 0;
#pragma unroll
            for (int i = 0; i < NO; ++i) m[i] = p[i] = kInfBits;
            // a1: V_s = v + D(nu_s., H) from the history rows; Lq = hb_s V_s -> own row
            __syncwarp();  // converged for the DMMAs (after the divergent sample above)
            double Dv[d2];
            {
                double b0[T], b1[T];
                n8m_frags<T>(X, fb0, fb1, b0, b1);
                n8m_contract<T>(Dv, aN0, aN1, b0, b1);
            }
            __syncwarp();  // fragments read before the rows are overwritten
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const double2 vv = *reinterpret_cast<const double2 *>(&qv[VO + 2 * t]);
                *reinterpret_cast<double2 *>(&X[myrow + 2 * t]) =
                    make_double2(dmul(hb_s, dadd(vv.x, Dv[2 * t])), dmul(hb_s, dadd(vv.y, Dv[2 * t + 1])));
            }
        }
        if (live) ++k;
        // the stop test runs from the second sweep of a step (Delta^[1] is not tested):
        // sweeps where no trajectory of the slot tests skip the E tile
        const bool k2 = live && k >= 2;
        const bool anyk2 = __any_sync(FULL, k2);
        __syncwarp();  // Lq rows written
        // ---- a2: Q_s = q + D(mu_s., Lq) ; |Q_s - Q_s^old| -> own row of E ----
#if N8M_QKEEP
        double Qk[d2];  // this sweep's Q_s, kept for the RHS (the shared copy is next sweep's Q^old)
#endif
        {
            double b0[T], b1[T], Dq[d2];
            n8m_frags<T>(X, fb0, fb1, b0, b1);
            n8m_contract<T>(Dq, aM0, aM1, b0, b1);
#if N8M_A2SYNC
            __syncwarp();  // (a scheduling fence: the nine DMMA chains issue before their consumers)
#endif
#pragma unroll
            for (int t = 0; t < T; ++t) {
                const double d0 = Dq[2 * t], d1 = Dq[2 * t + 1];
                const double2 qq = *reinterpret_cast<const double2 *>(&qv[2 * t]);
                const double q0 = dadd(qq.x, d0), q1 = dadd(qq.y, d1);
                longlong2 e;
                e.x = absdiff_bits(q0, N8M_Q(2 * t));
                e.y = (2 * t + 1 < d) ? absdiff_bits(q1, N8M_Q(2 * t + 1)) : 0;
                if (anyk2) *reinterpret_cast<longlong2 *>(&E[myrow + 2 * t]) = e;
                N8M_Q(2 * t) = q0;
                N8M_Q(2 * t + 1) = q1;
#if N8M_QKEEP
                Qk[2 * t] = q0;
                Qk[2 * t + 1] = q1;
#endif
            }
        }
        __syncwarp();  // E rows written
        // ---- a5: Delta_l (NaN-ignoring max over the 8 stages) and reading R2 for the
        // owned components l = s + 8 i ----
        bool ok_lane = true;
#pragma unroll
        for (int i = 0; i < NO; ++i) {
            const int l = s + 8 * i;
            if (anyk2 && l < d) {
                int64_t ev[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) ev[j] = E[Tile::row(g, j) + l];
                const int64_t delta = delta_bits8(ev);
                ok_lane = ok_lane && ((delta == 0) || (m[i] <= imin64(delta, p[i])));
                m[i] = k2 ? imin64(p[i], m[i]) : m[i];
                p[i] = k2 ? delta : p[i];
            }
        }
        const unsigned notok = __ballot_sync(FULL, !ok_lane);
        const bool stop = k2 && ((notok & gmask) == 0u);
        const bool fin = live && (stop || k >= a.max_iters);
        const unsigned finmask = __ballot_sync(FULL, fin), livemask = __ballot_sync(FULL, live);
        const bool anyfin = finmask != 0u, allfin = (finmask & livemask) == livemask;
        // ---- a6 (positions): q += S(Lq) by the component owners, from the Lq tile ----
        unsigned expmax = 0;  // non-finite result <=> an exponent field of all ones
        if (fin) n8m_owner_update<d, NO, Tile>(qv, X, g, s, expmax);
        // ---- a3: F_s ; Lv_s = hb_s F_s -> own row ----
        {
            double F[d], Qs[d];
#pragma unroll
            for (int l = 0; l < d; ++l) {
#if N8M_QKEEP
                Qs[l] = Qk[l];
#else
                Qs[l] = N8M_Q(l);
#endif
            }
            bool ok = true;
#if N8M_DREUSE == 2
            n8m_accel_bodies<NB, G1>(Qs, F, P, N8M_CMASS ? P.m : sm, ok);
#elif N8M_DREUSE
            n8m_accel<NB, G1>(Qs, F, P, N8M_CMASS ? P.m : sm, ok);
#else
            n8_accel<NB, false, G1>(Qs, F, P, sm, ok);
#endif
#if N8M_UNIFORM_EXACT
            if (__any_sync(FULL, !ok && live)) {  // exact intrinsics, same bits (out of line, rare; warp-uniform)
#else
            if (!ok && live) {  // exact intrinsics, same bits (out of line, rare)
#endif
                double row[d];
#pragma unroll
                for (int l = 0; l < d; ++l) row[l] = Qs[l];
                n8_accel_exact_row<NB>(row, P, sm);
#pragma unroll
                for (int l = 0; l < d; ++l) F[l] = row[l];
            }
            __syncwarp();  // every lane has read its Lq fragments
#pragma unroll
            for (int t = 0; t < T; ++t)
                *reinterpret_cast<double2 *>(&X[myrow + 2 * t]) =
                    make_double2(dmul(hb_s, F[2 * t]), (2 * t + 1 < d) ? dmul(hb_s, F[2 * t + 1]) : 0.0);
        }
        __syncwarp();  // Lv rows written
        // ---- a4: D = W Lv (W per trajectory) ----
        double Dv[d2];
        {
            double b0[T], b1[T];
            n8m_frags<T>(X, fb0, fb1, b0, b1);
            // one pass with the slot's common W; a second (nu~) pass if the slot's
            // live trajectories disagree
            const bool nu = anyfin && allfin;
            const double w0 = nu ? aN0 : aM0, w1 = nu ? aN1 : aM1;
            n8m_contract<T>(Dv, w0, w1, b0, b1);
            if ((anyfin && !allfin)) {
                double Dn[d2];
                n8m_contract<T>(Dn, aN0, aN1, b0, b1);
#pragma unroll
                for (int l = 0; l < d2; ++l) Dv[l] = fin ? Dn[l] : Dv[l];
            }
        }
        if (fin) n8m_owner_update<d, NO, Tile>(qv + VO, X, g, s, expmax);  // a6 (velocities) from the Lv tile
        const unsigned nonfinite = __ballot_sync(FULL, expmax == 0x7ff00000u);  // (every lane votes)
        const bool bad = fin && ((nonfinite & gmask) != 0u);
        __syncwarp();  // v updated; every lane has read its Lv fragments
        if (fin) {
            ++n;
            sweeps += k;
            hits += stop ? 0 : 1;
            k = 0;
#pragma unroll
            for (int i = 0; i < NO; ++i) m[i] = p[i] = kInfBits;
        }
        const int64_t nloc = c * qa.qchunk + n;
        if (fin && (sample || a.local_energy) && s == 0) {  // (sample test first: no divergent branch per step)
            const bool due = sample && (nloc % a.energy_every) == 0;
            if (due || a.local_energy) {
                const double hn = n8m_energy<NB>(qv, qv + VO, P);
                if (due) a.energy[(nloc / a.energy_every) * B + b] = hn;
                if (a.local_energy) dhloc_update(hn, hprev, dhmax);
            }
        }
        const bool release = fin && (n == len || bad);
        if (release) {  // history row s = Lv_s (q block zeroed, R-4); state, stats
#pragma unroll
            for (int l = 0; l < d; ++l) {
                a.hist[((int64_t)s * D + l) * B + b] = 0.0;
                a.hist[((int64_t)s * D + d + l) * B + b] = X[myrow + l];
            }
            for (int l = s; l < D; l += 8) a.y[(int64_t)l * B + b] = qv[l < d ? l : VO + l - d];
            if (s == 0) {
                a.stats[0 * B + b] = __ldcg(&a.stats[0 * B + b]) + hits;
                if (bad) a.stats[1 * B + b] = n0 + nloc;
                a.stats[2 * B + b] = __ldcg(&a.stats[2 * B + b]) + sweeps;
                if (a.iters) a.iters[b] = (c == 0) ? sweeps : __ldcg(&a.iters[b]) + sweeps;
                if (a.local_energy) dhloc_store(&a.stats[3 * B + b], c == 0, dhmax);
            }
            live = false;
        }
        // V_s = v + D ; next sweep's Lq_s = hb_s V_s -> own row (own Lv row read above)
#pragma unroll
        for (int t = 0; t < T; ++t) {
            const double2 vv = *reinterpret_cast<const double2 *>(&qv[VO + 2 * t]);
            *reinterpret_cast<double2 *>(&X[myrow + 2 * t]) =
                make_double2(dmul(hb_s, dadd(vv.x, Dv[2 * t])), dmul(hb_s, dadd(vv.y, Dv[2 * t + 1])));
        }
        if (!__any_sync(FULL, live)) {  // slot unit done: publish it
            __threadfence();
            __syncwarp();
            if (L == 0) st_release(&qa.progress[w], (int32_t)(c + 1));
            w = -1;
        }
    }
}
#undef N8M_Q

}  // namespace irk
