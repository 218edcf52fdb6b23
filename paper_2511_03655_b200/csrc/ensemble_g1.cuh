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

#include "ens_common.cuh"
#include "fp64.cuh"

namespace irk {

#ifndef G1_BLOCK
#define G1_BLOCK 64
#endif
constexpr int G1_THREADS = G1_BLOCK;
#ifndef G1Q_QREG
#define G1Q_QREG 1  // the heavy ens_g1q keeps the stage positions in registers
#endif
#ifndef G1Q_HEAVY_MAXREG
#define G1Q_HEAVY_MAXREG 240  // ens_g1q at <= 5 blocks per SM (launch geometry in irk_api.cu launch_g1q)
#endif
#ifndef G1_MAXREG
#define G1_MAXREG 168    // measured best on config 2 (tools/variants.py): 128: 116 ms, 144: 136, 168: 107, 190+: 109-111
#endif
#ifndef G1_V_SMEM
#define G1_V_SMEM 0      // keep V^[k] in shared memory instead of registers
#endif
#ifndef G1_RHS_ILP
#define G1_RHS_ILP 8     // stages per trip of the RHS loop (8: 107 ms, 4: 145 ms at 168 regs)
#endif

template <class P>
__global__ void __maxnreg__(G1_MAXREG) ens_g1_kernel(const __grid_constant__ EnsArgs a,
                                                    const __grid_constant__ P prob) {
    constexpr int d = P::d, D = 2 * d;
    const int64_t B = a.batch;
    const int64_t slot = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    __shared__ __align__(16) double sW[2][64];  // [0] = mu~, [1] = nu~ (row-major)
    for (int e = threadIdx.x; e < 128; e += blockDim.x) sW[e >> 6][e & 63] = (e < 64) ? (&c_mu[0][0])[e] : (&c_nu[0][0])[e - 64];
    __syncthreads();
    if (slot >= a.nslots) return;
    const int64_t b = a.perm ? (int64_t)a.perm[slot] : slot;
    if (b < 0 || b >= B) return;

    int64_t bad = a.stats[1 * B + b];
    int64_t hits = 0, sweeps = 0;
    // Q^[k-1] (only compared against, once per sweep) and the stop-test history
    // (m, p) live in shared memory, [element][thread] so that the 64-bit accesses
    // of a warp hit 32 distinct banks; registers are kept for V, the fresh Q^[k]
    // and the RHS temporaries (ILP across the eight stages).
    __shared__ double sQ[8 * d][G1_THREADS], sL[8 * d][G1_THREADS], sM[d][G1_THREADS], sP[d][G1_THREADS];
    const int tx = threadIdx.x;
#if G1_V_SMEM
    __shared__ double sV[8 * d][G1_THREADS];  // V^[k] between a4 and the next a2
#define G1_V(i, l) sV[(i) * d + (l)][tx]
#else
    double V[8][d];
#define G1_V(i, l) V[i][l]
#endif
    double q[d], v[d];
#pragma unroll
    for (int l = 0; l < d; ++l) {
        q[l] = a.y[l * B + b];
        v[l] = a.y[(d + l) * B + b];
    }
    const int64_t n0 = *a.n_done;
    const bool sample = (a.energy != nullptr) && (a.energy_every > 0);
    if (sample && a.c0 == 0) a.energy[b] = prob.energy(q, v);
    double hprev = a.local_energy ? prob.energy(q, v) : 0.0, dhmax = 0.0;
    if (bad > 0 || a.nsteps == 0) {  // frozen (diverged at step `bad`, 1-based) or nothing to do
        if (a.local_energy && a.c0 == 0) a.stats[3 * B + b] = 0;
        if (a.iters && a.c0 == 0) a.iters[b] = 0;
        if (a.csweeps) a.csweeps[b] = 0;
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
                double acc = dmul(c_nu[i][0], H[0][l]);
#pragma unroll
                for (int j = 1; j < 8; ++j) acc = dfma(c_nu[i][j], H[j][l], acc);
                G1_V(i, l) = dadd(v[l], acc);
            }
    }
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
    for (int l = 0; l < d; ++l) sM[l][tx] = sP[l][tx] = kInf;

    int64_t n = 0;
    int k = 0;
    while (n < a.nsteps) {
        ++k;
        // a2: Lq_j = hb_j V_j ; Q_i^[k] = q + D(mu_i., Lq)   (+ a5 on the fly).
        // S(Lq) is formed here (same left-to-right order as the update needs) so
        // that Lq dies before the RHS: 16 fewer live doubles across a3.
        double Lq[8][d], sLq[d];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int l = 0; l < d; ++l) Lq[j][l] = dmul(a.hb[j], G1_V(j, l));
#pragma unroll
        for (int l = 0; l < d; ++l) {
            sLq[l] = Lq[0][l];
#pragma unroll
            for (int j = 1; j < 8; ++j) sLq[l] = dadd(sLq[l], Lq[j][l]);
        }
        bool stop = (k >= 2);
        double delta[d];
        {
            double ev[d][8];
            const double2 *M = reinterpret_cast<const double2 *>(&c_mu[0][0]);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double2 w[4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) w[jj] = M[i * 4 + jj];
#pragma unroll
                for (int l = 0; l < d; ++l) {
                    double acc = dmul(w[0].x, Lq[0][l]);
                    acc = dfma(w[0].y, Lq[1][l], acc);
#pragma unroll
                    for (int jj = 1; jj < 4; ++jj) {
                        acc = dfma(w[jj].x, Lq[2 * jj][l], acc);
                        acc = dfma(w[jj].y, Lq[2 * jj + 1][l], acc);
                    }
                    const double qn = dadd(q[l], acc);
                    ev[l][i] = dabs(dsub(qn, sQ[i * d + l][tx]));  // garbage at k = 1, unused
                    sQ[i * d + l][tx] = qn;
                }
            }
#pragma unroll
            for (int l = 0; l < d; ++l) delta[l] = delta_max8(ev[l]);
        }
        if (k >= 2) {  // a5, reading R2: Delta^[k] exists from k = 2
#pragma unroll
            for (int l = 0; l < d; ++l) {
                const double pl = sP[l][tx], ml = sM[l][tx];
                const double mn = (delta[l] < pl) ? delta[l] : pl;
                const bool ok = (delta[l] == 0.0) || (ml <= mn);
                sM[l][tx] = (pl < ml) ? pl : ml;
                sP[l][tx] = delta[l];
                stop = stop && ok;
            }
        }
        // a3 + a4 (first half): F_i = g(Q_i, t_i) ; Lv_i = hb_i F_i, G1_RHS_ILP stages per
        // trip (ILP for the ~20-deep dependent div/sqrt chains, bounded register use).
        const double tn1 = dadd(a.t0, dmul((double)(n0 + n), a.h));
        double Lv[8][d];
#if G1_RHS_ILP == 8
        {   // all eight stages in flight, results straight into registers
            bool ok = true;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double Qi[d];
#pragma unroll
                for (int l = 0; l < d; ++l) Qi[l] = sQ[i * d + l][tx];
                prob.template accel<false>(Qi, Lv[i], dadd(tn1, dmul(c_c[i], a.h)), ok);
            }
            if (!ok) {  // some stage needs the exact slow path of div/sqrt: redo all, same bits
#pragma unroll 1
                for (int i = 0; i < 8; ++i) {
                    double Qi[d], Fi[d];
#pragma unroll
                    for (int l = 0; l < d; ++l) Qi[l] = sQ[i * d + l][tx];
                    prob.template accel<true>(Qi, Fi, dadd(tn1, dmul(c_c[i], a.h)), ok);
#pragma unroll
                    for (int l = 0; l < d; ++l) sL[i * d + l][tx] = Fi[l];
                }
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int l = 0; l < d; ++l) Lv[i][l] = sL[i * d + l][tx];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int l = 0; l < d; ++l) Lv[i][l] = dmul(a.hb[i], Lv[i][l]);
        }
#else
        {
            bool ok = true;
#pragma unroll 1
            for (int i0 = 0; i0 < 8; i0 += G1_RHS_ILP) {
#pragma unroll
                for (int i = i0; i < i0 + G1_RHS_ILP; ++i) {
                    double Qi[d], Fi[d];
#pragma unroll
                    for (int l = 0; l < d; ++l) Qi[l] = sQ[i * d + l][tx];
                    prob.template accel<false>(Qi, Fi, dadd(tn1, dmul(c_c[i], a.h)), ok);
#pragma unroll
                    for (int l = 0; l < d; ++l) sL[i * d + l][tx] = dmul(a.hb[i], Fi[l]);
                }
            }
            if (!ok) {  // some stage needs the exact slow path of div/sqrt: redo all, same bits
#pragma unroll 1
                for (int i = 0; i < 8; ++i) {
                    double Qi[d], Fi[d];
#pragma unroll
                    for (int l = 0; l < d; ++l) Qi[l] = sQ[i * d + l][tx];
                    prob.template accel<true>(Qi, Fi, dadd(tn1, dmul(c_c[i], a.h)), ok);
#pragma unroll
                    for (int l = 0; l < d; ++l) sL[i * d + l][tx] = dmul(a.hb[i], Fi[l]);
                }
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int l = 0; l < d; ++l) Lv[i][l] = sL[i * d + l][tx];
#endif
        const bool fin = stop || (k >= a.max_iters);
        if (fin) {  // a6: update with the last iteration's L, history <- Lv
            bool finite = true;
#pragma unroll
            for (int l = 0; l < d; ++l) {
                double sv = Lv[0][l];
#pragma unroll
                for (int j = 1; j < 8; ++j) sv = dadd(sv, Lv[j][l]);
                q[l] = dadd(q[l], sLq[l]);
                v[l] = dadd(v[l], sv);
                finite = finite && isfinite(q[l]) && isfinite(v[l]);
            }
            ++n;
            sweeps += k;
            hits += stop ? 0 : 1;
            k = 0;
#pragma unroll
            for (int l = 0; l < d; ++l) sM[l][tx] = sP[l][tx] = kInf;
            if (sample && ((a.c0 + n) % a.energy_every) == 0)
                a.energy[((a.c0 + n) / a.energy_every) * B + b] = prob.energy(q, v);
            if (a.local_energy) dhloc_update(prob.energy(q, v), hprev, dhmax);
            if (n == a.nsteps || !finite) {  // history = Lv (Eq. IRK_init2 extrapolates only
                                             // velocities); the q block is zeroed (R-4)
#pragma unroll
                for (int j = 0; j < 8; ++j)
#pragma unroll
                    for (int l = 0; l < d; ++l) {
                        a.hist[((int64_t)j * D + l) * B + b] = 0.0;
                        a.hist[((int64_t)j * D + d + l) * B + b] = Lv[j][l];
                    }
                if (!finite) bad = n0 + n;
                break;
            }
        }
        // a4 (second half) / next step's a1: V_i = v + D(W_i., Lv), W = fin ? nu : mu.
        // Lanes of a warp disagree on `fin` almost every sweep, so W is read from a
        // shared-memory copy of both tables (two broadcast addresses per LDS.128)
        // instead of per-coefficient selects.
        {
            const double2 *W = reinterpret_cast<const double2 *>(&sW[fin ? 1 : 0][0]);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double2 w[4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) w[jj] = W[i * 4 + jj];
#pragma unroll
                for (int l = 0; l < d; ++l) {
                    double acc = dmul(w[0].x, Lv[0][l]);
                    acc = dfma(w[0].y, Lv[1][l], acc);
#pragma unroll
                    for (int jj = 1; jj < 4; ++jj) {
                        acc = dfma(w[jj].x, Lv[2 * jj][l], acc);
                        acc = dfma(w[jj].y, Lv[2 * jj + 1][l], acc);
                    }
                    G1_V(i, l) = dadd(v[l], acc);
                }
            }
        }
    }
#undef G1_V
#pragma unroll
    for (int l = 0; l < d; ++l) {
        a.y[l * B + b] = q[l];
        a.y[(d + l) * B + b] = v[l];
    }
    a.stats[0 * B + b] += hits;
    a.stats[1 * B + b] = bad;
    a.stats[2 * B + b] += sweeps;
    if (a.iters) a.iters[b] = (a.c0 == 0) ? sweeps : a.iters[b] + sweeps;
    if (a.csweeps) a.csweeps[b] = (int32_t)sweeps;
    if (a.local_energy) dhloc_store(&a.stats[3 * B + b], a.c0 == 0, dhmax);
}

}  // namespace irk

namespace irk {

// ---------------------------------------------------------------------------
// ens_g1q: the g1 mapping as ONE persistent launch with a per-lane work queue.
//
// The chunked ens_g1 launches B threads per chunk; at 168 registers a B200 holds
// 148 x 384 = 56,832 of them, so config 2 (B = 65,536) runs 1.15 waves and the
// partial wave idles most of the GPU (ncu, profiles/r1: 87% of cycles active).
// Here the grid is exactly the resident capacity and every lane pulls work
// units u = c*B + b (trajectory b, step chunk c of `qchunk` steps) from a global
// counter; a lane that finishes a unit stores (y, history, stats), publishes
// progress[b] = c + 1 and pulls the next unit in the same sweep-granular loop,
// so lanes stay busy until the queue drains (tail <= one unit).  Unit (b, c)
// waits (idle trips) until unit (b, c-1) is published; it was issued B units
// earlier, so this is rare.  Each unit does exactly the arithmetic of the
// corresponding chunk of ens_g1 (same nu-init from the stored history, same
// absolute step index), so results are bitwise those of any other schedule.
//
// The stop test's comparisons run on the integer pipe: every operand is a
// non-negative, non-NaN double (|.|, NaN mapped to 0 as the canonical
// NaN-ignoring max does, +inf for "no history"), whose IEEE order is the order
// of the bit patterns as int64.

__device__ __forceinline__ int64_t dbits(double x) { return __double_as_longlong(x); }
// |a - b| as bits (NaN stays above +inf: a NaN-ignoring max is taken separately)
__device__ __forceinline__ int64_t absdiff_bits(double a, double b) {
    return dabs_bits(dsub(a, b));  // integer-pipe mask (fp64.cuh)
}
__device__ __forceinline__ int64_t imax64(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
constexpr int64_t kInfBits = 0x7ff0000000000000LL;
// Delta = NaN-ignoring max of eight |differences| (the canonical left-to-right
// `(e > d) ? e : d` from d = 0).  Plain max first; only if it is a NaN pattern
// (a diverging trajectory) are the NaNs dropped, so the common case costs 7
// int64 max operations.
__device__ __forceinline__ int64_t delta_bits8(const int64_t *e) {
    int64_t t = imax64(imax64(imax64(e[0], e[1]), imax64(e[2], e[3])), imax64(imax64(e[4], e[5]), imax64(e[6], e[7])));
    if (t > kInfBits) {
        t = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) t = (e[i] > kInfBits) ? t : imax64(t, e[i]);
    }
    return t;
}

template <class P, int MAXREG = G1_MAXREG>
__global__ void __maxnreg__(MAXREG) ens_g1q_kernel(const __grid_constant__ EnsArgs a,
                                                     const __grid_constant__ QueueArgs qa,
                                                     const __grid_constant__ P prob) {
    constexpr int d = P::d, D = 2 * d;
    const int64_t B = a.batch;
    // mu~ at [0, 64), nu~ at [66, 130): the 2-double gap puts the two tables in
    // different banks, so the per-lane (mu or nu) LDS.128 of a4 is conflict-free
    // (unpadded: 7.65 instead of 3.9 shared wavefronts per load, ncu)
    constexpr int kNuOff = 66;
    __shared__ __align__(16) double sW[kNuOff + 64];
    for (int e = threadIdx.x; e < 128; e += blockDim.x)
        sW[(e < 64) ? e : kNuOff + e - 64] = (e < 64) ? (&c_mu[0][0])[e] : (&c_nu[0][0])[e - 64];
    __syncthreads();
    // Q^[k] (read by the RHS and, as Q^[k-1], by the next sweep's Delta): in registers
    // when the register budget allows (the <= 5-blocks-per-SM instantiation), else in
    // shared memory [element][thread] (conflict-free)
    constexpr bool QREG = MAXREG >= 200 && G1Q_QREG;
    __shared__ double sQ[QREG ? 1 : 8 * d][G1_THREADS], sL[8 * d][G1_THREADS];
    double Qr[8][d];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int l = 0; l < d; ++l) Qr[i][l] = 0.0;
    // stop-test state (m, p) per component: registers in the heavy instantiation
    __shared__ int64_t sM[QREG ? 1 : d][G1_THREADS], sP[QREG ? 1 : d][G1_THREADS];
    int64_t rM[d], rP[d];
#pragma unroll
    for (int l = 0; l < d; ++l) rM[l] = rP[l] = 0x7ff0000000000000LL;
#define G1Q_M(l) (*(QREG ? &rM[l] : &sM[l][tx]))
#define G1Q_P(l) (*(QREG ? &rP[l] : &sP[l][tx]))
    const int tx = threadIdx.x;
    const int64_t n0 = *a.n_done;
    const bool sample = (a.energy != nullptr) && (a.energy_every > 0);
    const int64_t total = B * qa.nchunks;

    double q[d], v[d], V[8][d];
    int32_t b = -1;  // trajectory of the held unit (-1: none)
    int64_t c = 0, len = 0, n = 0, hits = 0, sweeps = 0, u = -1;
    double hprev = 0.0, dhmax = 0.0;
    int k = 0;
    int32_t bb = 0;
#ifdef IRK_TRACE
    unsigned long long t_fetch = 0, t_start = 0;
#endif
    for (;;) {
        if (b < 0) {  // ---- acquire the next unit (divergent, once per unit) ----
            if (u < 0) {
                u = (int64_t)atomicAdd(qa.counter, 1ull);
                if (u >= total) break;
                c = u / B;
                bb = (int32_t)(u - c * B);
#ifdef IRK_TRACE
                t_fetch = irk_now();
#endif
            }
            if (c > 0 && ld_acquire(&qa.progress[bb]) < c) {  // predecessor unit still running
                __nanosleep(1024);
                continue;
            }
#ifdef IRK_TRACE
            t_start = irk_now();
#endif
            u = -1;
            b = bb;
            const int64_t c0 = c * qa.qchunk;
            len = (a.nsteps - c0 < qa.qchunk) ? a.nsteps - c0 : qa.qchunk;
#pragma unroll
            for (int l = 0; l < d; ++l) {
                q[l] = __ldcg(&a.y[l * B + b]);  // L2: written by another SM's unit
                v[l] = __ldcg(&a.y[(d + l) * B + b]);
            }
            if (sample && c == 0) a.energy[b] = prob.energy(q, v);
            hprev = a.local_energy ? prob.energy(q, v) : 0.0;
            dhmax = 0.0;
            if (__ldcg(&a.stats[1 * B + b]) > 0 || len <= 0) {  // frozen (diverged earlier): nothing to do
                if (c == 0) {
                    if (a.local_energy) a.stats[3 * B + b] = 0;
                    if (a.iters) a.iters[b] = 0;
                }
                st_release(&qa.progress[b], (int32_t)(c + 1));
                b = -1;
                continue;
            }
            {   // a1: nu-init from the history (zeros = first step of the run)
                double H[8][d];
#pragma unroll
                for (int j = 0; j < 8; ++j)
#pragma unroll
                    for (int l = 0; l < d; ++l) H[j][l] = __ldcg(&a.hist[((int64_t)j * D + d + l) * B + b]);
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int l = 0; l < d; ++l) {
                        double acc = dmul(c_nu[i][0], H[0][l]);
#pragma unroll
                        for (int j = 1; j < 8; ++j) acc = dfma(c_nu[i][j], H[j][l], acc);
                        V[i][l] = dadd(v[l], acc);
                    }
            }
#pragma unroll
            for (int l = 0; l < d; ++l) G1Q_M(l) = G1Q_P(l) = kInfBits;
            n = hits = sweeps = 0;
            k = 0;
        }
        ++k;
        // a2: Lq_j = hb_j V_j ; Q_i^[k] = q + D(mu_i., Lq)  (+ a5 on the fly)
        double Lq[8][d], sLq[d];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int l = 0; l < d; ++l) Lq[j][l] = dmul(a.hb[j], V[j][l]);
#pragma unroll
        for (int l = 0; l < d; ++l) {
            sLq[l] = Lq[0][l];
#pragma unroll
            for (int j = 1; j < 8; ++j) sLq[l] = dadd(sLq[l], Lq[j][l]);
        }
        bool stop = (k >= 2);
        int64_t delta[d];
        {
            int64_t ev[d][8];
            const double2 *M = reinterpret_cast<const double2 *>(&c_mu[0][0]);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double2 w[4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) w[jj] = M[i * 4 + jj];
#pragma unroll
                for (int l = 0; l < d; ++l) {
                    double acc = dmul(w[0].x, Lq[0][l]);
                    acc = dfma(w[0].y, Lq[1][l], acc);
#pragma unroll
                    for (int jj = 1; jj < 4; ++jj) {
                        acc = dfma(w[jj].x, Lq[2 * jj][l], acc);
                        acc = dfma(w[jj].y, Lq[2 * jj + 1][l], acc);
                    }
                    const double qn = dadd(q[l], acc);
                    if (QREG) {
                        ev[l][i] = absdiff_bits(qn, Qr[i][l]);  // garbage at k = 1, unused
                        Qr[i][l] = qn;
                    } else {
                        ev[l][i] = absdiff_bits(qn, sQ[i * d + l][tx]);
                        sQ[i * d + l][tx] = qn;
                    }
                }
            }
#pragma unroll
            for (int l = 0; l < d; ++l) delta[l] = delta_bits8(ev[l]);
        }
        {   // a5, reading R2 (Delta^[k] exists from k = 2), on the bit patterns; branch-free
            // (selects) so that lanes at k = 1 and k >= 2 do not diverge
            const bool k2 = k >= 2;
#pragma unroll
            for (int l = 0; l < d; ++l) {
                const int64_t pl = G1Q_P(l), ml = G1Q_M(l);
                const bool ok = (delta[l] == 0) || (ml <= imin64(delta[l], pl));
                G1Q_M(l) = k2 ? imin64(pl, ml) : ml;
                G1Q_P(l) = k2 ? delta[l] : pl;
                stop = stop && ok;   // (stop starts as k >= 2)
            }
        }
        // a3 + a4 (first half): F_i = g(Q_i, t_i) ; Lv_i = hb_i F_i, all eight stages in flight
        const int64_t nabs = n0 + c * qa.qchunk + n;  // absolute index of the step being taken
        const double tn1 = dadd(a.t0, dmul((double)nabs, a.h));
        double Lv[8][d];
        {
            bool ok = true;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double Qi[d];
#pragma unroll
                for (int l = 0; l < d; ++l) Qi[l] = QREG ? Qr[i][l] : sQ[i * d + l][tx];
                prob.template accel<false>(Qi, Lv[i], dadd(tn1, dmul(c_c[i], a.h)), ok);
            }
            if (!ok) {  // some stage needs the exact slow path of div/sqrt: redo all, same bits
                if (QREG)  // through shared memory (a register array indexed in a rolled loop would
#pragma unroll             // put Qr in local memory for the whole kernel)
                    for (int i = 0; i < 8; ++i)
#pragma unroll
                        for (int l = 0; l < d; ++l) sL[i * d + l][tx] = Qr[i][l];
#pragma unroll 1
                for (int i = 0; i < 8; ++i) {
                    double Qi[d], Fi[d];
#pragma unroll
                    for (int l = 0; l < d; ++l) Qi[l] = QREG ? sL[i * d + l][tx] : sQ[i * d + l][tx];
                    prob.template accel<true>(Qi, Fi, dadd(tn1, dmul(c_c[i], a.h)), ok);
#pragma unroll
                    for (int l = 0; l < d; ++l) sL[i * d + l][tx] = Fi[l];
                }
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int l = 0; l < d; ++l) Lv[i][l] = sL[i * d + l][tx];
            }
#pragma unroll
            for (int i = 0; i < 8; ++i)
#pragma unroll
                for (int l = 0; l < d; ++l) Lv[i][l] = dmul(a.hb[i], Lv[i][l]);
        }
        const bool fin = stop || (k >= a.max_iters);
        if (fin) {  // a6: update with the last iteration's L, history <- Lv
            bool finite = true;
#pragma unroll
            for (int l = 0; l < d; ++l) {
                double sv = Lv[0][l];
#pragma unroll
                for (int j = 1; j < 8; ++j) sv = dadd(sv, Lv[j][l]);
                q[l] = dadd(q[l], sLq[l]);
                v[l] = dadd(v[l], sv);
                finite = finite && isfinite(q[l]) && isfinite(v[l]);
            }
            ++n;
            sweeps += k;
            hits += stop ? 0 : 1;
            k = 0;
#pragma unroll
            for (int l = 0; l < d; ++l) G1Q_M(l) = G1Q_P(l) = kInfBits;
            const int64_t nloc = c * qa.qchunk + n;  // call-local step index just completed
            if (sample && (nloc % a.energy_every) == 0)
                a.energy[(nloc / a.energy_every) * B + b] = prob.energy(q, v);
            if (a.local_energy) dhloc_update(prob.energy(q, v), hprev, dhmax);
            if (n == len || !finite) {  // ---- release the unit ----
#pragma unroll
                for (int j = 0; j < 8; ++j)
#pragma unroll
                    for (int l = 0; l < d; ++l) {
                        a.hist[((int64_t)j * D + l) * B + b] = 0.0;
                        a.hist[((int64_t)j * D + d + l) * B + b] = Lv[j][l];
                    }
#pragma unroll
                for (int l = 0; l < d; ++l) {
                    a.y[l * B + b] = q[l];
                    a.y[(d + l) * B + b] = v[l];
                }
                a.stats[0 * B + b] = __ldcg(&a.stats[0 * B + b]) + hits;
                if (!finite) a.stats[1 * B + b] = n0 + nloc;
                a.stats[2 * B + b] = __ldcg(&a.stats[2 * B + b]) + sweeps;
                if (a.iters) a.iters[b] = (c == 0) ? sweeps : __ldcg(&a.iters[b]) + sweeps;
                if (a.local_energy) dhloc_store(&a.stats[3 * B + b], c == 0, dhmax);
                st_release(&qa.progress[b], (int32_t)(c + 1));
#ifdef IRK_TRACE
                irk_trace_unit(c, b, t_fetch, t_start, sweeps);
#endif
                b = -1;
                continue;
            }
        }
        // a4 (second half) / next step's a1: V_i = v + D(W_i., Lv), W = fin ? nu : mu
        {
            const double2 *W = reinterpret_cast<const double2 *>(&sW[fin ? kNuOff : 0]);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double2 w[4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) w[jj] = W[i * 4 + jj];
#pragma unroll
                for (int l = 0; l < d; ++l) {
                    double acc = dmul(w[0].x, Lv[0][l]);
                    acc = dfma(w[0].y, Lv[1][l], acc);
#pragma unroll
                    for (int jj = 1; jj < 4; ++jj) {
                        acc = dfma(w[jj].x, Lv[2 * jj][l], acc);
                        acc = dfma(w[jj].y, Lv[2 * jj + 1][l], acc);
                    }
                    V[i][l] = dadd(v[l], acc);
                }
            }
        }
    }
}

#undef G1Q_M
#undef G1Q_P

// First-order mode (Eqs. IRK_init / IRK_FP) for the per-thread
// problems: all D = 2d components are extrapolated (a1 over y), each sweep
// evaluates F_i = (V-part of Y_i, g(Q-part of Y_i, t_i)), L = hb o F,
// Y_i = y + D(mu_i, L), and the stop test runs over all D components from k = 1
// (Delta^[1] = |Y^[1] - Y^[0]| exists here).  Reading R-6 of DESIGN.md: this form
// can false-stop on second-order systems (SURVEY C-6), so partitioned mode is the
// default; this kernel serves IRK_OPT_MODE = 1.  One thread per trajectory,
// per-step loop (not performance-tuned).
template <class P>
__global__ void __launch_bounds__(64) ens_g1fo_kernel(const __grid_constant__ EnsArgs a,
                                                      const __grid_constant__ P prob) {
    constexpr int d = P::d, D = 2 * d;
    const int64_t B = a.batch;
    const int64_t slot = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (slot >= a.nslots) return;
    const int64_t b = a.perm ? (int64_t)a.perm[slot] : slot;
    if (b < 0 || b >= B) return;
    double y[D];
#pragma unroll
    for (int l = 0; l < D; ++l) y[l] = a.y[l * B + b];
    int64_t bad = a.stats[1 * B + b];
    const int64_t n0 = *a.n_done;
    const bool sample = (a.energy != nullptr) && (a.energy_every > 0);
    if (sample && a.c0 == 0) a.energy[b] = prob.energy(y, y + d);
    double hprev = a.local_energy ? prob.energy(y, y + d) : 0.0, dhmax = 0.0;
    if (bad > 0 || a.nsteps == 0) {
        if (a.local_energy && a.c0 == 0) a.stats[3 * B + b] = 0;
        if (a.iters && a.c0 == 0) a.iters[b] = 0;
        if (a.csweeps) a.csweeps[b] = 0;
        return;
    }
    double L[8][D];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int l = 0; l < D; ++l) L[j][l] = a.hist[((int64_t)j * D + l) * B + b];
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    int64_t hits = 0, sweeps = 0, n = 0;
    for (; n < a.nsteps;) {
        double Y[8][D], m[D], p[D];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int l = 0; l < D; ++l) {
                double acc = dmul(c_nu[i][0], L[0][l]);
#pragma unroll
                for (int j = 1; j < 8; ++j) acc = dfma(c_nu[i][j], L[j][l], acc);
                Y[i][l] = dadd(y[l], acc);
            }
#pragma unroll
        for (int l = 0; l < D; ++l) m[l] = p[l] = kInf;
        const double tn1 = dadd(a.t0, dmul((double)(n0 + n), a.h));
        int k = 0;
        bool stop = false;
        for (;;) {
            ++k;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                bool ok = true;
                if constexpr (P::first_order) {  // f(y) of a non-separable problem
                    double F[D];
                    prob.template rhs<true>(Y[i], F, dadd(tn1, dmul(c_c[i], a.h)), ok);
#pragma unroll
                    for (int l = 0; l < D; ++l) L[i][l] = dmul(a.hb[i], F[l]);
                } else {                         // f(y) = (v, g(q, t))
                    double F[d];
                    prob.template accel<true>(Y[i], F, dadd(tn1, dmul(c_c[i], a.h)), ok);
#pragma unroll
                    for (int l = 0; l < d; ++l) {
                        L[i][l] = dmul(a.hb[i], Y[i][d + l]);
                        L[i][d + l] = dmul(a.hb[i], F[l]);
                    }
                }
            }
            stop = true;
#pragma unroll
            for (int l = 0; l < D; ++l) {
                double delta = 0.0;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    double acc = dmul(c_mu[i][0], L[0][l]);
#pragma unroll
                    for (int j = 1; j < 8; ++j) acc = dfma(c_mu[i][j], L[j][l], acc);
                    const double yn = dadd(y[l], acc);
                    const double e = dabs(dsub(yn, Y[i][l]));
                    delta = (e > delta) ? e : delta;
                    Y[i][l] = yn;
                }
                const double mn = (delta < p[l]) ? delta : p[l];
                const bool okc = (delta == 0.0) || (m[l] <= mn);
                m[l] = (p[l] < m[l]) ? p[l] : m[l];
                p[l] = delta;
                stop = stop && okc;
            }
            if (stop || k >= a.max_iters) break;
        }
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
        if (sample && ((a.c0 + n) % a.energy_every) == 0)
            a.energy[((a.c0 + n) / a.energy_every) * B + b] = prob.energy(y, y + d);
        if (a.local_energy) dhloc_update(prob.energy(y, y + d), hprev, dhmax);
        if (!finite) {
            bad = n0 + n;
            break;
        }
    }
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int l = 0; l < D; ++l) a.hist[((int64_t)j * D + l) * B + b] = L[j][l];
#pragma unroll
    for (int l = 0; l < D; ++l) a.y[l * B + b] = y[l];
    a.stats[0 * B + b] += hits;
    a.stats[1 * B + b] = bad;
    a.stats[2 * B + b] += sweeps;
    if (a.iters) a.iters[b] = (a.c0 == 0) ? sweeps : a.iters[b] + sweeps;
    if (a.csweeps) a.csweeps[b] = (int32_t)sweeps;
    if (a.local_energy) dhloc_store(&a.stats[3 * B + b], a.c0 == 0, dhmax);
}

}  // namespace irk
