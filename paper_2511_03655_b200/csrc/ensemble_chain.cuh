// Ensemble kernel, mapping "site-per-lane" (config 4, FPU-beta chains): one warp
// per chain of N = 32*SPL sites, lane L owns sites L*SPL .. L*SPL+SPL-1 (their
// positions and velocities for all 8 stages).
//
// Both 8x8 contractions are thread-local (components are independent); the
// RHS of a site needs its neighbours' stage positions, read from a shared-memory
// copy of Q^[k] that also serves as Q^[k-1] for the stop test.  A warp is one
// trajectory, so the sweep loop has no divergence at all; the stop test is a
// warp vote.
//
// Canonical RHS (oracle/CANON.md "Right-hand sides", oracle accel_fpu): bond b
// (b = 0..N, q_{-1} = q_N = 0 in 0-based sites) has D_b = q_b - q_{b-1} and
// f_b = fma(beta*(D_b*D_b), D_b, D_b); site s gets a_s = f_{s+1} - f_s.  A bond
// shared by two lanes is evaluated by both with identical operations.
#pragma once
#include <cstdint>

#include "ens_common.cuh"
#include "fp64.cuh"

namespace irk {

constexpr int CH_THREADS = 64;  // 2 chains per block

__device__ __forceinline__ double fpu_bond(double dl, double beta) {
    return dfma(dmul(beta, dmul(dl, dl)), dl, dl);
}

// H = sum p^2/2 + sum_b (D^2/2 + beta D^4/4), Neumaier, canonical order (oracle).
template <int N>
__device__ double fpu_energy(const double *q, const double *v, double beta) {
    Neumaier n;
    for (int i = 0; i < N; ++i) n.add(dmul(0.5, dmul(v[i], v[i])));
    for (int bnd = 0; bnd <= N; ++bnd) {
        const double ql = (bnd == 0) ? 0.0 : q[bnd - 1];
        const double qr = (bnd == N) ? 0.0 : q[bnd];
        const double dl = dsub(qr, ql);
        const double d2 = dmul(dl, dl);
        n.add(dadd(dmul(0.5, d2), dmul(dmul(0.25, beta), dmul(d2, d2))));
    }
    return n.result();
}

// Site index -> shared-memory slot of a chain's stage tile: site L*SPL + s of lane L
// lives at s*32 + L, so own-site and neighbour-site accesses of a warp hit 32
// consecutive doubles (conflict-free; the site-major layout was 2-way conflicted
// for SPL = 2).
template <int SPL, int WPC = 1>
__device__ __forceinline__ int ch_slot(int site) { return (site % SPL) * (32 * WPC) + site / SPL; }

// barrier over the WPC warps of one chain (WPC > 1: the block is one chain)
template <int WPC>
__device__ __forceinline__ void chain_sync() {
    if (WPC == 1) __syncwarp();
    else __syncthreads();
}

// WPC warps (one warp when WPC = 1) integrate chain b over the call-local steps
// [c0, c0 + nsteps); thread tid of the chain owns sites tid*SPL .. tid*SPL+SPL-1.
// WPC > 1 (small batches: more lanes per chain, shorter sweeps): the block is the
// chain, the stage tile and the votes are exchanged with block barriers.
template <int SPL, int WPC = 1>
__device__ __forceinline__ void chain_unit(const EnsArgs &a, const double beta, const int64_t b, const int64_t c0,
                                           const int64_t nsteps, double (*sQ)[32 * SPL * WPC], double *sQV,
                                           const double (*sW)[64], int *sVote = nullptr) {
    constexpr int N = 32 * SPL * WPC, d = N, D = 2 * N, TPC = 32 * WPC;
    const unsigned FULL = 0xffffffffu;
    const int64_t B = a.batch;
    const int lane = threadIdx.x % TPC;  // thread index within the chain
    const int wic = lane >> 5;           // warp index within the chain
    const int s0 = lane * SPL;
    // AND of a per-warp vote over the chain's warps (every thread calls it)
    auto chain_all = [&](bool warp_vote) -> bool {
        if (WPC == 1) return warp_vote;
        if ((lane & 31) == 0) sVote[wic] = warp_vote ? 1 : 0;
        chain_sync<WPC>();
        bool all = true;
#pragma unroll
        for (int w = 0; w < WPC; ++w) all = all && sVote[w] != 0;
        chain_sync<WPC>();  // votes read before the next write
        return all;
    };

    double q[SPL], v[SPL];
#pragma unroll
    for (int s = 0; s < SPL; ++s) {  // L2 loads: the previous unit may have run on another SM
        q[s] = __ldcg(&a.y[(int64_t)(s0 + s) * B + b]);
        v[s] = __ldcg(&a.y[(int64_t)(d + s0 + s) * B + b]);
    }
    int64_t bad = __ldcg(&a.stats[1 * B + b]);
    const int64_t n0 = *a.n_done;
    const bool sample = (a.energy != nullptr) && (a.energy_every > 0);
    double hprev = 0.0, dhmax = 0.0;  // lane 0: DH^loc tracking
    // H(y) of the chain (lane 0 sums the canonical terms); idx >= 0 stores a sample
    auto energy_at = [&](int64_t idx, bool track) {
#pragma unroll
        for (int s = 0; s < SPL; ++s) {
            sQV[s0 + s] = q[s];
            sQV[N + s0 + s] = v[s];
        }
        chain_sync<WPC>();
        if (lane == 0) {
            const double hn = fpu_energy<N>(sQV, sQV + N, beta);
            if (idx >= 0) a.energy[idx * B + b] = hn;
            if (track) dhloc_update(hn, hprev, dhmax);
            else hprev = hn;
        }
        chain_sync<WPC>();
    };
    if ((sample && c0 == 0) || a.local_energy) energy_at((sample && c0 == 0) ? 0 : -1, false);
    if (bad > 0 || nsteps == 0) {
        if (lane == 0) {
            if (a.iters && c0 == 0) a.iters[b] = 0;
            if (a.csweeps) a.csweeps[b] = 0;
            if (a.local_energy && c0 == 0) a.stats[3 * B + b] = 0;
        }
        return;
    }
    double V[8][SPL];
    {
        double H[8][SPL];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int s = 0; s < SPL; ++s) H[j][s] = __ldcg(&a.hist[((int64_t)j * D + d + s0 + s) * B + b]);
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int s = 0; s < SPL; ++s) {
                double acc = dmul(c_nu[i][0], H[0][s]);
#pragma unroll
                for (int j = 1; j < 8; ++j) acc = dfma(c_nu[i][j], H[j][s], acc);
                V[i][s] = dadd(v[s], acc);
            }
    }
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    double m[SPL], p[SPL];
#pragma unroll
    for (int s = 0; s < SPL; ++s) m[s] = p[s] = kInf;
    int64_t n = 0, hits = 0, sweeps = 0;
    int k = 0;
    while (n < nsteps) {  // warp-uniform
        ++k;
        // a2 + Delta
        double Lq[8][SPL], sLq[SPL], delta[SPL];
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int s = 0; s < SPL; ++s) Lq[j][s] = dmul(a.hb[j], V[j][s]);
#pragma unroll
        for (int s = 0; s < SPL; ++s) {
            sLq[s] = Lq[0][s];
#pragma unroll
            for (int j = 1; j < 8; ++j) sLq[s] = dadd(sLq[s], Lq[j][s]);
            delta[s] = 0.0;
        }
        chain_sync<WPC>();  // previous sweep's neighbour reads of sQ are done
        {
            const double2 *M = reinterpret_cast<const double2 *>(&c_mu[0][0]);
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double2 w[4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) w[jj] = M[i * 4 + jj];
#pragma unroll
                for (int s = 0; s < SPL; ++s) {
                    double acc = dmul(w[0].x, Lq[0][s]);
                    acc = dfma(w[0].y, Lq[1][s], acc);
#pragma unroll
                    for (int jj = 1; jj < 4; ++jj) {
                        acc = dfma(w[jj].x, Lq[2 * jj][s], acc);
                        acc = dfma(w[jj].y, Lq[2 * jj + 1][s], acc);
                    }
                    const double qn = dadd(q[s], acc);
                    const double e = dabs(dsub(qn, sQ[i][s * TPC + lane]));
                    delta[s] = (e > delta[s]) ? e : delta[s];
                    sQ[i][s * TPC + lane] = qn;
                }
            }
        }
        bool ok_lane = true;
        if (k >= 2) {
#pragma unroll
            for (int s = 0; s < SPL; ++s) {
                const double mn = (delta[s] < p[s]) ? delta[s] : p[s];
                const bool oks = (delta[s] == 0.0) || (m[s] <= mn);
                m[s] = (p[s] < m[s]) ? p[s] : m[s];
                p[s] = delta[s];
                ok_lane = ok_lane && oks;
            }
        }
        // every lane votes (k is chain-uniform here); the chain barrier inside
        // chain_all (or the warp barrier) also publishes this sweep's sQ writes
        const bool all_ok = chain_all(__all_sync(FULL, ok_lane));
        const bool stop = (k >= 2) && all_ok;
        if (WPC == 1) __syncwarp();
        // a3: bond forces of the lane's sites for every stage
        double Lv[8][SPL];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double *Qi = sQ[i];
            double qs[SPL + 2];
            qs[0] = (s0 == 0) ? 0.0 : Qi[ch_slot<SPL, WPC>(s0 - 1)];
#pragma unroll
            for (int s = 0; s < SPL; ++s) qs[s + 1] = Qi[s * TPC + lane];
            qs[SPL + 1] = (s0 + SPL == N) ? 0.0 : Qi[ch_slot<SPL, WPC>(s0 + SPL)];
            double f[SPL + 1];
#pragma unroll
            for (int t = 0; t <= SPL; ++t) f[t] = fpu_bond(dsub(qs[t + 1], qs[t]), beta);
#pragma unroll
            for (int s = 0; s < SPL; ++s) Lv[i][s] = dmul(a.hb[i], dsub(f[s + 1], f[s]));
        }
        const bool fin = stop || (k >= a.max_iters);
        if (fin) {
            bool finite = true;
#pragma unroll
            for (int s = 0; s < SPL; ++s) {
                double sv = Lv[0][s];
#pragma unroll
                for (int j = 1; j < 8; ++j) sv = dadd(sv, Lv[j][s]);
                q[s] = dadd(q[s], sLq[s]);
                v[s] = dadd(v[s], sv);
                finite = finite && isfinite(q[s]) && isfinite(v[s]);
            }
            finite = chain_all(__all_sync(FULL, finite));
            ++n;
            sweeps += k;
            hits += stop ? 0 : 1;
            k = 0;
#pragma unroll
            for (int s = 0; s < SPL; ++s) m[s] = p[s] = kInf;
            const bool due = sample && ((c0 + n) % a.energy_every) == 0;
            if (due || a.local_energy) energy_at(due ? (c0 + n) / a.energy_every : -1, a.local_energy != 0);
            if (n == nsteps || !finite) {
#pragma unroll
                for (int j = 0; j < 8; ++j)
#pragma unroll
                    for (int s = 0; s < SPL; ++s) {
                        a.hist[((int64_t)j * D + s0 + s) * B + b] = 0.0;
                        a.hist[((int64_t)j * D + d + s0 + s) * B + b] = Lv[j][s];
                    }
                if (!finite) bad = n0 + n;
                break;
            }
        }
        {
            const double2 *W = reinterpret_cast<const double2 *>(&sW[fin ? 1 : 0][0]);  // warp-uniform
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                double2 w[4];
#pragma unroll
                for (int jj = 0; jj < 4; ++jj) w[jj] = W[i * 4 + jj];
#pragma unroll
                for (int s = 0; s < SPL; ++s) {
                    double acc = dmul(w[0].x, Lv[0][s]);
                    acc = dfma(w[0].y, Lv[1][s], acc);
#pragma unroll
                    for (int jj = 1; jj < 4; ++jj) {
                        acc = dfma(w[jj].x, Lv[2 * jj][s], acc);
                        acc = dfma(w[jj].y, Lv[2 * jj + 1][s], acc);
                    }
                    V[i][s] = dadd(v[s], acc);
                }
            }
        }
    }
#pragma unroll
    for (int s = 0; s < SPL; ++s) {
        a.y[(int64_t)(s0 + s) * B + b] = q[s];
        a.y[(int64_t)(d + s0 + s) * B + b] = v[s];
    }
    if (lane == 0) {
        a.stats[0 * B + b] = __ldcg(&a.stats[0 * B + b]) + hits;
        a.stats[1 * B + b] = bad;
        a.stats[2 * B + b] = __ldcg(&a.stats[2 * B + b]) + sweeps;
        if (a.iters) a.iters[b] = (c0 == 0) ? sweeps : __ldcg(&a.iters[b]) + sweeps;
        if (a.csweeps) a.csweeps[b] = (int32_t)sweeps;
        if (a.local_energy) dhloc_store(&a.stats[3 * B + b], c0 == 0, dhmax);
    }
}

#ifndef CH_MAXREG
#define CH_MAXREG 255
#endif
template <int SPL>
__global__ void __maxnreg__(CH_MAXREG) ens_chain_kernel(const __grid_constant__ EnsArgs a, const double beta) {
    constexpr int N = 32 * SPL, CPB = CH_THREADS / 32;
    __shared__ __align__(16) double sW[2][64];
    __shared__ double sQ[CPB][8][N];   // Q^[k] of the chain (neighbour reads + Delta), slots ch_slot()
    __shared__ double sQV[CPB][2 * N]; // (q, v) for energy samples
    for (int e = threadIdx.x; e < 128; e += blockDim.x)
        sW[e >> 6][e & 63] = (e < 64) ? (&c_mu[0][0])[e] : (&c_nu[0][0])[e - 64];
    __syncthreads();
    const int cib = threadIdx.x >> 5;
    const int64_t slot = (int64_t)blockIdx.x * CPB + cib;
    if (slot >= a.nslots) return;  // warp-uniform
    const int64_t b = a.perm ? (int64_t)a.perm[slot] : slot;
    if (b < 0 || b >= a.batch) return;   // warp-uniform
    chain_unit<SPL>(a, beta, b, a.c0, a.nsteps, sQ[cib], sQV[cib], sW);
}

// Small batches: WPC warps per chain, one chain per block (SPL * WPC * 32 = N), a
// single launch over the whole call.  Half (WPC = 2) the sites per lane, so a sweep
// of one chain is shorter: the mapping for the per-GPU shares of strong scaling.
template <int SPL, int WPC>
__global__ void __launch_bounds__(32 * WPC) ens_chainw_kernel(const __grid_constant__ EnsArgs a, const double beta) {
    constexpr int N = 32 * SPL * WPC;
    __shared__ __align__(16) double sW[2][64];
    __shared__ double sQ[8][N];
    __shared__ double sQV[2 * N];
    __shared__ int sVote[WPC];
    for (int e = threadIdx.x; e < 128; e += blockDim.x)
        sW[e >> 6][e & 63] = (e < 64) ? (&c_mu[0][0])[e] : (&c_nu[0][0])[e - 64];
    __syncthreads();
    const int64_t b = blockIdx.x;
    if (b >= a.batch) return;  // block-uniform
    chain_unit<SPL, WPC>(a, beta, b, a.c0, a.nsteps, sQ, sQV, sW, sVote);
}

// Persistent work-queue version (IRK_OPT_SCHEDULE 0/2; see ens_g1q): every warp
// pulls (chain, step-chunk) units until the queue drains; unit (b, c) waits for
// progress[b] = c.  Same arithmetic per unit, so bitwise any schedule.
#ifndef CHQ_MAXREG
#define CHQ_MAXREG 192  // config 4 at 20,000 steps: 164 regs (unbounded) 371 ms, 158: 382, 174: 326.7, cap 192 (176 used): 324.3
#endif
template <int SPL>
__global__ void __maxnreg__(CHQ_MAXREG) ens_chain_q_kernel(const __grid_constant__ EnsArgs a,
                                                                const __grid_constant__ QueueArgs qa,
                                                                const double beta) {
    constexpr int N = 32 * SPL, CPB = CH_THREADS / 32;
    __shared__ __align__(16) double sW[2][64];
    __shared__ double sQ[CPB][8][N];
    __shared__ double sQV[CPB][2 * N];
    for (int e = threadIdx.x; e < 128; e += blockDim.x)
        sW[e >> 6][e & 63] = (e < 64) ? (&c_mu[0][0])[e] : (&c_nu[0][0])[e - 64];
    __syncthreads();
    const int cib = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t B = a.batch, total = B * qa.nchunks;
    for (;;) {
        unsigned long long u = 0;
        if (lane == 0) u = atomicAdd(qa.counter, 1ull);
        u = __shfl_sync(0xffffffffu, u, 0);
        if ((int64_t)u >= total) break;
        const int64_t c = (int64_t)u / B, b = (int64_t)u - c * B;
        if (lane == 0 && c > 0)
            while (ld_acquire(&qa.progress[b]) < c) __nanosleep(1024);
        __syncwarp();
        const int64_t c0 = c * qa.qchunk;
        const int64_t len = (a.nsteps - c0 < qa.qchunk) ? a.nsteps - c0 : qa.qchunk;
        chain_unit<SPL>(a, beta, b, c0, len, sQ[cib], sQV[cib], sW);
        __threadfence();  // this warp's stores of the unit, before the hand-off
        __syncwarp();
        if (lane == 0) st_release(&qa.progress[b], (int32_t)(c + 1));
    }
}

}  // namespace irk
