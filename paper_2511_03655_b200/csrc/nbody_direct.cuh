// Large-N single-system path (config 5, IRK_NBODY_DIRECT), body-sharded.
//
// One gravitational system of N bodies split into P shards of nloc = N/P
// bodies (P = 1 on one GPU; P = nranks under NCCL; or P "virtual" shards driven
// by one process on one GPU to exercise the sharded layout).  Per fixed-point
// sweep, per shard:
//
//   nbd_pos    (a2 + a5)  component-parallel over the shard's 3*nloc components:
//                         Lq = hb o V, Q_i = q + D(mu_i, Lq), Delta vs Q^[k-1],
//                         stop-test state (m, p); the shard's Q^[k] is written
//                         straight into its slot of the gathered buffer Qg, plus
//                         a "not converged" flag at the end of the slot.
//   (exchange)            ncclAllGather in place on Qg (NCCL mode) -- the one
//                         data-path collective, once per iteration;
//                         nothing to do for virtual shards (shared buffer).
//   nbd_or                global stop = no flag set in any slot (same on every rank).
//   nbd_force  (a3)       (local body, stage, j-block) parallel: the canonical blocked
//                         direct sum (R-8) over ALL N bodies read from Qg,
//                         one thread = one partial sum over NBD_JBLOCK = 1024 bodies j
//                         staged in shared memory (broadcast reads).
//   nbd_vel    (a4 + a6)  acc = ((0 + P_0) + P_1) + ... , Lv = hb o acc, then
//                         V = v + D(mu, Lv) or (converged) update + history + nu-init.
//   nbd_ctl    (1 thread) sweep / step counters (identical decisions on all ranks).
//
// The arithmetic is the oracle's canonical sequence (accel_direct_body,
// step_partitioned); the j-order does not depend on P, so every P gives the same
// bits as the oracle.
#pragma once
#include <cstdint>

#include "ens_common.cuh"
#include "fp64.cuh"

namespace irk {

constexpr int NBD_JBLOCK = 1024;  // canonical j-block (oracle NB_BLOCK)
constexpr int NBD_FORCE_THREADS = 128;

struct NbdCtl {           // device-side control block (one per process)
    int64_t n;            // steps completed in this call
    int32_t k;            // sweeps completed in the current step
    int32_t notok;        // global: some component failed the stop test this sweep
    int32_t fin;          // last sweep finished a step
    int32_t nonfinite;    // global (after an exchange): some component became non-finite
    int32_t halt;         // stop integrating (divergence)
    int32_t pad;
    int64_t sweeps, hits;
    int64_t target;       // device-driven loop: run sweeps until n == target (or halt)
};

// Per-shard arguments.  Component index l in [0, 3*nloc) of shard s is global
// position component 3*b0 + l.
struct NbdArgs {
    double hb[8];
    double *yq, *yv;      // shard's q and v blocks (3*nloc each)
    double *hist;         // history base; rows j*hdim + hq + l (q block), j*hdim + hv + l (v block)
    int64_t hdim, hq, hv;
    double *Qg;           // gathered stage positions [P][stride]; slot s = [8][3*nloc] + 2 flags
    int64_t stride;       // doubles per slot (8*3*nloc + 2): flags {not converged, non-finite}
    double *V;            // [8][3*nloc]
    double *M, *Pst;      // [3*nloc] stop-test state
    double *sLq;          // [3*nloc]
    double *part;         // [nj][8][3*nloc] block partial sums
    const double *mass;   // [N]
    NbdCtl *ctl;
    int64_t nbody, nloc, b0;
    int shard, nshards;
    double G, eps2;
    int max_iters;
};

__device__ __forceinline__ double *nbd_slot(const NbdArgs &a, int s) { return a.Qg + (int64_t)s * a.stride; }
__device__ __forceinline__ int64_t nbd_flag_index(const NbdArgs &a) { return 24 * a.nloc; }

__global__ void nbd_init_kernel(const __grid_constant__ NbdArgs a) {
    const int64_t dl = 3 * a.nloc;
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l == 0) {
        nbd_slot(a, a.shard)[nbd_flag_index(a)] = 0.0;
        nbd_slot(a, a.shard)[nbd_flag_index(a) + 1] = 0.0;
    }
    if (l >= dl) return;
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    const double v = a.yv[l];
    double H[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) H[j] = a.hist[(int64_t)j * a.hdim + a.hv + l];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        double acc = dmul(c_nu[i][0], H[0]);
#pragma unroll
        for (int j = 1; j < 8; ++j) acc = dfma(c_nu[i][j], H[j], acc);
        a.V[(int64_t)i * dl + l] = dadd(v, acc);
    }
    a.M[l] = kInf;
    a.Pst[l] = kInf;
}

__global__ void nbd_pos_kernel(const __grid_constant__ NbdArgs a) {
    const int64_t dl = 3 * a.nloc;
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= dl) return;
    const int k = a.ctl->k + 1;
    double *Q = nbd_slot(a, a.shard);
    const double q = a.yq[l];
    double Lq[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) Lq[j] = dmul(a.hb[j], a.V[(int64_t)j * dl + l]);
    double s = Lq[0];
#pragma unroll
    for (int j = 1; j < 8; ++j) s = dadd(s, Lq[j]);
    a.sLq[l] = s;
    double delta = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        double acc = dmul(c_mu[i][0], Lq[0]);
#pragma unroll
        for (int j = 1; j < 8; ++j) acc = dfma(c_mu[i][j], Lq[j], acc);
        const double qn = dadd(q, acc);
        const double e = dabs(dsub(qn, Q[(int64_t)i * dl + l]));
        delta = (e > delta) ? e : delta;
        Q[(int64_t)i * dl + l] = qn;
    }
    if (k >= 2) {
        const double pl = a.Pst[l], ml = a.M[l];
        const double mn = (delta < pl) ? delta : pl;
        const bool ok = (delta == 0.0) || (ml <= mn);
        a.M[l] = (pl < ml) ? pl : ml;
        a.Pst[l] = delta;
        if (!ok) Q[nbd_flag_index(a)] = 1.0;  // benign race: every writer stores 1
    }
}

// global flags from every slot (after the exchange)
__global__ void nbd_or_kernel(const __grid_constant__ NbdArgs a) {
    int any = 0, bad = 0;
    for (int s = 0; s < a.nshards; ++s) {
        any |= (nbd_slot(a, s)[nbd_flag_index(a)] != 0.0);
        bad |= (nbd_slot(a, s)[nbd_flag_index(a) + 1] != 0.0);
    }
    a.ctl->notok = any;
    a.ctl->nonfinite = bad;
}

// grid: x = local body tile (NBD_FORCE_THREADS bodies), y = stage i, z = j-block
__global__ void __launch_bounds__(NBD_FORCE_THREADS) nbd_force_kernel(const __grid_constant__ NbdArgs a) {
    __shared__ double4 sj[NBD_JBLOCK];
    const int64_t N = a.nbody, nloc = a.nloc, dl = 3 * nloc;
    const int i = blockIdx.y, J = blockIdx.z;
    const int64_t j0 = (int64_t)J * NBD_JBLOCK;
    const int nj = (int)((N - j0) < NBD_JBLOCK ? (N - j0) : NBD_JBLOCK);
    for (int t = threadIdx.x; t < nj; t += blockDim.x) {
        const int64_t j = j0 + t;
        const double *Qj = nbd_slot(a, (int)(j / nloc)) + (int64_t)i * dl + 3 * (j % nloc);
        sj[t] = make_double4(Qj[0], Qj[1], Qj[2], a.mass[j]);
    }
    __syncthreads();
    const int64_t body = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // local index
    if (body >= nloc) return;
    const double *Qa = nbd_slot(a, a.shard) + (int64_t)i * dl + 3 * body;
    const double qx = Qa[0], qy = Qa[1], qz = Qa[2];
    double px = 0.0, py = 0.0, pz = 0.0;
    bool ok = true;
#pragma unroll 4
    for (int t = 0; t < nj; ++t) {
        const double4 pj = sj[t];
        const double dx = dsub(pj.x, qx), dy = dsub(pj.y, qy), dz = dsub(pj.z, qz);
        const double r2 = dfma(dz, dz, dfma(dy, dy, dfma(dx, dx, a.eps2)));
        const double w = ddiv_fast(a.G, dmul(r2, dsqrt_fast(r2, ok)), ok);
        const double s = dmul(pj.w, w);
        px = dfma(s, dx, px);
        py = dfma(s, dy, py);
        pz = dfma(s, dz, pz);
    }
    if (!ok) {  // an operand outside the fast-path range: exact intrinsics, same bits
        px = py = pz = 0.0;
        for (int t = 0; t < nj; ++t) {
            const double4 pj = sj[t];
            const double dx = dsub(pj.x, qx), dy = dsub(pj.y, qy), dz = dsub(pj.z, qz);
            const double r2 = dfma(dz, dz, dfma(dy, dy, dfma(dx, dx, a.eps2)));
            const double w = ddiv(a.G, dmul(r2, dsqrt(r2)));
            const double s = dmul(pj.w, w);
            px = dfma(s, dx, px);
            py = dfma(s, dy, py);
            pz = dfma(s, dz, pz);
        }
    }
    double *P = a.part + ((int64_t)J * 8 + i) * dl;
    P[3 * body] = px;
    P[3 * body + 1] = py;
    P[3 * body + 2] = pz;
}

__global__ void nbd_vel_kernel(const __grid_constant__ NbdArgs a) {
    const int64_t dl = 3 * a.nloc;
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= dl) return;
    if (a.ctl->nonfinite) return;  // diverged at the previous step: frozen (R-10)
    const int nj = (int)((a.nbody + NBD_JBLOCK - 1) / NBD_JBLOCK);
    const int k = a.ctl->k + 1;
    const bool stop = (k >= 2) && (a.ctl->notok == 0);
    const bool fin = stop || (k >= a.max_iters);
    double Lv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        double acc = 0.0;
        for (int J = 0; J < nj; ++J) acc = dadd(acc, a.part[((int64_t)J * 8 + i) * dl + l]);
        Lv[i] = dmul(a.hb[i], acc);
    }
    double v = a.yv[l];
    if (fin) {
        double sv = Lv[0];
#pragma unroll
        for (int j = 1; j < 8; ++j) sv = dadd(sv, Lv[j]);
        const double q = dadd(a.yq[l], a.sLq[l]);
        v = dadd(v, sv);
        a.yq[l] = q;
        a.yv[l] = v;
        if (!isfinite(q) || !isfinite(v)) nbd_slot(a, a.shard)[nbd_flag_index(a) + 1] = 1.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            a.hist[(int64_t)j * a.hdim + a.hq + l] = 0.0;
            a.hist[(int64_t)j * a.hdim + a.hv + l] = Lv[j];
        }
        const double kInf = __longlong_as_double(0x7ff0000000000000LL);
        a.M[l] = kInf;
        a.Pst[l] = kInf;
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        double acc = dmul(fin ? c_nu[i][0] : c_mu[i][0], Lv[0]);
#pragma unroll
        for (int j = 1; j < 8; ++j) acc = dfma(fin ? c_nu[i][j] : c_mu[i][j], Lv[j], acc);
        a.V[(int64_t)i * dl + l] = dadd(v, acc);
    }
}

// after the last shard's nbd_vel of the sweep: counters, stats, reset local flags;
// inside the device-driven loop (use_cond) also the WHILE condition of the graph
// (no host round trip per fixed-point iteration)
__global__ void nbd_ctl_kernel(const __grid_constant__ NbdArgs a, int first_local, int nlocal, int64_t *n_done,
                               int64_t *stats, cudaGraphConditionalHandle cond, int use_cond) {
    NbdCtl *c = a.ctl;
    for (int s = first_local; s < first_local + nlocal; ++s) nbd_slot(a, s)[nbd_flag_index(a)] = 0.0;
    if (c->nonfinite) {  // some shard diverged at the last completed step
        if (stats[1] == 0) stats[1] = *n_done;
        c->halt = 1;
        c->fin = 0;
        if (use_cond) cudaGraphSetConditional(cond, 0);
        return;
    }
    const int k = c->k + 1;
    const bool stop = (k >= 2) && (c->notok == 0);
    const bool fin = stop || (k >= a.max_iters);
    c->notok = 0;
    c->fin = fin ? 1 : 0;
    if (fin) {
        c->n += 1;
        c->sweeps += k;
        c->hits += stop ? 0 : 1;
        c->k = 0;
        *n_done += 1;
        stats[0] += stop ? 0 : 1;
        stats[2] += k;
    } else {
        c->k = k;
    }
    if (use_cond) cudaGraphSetConditional(cond, (c->n < c->target) ? 1u : 0u);
}

// after the final exchange of a call: record a divergence at the last step
__global__ void nbd_final_kernel(const __grid_constant__ NbdArgs a, int64_t *n_done, int64_t *stats) {
    int bad = 0;
    for (int s = 0; s < a.nshards; ++s) bad |= (nbd_slot(a, s)[nbd_flag_index(a) + 1] != 0.0);
    if (bad && stats[1] == 0) stats[1] = *n_done;
}

// ---- energy (canonical: kinetic terms, then row sums over j > i, Neumaier) ----
// Qall: all N positions (3N, gathered); each shard writes its kinetic terms and
// row sums into its slot [kin(nloc) | row(nloc)] of `terms` ([P][2*nloc]); the
// total is added by one thread over all kinetic terms, then all rows, in order.
__global__ void nbd_energy_terms_kernel(const double *Qall, const double *vloc, const double *mass, int64_t N,
                                        int64_t b0, int64_t nloc, double G, double eps2, double *slot) {
    const int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (r >= nloc) return;
    const int64_t i = b0 + r;
    const double *q = Qall, *v = vloc + 3 * r;
    const double k = dfma(v[2], v[2], dfma(v[1], v[1], dmul(v[0], v[0])));
    slot[r] = dmul(dmul(0.5, mass[i]), k);
    Neumaier row;
    for (int64_t j = i + 1; j < N; ++j) {
        const double dx = dsub(q[3 * j], q[3 * i]);
        const double dy = dsub(q[3 * j + 1], q[3 * i + 1]);
        const double dz = dsub(q[3 * j + 2], q[3 * i + 2]);
        const double r2 = dfma(dz, dz, dfma(dy, dy, dfma(dx, dx, eps2)));
        row.add(-ddiv(dmul(G, dmul(mass[i], mass[j])), dsqrt(r2)));
    }
    slot[nloc + r] = row.result();
}

__global__ void nbd_energy_sum_kernel(const double *terms, int P, int64_t nloc, double *out) {
    Neumaier tot;
    for (int s = 0; s < P; ++s)
        for (int64_t r = 0; r < nloc; ++r) tot.add(terms[(int64_t)s * 2 * nloc + r]);
    for (int s = 0; s < P; ++s)
        for (int64_t r = 0; r < nloc; ++r) tot.add(terms[(int64_t)s * 2 * nloc + nloc + r]);
    *out = tot.result();
}

}  // namespace irk
