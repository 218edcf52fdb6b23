// Large-N single-system path (config 5, IRK_NBODY_DIRECT): one gravitational
// system of N bodies (d = 3N position components), all 8 stages, split into
// three kernels per fixed-point sweep plus a one-thread control kernel:
//
//   nbd_pos    (a2 + a5)  component-parallel: Lq = hb o V, Q_i = q + D(mu_i, Lq),
//                         Delta vs Q^[k-1], stop-test state (m, p) per component,
//                         a global "not converged" flag.
//   nbd_force  (a3)       (stage, body, j-block) parallel: the canonical blocked
//                         direct sum (R-8): one thread = one partial sum
//                         over a block of NBD_JBLOCK = 1024 bodies j, with the
//                         block's positions and masses staged in shared memory
//                         (every lane reads the same j: broadcast).
//   nbd_vel    (a4 + a6)  component-parallel: acc = ((0 + P_0) + P_1) + ... (blocks
//                         left to right), Lv = hb o acc, then either V = v + D(mu, Lv)
//                         or, when the step converged, the update q += S(Lq),
//                         v += S(Lv), history <- Lv and the next nu-init.
//   nbd_ctl    (1 thread) advances the sweep / step counters.
//
// All arithmetic follows the oracle's canonical sequence (accel_direct_body and
// step_partitioned), so the result is bitwise the oracle's for any N.
#pragma once
#include <cstdint>

#include "ens_common.cuh"
#include "fp64.cuh"

namespace irk {

constexpr int NBD_JBLOCK = 1024;  // canonical j-block (oracle NB_BLOCK)
constexpr int NBD_FORCE_THREADS = 128;

struct NbdCtl {           // device-side control block (in the workspace)
    int64_t n;            // steps completed in this call
    int32_t k;            // sweeps completed in the current step
    int32_t notok;        // any component failed the stop test in this sweep
    int32_t fin;          // last sweep finished a step (for the host / energy)
    int32_t nonfinite;    // a component became non-finite at the last update
    int64_t sweeps, hits, bad;
};

struct NbdArgs {
    double hb[8];
    double *y;            // [6N] (batch = 1): q then v
    double *hist;         // [8][6N]
    double *Q;            // [8][3N]
    double *V;            // [8][3N]
    double *M, *Pst;      // [3N] stop-test state
    double *sLq;          // [3N]
    double *part;         // [nj][8][3N] block partial sums
    const double *mass;   // [N]
    NbdCtl *ctl;
    int64_t nbody, nsteps;
    double G, eps2;
    int max_iters;
};

__global__ void nbd_init_kernel(const __grid_constant__ NbdArgs a) {
    const int64_t d = 3 * a.nbody;
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= d) return;
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    const double v = a.y[d + l];
    double H[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) H[j] = a.hist[(int64_t)j * 2 * d + d + l];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        double acc = dmul(c_nu[i][0], H[0]);
#pragma unroll
        for (int j = 1; j < 8; ++j) acc = dfma(c_nu[i][j], H[j], acc);
        a.V[(int64_t)i * d + l] = dadd(v, acc);
    }
    a.M[l] = kInf;
    a.Pst[l] = kInf;
}

__global__ void nbd_pos_kernel(const __grid_constant__ NbdArgs a) {
    const int64_t d = 3 * a.nbody;
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= d) return;
    const int k = a.ctl->k + 1;
    const double q = a.y[l];
    double Lq[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) Lq[j] = dmul(a.hb[j], a.V[(int64_t)j * d + l]);
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
        const double e = dabs(dsub(qn, a.Q[(int64_t)i * d + l]));
        delta = (e > delta) ? e : delta;
        a.Q[(int64_t)i * d + l] = qn;
    }
    if (k >= 2) {
        const double pl = a.Pst[l], ml = a.M[l];
        const double mn = (delta < pl) ? delta : pl;
        const bool ok = (delta == 0.0) || (ml <= mn);
        a.M[l] = (pl < ml) ? pl : ml;
        a.Pst[l] = delta;
        if (!ok) a.ctl->notok = 1;  // benign race: every writer stores 1
    }
}

// grid: x = body tile (NBD_FORCE_THREADS bodies), y = stage i, z = j-block
__global__ void __launch_bounds__(NBD_FORCE_THREADS) nbd_force_kernel(const __grid_constant__ NbdArgs a) {
    __shared__ double4 sj[NBD_JBLOCK];
    const int64_t N = a.nbody, d = 3 * N;
    const int i = blockIdx.y, J = blockIdx.z;
    const int64_t j0 = (int64_t)J * NBD_JBLOCK;
    const int nj = (int)((N - j0) < NBD_JBLOCK ? (N - j0) : NBD_JBLOCK);
    const double *Qi = a.Q + (int64_t)i * d;
    for (int t = threadIdx.x; t < nj; t += blockDim.x) {
        const int64_t j = j0 + t;
        sj[t] = make_double4(Qi[3 * j], Qi[3 * j + 1], Qi[3 * j + 2], a.mass[j]);
    }
    __syncthreads();
    const int64_t body = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (body >= N) return;
    const double qx = Qi[3 * body], qy = Qi[3 * body + 1], qz = Qi[3 * body + 2];
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
    if (!ok) {  // some operand outside the fast-path range: exact intrinsics, same bits
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
    double *P = a.part + ((int64_t)J * 8 + i) * d;
    P[3 * body] = px;
    P[3 * body + 1] = py;
    P[3 * body + 2] = pz;
}

__global__ void nbd_vel_kernel(const __grid_constant__ NbdArgs a) {
    const int64_t d = 3 * a.nbody;
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= d) return;
    const int nj = (int)((a.nbody + NBD_JBLOCK - 1) / NBD_JBLOCK);
    const int k = a.ctl->k + 1;
    const bool stop = (k >= 2) && (a.ctl->notok == 0);
    const bool fin = stop || (k >= a.max_iters);
    double Lv[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        double acc = 0.0;
        for (int J = 0; J < nj; ++J) acc = dadd(acc, a.part[((int64_t)J * 8 + i) * d + l]);
        Lv[i] = dmul(a.hb[i], acc);
    }
    double v = a.y[d + l];
    if (fin) {
        double sv = Lv[0];
#pragma unroll
        for (int j = 1; j < 8; ++j) sv = dadd(sv, Lv[j]);
        const double q = dadd(a.y[l], a.sLq[l]);
        v = dadd(v, sv);
        a.y[l] = q;
        a.y[d + l] = v;
        if (!isfinite(q) || !isfinite(v)) a.ctl->nonfinite = 1;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            a.hist[(int64_t)j * 2 * d + l] = 0.0;
            a.hist[(int64_t)j * 2 * d + d + l] = Lv[j];
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
        a.V[(int64_t)i * d + l] = dadd(v, acc);
    }
}

__global__ void nbd_ctl_kernel(const __grid_constant__ NbdArgs a, int64_t *n_done, int64_t *stats) {
    NbdCtl *c = a.ctl;
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
        if (c->nonfinite && stats[1] == 0) stats[1] = *n_done;
    } else {
        c->k = k;
    }
}

// H of the system (canonical: kinetic terms, then row sums over j > i, Neumaier).
// Pass 1: one thread per row i writes its Neumaier row sum; pass 2 (one thread)
// adds the kinetic terms and the rows in order.
__global__ void nbd_energy_rows_kernel(const double *y, const double *mass, int64_t N, double G, double eps2,
                                       double *rows) {
    const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (i >= N) return;
    const double *q = y;
    Neumaier row;
    for (int64_t j = i + 1; j < N; ++j) {
        const double dx = dsub(q[3 * j], q[3 * i]);
        const double dy = dsub(q[3 * j + 1], q[3 * i + 1]);
        const double dz = dsub(q[3 * j + 2], q[3 * i + 2]);
        const double r2 = dfma(dz, dz, dfma(dy, dy, dfma(dx, dx, eps2)));
        row.add(-ddiv(dmul(G, dmul(mass[i], mass[j])), dsqrt(r2)));
    }
    rows[i] = row.result();
}

__global__ void nbd_energy_sum_kernel(const double *y, const double *mass, int64_t N, const double *rows,
                                      double *out) {
    const double *v = y + 3 * N;
    Neumaier tot;
    for (int64_t i = 0; i < N; ++i) {
        const double k = dfma(v[3 * i + 2], v[3 * i + 2], dfma(v[3 * i + 1], v[3 * i + 1], dmul(v[3 * i], v[3 * i])));
        tot.add(dmul(dmul(0.5, mass[i]), k));
    }
    for (int64_t i = 0; i < N; ++i) tot.add(rows[i]);
    *out = tot.result();
}

}  // namespace irk
