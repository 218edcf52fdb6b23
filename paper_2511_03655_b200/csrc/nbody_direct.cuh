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
//                         Fused mode (IRK_OPT_EXCHANGE = 1, NEXT f3): no separate
//                         collective -- nbd_pos stores each Q^[k] value straight into
//                         every rank's copy of its slot (NVLink peer pointers of a
//                         symmetric NCCL window) and its last CTA signals arrival to
//                         every rank; see the fused-exchange helpers below.
//   nbd_or                global stop = no flag set in any slot (same on every rank);
//                         fused mode: first waits for every rank's arrival (the
//                         j-blocks of the rank's own bodies are summed before it).
//   nbd_force  (a3)       (local body, stage, j-block) parallel: the canonical blocked
//                         direct sum (R-8) over ALL N bodies read from Qg,
//                         one thread = one partial sum over NBD_JBLOCK = 1024 bodies j
//                         staged in shared memory by TMA bulk copies (broadcast reads).
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
#ifndef NBD_FORCE_BLOCK
#define NBD_FORCE_BLOCK 256  // config 5, 100 steps: 64 threads 531 ms, 128: 524, 256: 519 (the j-block fill amortised over more bodies)
#endif
constexpr int NBD_FORCE_THREADS = NBD_FORCE_BLOCK;

struct NbdCtl {           // device-side control block (one per process)
    int64_t n;            // steps completed in this call
    int32_t k;            // sweeps completed in the current step
    int32_t notok;        // global: some component failed the stop test this sweep
    int32_t fin;          // last sweep finished a step
    int32_t nonfinite;    // global (after an exchange): some component became non-finite
    int32_t halt;         // stop integrating (divergence)
    int32_t xerr;         // fused exchange: a peer's arrival timed out (IRK_E_COMM)
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
    // fused exchange (xmode = 1): Qg is this rank's view of a symmetric NCCL window
    // holding two buffers [2][P][stride]; the sweep of exchange epoch e uses buffer
    // e & 1.  peerQ[r] = rank r's Qg and peerHdr[r] = rank r's header, both through
    // the NVLink (LSA) mapping; xhdr = this rank's header (see kX* below).
    int xmode, rank;
    double *const *peerQ;
    int64_t *const *peerHdr;
    int64_t *xhdr;
    int64_t qbuf;         // doubles per buffer (P * stride)
};

// Fused exchange header (int64 words of the window, before the Q buffers):
// [0, P) arrival epochs written by the peers (word r: rank r's last arrival),
// then local words: the epoch (barriers passed), the CTA counter of nbd_pos and
// the OR of its CTAs' "not converged" votes.
__device__ __forceinline__ int64_t *nbd_xepoch(const NbdArgs &a) { return a.xhdr + a.nshards; }
__device__ __forceinline__ int64_t *nbd_xcount(const NbdArgs &a) { return a.xhdr + a.nshards + 1; }
__device__ __forceinline__ int64_t *nbd_xnotok(const NbdArgs &a) { return a.xhdr + a.nshards + 2; }
constexpr int kXHeaderExtra = 3;

// gathered-slot buffer of the current sweep (buffer 0 unless fused)
__device__ __forceinline__ double *nbd_cur(const NbdArgs &a) {
    return a.xmode ? a.Qg + (*nbd_xepoch(a) & 1) * a.qbuf : a.Qg;
}
__device__ __forceinline__ double *nbd_slot(const NbdArgs &a, double *buf, int s) { return buf + (int64_t)s * a.stride; }
__device__ __forceinline__ const double *nbd_slot(const NbdArgs &a, const double *buf, int s) {
    return buf + (int64_t)s * a.stride;
}
__device__ __forceinline__ double *nbd_slot(const NbdArgs &a, int s) { return nbd_slot(a, nbd_cur(a), s); }
__device__ __forceinline__ int64_t nbd_flag_index(const NbdArgs &a) { return 24 * a.nloc; }
// element o of this rank's slot in buffer b of rank r's window (NVLink store target)
__device__ __forceinline__ double *nbd_peer(const NbdArgs &a, int r, int64_t b, int64_t o) {
    return a.peerQ[r] + (b & 1) * a.qbuf + (int64_t)a.shard * a.stride + o;
}

__device__ __forceinline__ int64_t ld_acquire_sys(const int64_t *p) {
    int64_t v;
    asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t nbd_globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
constexpr uint64_t kXTimeoutNs = 60ull * 1000000000ull;  // a peer that has not arrived in 60 s: IRK_E_COMM

// Barrier wait of the fused exchange (one thread): every rank's arrival word >= e + 1.
__device__ __forceinline__ bool nbd_xwait(const NbdArgs &a, int64_t e) {
    const uint64_t t0 = nbd_globaltimer();
    for (int r = 0; r < a.nshards; ++r)
        while (ld_acquire_sys(a.xhdr + r) < e + 1) {
            if (nbd_globaltimer() - t0 > kXTimeoutNs) return false;
            __nanosleep(64);
        }
    return true;
}
// Barrier arrival (one thread): publish e + 1 to every rank (release pattern: a
// system-scope fence, cumulative over every store that happens before it, then
// relaxed stores; the waiter's ld.acquire.sys completes the synchronisation).
__device__ __forceinline__ void nbd_xarrive(const NbdArgs &a, int64_t e) {
    asm volatile("fence.acq_rel.sys;" ::: "memory");  // one release fence, then relaxed stores
    for (int r = 0; r < a.nshards; ++r)
        asm volatile("st.relaxed.sys.global.b64 [%0], %1;" ::"l"(a.peerHdr[r] + a.rank), "l"(e + 1) : "memory");
}
// After barrier e: read the flags of buffer e & 1 from every slot, then clear this
// rank's flags in buffer (e + 1) & 1 of every rank (their last readers, the barrier
// e - 1 waits, are all behind barrier e; their next writers are this rank's own
// nbd_vel of this sweep and nbd_pos of the next, both later in stream order).
__device__ __forceinline__ void nbd_xflags(const NbdArgs &a, int64_t e, int &notok, int &bad) {
    double *buf = a.Qg + (e & 1) * a.qbuf;
    notok = bad = 0;
    for (int s = 0; s < a.nshards; ++s) {
        notok |= (__ldcv(nbd_slot(a, buf, s) + nbd_flag_index(a)) != 0.0);
        bad |= (__ldcv(nbd_slot(a, buf, s) + nbd_flag_index(a) + 1) != 0.0);
    }
    for (int r = 0; r < a.nshards; ++r) {
        *nbd_peer(a, r, e + 1, nbd_flag_index(a)) = 0.0;
        *nbd_peer(a, r, e + 1, nbd_flag_index(a) + 1) = 0.0;
    }
}

__global__ void nbd_init_kernel(const __grid_constant__ NbdArgs a) {
    const int64_t dl = 3 * a.nloc;
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l == 0 && !a.xmode) {  // fused: cleared by the previous barrier (nbd_xflags)
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
    const int k = a.ctl->k + 1;
    const int64_t e = a.xmode ? *nbd_xepoch(a) : 0;
    // own slot: Q^[k-1] is read from it; Q^[k] goes to it (NCCL / one GPU) or, fused,
    // to this rank's slot of buffer e & 1 in every rank's window (Q^[k-1] is in e - 1)
    double *Q = a.xmode ? nbd_slot(a, a.Qg + ((e + 1) & 1) * a.qbuf, a.shard) : nbd_slot(a, a.shard);
    bool ok = true;
    if (l < dl) {
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
            const double d = dabs(dsub(qn, Q[(int64_t)i * dl + l]));
            delta = (d > delta) ? d : delta;
            if (a.xmode) {
#ifdef NBD_XSELF_LOCAL
                a.Qg[(e & 1) * a.qbuf + (int64_t)a.shard * a.stride + (int64_t)i * dl + l] = qn;
                for (int r = 0; r < a.nshards; ++r)
                    if (r != a.rank) *nbd_peer(a, r, e, (int64_t)i * dl + l) = qn;
#else
                for (int r = 0; r < a.nshards; ++r) *nbd_peer(a, r, e, (int64_t)i * dl + l) = qn;
#endif
            } else {
                Q[(int64_t)i * dl + l] = qn;
            }
        }
        if (k >= 2) {
            const double pl = a.Pst[l], ml = a.M[l];
            const double mn = (delta < pl) ? delta : pl;
            ok = (delta == 0.0) || (ml <= mn);
            a.M[l] = (pl < ml) ? pl : ml;
            a.Pst[l] = delta;
            if (!ok && !a.xmode) Q[nbd_flag_index(a)] = 1.0;  // benign race: every writer stores 1
        }
    }
    if (!a.xmode) return;
    // Fused exchange epilogue: the CTA's threads' votes are OR-ed at the CTA barrier
    // (which also orders their stores before thread 0's); thread 0 takes a ticket
    // with an acq_rel atomic; the CTA with the last ticket pushes the "not
    // converged" flag and signals arrival e + 1 to every rank after a system-scope
    // release fence (cumulative: every CTA's stores happen before the arrival -- the
    // CTA-barrier-then-release pattern of NCCL's own LSA barrier).
    const int bad = __syncthreads_or(!ok);
    if (threadIdx.x == 0) {
        unsigned long long *cnt = reinterpret_cast<unsigned long long *>(nbd_xcount(a));
        unsigned long long *nok = reinterpret_cast<unsigned long long *>(nbd_xnotok(a));
        if (bad) atomicOr(nok, 1ull);
        // acq_rel at gpu scope: this CTA's stores are released to, and every earlier
        // CTA's acquired by, the CTA that takes the last ticket
        unsigned long long prev;
        asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(prev) : "l"(cnt) : "memory");
        if (prev == gridDim.x - 1) {
            const bool any = atomicExch(nok, 0ull) != 0ull;
            *cnt = 0ull;
            if (any)
                for (int r = 0; r < a.nshards; ++r) *nbd_peer(a, r, e, nbd_flag_index(a)) = 1.0;
            nbd_xarrive(a, e);
        }
    }
}

// global flags from every slot (after the exchange)
__global__ void nbd_or_kernel(const __grid_constant__ NbdArgs a) {
    int any = 0, bad = 0;
    if (a.xmode) {  // fused: barrier e (every rank's Q^[k] and flags are in), then the flags
        const int64_t e = *nbd_xepoch(a);
        if (!nbd_xwait(a, e)) {
            a.ctl->xerr = 1;
            return;
        }
        nbd_xflags(a, e, any, bad);
        a.ctl->notok = any;
        a.ctl->nonfinite = bad;
        return;
    }
    for (int s = 0; s < a.nshards; ++s) {
        any |= (nbd_slot(a, s)[nbd_flag_index(a)] != 0.0);
        bad |= (nbd_slot(a, s)[nbd_flag_index(a) + 1] != 0.0);
    }
    a.ctl->notok = any;
    a.ctl->nonfinite = bad;
}

// grid: x = local body tile (NBD_FORCE_THREADS bodies), y = stage i, z = j-block.
// The j-block's positions and masses are staged in shared memory as packed
// xyz[3 x 1024] and m[1024]: by two TMA bulk copies (cp.async.bulk, completion on
// an mbarrier) when the block's bodies are contiguous in one slot of the gathered
// buffer and 16-byte aligned -- every j-block of config 5 -- else by a gather.
// The pair loop reads them as broadcast double2 loads, two bodies per trip, in j
// order (the canonical per-block sum).
#ifndef NBD_FORCE_MINB
#define NBD_FORCE_MINB 1
#endif
template <bool EXACT, bool G1>
__device__ __forceinline__ void nbd_pair(double xj, double yj, double zj, double mj, double qx, double qy, double qz,
                                         double G, double eps2, double &px, double &py, double &pz, bool &ok) {
    const double dx = dsub(xj, qx), dy = dsub(yj, qy), dz = dsub(zj, qz);
    const double r2 = dfma(dz, dz, dfma(dy, dy, dfma(dx, dx, eps2)));
    const double w = EXACT ? ddiv(G, dmul(r2, dsqrt(r2)))
                           : (G1 ? drcp_fast(dmul(r2, dsqrt_fast(r2, ok)), ok)   // G == 1: same bits
                                 : ddiv_fast(G, dmul(r2, dsqrt_fast(r2, ok)), ok));
    const double s = dmul(mj, w);
    px = dfma(s, dx, px);
    py = dfma(s, dy, py);
    pz = dfma(s, dz, pz);
}
template <bool EXACT, bool G1>
__device__ __forceinline__ void nbd_pairs(const double *sxyz, const double *sm, int n, double qx, double qy, double qz,
                                          double G, double eps2, double &px, double &py, double &pz, bool &ok) {
    const double2 *x2 = reinterpret_cast<const double2 *>(sxyz);
    const double2 *m2 = reinterpret_cast<const double2 *>(sm);
#pragma unroll 2
    for (int t2 = 0; t2 < n / 2; ++t2) {  // bodies 2 t2 and 2 t2 + 1
        const double2 a0 = x2[3 * t2], a1 = x2[3 * t2 + 1], a2 = x2[3 * t2 + 2], mm = m2[t2];
        nbd_pair<EXACT, G1>(a0.x, a0.y, a1.x, mm.x, qx, qy, qz, G, eps2, px, py, pz, ok);
        nbd_pair<EXACT, G1>(a1.y, a2.x, a2.y, mm.y, qx, qy, qz, G, eps2, px, py, pz, ok);
    }
    if (n & 1) {
        const int t = n - 1;
        nbd_pair<EXACT, G1>(sxyz[3 * t], sxyz[3 * t + 1], sxyz[3 * t + 2], sm[t], qx, qy, qz, G, eps2, px, py, pz, ok);
    }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <bool G1>
__global__ void __launch_bounds__(NBD_FORCE_THREADS, NBD_FORCE_MINB) nbd_force_kernel(const __grid_constant__ NbdArgs a,
                                                                                      int jbase) {
    __shared__ __align__(128) double sxyz[3 * NBD_JBLOCK];
    __shared__ __align__(16) double smass[NBD_JBLOCK];
    __shared__ __align__(8) uint64_t mbar;
    const int64_t N = a.nbody, nloc = a.nloc, dl = 3 * nloc;
    const int i = blockIdx.y, J = jbase + (int)blockIdx.z;  // j-blocks [jbase, jbase + gridDim.z)
    const int64_t j0 = (int64_t)J * NBD_JBLOCK;
    const int nj = (int)((N - j0) < NBD_JBLOCK ? (N - j0) : NBD_JBLOCK);
    const double *cur = nbd_cur(a);
    // ---- stage the j-block ----
    const int s0 = (int)(j0 / nloc);
    const double *src = nbd_slot(a, cur, s0) + (int64_t)i * dl + 3 * (j0 - (int64_t)s0 * nloc);
    const double *msrc = a.mass + j0;
    const bool bulk = ((j0 + nj - 1) / nloc == s0) && !(nj & 1) &&
                      !((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(msrc)) & 15);
    if (bulk) {
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            const uint32_t bx = 24u * (uint32_t)nj, bm = 8u * (uint32_t)nj;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&mbar)), "r"(bx + bm)
                         : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(sxyz)),
                "l"(src), "r"(bx), "r"(smem_u32(&mbar))
                : "memory");
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    smem_u32(smass)),
                "l"(msrc), "r"(bm), "r"(smem_u32(&mbar))
                : "memory");
        }
    } else {
        for (int t = threadIdx.x; t < nj; t += blockDim.x) {
            const int64_t j = j0 + t;
            const double *Qj = nbd_slot(a, cur, (int)(j / nloc)) + (int64_t)i * dl + 3 * (j % nloc);
            sxyz[3 * t] = Qj[0];
            sxyz[3 * t + 1] = Qj[1];
            sxyz[3 * t + 2] = Qj[2];
            smass[t] = a.mass[j];
        }
    }
    const int64_t body = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;  // local index
    const bool act = body < nloc;
    double qx = 0.0, qy = 0.0, qz = 0.0;
    if (act) {  // (overlaps the bulk copies)
        const double *Qa = nbd_slot(a, cur, a.shard) + (int64_t)i * dl + 3 * body;
        qx = Qa[0], qy = Qa[1], qz = Qa[2];
    }
    __syncthreads();  // gather stores visible / mbarrier initialised before anyone waits on it
    if (bulk) {
        asm volatile(
            "{\n"
            ".reg .pred P1;\n"
            "WAIT_%=:\n"
            "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0;\n"
            "@!P1 bra WAIT_%=;\n"
            "}\n" ::"r"(smem_u32(&mbar))
            : "memory");
    }
    // ---- range pre-check: with every coordinate of the block's bodies j and i finite
    // and below 2^290 in magnitude, eps^2 >= 2^-600 and 2^-100 <= G <= 2^100, every
    // pair has eps^2 <= r2 < 2^600 (r2 is an fma chain of non-negative terms added to
    // eps^2, rounding is monotone), so r2 * sqrt(r2) and the weight stay normal and
    // the fast division / square root paths are valid for every pair: the per-pair
    // range predicates can be skipped (same bits, nbd_force)
    bool in_range = !act || (fabs(qx) < 0x1p290 && fabs(qy) < 0x1p290 && fabs(qz) < 0x1p290);
    for (int t = threadIdx.x; t < 3 * nj; t += blockDim.x) in_range = in_range && fabs(sxyz[t]) < 0x1p290;
    const bool unchecked = __syncthreads_and(in_range) && a.eps2 >= 0x1p-600 && a.G >= 0x1p-100 && a.G <= 0x1p100;
    double px = 0.0, py = 0.0, pz = 0.0;
    if (unchecked) {
        bool dummy = true;
        if (act) nbd_pairs<false, G1>(sxyz, smass, nj, qx, qy, qz, a.G, a.eps2, px, py, pz, dummy);
        if (!act) return;
        double *P = a.part + ((int64_t)J * 8 + i) * dl;
        P[3 * body] = px;
        P[3 * body + 1] = py;
        P[3 * body + 2] = pz;
        return;
    }
    // ---- the block's pair sums (pass 1 only if an operand left the fast-path range) ----
    bool ok = true;
    if (act) nbd_pairs<false, G1>(sxyz, smass, nj, qx, qy, qz, a.G, a.eps2, px, py, pz, ok);
    if (__syncthreads_or(!ok)) {  // exact intrinsics, same bits, for the whole block
        px = py = pz = 0.0;
        if (act) nbd_pairs<true, G1>(sxyz, smass, nj, qx, qy, qz, a.G, a.eps2, px, py, pz, ok);
    }
    if (!act) return;
    double *P = a.part + ((int64_t)J * 8 + i) * dl;
    P[3 * body] = px;
    P[3 * body + 1] = py;
    P[3 * body + 2] = pz;
}

__global__ void nbd_vel_kernel(const __grid_constant__ NbdArgs a) {
    const int64_t dl = 3 * a.nloc;
    const int64_t l = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (l >= dl) return;
    if (a.ctl->nonfinite || a.ctl->xerr) return;  // diverged at the previous step: frozen (R-10)
    const int nj = (int)((a.nbody + NBD_JBLOCK - 1) / NBD_JBLOCK);
    const int k = a.ctl->k + 1;
    const bool stop = (k >= 2) && (a.ctl->notok == 0);
    const bool fin = stop || (k >= a.max_iters);
    double Lv[8];
    if (nj <= 8) {  // (N <= 8,192: all 64 partial sums loaded before the dadd chains -- one
                    // memory latency per thread instead of one per j-block)
        double pv[8][8];
#pragma unroll
        for (int J = 0; J < 8; ++J)
#pragma unroll
            for (int i = 0; i < 8; ++i) pv[J][i] = J < nj ? __ldcg(&a.part[((int64_t)J * 8 + i) * dl + l]) : 0.0;
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            double acc = 0.0;
#pragma unroll
            for (int J = 0; J < 8; ++J)
                if (J < nj) acc = dadd(acc, pv[J][i]);
            Lv[i] = dmul(a.hb[i], acc);
        }
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            double acc = 0.0;
            for (int J = 0; J < nj; ++J) acc = dadd(acc, a.part[((int64_t)J * 8 + i) * dl + l]);
            Lv[i] = dmul(a.hb[i], acc);
        }
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
        if (!isfinite(q) || !isfinite(v)) {
            if (a.xmode) {  // into buffer e + 1, read after the next barrier
                const int64_t e = *nbd_xepoch(a);
                for (int r = 0; r < a.nshards; ++r) *nbd_peer(a, r, e + 1, nbd_flag_index(a) + 1) = 1.0;
            } else {
                nbd_slot(a, a.shard)[nbd_flag_index(a) + 1] = 1.0;
            }
        }
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
    if (a.xmode) {
        *nbd_xepoch(a) += 1;  // barrier e passed: the next sweep uses the other buffer
    } else {
        for (int s = first_local; s < first_local + nlocal; ++s) nbd_slot(a, s)[nbd_flag_index(a)] = 0.0;
    }
    if (c->nonfinite || c->xerr) {  // some shard diverged at the last completed step (or a peer is gone)
        if (c->nonfinite && stats[1] == 0) stats[1] = *n_done;
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

// fused mode, after a call's last sweep: one more barrier (epoch e) so that a
// divergence at the last step (nbd_vel's flag in buffer e & 1) is seen by every
// rank, exactly as the NCCL mode's final all-gather
__global__ void nbd_xfinal_kernel(const __grid_constant__ NbdArgs a, int64_t *n_done, int64_t *stats) {
    const int64_t e = *nbd_xepoch(a);
    nbd_xarrive(a, e);
    if (!nbd_xwait(a, e)) {
        a.ctl->xerr = 1;
        return;
    }
    int notok, bad;
    nbd_xflags(a, e, notok, bad);
    *nbd_xepoch(a) = e + 1;
    if (bad && stats[1] == 0) stats[1] = *n_done;
}

// ---- energy (canonical: kinetic terms, then row sums over j > i, Neumaier) ----
// Qall: all N positions (3N, gathered); each shard writes its kinetic terms and
// row sums into its slot [kin(nloc) | row(nloc)] of `terms` ([P][2*nloc]); the
// total is added by one thread over all kinetic terms, then all rows, in order
// (one compensated sum in the oracle's order: sequential by definition).
// Row r of the shard (body i = b0 + r) is the in-order Neumaier sum over j > i of
// -G m_i m_j / sqrt(r_ij^2 + eps^2).  The terms of a row are independent, only
// their sum is sequential: a block takes 32 rows, its 256 threads evaluate the
// terms of a 32 x 128 tile (rows x consecutive j) into shared memory, and lane r of
// warp 0 adds row r's 128 terms in j order -- the same Neumaier sequence, so the
// same bits as one thread per row, with the divisions and square roots of a tile
// in flight at once.  Launch ceil(nloc / 32) blocks of NBD_EROW_THREADS threads.
constexpr int NBD_EROW_THREADS = 256, NBD_EROW_ROWS = 32, NBD_EROW_COLS = 128;
__global__ void __launch_bounds__(NBD_EROW_THREADS) nbd_energy_terms_kernel(const double *Qall, const double *vloc,
                                                                            const double *mass, int64_t N, int64_t b0,
                                                                            int64_t nloc, double G, double eps2,
                                                                            double *slot) {
    __shared__ double T[NBD_EROW_ROWS][NBD_EROW_COLS + 1];
    const double *q = Qall;
    const int64_t r0 = (int64_t)blockIdx.x * NBD_EROW_ROWS;
    const int tx = threadIdx.x;
    if (tx < NBD_EROW_ROWS && r0 + tx < nloc) {  // kinetic terms
        const int64_t r = r0 + tx;
        const double *v = vloc + 3 * r;
        const double k = dfma(v[2], v[2], dfma(v[1], v[1], dmul(v[0], v[0])));
        slot[r] = dmul(dmul(0.5, mass[b0 + r]), k);
    }
    Neumaier row;  // (lane tx < 32 of warp 0: row r0 + tx)
    const int64_t ilo = b0 + r0;
    for (int64_t jc = ilo + 1; jc < N; jc += NBD_EROW_COLS) {
        for (int e = tx; e < NBD_EROW_ROWS * NBD_EROW_COLS; e += NBD_EROW_THREADS) {
            const int rr = e / NBD_EROW_COLS, cc = e % NBD_EROW_COLS;
            const int64_t i = ilo + rr, j = jc + cc;
            if (r0 + rr < nloc && j > i && j < N) {
                const double dx = dsub(q[3 * j], q[3 * i]);
                const double dy = dsub(q[3 * j + 1], q[3 * i + 1]);
                const double dz = dsub(q[3 * j + 2], q[3 * i + 2]);
                const double r2 = dfma(dz, dz, dfma(dy, dy, dfma(dx, dx, eps2)));
                T[rr][cc] = -ddiv(dmul(G, dmul(mass[i], mass[j])), dsqrt(r2));
            }
        }
        __syncthreads();
        if (tx < NBD_EROW_ROWS && r0 + tx < nloc) {
            const int64_t i = ilo + tx;
            const int64_t c0 = (i + 1 > jc) ? i + 1 - jc : 0;
            const int64_t c1 = (N - jc < NBD_EROW_COLS) ? N - jc : NBD_EROW_COLS;
            for (int64_t cc = c0; cc < c1; ++cc) row.add(T[tx][cc]);
        }
        __syncthreads();
    }
    if (tx < NBD_EROW_ROWS && r0 + tx < nloc) slot[nloc + r0 + tx] = row.result();
}

// One block: the terms are staged through shared memory in chunks by all threads
// (coalesced), and thread 0 runs the compensated sum over each chunk in order --
// the oracle's order (every kinetic term, then every row, shard by shard), so the
// same bits as one thread reading global memory, without a global-load latency
// per term.  Launch with NBD_ESUM_THREADS threads.
constexpr int NBD_ESUM_THREADS = 256, NBD_ESUM_CHUNK = 4096;
__global__ void __launch_bounds__(NBD_ESUM_THREADS) nbd_energy_sum_kernel(const double *terms, int P, int64_t nloc,
                                                                          double *out) {
    __shared__ double buf[NBD_ESUM_CHUNK];
    const int64_t total = 2 * (int64_t)P * nloc;
    Neumaier tot;
    for (int64_t k0 = 0; k0 < total; k0 += NBD_ESUM_CHUNK) {
        const int n = (int)((total - k0) < NBD_ESUM_CHUNK ? (total - k0) : NBD_ESUM_CHUNK);
        for (int t = threadIdx.x; t < n; t += blockDim.x) {
            const int64_t k = k0 + t, half = (int64_t)P * nloc;  // k-th term of the summation order
            const int64_t kk = k < half ? k : k - half, sh = kk / nloc, r = kk - sh * nloc;
            buf[t] = terms[sh * 2 * nloc + (k < half ? 0 : nloc) + r];
        }
        __syncthreads();
        if (threadIdx.x == 0)
            for (int t = 0; t < n; ++t) tot.add(buf[t]);
        __syncthreads();
    }
    if (threadIdx.x == 0) *out = tot.result();
}

}  // namespace irk
