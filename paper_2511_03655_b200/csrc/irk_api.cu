// C ABI of the IRKGL16 library (include/irk.h): context, workspace, dispatch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges for nsys timelines (no-op without a tool)

#include "../../include/irk.h"
#include "balance.cuh"
#ifndef G1Q_UNITS
#define G1Q_UNITS 16  // step chunks per trajectory of the ens_g1q work queue (config 2: 16 -> 81.4 ms, 12: 81.8, 32: 82.0, 8: 83.1)
#endif
#ifndef G1Q_MAX_BPS
#define G1Q_MAX_BPS 0  // > 0: force the heavy ens_g1q kernel at this many blocks per SM (A/B builds); 0: auto
#endif
#include "ensemble_g1.cuh"
#include "ensemble_g8.cuh"
#include "ensemble_g8m.cuh"
#include "ensemble_fo.cuh"
#include "ensemble_nbody.cuh"
#include "ensemble_nbody8.cuh"
#include "ensemble_nbody8m.cuh"
#include "ensemble_chain.cuh"
#include "nbody_direct.cuh"
#include "problems.cuh"
#include "tableau.h"

using irk::EnsArgs;
using irk::Tableau;

static thread_local std::string g_create_error;

struct irk_ctx {
    int problem = 0, dim = 0;
    double h = 0.0;
    int64_t nsteps = 0, batch = 0;
    std::vector<double> params;
    bool have_params = false;
    int mode = 0, max_iters = 100, mapping = 0;
    int64_t balance = -1;  // IRK_OPT_BALANCE: -1 auto, 0 off, >0 chunk length
    int schedule = 0;      // IRK_OPT_SCHEDULE: 0 auto, 1 chunked launches, 2 persistent work queue
    int g1q_blocks_per_sm = 0;  // occupancy of the work-queue kernels (queried once)
    int g1q_heavy_blocks_per_sm = 0;
    int chain_blocks_per_sm[5] = {0, 0, 0, 0, 0};
    int nbody_blocks_per_sm[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    int fo_blocks_per_sm = 0;
    int nbody8_blocks_per_sm[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    int nbody8m_blocks_per_sm[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    int nbody8m_hi_blocks_per_sm[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0};
    int local_energy = 0;  // IRK_OPT_LOCAL_ENERGY
    int64_t energy_every = 0;
    Tableau T;
    std::string err;
    // buffers owned by the ctx for irk_integrate_host
    double *d_y = nullptr, *d_energy = nullptr;
    int64_t *d_iters = nullptr;
    void *d_ws = nullptr;
    size_t cap_y = 0, cap_energy = 0, cap_ws = 0;
    int64_t cap_iters = 0;
    // large-N path
    double *d_mass = nullptr, *d_rows = nullptr;
    irk::NbdCtl *h_ctl = nullptr;  // pinned readback of the control block
    int nranks = 1, rank = 0;      // NCCL body sharding (irk_set_comm)
    int vshards = 1;               // virtual shards on one GPU (IRK_OPT_VSHARDS)
    int device_loop = 1;           // IRK_OPT_DEVICE_LOOP (large-N path)
    int device_loop_used = 0;      // IRK_INFO_DEVICE_LOOP_USED: the last call ran the graph loop
    int mapping_used = 0;          // IRK_INFO_MAPPING_USED: the IRK_MAP_* the last call resolved to
    void *nccl_comm = nullptr;
    // fused exchange (IRK_OPT_EXCHANGE = 1): symmetric NCCL window [header | 2 x P x stride]
    int exchange = 0;
    void *xbuf = nullptr, *xwin = nullptr;
    size_t xbytes = 0, xqoff = 0;
    void **d_xpeers = nullptr;  // [2P]: rank r's Q buffers, rank r's header (NVLink mapping)
};

namespace {

constexpr size_t kHeader = 64;
#ifndef IRK_UNIT_G
#define IRK_UNIT_G 1  // G = 1 / GM = 1 kernels use the reciprocal form of the division (fp64.cuh drcp_fast)
#endif
#ifndef IRK_CHAINW_MAX
#define IRK_CHAINW_MAX 384  // FPU chains: two warps per chain up to this batch (20,000 steps, 1 / 2 warps: 256 chains 59.0 / 51.1 ms, 512: 59.3 / 65.1, 1,024: 99.9 / 112.5)
#endif
#ifndef IRK_G8_AUTO_MAX
#define IRK_G8_AUTO_MAX 6144
#endif
#ifndef IRK_G4_AUTO_MAX
#define IRK_G4_AUTO_MAX 12288
#endif
#ifndef IRK_G2_AUTO_MAX
#define IRK_G2_AUTO_MAX 0  // g2 is not chosen by auto any more (g1 on 2 blocks per SM beats it)
#endif
// IRK_OPT_MAPPING auto (Kepler, HH): g8m (stage per lane, DMMA contractions; faster than
// g8 at every batch up to 8,192: config 1 13.8 -> 13.1 ms, 6,144: 22.2 -> 20.9 ms) up to
// kG8AutoMaxBatch, g4 up to kG4AutoMaxBatch, then g1
// (ens_g1q, launch geometry in launch_g1q).  Measured with tools/ab.py, config-2 generator,
// 10,000 steps (profiles/r2/ab_mapping_crossover.json), g1 / g2 / g4 / g8 ms:
// 4,096: 38.9/31.2/22.2/19.3; 6,144: 38.9/31.6/26.8/23.9; 8,192: 38.7/31.5/27.0/29.6;
// 12,288: 39.5/42.5/34.7/45.0; 16,384: 39.2/42.9/56.1/54.3; 24,576: 43.2/56.8/67.4/76.6
// (g1 at 2 blocks per SM from 16,384 on).
constexpr int64_t kG8AutoMaxBatch = IRK_G8_AUTO_MAX;
constexpr int64_t kG4AutoMaxBatch = IRK_G4_AUTO_MAX;
constexpr int64_t kG2AutoMaxBatch = IRK_G2_AUTO_MAX;
#ifndef IRK_N8M_HIREG_MAX
#define IRK_N8M_HIREG_MAX 6144
#endif
constexpr int64_t kN8mHiRegMaxBatch = IRK_N8M_HIREG_MAX;  // ens_nbody8m at 255 registers up to this batch
constexpr int64_t kFo8AutoMaxBatch = INT64_MAX;  // first-order mode: stage per lane at every measured batch
                                                 // (tools/fo_bench.py: 1 to 65,536 trajectories)

int fail(irk_ctx *c, int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    return code;
}

int cuda_check(irk_ctx *c, cudaError_t e, const char *what) {
    if (e == cudaSuccess) return IRK_OK;
    return fail(c, IRK_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

// NVTX range for the phases of a call (irk_integrate, config-5 segments, exchanges).
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

// rows of y / history held by this process (the local bodies' 6N/P rows when sharded under NCCL)
int64_t local_dim(const irk_ctx *c) {
    return (c->problem == IRK_NBODY_DIRECT && c->nccl_comm) ? c->dim / c->nranks : c->dim;
}
size_t hist_bytes(const irk_ctx *c) { return sizeof(double) * 8 * (size_t)local_dim(c) * c->batch; }
size_t stats_bytes(const irk_ctx *c) { return sizeof(int64_t) * 4 * (size_t)c->batch; }

int n_params_expected(int problem, int dim) {
    switch (problem) {
    case IRK_KEPLER: return 1;
    case IRK_HENON_HEILES: return 2;
    case IRK_FPU_BETA: return 1;
    case IRK_SCHWARZSCHILD: return 3;
    case IRK_NBODY:
    case IRK_NBODY_DIRECT: return 2 + dim / 6;
    }
    return -1;
}

// mu~, nu~, c~ into the constant bank of the current device, enqueued on the
// call's stream every call (1.1 KB).  The values are the same for every ctx
// (one fixed tableau), so concurrent calls on other streams read the same bits;
// uploading per call (not once per device index) survives a cudaDeviceReset,
// which would otherwise leave the bank zeroed behind a stale "done" flag.
int upload_constants(irk_ctx *c, cudaStream_t st) {
    int rc;
    if ((rc = cuda_check(c, cudaMemcpyToSymbolAsync(irk::c_mu, c->T.mu, sizeof c->T.mu, 0, cudaMemcpyHostToDevice, st),
                         "upload mu")))
        return rc;
    if ((rc = cuda_check(c, cudaMemcpyToSymbolAsync(irk::c_nu, c->T.nu, sizeof c->T.nu, 0, cudaMemcpyHostToDevice, st),
                         "upload nu")))
        return rc;
    return cuda_check(c, cudaMemcpyToSymbolAsync(irk::c_c, c->T.c, sizeof c->T.c, 0, cudaMemcpyHostToDevice, st),
                      "upload c");
}

__global__ void advance_n_kernel(int64_t *n_done, int64_t nsteps) { *n_done += nsteps; }

// Workspace regions after the stats block (irk_workspace_bytes).
struct Sched {
    int32_t *perm, *csweeps, *sorted, *bins;
};
// thread-slot capacity of the scheduler's permutation (>= slots of any ensemble kernel)
// >= the thread slots of every mapping: blocks x (warps x slots per warp) rounds B up
// by less than one block (< 64 slots; e.g. ens_nbody: 10 slots per block, B = 16,384
// -> 16,390 slots).  (Round 1 used round_up(B, 256), which the nbody mapping
// overran into the csweeps array: a chunked, cost-sorted launch could then run a
// trajectory in two groups at once.)
int64_t perm_slots(int64_t B) { return (B + 64 + 255) / 256 * 256; }
size_t sched_bytes(const irk_ctx *c) {
    return sizeof(int32_t) * ((size_t)perm_slots(c->batch) + 2 * (size_t)c->batch + irk::kCostBins);
}
Sched sched_of(const irk_ctx *c, char *ws) {
    Sched s;
    s.perm = reinterpret_cast<int32_t *>(ws + kHeader + hist_bytes(c) + stats_bytes(c));
    s.csweeps = s.perm + perm_slots(c->batch);
    s.sorted = s.csweeps + c->batch;
    s.bins = s.sorted + c->batch;
    return s;
}

// chunk length of the cost-balanced schedule (0 = one launch, identity order)
int64_t balance_chunk(const irk_ctx *c) {
    if (c->balance == 0 || c->nsteps == 0) return 0;
    if (c->balance > 0) return c->balance < c->nsteps ? c->balance : 0;
    if (c->batch < 8192) return 0;  // auto: only worth it with many warps per SM
    int64_t ch = (c->nsteps + 7) / 8;
    return ch < c->nsteps ? ch : 0;
}

// Runs the call's nsteps in (cost-balanced) chunks.  `launch(args, nblocks)` starts
// one ensemble kernel over `nblocks` blocks; a block holds `wpb` warps of `spw`
// trajectory slots each.
template <class LaunchFn>
int run_chunks(irk_ctx *c, EnsArgs &a, char *ws, int64_t nblocks, int wpb, int spw, cudaStream_t st,
               LaunchFn launch) {
    const int64_t chunk = balance_chunk(c);
    const int64_t nslots = nblocks * wpb * spw;
    if (chunk == 0) {  // one launch over all steps, identity assignment
        a.nsteps = c->nsteps;
        a.c0 = 0;
        a.csweeps = nullptr;
        a.perm = nullptr;
        a.nslots = c->batch;
        launch(a, nblocks);
        int rc = cuda_check(c, cudaGetLastError(), "ensemble kernel launch");
        if (rc) return rc;
        advance_n_kernel<<<1, 1, 0, st>>>(reinterpret_cast<int64_t *>(ws), c->nsteps);
        return cuda_check(c, cudaGetLastError(), "advance_n launch");
    }
    Sched sc = sched_of(c, ws);
    // auto schedule: a short unsorted pilot chunk (1/4 of a chunk) measures the
    // costs, then full chunks run cost-sorted; an explicit BALANCE = C uses C throughout
    const int64_t pilot = (c->balance < 0) ? (chunk + 3) / 4 : chunk;
    int64_t prev_steps = 0;
    for (int64_t c0 = 0; c0 < c->nsteps;) {
        const int64_t want = (c0 == 0) ? pilot : chunk;
        const int64_t steps = (c->nsteps - c0 < want) ? c->nsteps - c0 : want;
        a.nsteps = steps;
        a.c0 = c0;
        a.csweeps = sc.csweeps;
        if (c0 == 0) {
            a.perm = nullptr;
            a.nslots = c->batch;
        } else {  // sort by the previous chunk's sweeps per step, deal warps to blocks
            const unsigned sb = (unsigned)((c->batch + 255) / 256 < 1184 ? (c->batch + 255) / 256 : 1184);
            const int rcm = cuda_check(c, cudaMemsetAsync(sc.bins, 0, sizeof(int32_t) * irk::kCostBins, st), "memset bins");
            if (rcm) return rcm;
            irk::cost_hist_kernel<<<sb, 256, 0, st>>>(sc.csweeps, c->batch, prev_steps, sc.bins);
            irk::cost_scan_kernel<<<1, irk::kCostBins, 0, st>>>(sc.bins);
            irk::cost_scatter_kernel<<<sb, 256, 0, st>>>(sc.csweeps, c->batch, prev_steps, sc.bins, sc.sorted);
            irk::cost_perm_kernel<<<(unsigned)((nslots + 255) / 256), 256, 0, st>>>(sc.sorted, c->batch, nblocks, wpb,
                                                                                      spw, sc.perm);
            a.perm = sc.perm;
            a.nslots = nslots;
        }
        prev_steps = steps;
        c0 += steps;
        launch(a, nblocks);
        int rc = cuda_check(c, cudaGetLastError(), "ensemble kernel launch");
        if (rc) return rc;
        advance_n_kernel<<<1, 1, 0, st>>>(reinterpret_cast<int64_t *>(ws), steps);
        if ((rc = cuda_check(c, cudaGetLastError(), "advance_n launch"))) return rc;
    }
    return IRK_OK;
}

// ---- large-N single system (IRK_NBODY_DIRECT), body-sharded ----
int64_t nbd_nj(int64_t N) { return (N + irk::NBD_JBLOCK - 1) / irk::NBD_JBLOCK; }
int nbd_P(const irk_ctx *c) { return c->nccl_comm ? c->nranks : (c->vshards > 1 ? c->vshards : 1); }
int nbd_nlocal(const irk_ctx *c) { return c->nccl_comm ? 1 : nbd_P(c); }  // shards driven by this process
int64_t nbd_stride(const irk_ctx *c) { return 24 * ((int64_t)c->dim / 6 / nbd_P(c)) + 2; }
size_t nbd_bytes(const irk_ctx *c) {
    if (c->problem != IRK_NBODY_DIRECT) return 0;
    const int P = nbd_P(c);
    const size_t N = (size_t)c->dim / 6, nloc = N / P, dl = 3 * nloc;
    const size_t per_shard = 8 * dl + 3 * dl + (size_t)nbd_nj(N) * 8 * dl;
    return 256 + sizeof(double) * ((size_t)P * nbd_stride(c) + nbd_nlocal(c) * per_shard + 3 * N + 2 * N);
}

int nccl_check(irk_ctx *c, int r, const char *what);
int nccl_allgather_inplace(irk_ctx *c, double *buf, size_t count_per_rank, cudaStream_t st);
int xsetup(irk_ctx *c, size_t qbytes, double *scratch, cudaStream_t st);

int launch_direct(irk_ctx *c, double *y, double t0, char *ws, double *energy, int64_t *iters, cudaStream_t st) {
    (void)t0;
    const int64_t N = c->dim / 6;
    const int P = nbd_P(c), nlocal = nbd_nlocal(c);
    const int first = c->nccl_comm ? c->rank : 0;
    const int64_t nloc = N / P, dl = 3 * nloc, stride = nbd_stride(c);
    const bool nccl = c->nccl_comm != nullptr;
    const bool fused = nccl && c->exchange == 1;
    int rc;
    if (c->exchange == 1 && !nccl)
        return fail(c, IRK_E_STATE, "irk_integrate: IRK_OPT_EXCHANGE = 1 needs a communicator (irk_set_comm)");
    // The fused exchange's cross-GPU memory ordering has only run at one rank
    // (DESIGN.md section 8); more ranks need an explicit opt-in until it has run there.
    if (fused && c->nranks > 1) {
        const char *ok = getenv("IRK_EXPERIMENTAL_FUSED_EXCHANGE");
        if (!ok || strcmp(ok, "1") != 0)
            return fail(c, IRK_E_STATE, "irk_integrate: IRK_OPT_EXCHANGE = 1 with %d ranks is experimental "
                                        "(never run across GPUs); set IRK_EXPERIMENTAL_FUSED_EXCHANGE=1 to use it",
                        c->nranks);
    }
    if (!c->d_mass) {
        if ((rc = cuda_check(c, cudaMalloc(&c->d_mass, sizeof(double) * N), "cudaMalloc mass"))) return rc;
        if ((rc = cuda_check(c, cudaMallocHost(&c->h_ctl, sizeof(irk::NbdCtl)), "cudaMallocHost ctl"))) return rc;
    }
    if ((rc = cuda_check(c, cudaMemcpyAsync(c->d_mass, c->params.data() + 2, sizeof(double) * N, cudaMemcpyHostToDevice, st),
                         "H2D mass")))
        return rc;
    char *base = ws + kHeader + hist_bytes(c) + stats_bytes(c) + sched_bytes(c);
    irk::NbdCtl *ctl = reinterpret_cast<irk::NbdCtl *>(base);
    double *Qg = reinterpret_cast<double *>(base + 256);
    double *shard_mem = Qg + (size_t)P * stride;
    const size_t per_shard = 8 * dl + 3 * dl + (size_t)nbd_nj(N) * 8 * dl;
    double *Qall = shard_mem + (size_t)nlocal * per_shard;   // [3N] positions for energy samples
    double *terms = Qall + 3 * N;                            // [P][2*nloc]
    int64_t *n_done = reinterpret_cast<int64_t *>(ws);
    int64_t *stats = reinterpret_cast<int64_t *>(ws + kHeader + hist_bytes(c));
    const int64_t ldim = nccl ? 6 * nloc : 6 * N;  // rows of this process's y / history
    std::vector<irk::NbdArgs> A(nlocal);
    for (int t = 0; t < nlocal; ++t) {
        irk::NbdArgs &a = A[t];
        const int sh = first + t;
        for (int j = 0; j < 8; ++j) a.hb[j] = c->T.hb[j];
        const int64_t qoff = nccl ? 0 : 3 * (int64_t)sh * nloc, voff = nccl ? 3 * nloc : 3 * N + 3 * (int64_t)sh * nloc;
        a.yq = y + qoff;
        a.yv = y + voff;
        a.hist = reinterpret_cast<double *>(ws + kHeader);
        a.hdim = ldim;
        a.hq = qoff;
        a.hv = voff;
        a.Qg = Qg;
        a.stride = stride;
        double *m = shard_mem + (size_t)t * per_shard;
        a.V = m;
        a.M = m + 8 * dl;
        a.Pst = a.M + dl;
        a.sLq = a.Pst + dl;
        a.part = a.sLq + dl;
        a.mass = c->d_mass;
        a.ctl = ctl;
        a.nbody = N;
        a.nloc = nloc;
        a.b0 = (int64_t)sh * nloc;
        a.shard = sh;
        a.nshards = P;
        a.G = c->params[0];
        a.eps2 = c->params[1] * c->params[1];
        a.max_iters = c->max_iters;
        a.xmode = 0;
        a.rank = c->rank;
        a.peerQ = nullptr;
        a.peerHdr = nullptr;
        a.xhdr = nullptr;
        a.qbuf = (int64_t)P * stride;
    }
    if (fused) {
        // the symmetric window is created on the first fused call (collective: every
        // rank integrates); one scratch double of `terms` serves the set-up barrier
        if (!c->xwin && (rc = xsetup(c, sizeof(double) * 2 * (size_t)P * stride, terms, st))) return rc;
        A[0].xmode = 1;
        A[0].Qg = reinterpret_cast<double *>(static_cast<char *>(c->xbuf) + c->xqoff);
        A[0].peerQ = reinterpret_cast<double *const *>(c->d_xpeers);
        A[0].peerHdr = reinterpret_cast<int64_t *const *>(c->d_xpeers + P);
        A[0].xhdr = static_cast<int64_t *>(c->xbuf);
    }
    const unsigned cb = (unsigned)((dl + 127) / 128);
    const int64_t E = c->energy_every;
    auto sample = [&](int64_t idx) -> int {
        NvtxRange range("irk:energy_sample");
        for (int t = 0; t < nlocal; ++t) {
            const int r = cuda_check(c, cudaMemcpyAsync(Qall + 3 * A[t].b0, A[t].yq, sizeof(double) * dl,
                                                        cudaMemcpyDeviceToDevice, st), "energy sample: positions");
            if (r) return r;
        }
        if (nccl) {
            int r = nccl_allgather_inplace(c, Qall, (size_t)dl, st);
            if (r) return r;
        }
        for (int t = 0; t < nlocal; ++t)
            irk::nbd_energy_terms_kernel<<<(unsigned)((nloc + irk::NBD_EROW_ROWS - 1) / irk::NBD_EROW_ROWS), irk::NBD_EROW_THREADS, 0, st>>>(
                Qall, A[t].yv, c->d_mass, N, A[t].b0, nloc, A[t].G, A[t].eps2, terms + 2 * A[t].b0);
        if (nccl) {
            int r = nccl_allgather_inplace(c, terms, (size_t)(2 * nloc), st);
            if (r) return r;
        }
        irk::nbd_energy_sum_kernel<<<1, irk::NBD_ESUM_THREADS, 0, st>>>(terms, P, nloc, energy + idx);
        return cuda_check(c, cudaGetLastError(), "energy sample");
    };
    if (E > 0 && energy && (rc = sample(0))) return rc;
    if ((rc = cuda_check(c, cudaMemsetAsync(ctl, 0, sizeof(irk::NbdCtl), st), "memset ctl"))) return rc;
    int64_t bad0 = 0;  // frozen (diverged in an earlier call)?
    if ((rc = cuda_check(c, cudaMemcpyAsync(&bad0, stats + 1, sizeof(int64_t), cudaMemcpyDeviceToHost, st), "D2H bad")))
        return rc;
    if ((rc = cuda_check(c, cudaStreamSynchronize(st), "sync"))) return rc;
    if (bad0 > 0 || c->nsteps == 0) {
        if (iters && (rc = cuda_check(c, cudaMemsetAsync(iters, 0, sizeof(int64_t), st), "memset iters"))) return rc;
        return cuda_check(c, cudaGetLastError(), "direct: frozen");
    }
    for (int t = 0; t < nlocal; ++t) irk::nbd_init_kernel<<<cb, 128, 0, st>>>(A[t]);
    const int nj = (int)nbd_nj(N);
    auto force = [&](cudaStream_t s, const irk::NbdArgs &aa, int j_lo, int j_hi) {
        if (j_hi <= j_lo) return;
        const dim3 g((unsigned)((nloc + irk::NBD_FORCE_THREADS - 1) / irk::NBD_FORCE_THREADS), 8, (unsigned)(j_hi - j_lo));
        if (IRK_UNIT_G && aa.G == 1.0)  // the reciprocal form of the same correctly rounded division
            irk::nbd_force_kernel<true><<<g, irk::NBD_FORCE_THREADS, 0, s>>>(aa, j_lo);
        else
            irk::nbd_force_kernel<false><<<g, irk::NBD_FORCE_THREADS, 0, s>>>(aa, j_lo);
    };
    // Fused exchange: the j-blocks made only of this rank's bodies need no peer
    // data, so they run before the arrival wait (overlapping the exchange, SURVEY
    // 8(e)); the others after it.  Partial sums are per j-block, so the bits do
    // not depend on the launch order.
    int jl0 = 0, jl1 = 0;
    if (fused) {
        const int64_t b0 = A[0].b0, b1 = A[0].b0 + nloc;
        jl0 = (int)((b0 + irk::NBD_JBLOCK - 1) / irk::NBD_JBLOCK);
        jl1 = jl0;
        while (jl1 < nj && (int64_t)jl1 * irk::NBD_JBLOCK >= b0 &&
               std::min<int64_t>((int64_t)(jl1 + 1) * irk::NBD_JBLOCK, N) <= b1)
            ++jl1;
    }
    // one fixed-point sweep of every local shard (a2+a5, exchange, a3, a4+a6, counters)
    auto enqueue_sweep = [&](cudaStream_t s, cudaGraphConditionalHandle cond, int use_cond) -> int {
        for (int t = 0; t < nlocal; ++t) irk::nbd_pos_kernel<<<cb, 128, 0, s>>>(A[t]);
        if (nccl && !fused) {
            int r = nccl_allgather_inplace(c, Qg, (size_t)stride, s);  // the exchange
            if (r) return r;
        }
        if (fused) force(s, A[0], jl0, jl1);  // local x local, before the wait
        irk::nbd_or_kernel<<<1, 1, 0, s>>>(A[0]);
        if (fused) {
            force(s, A[0], 0, jl0);
            force(s, A[0], jl1, nj);
        } else {
            for (int t = 0; t < nlocal; ++t) force(s, A[t], 0, nj);
        }
        for (int t = 0; t < nlocal; ++t) irk::nbd_vel_kernel<<<cb, 128, 0, s>>>(A[t]);
        irk::nbd_ctl_kernel<<<1, 1, 0, s>>>(A[0], first, nlocal, n_done, stats, cond, use_cond);
        return cuda_check(c, cudaGetLastError(), "direct sweep launch");
    };
    // Device-driven loop (IRK_OPT_DEVICE_LOOP, default on): the sweep captured once
    // into the body of a CUDA-graph conditional WHILE node; nbd_ctl sets the
    // condition, so the GPU runs sweep after sweep until n reaches the segment
    // target (the next energy sample or nsteps) or the system diverges, and the
    // host syncs once per segment instead of once per sweep.  Falls back to the
    // host loop if the graph cannot be built (e.g. NCCL refusing capture).
    cudaGraphExec_t gexec = nullptr;
    if (c->device_loop) {
        cudaGraph_t g = nullptr, body = nullptr;
        cudaStream_t cs = nullptr;
        cudaGraphConditionalHandle cond = 0;
        bool okg = cudaGraphCreate(&g, 0) == cudaSuccess &&
                   cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
        if (okg) {
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = cond;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            cudaGraphNode_t node;
            okg = cudaGraphAddNode(&node, g, nullptr, 0, &cp) == cudaSuccess;
            if (okg) body = cp.conditional.phGraph_out[0];
        }
        okg = okg && cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking) == cudaSuccess &&
              cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal) ==
                  cudaSuccess;
        if (okg) {
            const int r = enqueue_sweep(cs, cond, 1);
            cudaGraph_t captured = nullptr;
            okg = (cudaStreamEndCapture(cs, &captured) == cudaSuccess) && r == IRK_OK &&
                  cudaGraphInstantiate(&gexec, g, 0) == cudaSuccess;
        }
        if (!okg && gexec) {
            cudaGraphExecDestroy(gexec);
            gexec = nullptr;
        }
        if (cs) cudaStreamDestroy(cs);
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();  // a failed attempt leaves no sticky error: use the host loop
        c->err.clear();
    }
    int64_t n = 0;
    c->device_loop_used = gexec ? 1 : 0;
    if (gexec) {
        while (n < c->nsteps) {
            NvtxRange range("irk:device_loop_segment");
            const int64_t target = (E > 0 && energy) ? ((n / E + 1) * E < c->nsteps ? (n / E + 1) * E : c->nsteps)
                                                     : c->nsteps;
            c->h_ctl->target = target;
            if ((rc = cuda_check(c, cudaMemcpyAsync(&ctl->target, &c->h_ctl->target, sizeof(int64_t),
                                                    cudaMemcpyHostToDevice, st), "H2D loop target")) ||
                (rc = cuda_check(c, cudaGraphLaunch(gexec, st), "device loop graph launch")) ||
                (rc = cuda_check(c, cudaMemcpyAsync(c->h_ctl, ctl, offsetof(irk::NbdCtl, target), cudaMemcpyDeviceToHost, st),
                                 "D2H loop control")) ||
                (rc = cuda_check(c, cudaStreamSynchronize(st), "direct device loop"))) {
                cudaGraphExecDestroy(gexec);
                return rc;
            }
            if (c->h_ctl->halt) break;
            n = c->h_ctl->n;
            if (E > 0 && energy && n % E == 0 && (rc = sample(n / E))) {
                cudaGraphExecDestroy(gexec);
                return rc;
            }
        }
        cudaGraphExecDestroy(gexec);
    } else {
        while (n < c->nsteps) {
            NvtxRange range("irk:host_loop_sweep");
            if ((rc = enqueue_sweep(st, 0, 0))) return rc;
            if ((rc = cuda_check(c, cudaMemcpyAsync(c->h_ctl, ctl, sizeof(irk::NbdCtl), cudaMemcpyDeviceToHost, st),
                                 "D2H sweep control")))
                return rc;
            if ((rc = cuda_check(c, cudaStreamSynchronize(st), "direct sweep"))) return rc;
            if (c->h_ctl->halt) break;
            if (c->h_ctl->fin) {
                n = c->h_ctl->n;
                if (E > 0 && energy && n % E == 0 && (rc = sample(n / E))) return rc;
            }
        }
    }
    if (fused && c->h_ctl->xerr) return fail(c, IRK_E_COMM, "fused exchange: a peer did not arrive within 60 s");
    // final exchange: a divergence at the call's last step is recorded on every rank
    if (fused) {
        irk::nbd_xfinal_kernel<<<1, 1, 0, st>>>(A[0], n_done, stats);
        if ((rc = cuda_check(c, cudaMemcpyAsync(c->h_ctl, ctl, sizeof(irk::NbdCtl), cudaMemcpyDeviceToHost, st),
                             "D2H final control")))
            return rc;
        if ((rc = cuda_check(c, cudaStreamSynchronize(st), "fused exchange final barrier"))) return rc;
        if (c->h_ctl->xerr)
            return fail(c, IRK_E_COMM, "fused exchange: a peer did not arrive within %d s", 60);
    } else {
        if (nccl && (rc = nccl_allgather_inplace(c, Qg, (size_t)stride, st))) return rc;
        irk::nbd_final_kernel<<<1, 1, 0, st>>>(A[0], n_done, stats);
    }
    if (iters && (rc = cuda_check(c, cudaMemcpyAsync(iters, &ctl->sweeps, sizeof(int64_t), cudaMemcpyDeviceToDevice, st),
                                  "sweeps -> iters")))
        return rc;
    return cuda_check(c, cudaGetLastError(), "direct launch");
}

EnsArgs ens_args(irk_ctx *c, double *y, double t0, char *ws, double *energy, int64_t *iters) {
    EnsArgs a;
    for (int j = 0; j < 8; ++j) a.hb[j] = c->T.hb[j];
    a.y = y;
    a.n_done = reinterpret_cast<const int64_t *>(ws);
    a.hist = reinterpret_cast<double *>(ws + kHeader);
    a.stats = reinterpret_cast<int64_t *>(ws + kHeader + hist_bytes(c));
    a.energy = energy;
    a.iters = iters;
    a.batch = c->batch;
    a.energy_every = c->energy_every;
    a.h = c->h;
    a.t0 = t0;
    a.max_iters = c->max_iters;
    a.local_energy = c->local_energy;
    return a;
}

// Persistent work-queue launches (IRK_OPT_SCHEDULE auto / 2): grid = resident
// capacity of `kernel`, `spb` trajectory slots per block; units of `qchunk` steps
// (one unit per trajectory when every trajectory has its own slot, else ~32).
template <class KernelPtr, class LaunchFn>
int launch_queue(irk_ctx *c, KernelPtr kernel, int threads, int spb, int *bps_cache, EnsArgs &a, char *ws,
                 cudaStream_t st, LaunchFn launch, int units = 32, int max_bps = 0, int64_t unit_steps = 0) {
    int rc;
    if (!*bps_cache &&
        (rc = cuda_check(c, cudaOccupancyMaxActiveBlocksPerMultiprocessor(bps_cache, kernel, threads, 0), "occupancy")))
        return rc;
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int bps = *bps_cache > 0 ? *bps_cache : 1;
    if (max_bps > 0 && bps > max_bps) bps = max_bps;
    const int64_t resident_blocks = (int64_t)sms * bps;
    const int64_t need = (c->batch + spb - 1) / spb;
    const int64_t blocks = need < resident_blocks ? need : resident_blocks;
    irk::QueueArgs qa;
    Sched sc = sched_of(c, ws);
    qa.progress = sc.perm;
    qa.orphan = sc.csweeps;
    qa.counter = reinterpret_cast<unsigned long long *>(sc.bins);
    int64_t chunk = c->nsteps;
    if (c->balance > 0) chunk = c->balance;
    else if (c->balance < 0 && unit_steps > 0) chunk = unit_steps;
    else if (c->balance < 0 && c->batch > resident_blocks * spb) chunk = (c->nsteps + units - 1) / units;
    if (chunk < 1) chunk = 1;
    qa.qchunk = chunk;
    qa.nchunks = c->nsteps > 0 ? (c->nsteps + chunk - 1) / chunk : 1;
    // progress[] / orphan[] hold chunk indices + 1 as int32
    if (qa.nchunks >= INT32_MAX)
        return fail(c, IRK_E_ARG, "irk_integrate: %lld step chunks per call exceed the work queue's int32 counters "
                                  "(raise IRK_OPT_BALANCE or split the call)", (long long)qa.nchunks);
    a.nsteps = c->nsteps;
    a.c0 = 0;
    a.csweeps = nullptr;
    a.perm = nullptr;
    a.nslots = c->batch;
    if ((rc = cuda_check(c, cudaMemsetAsync(sc.perm, 0, sizeof(int32_t) * c->batch, st), "memset progress"))) return rc;
    if ((rc = cuda_check(c, cudaMemsetAsync(sc.csweeps, 0, sizeof(int32_t) * c->batch, st), "memset orphan"))) return rc;
    if ((rc = cuda_check(c, cudaMemsetAsync(sc.bins, 0, sizeof(unsigned long long), st), "memset counter"))) return rc;
    launch(a, qa, (unsigned)blocks);
    if ((rc = cuda_check(c, cudaGetLastError(), "work-queue kernel launch"))) return rc;
    advance_n_kernel<<<1, 1, 0, st>>>(reinterpret_cast<int64_t *>(ws), c->nsteps);
    return cuda_check(c, cudaGetLastError(), "advance_n launch");
}

// ens_g1q launch geometry.  The makespan of the queue is max(total work / lanes,
// the slowest trajectory's serial chain): a trajectory's units run one after the
// other, each at the per-lane speed of its SM, so with lanes ~ batch the slowest
// trajectory (config 2: 1.29x the mean sweeps) outlasts the average lane and its
// successors' units are fetched early and wait (unit trace of the round-1 launch:
// 7.3 % of lane time waiting, 7.4 % idle; tools/unit_trace.py).  Fewer resident
// lanes shorten the chains (each lane gets a larger share of its SM's FP64 pipe)
// at some cost in throughput, so below 1.5 x the light kernel's resident lanes the
// kernel runs 2-4 blocks of 64 per SM (from the batch) at up to 240 registers
// (config 2: 92.2 -> 81.4 ms, with 16 units per trajectory instead of 32); above
// it, 6 blocks at 168 registers (B = 262,144 x 2,500 steps: 76.8 ms vs 85.1 ms at
// 4 blocks).  Bitwise-neutral: every unit does the same arithmetic.
template <class P>
int launch_g1q(irk_ctx *c, const P &prob, EnsArgs &a, char *ws, cudaStream_t st) {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int &bps_light = c->g1q_blocks_per_sm;
    if (!bps_light)
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_light, irk::ens_g1q_kernel<P>, irk::G1_THREADS, 0);
    const int64_t light_lanes = (int64_t)sms * (bps_light > 0 ? bps_light : 1) * irk::G1_THREADS;
    if (G1Q_MAX_BPS == 0 && 2 * c->batch >= 3 * light_lanes)
        return launch_queue(c, irk::ens_g1q_kernel<P>, irk::G1_THREADS, irk::G1_THREADS, &c->g1q_blocks_per_sm, a, ws,
                            st, [&](const EnsArgs &aa, const irk::QueueArgs &qa, unsigned nb) {
                                irk::ens_g1q_kernel<P><<<nb, irk::G1_THREADS, 0, st>>>(aa, qa, prob);
                            }, G1Q_UNITS);
    // blocks per SM from the batch (measured, config-2 generator, 10,000 steps, ms at
    // 2 / 3 / 4 blocks: 24,576: 43.2/60.7/60.0; 32,768: 56.5/59.9/60.5; 40,960:
    // 70.2/63.6/64.7; 49,152: 84.0/71.3/66.1; 57,344: 97.7/82.1/71.2; 65,536: -/-/80.1)
    int64_t cap = c->batch / ((int64_t)sms * 83);
    cap = cap < 2 ? 2 : (cap > 4 ? 4 : cap);
    if (G1Q_MAX_BPS > 0) cap = G1Q_MAX_BPS;
    auto heavy = irk::ens_g1q_kernel<P, G1Q_HEAVY_MAXREG>;
    return launch_queue(c, heavy, irk::G1_THREADS, irk::G1_THREADS, &c->g1q_heavy_blocks_per_sm, a, ws, st,
                        [&](const EnsArgs &aa, const irk::QueueArgs &qa, unsigned nb) {
                            heavy<<<nb, irk::G1_THREADS, 0, st>>>(aa, qa, prob);
                        }, G1Q_UNITS, (int)cap);
}

// Stage-per-lane mappings (ensemble_g8.cuh): one launch, one group of G lanes per
// trajectory (G = 8: one stage per lane; G = 4: two).
template <class P, int G>
int launch_gs(irk_ctx *c, const P &prob, EnsArgs &a, char *ws, cudaStream_t st) {
    a.nsteps = c->nsteps;
    a.c0 = 0;
    a.csweeps = nullptr;
    a.perm = nullptr;
    a.nslots = c->batch;
    const int64_t blocks = (c->batch * G + irk::G8_THREADS - 1) / irk::G8_THREADS;
    irk::ens_gs_kernel<P, G><<<(unsigned)blocks, irk::G8_THREADS, 0, st>>>(a, prob);
    int rc = cuda_check(c, cudaGetLastError(), "ens_gs launch");
    if (rc) return rc;
    advance_n_kernel<<<1, 1, 0, st>>>(reinterpret_cast<int64_t *>(ws), c->nsteps);
    return cuda_check(c, cudaGetLastError(), "advance_n launch");
}

// Stage per lane with DMMA contractions (ensemble_g8m.cuh): one launch, one slot of
// 4 trajectories per warp.
template <class P>
int launch_gsm(irk_ctx *c, const P &prob, EnsArgs &a, char *ws, cudaStream_t st) {
    a.nsteps = c->nsteps;
    a.c0 = 0;
    a.csweeps = nullptr;
    a.perm = nullptr;
    a.nslots = c->batch;
    const int64_t blocks = (c->batch * 8 + irk::G8M_THREADS - 1) / irk::G8M_THREADS;
    if (c->batch <= 4)  // one slot: the latency-bound single-trajectory case (config 1)
        irk::ens_gsm_kernel<P, true, false><<<(unsigned)blocks, irk::G8M_THREADS, 0, st>>>(a, prob);
    else
        irk::ens_gsm_kernel<P, false, true><<<(unsigned)blocks, irk::G8M_THREADS, 0, st>>>(a, prob);
    int rc = cuda_check(c, cudaGetLastError(), "ens_gsm launch");
    if (rc) return rc;
    advance_n_kernel<<<1, 1, 0, st>>>(reinterpret_cast<int64_t *>(ws), c->nsteps);
    return cuda_check(c, cudaGetLastError(), "advance_n launch");
}

// IRK_OPT_MAPPING auto for the N-body ensembles, from tools/nb_map_ab.py (1,000
// steps at batches 2,048 / 6,144 / 16,384 / 65,536, all three mappings;
// profiles/r2/nb_map_ab_r2.json): stage per lane with DMMA contractions
// (ens_nbody8m) for N = 3..6 at every batch and N = 2 up to 32,768 (config 3:
// 30.6 vs 39.1 ms shared-memory stage per lane, 46.0 ms body per lane); N = 7, 8
// keep the round-1 choice (ens_nbody8m's tiles do not fit unpadded in registers
// and shared memory there: slower): stage per lane for N = 7, and for N = 8
// except near 6,144; body per lane for N = 2 beyond 32,768.
int nbody_auto_mapping(int NB, int64_t batch) {
    switch (NB) {
    case 2: return batch <= 32768 ? IRK_MAP_G8M : IRK_MAP_G1;
    case 7: return IRK_MAP_G8;
    case 8: return (batch <= 4096 || batch >= 12288) ? IRK_MAP_G8 : IRK_MAP_G1;
    default: return IRK_MAP_G8M;
    }
}

// IRK_OPT_MAPPING auto for the per-thread problems (partitioned mode): lanes per
// trajectory G = 8 while the batch leaves most g1 lanes of the GPU empty, then
// G = 4, then one trajectory per lane ("ens_gs": measured crossovers).
int lanes_per_trajectory(const irk_ctx *c) {
    if (c->mapping == IRK_MAP_G8M) return IRK_MAP_G8M;
    if (c->mapping == IRK_MAP_G8) return 8;
    if (c->mapping == IRK_MAP_G4) return 4;
    if (c->mapping == IRK_MAP_G2) return 2;
    if (c->mapping == IRK_MAP_G1) return 1;
    if (c->batch <= kG8AutoMaxBatch) return IRK_MAP_G8M;
    if (c->batch <= kG4AutoMaxBatch) return 4;
    if (c->batch > kG4AutoMaxBatch * 5 / 4 && c->batch <= kG2AutoMaxBatch) return 2;  // g1 ~ g4 in between
    return 1;
}

// First-order mode (IRK_OPT_MODE = 1; the only mode of non-separable problems):
// the sweep-granular work-queue kernel, or the chunked per-step kernel (SCHEDULE = 1).
template <class P>
int launch_first_order(irk_ctx *c, const P &prob, double *y, double t0, char *ws, double *energy, int64_t *iters,
                       cudaStream_t st) {
    EnsArgs a = ens_args(c, y, t0, ws, energy, iters);
    const bool fo8 = c->mapping == IRK_MAP_G8 || (c->mapping == IRK_MAP_AUTO && c->batch <= kFo8AutoMaxBatch);
    c->mapping_used = fo8 ? IRK_MAP_G8 : IRK_MAP_G1;
    if (fo8) {
        a.nsteps = c->nsteps;  // stage per lane: one launch, one group of 8 lanes per trajectory
        a.c0 = 0;
        a.csweeps = nullptr;
        a.perm = nullptr;
        a.nslots = c->batch;
        const int64_t blocks = (c->batch * 8 + irk::FO8_THREADS - 1) / irk::FO8_THREADS;
        irk::ens_fo8_kernel<P><<<(unsigned)blocks, irk::FO8_THREADS, 0, st>>>(a, prob);
        int rc = cuda_check(c, cudaGetLastError(), "ens_fo8 launch");
        if (rc) return rc;
        advance_n_kernel<<<1, 1, 0, st>>>(reinterpret_cast<int64_t *>(ws), c->nsteps);
        return cuda_check(c, cudaGetLastError(), "advance_n launch");
    }
    if (c->schedule != 1)
        return launch_queue(c, irk::ens_fo_q_kernel<P>, irk::FO_THREADS, irk::FO_THREADS, &c->fo_blocks_per_sm, a, ws, st,
                            [&](const EnsArgs &aa, const irk::QueueArgs &qa, unsigned nb) {
                                irk::ens_fo_q_kernel<P><<<nb, irk::FO_THREADS, 0, st>>>(aa, qa, prob);
                            });
    const int64_t blocks = (c->batch + irk::G1_THREADS - 1) / irk::G1_THREADS;
    return run_chunks(c, a, ws, blocks, irk::G1_THREADS / 32, 32, st, [&](const EnsArgs &aa, int64_t nb) {
        irk::ens_g1fo_kernel<P><<<(unsigned)nb, irk::G1_THREADS, 0, st>>>(aa, prob);
    });
}

template <class P>
int launch_g1(irk_ctx *c, const P &prob, double *y, double t0, char *ws, double *energy,
              int64_t *iters, cudaStream_t st) {
    EnsArgs a = ens_args(c, y, t0, ws, energy, iters);
    const int64_t blocks = (c->batch + irk::G1_THREADS - 1) / irk::G1_THREADS;
    c->mapping_used = c->mode == 0 ? lanes_per_trajectory(c) : IRK_MAP_G1;  // (first-order: set below)
    if (c->mode == 0 && lanes_per_trajectory(c) == IRK_MAP_G8M) return launch_gsm(c, prob, a, ws, st);
    if (c->mode == 0 && lanes_per_trajectory(c) == 8) return launch_gs<P, 8>(c, prob, a, ws, st);
    if (c->mode == 0 && lanes_per_trajectory(c) == 4) return launch_gs<P, 4>(c, prob, a, ws, st);
    if (c->mode == 0 && lanes_per_trajectory(c) == 2) return launch_gs<P, 2>(c, prob, a, ws, st);
    if (c->mode == 0 && c->schedule != 1) return launch_g1q(c, prob, a, ws, st);
    if (c->mode == 1) return launch_first_order(c, prob, y, t0, ws, energy, iters, st);
    return run_chunks(c, a, ws, blocks, irk::G1_THREADS / 32, 32, st, [&](const EnsArgs &aa, int64_t nb) {
        irk::ens_g1_kernel<P><<<(unsigned)nb, irk::G1_THREADS, 0, st>>>(aa, prob);
    });
}

template <int NB>
int launch_nbody_t(irk_ctx *c, double *y, double t0, char *ws, double *energy, int64_t *iters, cudaStream_t st) {
    irk::NBodyParams P;
    P.G = c->params[0];
    P.eps2 = c->params[1] * c->params[1];
    for (int i = 0; i < 16; ++i) P.m[i] = i < NB ? c->params[2 + i] : 0.0;
    EnsArgs a = ens_args(c, y, t0, ws, energy, iters);
    constexpr int GPW = 32 / NB, WPB = irk::NB_THREADS / 32;
    const int64_t blocks = (c->batch + GPW * WPB - 1) / (GPW * WPB);
    // stage-per-lane (ensemble_nbody8.cuh) when asked or where auto measured it faster; the
    // chunked schedule (IRK_OPT_SCHEDULE = 1) keeps body-per-lane
    const int autom = (c->mapping == IRK_MAP_AUTO && c->schedule != 1) ? nbody_auto_mapping(NB, c->batch) : 0;
    const bool stage_per_lane = c->mapping == IRK_MAP_G8 || autom == IRK_MAP_G8;
    const bool dmma = c->mapping == IRK_MAP_G8M || autom == IRK_MAP_G8M;
    c->mapping_used = dmma ? IRK_MAP_G8M : stage_per_lane ? IRK_MAP_G8 : IRK_MAP_G1;
    if (dmma) {
        // units of 50 steps at every batch: a slot's 4 trajectories restart in step at
        // each unit (they share the contraction's coefficient fragment; drifted apart,
        // the velocity contraction runs twice): config 3 1.70 s with 32 units per
        // trajectory (1,563 steps), 1.58 / 1.53 / 1.52 / 1.53 s at 250 / 100 / 50 / 25
        constexpr int64_t kUnitSteps = 50;
        constexpr int SPB = irk::N8M_THREADS / 32 * 4;  // trajectories per block
        // small batches: the 255-register instantiation (few warps per SM; config-3
        // generator, 5,000 steps, ms at 168 / 255 registers: 2,048 42.4 / 37.7,
        // 4,096 50.9 / 46.5, 8,192 73.0 / 79.9)
        const bool hi = c->batch <= kN8mHiRegMaxBatch;
        int *bps = hi ? &c->nbody8m_hi_blocks_per_sm[NB] : &c->nbody8m_blocks_per_sm[NB];
        auto run = [&](auto kern) {
            return launch_queue(c, kern, irk::N8M_THREADS, SPB, bps, a, ws, st,
                                [&](const EnsArgs &aa, const irk::QueueArgs &qa, unsigned nb) {
                                    kern<<<nb, irk::N8M_THREADS, 0, st>>>(aa, qa, P);
                                }, 32, 0, kUnitSteps);
        };
        if (IRK_UNIT_G && P.G == 1.0)
            return hi ? run(irk::ens_nbody8m_kernel<NB, true, 255>) : run(irk::ens_nbody8m_kernel<NB, true>);
        return hi ? run(irk::ens_nbody8m_kernel<NB, false, 255>) : run(irk::ens_nbody8m_kernel<NB, false>);
    }
    if (stage_per_lane)
        return (IRK_UNIT_G && P.G == 1.0)
                   ? launch_queue(c, irk::ens_nbody8_kernel<NB, true>, irk::N8_THREADS, irk::N8_THREADS / 8,
                                  &c->nbody8_blocks_per_sm[NB], a, ws, st,
                                  [&](const EnsArgs &aa, const irk::QueueArgs &qa, unsigned nb) {
                                      irk::ens_nbody8_kernel<NB, true><<<nb, irk::N8_THREADS, 0, st>>>(aa, qa, P);
                                  })
                   : launch_queue(c, irk::ens_nbody8_kernel<NB, false>, irk::N8_THREADS, irk::N8_THREADS / 8,
                                  &c->nbody8_blocks_per_sm[NB], a, ws, st,
                                  [&](const EnsArgs &aa, const irk::QueueArgs &qa, unsigned nb) {
                                      irk::ens_nbody8_kernel<NB, false><<<nb, irk::N8_THREADS, 0, st>>>(aa, qa, P);
                                  });
    if (c->schedule != 1)
        return launch_queue(c, irk::ens_nbody_q_kernel<NB>, irk::NB_THREADS, GPW * WPB, &c->nbody_blocks_per_sm[NB], a,
                            ws, st, [&](const EnsArgs &aa, const irk::QueueArgs &qa, unsigned nb) {
                                irk::ens_nbody_q_kernel<NB><<<nb, irk::NB_THREADS, 0, st>>>(aa, qa, P);
                            }, 128);  // config 3: 32 units 2.16 s, 64: 2.15, 128: 2.14 (with hand-off)
    return run_chunks(c, a, ws, blocks, WPB, GPW, st, [&](const EnsArgs &aa, int64_t nb) {
        irk::ens_nbody_kernel<NB><<<(unsigned)nb, irk::NB_THREADS, 0, st>>>(aa, P);
    });
}

template <int SPL>
int launch_chain_t(irk_ctx *c, double *y, double t0, char *ws, double *energy, int64_t *iters, cudaStream_t st) {
    EnsArgs a = ens_args(c, y, t0, ws, energy, iters);
    // small batches (strong-scaling shares): two warps per chain, one launch
    if (SPL % 2 == 0 && c->schedule == 0 && c->batch <= IRK_CHAINW_MAX) {
        constexpr int SPLW = SPL / 2 > 0 ? SPL / 2 : 1;
        a.nsteps = c->nsteps;
        a.c0 = 0;
        a.csweeps = nullptr;
        a.perm = nullptr;
        a.nslots = c->batch;
        irk::ens_chainw_kernel<SPLW, 2><<<(unsigned)c->batch, 64, 0, st>>>(a, c->params[0]);
        int rc = cuda_check(c, cudaGetLastError(), "ens_chainw launch");
        if (rc) return rc;
        advance_n_kernel<<<1, 1, 0, st>>>(reinterpret_cast<int64_t *>(ws), c->nsteps);
        return cuda_check(c, cudaGetLastError(), "advance_n launch");
    }
    constexpr int CPB = irk::CH_THREADS / 32;
    const int64_t blocks = (c->batch + CPB - 1) / CPB;
    const double beta = c->params[0];
    // Auto: the work queue, except for batches between one and two resident waves
    // of warps, where its step-chunk units leave the SMs unevenly loaded (one warp
    // per chain, chains handed between warps): config 4, 20,000 steps, at 1,536 /
    // 2,048 chains 212 / 221 ms queued vs 146 / 191 ms chunked, at 3,072 245 vs 281.
    bool queue = c->schedule != 1;
    if (c->schedule == 0 && c->balance < 0) {
        int &bps = c->chain_blocks_per_sm[SPL];
        if (!bps) cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, irk::ens_chain_q_kernel<SPL>, irk::CH_THREADS, 0);
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const int64_t resident = (int64_t)sms * (bps > 0 ? bps : 1) * CPB;
        if (c->batch > resident && c->batch <= 2 * resident) queue = false;
    }
    if (queue)
        return launch_queue(c, irk::ens_chain_q_kernel<SPL>, irk::CH_THREADS, CPB, &c->chain_blocks_per_sm[SPL], a, ws,
                            st, [&](const EnsArgs &aa, const irk::QueueArgs &qa, unsigned nb) {
                                irk::ens_chain_q_kernel<SPL><<<nb, irk::CH_THREADS, 0, st>>>(aa, qa, beta);
                            });
    return run_chunks(c, a, ws, blocks, CPB, 1, st, [&](const EnsArgs &aa, int64_t nb) {
        irk::ens_chain_kernel<SPL><<<(unsigned)nb, irk::CH_THREADS, 0, st>>>(aa, beta);
    });
}

int launch_chain(irk_ctx *c, double *y, double t0, char *ws, double *energy, int64_t *iters, cudaStream_t st) {
    switch (c->dim / 2) {
    case 32: return launch_chain_t<1>(c, y, t0, ws, energy, iters, st);
    case 64: return launch_chain_t<2>(c, y, t0, ws, energy, iters, st);
    case 96: return launch_chain_t<3>(c, y, t0, ws, energy, iters, st);
    case 128: return launch_chain_t<4>(c, y, t0, ws, energy, iters, st);
    }
    return fail(c, IRK_E_ARG, "irk_integrate: IRK_FPU_BETA supports N in {32, 64, 96, 128} sites");
}

int launch_nbody(irk_ctx *c, double *y, double t0, char *ws, double *energy, int64_t *iters, cudaStream_t st) {
    switch (c->dim / 6) {
    case 2: return launch_nbody_t<2>(c, y, t0, ws, energy, iters, st);
    case 3: return launch_nbody_t<3>(c, y, t0, ws, energy, iters, st);
    case 4: return launch_nbody_t<4>(c, y, t0, ws, energy, iters, st);
    case 5: return launch_nbody_t<5>(c, y, t0, ws, energy, iters, st);
    case 6: return launch_nbody_t<6>(c, y, t0, ws, energy, iters, st);
    case 7: return launch_nbody_t<7>(c, y, t0, ws, energy, iters, st);
    case 8: return launch_nbody_t<8>(c, y, t0, ws, energy, iters, st);
    }
    return fail(c, IRK_E_ARG, "irk_integrate: IRK_NBODY ensembles support N in {2,...,8} bodies");
}

template <int N>
__global__ void energy_fpu_kernel(const double *y, double *H, int64_t B, double beta) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= B) return;
    double q[N], v[N];
    for (int l = 0; l < N; ++l) {
        q[l] = y[l * B + b];
        v[l] = y[(N + l) * B + b];
    }
    H[b] = irk::fpu_energy<N>(q, v, beta);
}

template <int NB>
__global__ void energy_nbody_kernel(const double *y, double *H, int64_t B, const __grid_constant__ irk::NBodyParams P) {
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= B) return;
    double qv[6 * NB];
    for (int l = 0; l < 6 * NB; ++l) qv[l] = y[l * B + b];
    H[b] = irk::nbody_energy<NB>(qv, P);
}

template <int NB>
void launch_energy_nbody_t(irk_ctx *c, const double *y, double *H, cudaStream_t st) {
    irk::NBodyParams P;
    P.G = c->params[0];
    P.eps2 = c->params[1] * c->params[1];
    for (int i = 0; i < 16; ++i) P.m[i] = i < NB ? c->params[2 + i] : 0.0;
    energy_nbody_kernel<NB><<<(unsigned)((c->batch + 127) / 128), 128, 0, st>>>(y, H, c->batch, P);
}

template <class P>
__global__ void energy_g1_kernel(const double *y, double *H, int64_t B, const __grid_constant__ P prob) {
    constexpr int d = P::d;
    int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (b >= B) return;
    double q[d], v[d];
    for (int l = 0; l < d; ++l) {
        q[l] = y[l * B + b];
        v[l] = y[(d + l) * B + b];
    }
    H[b] = prob.energy(q, v);
}

}  // namespace

// ---- NCCL (loaded at run time: the library has no link-time NCCL dependency) ----
#include <dlfcn.h>
#include "nccl.h"
#include "nccl_device.h"  // ncclGetPeerPointer (device-inline window mapping) for the fused exchange

namespace {
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*getUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char *(*getErrorString)(ncclResult_t) = nullptr;
    // symmetric windows (fused exchange); absent in older NCCL: the option then fails
    ncclResult_t (*memAlloc)(void **, size_t) = nullptr;
    ncclResult_t (*memFree)(void *) = nullptr;
    ncclResult_t (*winRegister)(ncclComm_t, void *, size_t, ncclWindow_t *, int) = nullptr;
    ncclResult_t (*winDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
    ncclTeam_t (*teamLsa)(ncclComm_t) = nullptr;
};
std::mutex g_nccl_mu;
NcclApi g_nccl;

const char *load_nccl() {
    std::lock_guard<std::mutex> lk(g_nccl_mu);
    if (g_nccl.h) return nullptr;
    const char *env = getenv("IRK_NCCL_LIB");
    const char *cands[] = {env, "libnccl.so.2", "libnccl.so",
                           "/opt/prime-rl/.venv/lib/python3.12/site-packages/nvidia/nccl/lib/libnccl.so.2"};
    void *h = nullptr;
    for (const char *c : cands)
        if (c && (h = dlopen(c, RTLD_NOW | RTLD_GLOBAL))) break;
    if (!h) return "NCCL library not found (set IRK_NCCL_LIB)";
    g_nccl.getUniqueId = (decltype(g_nccl.getUniqueId))dlsym(h, "ncclGetUniqueId");
    g_nccl.commInitRank = (decltype(g_nccl.commInitRank))dlsym(h, "ncclCommInitRank");
    g_nccl.allGather = (decltype(g_nccl.allGather))dlsym(h, "ncclAllGather");
    g_nccl.commDestroy = (decltype(g_nccl.commDestroy))dlsym(h, "ncclCommDestroy");
    g_nccl.getErrorString = (decltype(g_nccl.getErrorString))dlsym(h, "ncclGetErrorString");
    g_nccl.memAlloc = (decltype(g_nccl.memAlloc))dlsym(h, "ncclMemAlloc");
    g_nccl.memFree = (decltype(g_nccl.memFree))dlsym(h, "ncclMemFree");
    g_nccl.winRegister = (decltype(g_nccl.winRegister))dlsym(h, "ncclCommWindowRegister");
    g_nccl.winDeregister = (decltype(g_nccl.winDeregister))dlsym(h, "ncclCommWindowDeregister");
    g_nccl.teamLsa = (decltype(g_nccl.teamLsa))dlsym(h, "ncclTeamLsa");
    if (!g_nccl.getUniqueId || !g_nccl.commInitRank || !g_nccl.allGather || !g_nccl.commDestroy)
        return "NCCL library lacks required symbols";
    g_nccl.h = h;
    return nullptr;
}

int nccl_check(irk_ctx *c, int r, const char *what) {
    if (r == 0) return IRK_OK;
    return fail(c, IRK_E_COMM, "%s: %s", what, g_nccl.getErrorString ? g_nccl.getErrorString((ncclResult_t)r) : "error");
}

int nccl_allgather_inplace(irk_ctx *c, double *buf, size_t count_per_rank, cudaStream_t st) {
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(c->nccl_comm);
    return nccl_check(c, g_nccl.allGather(buf + (size_t)c->rank * count_per_rank, buf, count_per_rank, ncclFloat64,
                                          comm, st),
                      "ncclAllGather");
}

// rank r's view of the window through the NVLink (LSA) mapping: its Q buffers and header
__global__ void xpeers_kernel(ncclWindow_t w, int P, size_t qoff, void **out) {
    const int r = threadIdx.x;
    if (r >= P) return;
    out[r] = ncclGetPeerPointer(w, qoff, r);
    out[P + r] = ncclGetPeerPointer(w, 0, r);
}

// Fused exchange set-up (collective over the communicator; NEXT f3): one symmetric
// window [header | Q buffer 0 | Q buffer 1] per rank from ncclMemAlloc, registered
// with NCCL_WIN_COLL_SYMMETRIC so that every rank reaches every other rank's copy
// through NVLink load/store; zero-filled, then a 1-double all-gather as a barrier
// so that no rank pushes into a window before its owner has cleared it.
int xsetup(irk_ctx *c, size_t qbytes, double *scratch, cudaStream_t st) {
    ncclComm_t comm = reinterpret_cast<ncclComm_t>(c->nccl_comm);
    const int P = c->nranks;
    if (!g_nccl.memAlloc || !g_nccl.memFree || !g_nccl.winRegister || !g_nccl.winDeregister)
        return fail(c, IRK_E_COMM, "fused exchange: this NCCL has no symmetric windows (needs >= 2.27)");
    if (g_nccl.teamLsa) {
        const ncclTeam_t lsa = g_nccl.teamLsa(comm);
        if (lsa.nRanks != P)
            return fail(c, IRK_E_COMM, "fused exchange: %d of %d ranks share a load/store (NVLink) domain", lsa.nRanks, P);
    }
    const size_t hdr = ((sizeof(int64_t) * (P + irk::kXHeaderExtra)) + 4095) / 4096 * 4096;
    const size_t bytes = (hdr + qbytes + 4095) / 4096 * 4096;
    void *buf = nullptr;
    int rc = nccl_check(c, g_nccl.memAlloc(&buf, bytes), "ncclMemAlloc");
    if (rc) return rc;
    if ((rc = cuda_check(c, cudaMemsetAsync(buf, 0, bytes, st), "memset window")) ||
        (rc = cuda_check(c, cudaStreamSynchronize(st), "memset window"))) {
        g_nccl.memFree(buf);
        return rc;
    }
    ncclWindow_t win = nullptr;
    if ((rc = nccl_check(c, g_nccl.winRegister(comm, buf, bytes, &win, NCCL_WIN_COLL_SYMMETRIC),
                         "ncclCommWindowRegister"))) {
        g_nccl.memFree(buf);
        return rc;
    }
    c->xbuf = buf;
    c->xwin = win;
    c->xbytes = bytes;
    c->xqoff = hdr;
    if ((rc = cuda_check(c, cudaMalloc(&c->d_xpeers, sizeof(void *) * 2 * P), "cudaMalloc peers"))) return rc;
    xpeers_kernel<<<1, (P + 31) / 32 * 32, 0, st>>>(win, P, hdr, c->d_xpeers);
    if ((rc = cuda_check(c, cudaGetLastError(), "peer pointers"))) return rc;
    if ((rc = nccl_allgather_inplace(c, scratch, 1, st))) return rc;
    return cuda_check(c, cudaStreamSynchronize(st), "window set-up barrier");
}
}  // namespace

extern "C" {

irk_ctx *irk_create(int problem, int dim, double h, int64_t nsteps, int64_t batch) {
    g_create_error.clear();
    auto bad = [](const char *m) -> irk_ctx * {
        g_create_error = m;
        return nullptr;
    };
    switch (problem) {
    case IRK_KEPLER:
    case IRK_HENON_HEILES:
        if (dim != 4) return bad("irk_create: Kepler/Henon-Heiles need dim == 4");
        break;
    case IRK_SCHWARZSCHILD:
        if (dim != 4) return bad("irk_create: Schwarzschild needs dim == 4 (r, theta, p_r, p_theta)");
        break;
    case IRK_FPU_BETA:
        if (dim < 2 || dim % 2) return bad("irk_create: FPU needs an even dim >= 2");
        if (dim / 2 != 32 && dim / 2 != 64 && dim / 2 != 96 && dim / 2 != 128)
            return bad("irk_create: IRK_FPU_BETA supports N in {32, 64, 96, 128} sites (one warp per chain)");
        break;
    case IRK_NBODY: {
        if (dim % 6 || dim < 12) return bad("irk_create: N-body needs dim = 6N, N >= 2");
        const int N = dim / 6;
        if (N > 8) return bad("irk_create: IRK_NBODY ensembles support N in {2,...,8}");
        break;
    }
    case IRK_NBODY_DIRECT:
        if (dim % 6 || dim < 12) return bad("irk_create: N-body needs dim = 6N, N >= 2");
        if (batch != 1) return bad("irk_create: IRK_NBODY_DIRECT integrates one system (batch must be 1)");
        break;
    default: return bad("irk_create: unknown problem");
    }
    if (!std::isfinite(h) || h == 0.0) return bad("irk_create: h must be finite and nonzero");
    if (nsteps < 0) return bad("irk_create: nsteps < 0");
    if (batch < 1) return bad("irk_create: batch < 1");
    if (batch > 0x7fffffffLL) return bad("irk_create: batch > 2^31 - 1 (int32 trajectory indices)");
    irk_ctx *c = new irk_ctx;
    c->problem = problem;
    c->dim = dim;
    c->h = h;
    c->nsteps = nsteps;
    c->batch = batch;
    if (problem == IRK_SCHWARZSCHILD) c->mode = 1;  // not separable: first-order iteration only
    char err[256];
    if (irk::build_tableau(h, &c->T, err, sizeof err)) {
        g_create_error = err;
        delete c;
        return nullptr;
    }
    return c;
}

int irk_set_params(irk_ctx *c, const double *p, int n) {
    if (!c) return IRK_E_ARG;
    if (c->problem == IRK_NBODY_DIRECT && p && n >= 2 && !(p[1] > 0.0))
        return fail(c, IRK_E_ARG, "irk_set_params: IRK_NBODY_DIRECT needs eps > 0");
    if (!p || n != n_params_expected(c->problem, c->dim))
        return fail(c, IRK_E_ARG, "irk_set_params: expected %d params", n_params_expected(c->problem, c->dim));
    for (int i = 0; i < n; ++i)
        if (!std::isfinite(p[i])) return fail(c, IRK_E_ARG, "irk_set_params: non-finite param %d", i);
    c->params.assign(p, p + n);
    c->have_params = true;
    return IRK_OK;
}

int irk_set_option(irk_ctx *c, int key, int64_t val) {
    if (!c) return IRK_E_ARG;
    switch (key) {
    case IRK_OPT_MODE:
        if (val != 0 && val != 1) return fail(c, IRK_E_ARG, "irk_set_option: MODE must be 0 or 1");
        if (val == 1 && c->problem != IRK_KEPLER && c->problem != IRK_HENON_HEILES && c->problem != IRK_SCHWARZSCHILD)
            return fail(c, IRK_E_ARG, "irk_set_option: first-order mode is built for Kepler, Henon-Heiles, Schwarzschild");
        if (val == 0 && c->problem == IRK_SCHWARZSCHILD)
            return fail(c, IRK_E_ARG, "irk_set_option: Schwarzschild is not separable (first-order mode only)");
        c->mode = (int)val;
        return IRK_OK;
    case IRK_OPT_MAX_ITERS:
        if (val < 1 || val > 1000000) return fail(c, IRK_E_ARG, "irk_set_option: MAX_ITERS out of range");
        c->max_iters = (int)val;
        return IRK_OK;
    case IRK_OPT_ENERGY_EVERY:
        if (val < 0) return fail(c, IRK_E_ARG, "irk_set_option: ENERGY_EVERY < 0");
        c->energy_every = val;
        return IRK_OK;
    case IRK_OPT_BALANCE:
        if (val < -1) return fail(c, IRK_E_ARG, "irk_set_option: bad BALANCE");
        c->balance = val;
        return IRK_OK;
    case IRK_OPT_LOCAL_ENERGY:
        if (val != 0 && val != 1) return fail(c, IRK_E_ARG, "irk_set_option: LOCAL_ENERGY must be 0 or 1");
        if (val && c->problem == IRK_NBODY_DIRECT)
            return fail(c, IRK_E_ARG, "irk_set_option: LOCAL_ENERGY is for the ensemble problems (use ENERGY_EVERY)");
        c->local_energy = (int)val;
        return IRK_OK;
    case IRK_OPT_VSHARDS:
        if (c->problem != IRK_NBODY_DIRECT || val < 1 || (c->dim / 6) % val || c->nccl_comm)
            return fail(c, IRK_E_ARG, "irk_set_option: VSHARDS needs IRK_NBODY_DIRECT, N %% P == 0, no NCCL comm");
        c->vshards = (int)val;
        return IRK_OK;
    case IRK_OPT_EXCHANGE:
        if (c->problem != IRK_NBODY_DIRECT || (val != 0 && val != 1))
            return fail(c, IRK_E_ARG, "irk_set_option: EXCHANGE is 0 or 1, for IRK_NBODY_DIRECT");
        c->exchange = (int)val;
        return IRK_OK;
    case IRK_OPT_DEVICE_LOOP:
        if (val != 0 && val != 1) return fail(c, IRK_E_ARG, "irk_set_option: DEVICE_LOOP must be 0 or 1");
        c->device_loop = (int)val;
        return IRK_OK;
    case IRK_OPT_SCHEDULE:
        if (val < 0 || val > 2) return fail(c, IRK_E_ARG, "irk_set_option: SCHEDULE must be 0, 1 or 2");
        c->schedule = (int)val;
        return IRK_OK;
    case IRK_OPT_MAPPING:
        if (val != IRK_MAP_AUTO && val != IRK_MAP_G1 && val != IRK_MAP_G2 && val != IRK_MAP_G4 && val != IRK_MAP_G8 &&
            val != IRK_MAP_G8M)
            return fail(c, IRK_E_ARG,
                        "irk_set_option: MAPPING must be 0 (auto), 1 (g1), 2 (g2), 4 (g4), 8 (g8) or 9 (g8m)");
        if (val == IRK_MAP_G8M && c->problem != IRK_NBODY && c->problem != IRK_KEPLER && c->problem != IRK_HENON_HEILES)
            return fail(c, IRK_E_ARG, "irk_set_option: the g8m mapping is built for Kepler, Henon-Heiles, N-body");
        if ((val == IRK_MAP_G4 || val == IRK_MAP_G2) && c->problem != IRK_KEPLER && c->problem != IRK_HENON_HEILES)
            return fail(c, IRK_E_ARG, "irk_set_option: the g2 / g4 mappings are built for Kepler and Henon-Heiles");
        if (val == IRK_MAP_G8 && c->problem != IRK_KEPLER && c->problem != IRK_HENON_HEILES && c->problem != IRK_NBODY &&
            c->problem != IRK_SCHWARZSCHILD)
            return fail(c, IRK_E_ARG, "irk_set_option: the g8 mapping is built for Kepler, Henon-Heiles, N-body");
        c->mapping = (int)val;
        return IRK_OK;
    }
    return fail(c, IRK_E_ARG, "irk_set_option: unknown key %d", key);
}

int irk_get_option(const irk_ctx *c, int key, int64_t *val) {
    if (!c || !val) return IRK_E_ARG;
    switch (key) {
    case IRK_OPT_MODE: *val = c->mode; return IRK_OK;
    case IRK_OPT_MAX_ITERS: *val = c->max_iters; return IRK_OK;
    case IRK_OPT_ENERGY_EVERY: *val = c->energy_every; return IRK_OK;
    case IRK_OPT_MAPPING: *val = c->mapping; return IRK_OK;
    case IRK_OPT_BALANCE: *val = c->balance; return IRK_OK;
    case IRK_OPT_VSHARDS: *val = c->vshards; return IRK_OK;
    case IRK_OPT_LOCAL_ENERGY: *val = c->local_energy; return IRK_OK;
    case IRK_OPT_SCHEDULE: *val = c->schedule; return IRK_OK;
    case IRK_OPT_DEVICE_LOOP: *val = c->device_loop; return IRK_OK;
    case IRK_OPT_EXCHANGE: *val = c->exchange; return IRK_OK;
    case IRK_INFO_DEVICE_LOOP_USED: *val = c->device_loop_used; return IRK_OK;
    case IRK_INFO_MAPPING_USED: *val = c->mapping_used; return IRK_OK;
    }
    return IRK_E_ARG;
}

size_t irk_workspace_bytes(const irk_ctx *c) {
    if (!c) return 0;
    return kHeader + hist_bytes(c) + stats_bytes(c) + sched_bytes(c) + nbd_bytes(c);
}

int irk_integrate(irk_ctx *c, double *y, double t0, void *workspace, double *energy, int64_t *iters,
                  void *stream) {
    if (!c) return IRK_E_ARG;
    if (!c->have_params) return fail(c, IRK_E_STATE, "irk_integrate: irk_set_params not called");
    if (!y || !workspace) return fail(c, IRK_E_ARG, "irk_integrate: null y or workspace");
    if (!std::isfinite(t0)) return fail(c, IRK_E_ARG, "irk_integrate: non-finite t0");
    if (c->energy_every > 0 && !energy) return fail(c, IRK_E_ARG, "irk_integrate: ENERGY_EVERY set but energy == NULL");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    char *ws = static_cast<char *>(workspace);
    static const char *kNames[] = {"irk_integrate", "irk_integrate:kepler", "irk_integrate:nbody",
                                   "irk_integrate:fpu_beta", "irk_integrate:henon_heiles",
                                   "irk_integrate:nbody_direct", "irk_integrate:schwarzschild"};
    NvtxRange range(kNames[(c->problem >= 1 && c->problem <= 6) ? c->problem : 0]);
    int rc = upload_constants(c, st);
    if (rc) return rc;
    switch (c->problem) {
    case IRK_KEPLER: {
        if (IRK_UNIT_G && c->params[0] == 1.0) {  // GM = 1: the reciprocal form of the same division
            irk::KeplerG1 P{c->params[0]};
            rc = launch_g1(c, P, y, t0, ws, energy, iters, st);
        } else {
            irk::Kepler P{c->params[0]};
            rc = launch_g1(c, P, y, t0, ws, energy, iters, st);
        }
        break;
    }
    case IRK_HENON_HEILES: {
        irk::HenonHeiles P{c->params[0], c->params[1]};
        rc = launch_g1(c, P, y, t0, ws, energy, iters, st);
        break;
    }
    case IRK_SCHWARZSCHILD: {
        irk::Schwarzschild P{c->params[0], c->params[1], c->params[2]};
        rc = launch_first_order(c, P, y, t0, ws, energy, iters, st);
        break;
    }
    case IRK_NBODY:
        rc = launch_nbody(c, y, t0, ws, energy, iters, st);
        break;
    case IRK_FPU_BETA:
        c->mapping_used = 0;
        rc = launch_chain(c, y, t0, ws, energy, iters, st);
        break;
    case IRK_NBODY_DIRECT:
        c->mapping_used = 0;
        rc = launch_direct(c, y, t0, ws, energy, iters, st);
        break;
    default: return fail(c, IRK_E_ARG, "irk_integrate: problem not supported");
    }
    return rc;
}

int irk_integrate_host(irk_ctx *c, double *y_host, double t0, double *energy_host, int64_t *iters_host,
                       void *stream) {
    if (!c) return IRK_E_ARG;
    if (!y_host) return fail(c, IRK_E_ARG, "irk_integrate_host: null y");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const size_t ybytes = sizeof(double) * (size_t)local_dim(c) * c->batch;
    const size_t wsb = irk_workspace_bytes(c);
    const size_t ebytes = c->energy_every > 0 ? sizeof(double) * (size_t)(c->nsteps / c->energy_every + 1) * c->batch : 0;
    int rc;
    if (c->cap_y < ybytes) {
        cudaFree(c->d_y);
        c->d_y = nullptr;
        c->cap_y = 0;
        if ((rc = cuda_check(c, cudaMalloc(&c->d_y, ybytes), "cudaMalloc y"))) return rc;
        c->cap_y = ybytes;
    }
    if (c->cap_ws < wsb) {
        cudaFree(c->d_ws);
        c->d_ws = nullptr;
        c->cap_ws = 0;
        if ((rc = cuda_check(c, cudaMalloc(&c->d_ws, wsb), "cudaMalloc workspace"))) return rc;
        c->cap_ws = wsb;
    }
    if (ebytes && c->cap_energy < ebytes) {
        cudaFree(c->d_energy);
        c->d_energy = nullptr;
        c->cap_energy = 0;
        if ((rc = cuda_check(c, cudaMalloc(&c->d_energy, ebytes), "cudaMalloc energy"))) return rc;
        c->cap_energy = ebytes;
    }
    if (iters_host && c->cap_iters < c->batch) {
        cudaFree(c->d_iters);
        c->d_iters = nullptr;
        c->cap_iters = 0;
        if ((rc = cuda_check(c, cudaMalloc(&c->d_iters, sizeof(int64_t) * c->batch), "cudaMalloc iters"))) return rc;
        c->cap_iters = c->batch;
    }
    if ((rc = cuda_check(c, cudaMemcpyAsync(c->d_y, y_host, ybytes, cudaMemcpyHostToDevice, st), "H2D y"))) return rc;
    if ((rc = cuda_check(c, cudaMemsetAsync(c->d_ws, 0, wsb, st), "memset workspace"))) return rc;
    if ((rc = irk_integrate(c, c->d_y, t0, c->d_ws, ebytes ? c->d_energy : nullptr,
                            iters_host ? c->d_iters : nullptr, stream)))
        return rc;
    if ((rc = cuda_check(c, cudaMemcpyAsync(y_host, c->d_y, ybytes, cudaMemcpyDeviceToHost, st), "D2H y"))) return rc;
    if (energy_host && ebytes &&
        (rc = cuda_check(c, cudaMemcpyAsync(energy_host, c->d_energy, ebytes, cudaMemcpyDeviceToHost, st), "D2H energy")))
        return rc;
    if (iters_host &&
        (rc = cuda_check(c, cudaMemcpyAsync(iters_host, c->d_iters, sizeof(int64_t) * c->batch, cudaMemcpyDeviceToHost, st),
                         "D2H iters")))
        return rc;
    return cuda_check(c, cudaStreamSynchronize(st), "irk_integrate_host sync");
}

int irk_energy(irk_ctx *c, const double *y, double *H, void *stream) {
    if (!c) return IRK_E_ARG;
    if (!c->have_params) return fail(c, IRK_E_STATE, "irk_energy: irk_set_params not called");
    if (!y || !H) return fail(c, IRK_E_ARG, "irk_energy: null pointer");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    const int threads = 128;
    const unsigned blocks = (unsigned)((c->batch + threads - 1) / threads);
    switch (c->problem) {
    case IRK_KEPLER:
        energy_g1_kernel<<<blocks, threads, 0, st>>>(y, H, c->batch, irk::Kepler{c->params[0]});
        break;
    case IRK_HENON_HEILES:
        energy_g1_kernel<<<blocks, threads, 0, st>>>(y, H, c->batch, irk::HenonHeiles{c->params[0], c->params[1]});
        break;
    case IRK_SCHWARZSCHILD:
        energy_g1_kernel<<<blocks, threads, 0, st>>>(y, H, c->batch,
                                                     irk::Schwarzschild{c->params[0], c->params[1], c->params[2]});
        break;
    case IRK_NBODY_DIRECT: {
        const int64_t N = c->dim / 6;
        const int P = c->nccl_comm ? c->nranks : 1;
        const int64_t nloc = N / P;
        int rc;
        if (!c->d_mass) {
            if ((rc = cuda_check(c, cudaMalloc(&c->d_mass, sizeof(double) * N), "cudaMalloc mass"))) return rc;
            if ((rc = cuda_check(c, cudaMallocHost(&c->h_ctl, sizeof(irk::NbdCtl)), "cudaMallocHost ctl"))) return rc;
        }
        if (!c->d_rows && (rc = cuda_check(c, cudaMalloc(&c->d_rows, sizeof(double) * 5 * N), "cudaMalloc energy")))
            return rc;
        double *Qall = c->d_rows, *terms = c->d_rows + 3 * N;
        const int64_t b0 = (int64_t)c->rank * nloc;
        if ((rc = cuda_check(c, cudaMemcpyAsync(c->d_mass, c->params.data() + 2, sizeof(double) * N,
                                                cudaMemcpyHostToDevice, st), "H2D mass")) ||
            (rc = cuda_check(c, cudaMemcpyAsync(Qall + 3 * b0, y, sizeof(double) * 3 * nloc, cudaMemcpyDeviceToDevice, st),
                             "energy: positions")))
            return rc;
        if (c->nccl_comm && (rc = nccl_allgather_inplace(c, Qall, (size_t)(3 * nloc), st))) return rc;
        const double *v = y + (c->nccl_comm ? 3 * nloc : 3 * N);
        irk::nbd_energy_terms_kernel<<<(unsigned)((nloc + irk::NBD_EROW_ROWS - 1) / irk::NBD_EROW_ROWS), irk::NBD_EROW_THREADS, 0, st>>>(
            Qall, v, c->d_mass, N, b0, nloc, c->params[0], c->params[1] * c->params[1], terms + 2 * b0);
        if (c->nccl_comm && (rc = nccl_allgather_inplace(c, terms, (size_t)(2 * nloc), st))) return rc;
        irk::nbd_energy_sum_kernel<<<1, irk::NBD_ESUM_THREADS, 0, st>>>(terms, P, nloc, H);
        break;
    }
    case IRK_FPU_BETA: {
        const unsigned nb = (unsigned)((c->batch + 127) / 128);
        switch (c->dim / 2) {
        case 32: energy_fpu_kernel<32><<<nb, 128, 0, st>>>(y, H, c->batch, c->params[0]); break;
        case 64: energy_fpu_kernel<64><<<nb, 128, 0, st>>>(y, H, c->batch, c->params[0]); break;
        case 96: energy_fpu_kernel<96><<<nb, 128, 0, st>>>(y, H, c->batch, c->params[0]); break;
        case 128: energy_fpu_kernel<128><<<nb, 128, 0, st>>>(y, H, c->batch, c->params[0]); break;
        default: return fail(c, IRK_E_ARG, "irk_energy: unsupported N");
        }
        break;
    }
    case IRK_NBODY:
        switch (c->dim / 6) {
        case 2: launch_energy_nbody_t<2>(c, y, H, st); break;
        case 3: launch_energy_nbody_t<3>(c, y, H, st); break;
        case 4: launch_energy_nbody_t<4>(c, y, H, st); break;
        case 5: launch_energy_nbody_t<5>(c, y, H, st); break;
        case 6: launch_energy_nbody_t<6>(c, y, H, st); break;
        case 7: launch_energy_nbody_t<7>(c, y, H, st); break;
        case 8: launch_energy_nbody_t<8>(c, y, H, st); break;
        default: return fail(c, IRK_E_ARG, "irk_energy: unsupported N");
        }
        break;
    default: return fail(c, IRK_E_ARG, "irk_energy: problem not supported");
    }
    return cuda_check(c, cudaGetLastError(), "energy kernel launch");
}

int irk_stats(irk_ctx *c, const void *workspace, void *stream, int64_t out[4]) {
    if (!c || !workspace || !out) return IRK_E_ARG;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
    std::vector<int64_t> s(4 * (size_t)c->batch);
    int rc = cuda_check(c,
                        cudaMemcpyAsync(s.data(), static_cast<const char *>(workspace) + kHeader + hist_bytes(c),
                                        stats_bytes(c), cudaMemcpyDeviceToHost, st),
                        "D2H stats");
    if (rc) return rc;
    if ((rc = cuda_check(c, cudaStreamSynchronize(st), "irk_stats sync"))) return rc;
    int64_t hit_traj = 0, div_traj = 0, first_bad = -1, total = 0;
    const int64_t B = c->batch;
    for (int64_t b = 0; b < B; ++b) {
        if (s[b] > 0) ++hit_traj;
        if (s[B + b] > 0) {  // diverged_step is 1-based; 0 = none
            ++div_traj;
            if (first_bad < 0 || s[B + b] < first_bad) first_bad = s[B + b];
        }
        total += s[2 * B + b];
    }
    out[0] = hit_traj;
    out[1] = div_traj;
    out[2] = first_bad;
    out[3] = total;
    if (div_traj) return IRK_E_DIVERGED;
    if (hit_traj) return IRK_W_MAXITER;
    return IRK_OK;
}

int irk_local_energy_error(irk_ctx *c, const void *workspace, double *out, void *stream) {
    if (!c || !workspace || !out) return IRK_E_ARG;
    if (!c->local_energy) return fail(c, IRK_E_STATE, "irk_local_energy_error: IRK_OPT_LOCAL_ENERGY not set");
    const char *src = static_cast<const char *>(workspace) + kHeader + hist_bytes(c) + sizeof(int64_t) * 3 * c->batch;
    return cuda_check(c, cudaMemcpyAsync(out, src, sizeof(double) * c->batch, cudaMemcpyDeviceToDevice,
                                         reinterpret_cast<cudaStream_t>(stream)),
                      "D2D dhloc");
}

int irk_tableau(double *c, double *b, double *mu, double *nu) {
    Tableau T;
    char err[256];
    if (irk::build_tableau(1.0, &T, err, sizeof err)) return IRK_E_ARG;
    if (c) memcpy(c, T.c, sizeof T.c);
    if (b) memcpy(b, T.b, sizeof T.b);
    if (mu) memcpy(mu, T.mu, sizeof T.mu);
    if (nu) memcpy(nu, T.nu, sizeof T.nu);
    return IRK_OK;
}

int irk_nccl_unique_id(void *out) {
    if (!out) return IRK_E_ARG;
    if (load_nccl()) return IRK_E_COMM;
    ncclUniqueId id;
    if (g_nccl.getUniqueId(&id) != ncclSuccess) return IRK_E_COMM;
    memcpy(out, &id, sizeof id);
    return IRK_OK;
}

int irk_set_comm(irk_ctx *c, const void *id, int rank, int nranks) {
    if (!c) return IRK_E_ARG;
    if (c->problem != IRK_NBODY_DIRECT) return fail(c, IRK_E_ARG, "irk_set_comm: only IRK_NBODY_DIRECT shards");
    if (!id || nranks < 1 || rank < 0 || rank >= nranks) return fail(c, IRK_E_ARG, "irk_set_comm: bad rank/nranks");
    if ((c->dim / 6) % nranks) return fail(c, IRK_E_ARG, "irk_set_comm: N must be divisible by nranks");
    if (c->nccl_comm) return fail(c, IRK_E_STATE, "irk_set_comm: communicator already set");
    if (const char *e = load_nccl()) return fail(c, IRK_E_COMM, "irk_set_comm: %s", e);
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof uid);
    ncclComm_t comm = nullptr;
    int rc = nccl_check(c, g_nccl.commInitRank(&comm, nranks, uid, rank), "ncclCommInitRank");
    if (rc) return rc;
    c->nccl_comm = comm;
    c->nranks = nranks;
    c->rank = rank;
    c->vshards = 1;
    return IRK_OK;
}

const char *irk_last_error(const irk_ctx *c) {
    if (!c) return g_create_error.c_str();
    return c->err.c_str();
}

void irk_destroy(irk_ctx *c) {
    if (!c) return;
    cudaFree(c->d_y);
    cudaFree(c->d_energy);
    cudaFree(c->d_iters);
    cudaFree(c->d_ws);
    cudaFree(c->d_mass);
    cudaFree(c->d_rows);
    cudaFree(c->d_xpeers);
    if (c->xwin && g_nccl.winDeregister)
        g_nccl.winDeregister(reinterpret_cast<ncclComm_t>(c->nccl_comm), reinterpret_cast<ncclWindow_t>(c->xwin));
    if (c->xbuf && g_nccl.memFree) g_nccl.memFree(c->xbuf);
    if (c->nccl_comm && g_nccl.commDestroy) g_nccl.commDestroy(reinterpret_cast<ncclComm_t>(c->nccl_comm));
    if (c->h_ctl) cudaFreeHost(c->h_ctl);
    delete c;
}

}  // extern "C"

#ifdef IRK_TRACE
// measurement builds only (tools/unit_trace.py): point the work-unit trace at a
// device buffer of cap records (6 x uint64 each) and reset its counter
extern "C" int irk_trace_set(void *buf, int64_t cap) {
    unsigned long long *p = static_cast<unsigned long long *>(buf), n = 0, c = (unsigned long long)cap;
    if (cudaMemcpyToSymbol(irk::g_irk_trace, &p, sizeof p) != cudaSuccess) return -1;
    if (cudaMemcpyToSymbol(irk::g_irk_trace_n, &n, sizeof n) != cudaSuccess) return -1;
    return cudaMemcpyToSymbol(irk::g_irk_trace_cap, &c, sizeof c) == cudaSuccess ? 0 : -1;
}
#endif

