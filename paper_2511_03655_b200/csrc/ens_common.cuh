// Shared declarations of the ensemble kernels: coefficient constants and the
// launch-argument block.
#pragma once
#include <cstdint>

#include "tableau.h"

namespace irk {

// mu~, nu~ and c~ do not depend on h: one copy per device in the constant bank
// (uploaded once per device by irk_api.cu), read as uniform operands.  hb~ =
// fl(h b~) depends on h and travels in the kernel parameters.
__constant__ double c_mu[8][8];
__constant__ double c_nu[8][8];
__constant__ double c_c[8];

struct EnsArgs {
    double hb[8];
    double *y;            // [dim][batch]
    double *hist;         // [8][dim][batch]
    int64_t *stats;       // [4][batch]
    const int64_t *n_done;
    double *energy;       // [(nsteps/E)+1][batch] or null
    int64_t *iters;       // [batch] or null (set on the first chunk, accumulated after)
    const int32_t *perm;  // thread slot -> trajectory (null = identity; < 0 = idle slot)
    int32_t *csweeps;     // [batch] sweeps of this chunk, for the cost sort (or null)
    int64_t batch, nsteps, energy_every;
    int64_t c0;           // call-local index of this chunk's first step
    int64_t nslots;       // launched thread slots (perm covers all of them)
    double h, t0;
    int max_iters;
    int local_energy;     // track Delta H^loc_max (Eq. DHlocmax) into stats[3] (as double bits)
};

// running max of the local relative energy error (Eq. DHlocmax):
// loc = |(H_n - H_{n-1}) / H_{n-1}|, NaN-ignoring max, same ops as the oracle
__device__ __forceinline__ void dhloc_update(double hn, double &hprev, double &dmax) {
    const double loc = fabs(__ddiv_rn(__dsub_rn(hn, hprev), hprev));
    dmax = (loc > dmax) ? loc : dmax;
    hprev = hn;
}
// Work queue of the persistent ensemble kernels (ens_g1q, ens_chain_q): units
// u = c * batch + b are (trajectory b, step chunk c of qchunk steps).
struct QueueArgs {
    unsigned long long *counter;  // next unit
    int32_t *progress;            // [batch] chunks completed in this call
    int32_t *orphan;              // [batch] c > 0: unit (w, c) was fetched while blocked and parked
                                  // for the warp finishing (w, c - 1); 0: none (ens_nbody_q)
    int64_t qchunk;               // steps per unit
    int64_t nchunks;              // units per trajectory
};

// Hand-off of a blocked unit.  Fetcher of (w, c), finding progress[w] < c: park it
// (orphan[w]: 0 -> c), fence, re-read progress; if still < c the predecessor's
// warp will run it, else reclaim it (orphan[w]: c -> 0).  Releaser of (w, c - 1):
// publish progress[w] = c, fence, claim (orphan[w]: c -> 0).  With sequentially
// consistent fences on both sides exactly one of the two runs the unit.
__device__ __forceinline__ bool claim_orphan(const QueueArgs &qa, int32_t w, int64_t c) {
    if (c >= qa.nchunks) return false;
    __threadfence();
    return atomicCAS(&qa.orphan[w], (int)c, 0) == (int)c;
}

// inter-unit hand-off of the work-queue kernels (gpu-scope release / acquire)
__device__ __forceinline__ int32_t ld_acquire(const int32_t *p) {
    int32_t v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int32_t *p, int32_t v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Work-unit trace (measurement builds only, -DIRK_TRACE; tools/unit_trace.py):
// per finished unit {c << 32 | b, smid << 48 | block << 16 | thread, t_fetch, t_start, t_end, sweeps}
// (globaltimer ns).  Absent from the product build.
#ifdef IRK_TRACE
__device__ unsigned long long *g_irk_trace;
__device__ unsigned long long g_irk_trace_n, g_irk_trace_cap;
__device__ __forceinline__ unsigned long long irk_now() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__device__ __forceinline__ void irk_trace_unit(int64_t c, int64_t b, unsigned long long tf, unsigned long long ts,
                                               int64_t sweeps) {
    const unsigned long long i = atomicAdd(&g_irk_trace_n, 1ull);
    if (!g_irk_trace || i >= g_irk_trace_cap) return;
    unsigned smid;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
    unsigned long long *r = g_irk_trace + 6 * i;
    r[0] = ((unsigned long long)c << 32) | (unsigned long long)b;
    r[1] = ((unsigned long long)smid << 48) | ((unsigned long long)blockIdx.x << 16) | threadIdx.x;
    r[2] = tf;
    r[3] = ts;
    r[4] = irk_now();
    r[5] = (unsigned long long)sweeps;
}
#endif

// combine this chunk's max with the call's running max stored in stats[3]
__device__ __forceinline__ void dhloc_store(int64_t *stats3, bool first_chunk, double dmax) {
    double prev = first_chunk ? 0.0 : __longlong_as_double(__ldcg(stats3));
    *stats3 = __double_as_longlong((dmax > prev) ? dmax : prev);
}

}  // namespace irk
