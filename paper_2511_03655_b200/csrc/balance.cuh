// Cost-balanced trajectory scheduling for the ensemble kernels.
//
// The fixed-point iteration takes a data-dependent number of sweeps per step
// (2-13 on config 2), so a warp of 32 random trajectories runs as long as its
// most expensive lane.  irk_integrate therefore runs the nsteps of a call in
// chunks; after each chunk the trajectories are counting-sorted by the sweeps
// they needed in it (bucket = sweeps per step in 1/64 units), consecutive ranks
// form a warp (similar cost), and warps are dealt to blocks in a mirrored order
// (block b gets warp b and warp 2*nblocks-1-b) so that every SM receives a mix
// of cheap and expensive warps.  The assignment only changes which thread
// integrates which trajectory: every trajectory's arithmetic, and so every
// result bit, is unchanged (the order inside a bucket is not even deterministic).
#pragma once
#include <cstdint>

namespace irk {

constexpr int kCostBins = 1024;  // sweeps/step in [0, 16) at 1/64 resolution (clamped)

__device__ __forceinline__ int cost_bin(int32_t sweeps, int64_t steps) {
    int64_t v = steps > 0 ? ((int64_t)sweeps * 64) / steps : 0;
    return (int)(v < 0 ? 0 : (v >= kCostBins ? kCostBins - 1 : v));
}

__global__ void cost_hist_kernel(const int32_t *csweeps, int64_t B, int64_t steps, int32_t *bins) {
    __shared__ int32_t h[kCostBins];
    for (int i = threadIdx.x; i < kCostBins; i += blockDim.x) h[i] = 0;
    __syncthreads();
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&h[cost_bin(csweeps[b], steps)], 1);
    __syncthreads();
    for (int i = threadIdx.x; i < kCostBins; i += blockDim.x)
        if (h[i]) atomicAdd(&bins[i], h[i]);
}

// exclusive scan of kCostBins counts, one block of kCostBins threads
__global__ void cost_scan_kernel(int32_t *bins) {
    __shared__ int32_t t[kCostBins];
    const int i = threadIdx.x;
    t[i] = bins[i];
    __syncthreads();
    for (int off = 1; off < kCostBins; off <<= 1) {
        int32_t v = (i >= off) ? t[i - off] : 0;
        __syncthreads();
        t[i] += v;
        __syncthreads();
    }
    bins[i] = t[i] - bins[i];
}

__global__ void cost_scatter_kernel(const int32_t *csweeps, int64_t B, int64_t steps, int32_t *bins,
                                    int32_t *sorted) {
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < B; b += (int64_t)gridDim.x * blockDim.x) {
        int pos = atomicAdd(&bins[cost_bin(csweeps[b], steps)], 1);
        sorted[pos] = (int32_t)b;
    }
}

// slot -> trajectory.  A kernel warp holds `spw` trajectory slots (32 for ens_g1,
// 32/NB groups for ens_nbody) and a block holds `wpb` warps.  Warp W of the
// sorted order holds ranks [spw*W, spw*W + spw); block blk runs warps blk*wpb/2..
// from the front of the order and as many from the back (mirrored dealing).
__global__ void cost_perm_kernel(const int32_t *sorted, int64_t B, int64_t nblocks, int wpb, int spw,
                                 int32_t *perm) {
    const int64_t slot = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t per_block = (int64_t)wpb * spw;
    if (slot >= nblocks * per_block) return;
    const int64_t blk = slot / per_block;
    const int wib = (int)((slot % per_block) / spw), s = (int)(slot % spw);
    const int64_t nw = nblocks * wpb;
    const int64_t kk = blk * wpb + wib;  // 0..nw-1
    const int64_t W = (wib % 2 == 0) ? (kk / 2) : (nw - 1 - kk / 2);
    const int64_t rank = W * spw + s;
    perm[slot] = (rank < B) ? sorted[rank] : -1;
}

}  // namespace irk
