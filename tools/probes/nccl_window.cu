// Probe: does NCCL 2.28 (torch wheel) register a symmetric window on a 1-rank
// communicator on this box, and does ncclGetPeerPointer(win, off, rank) give a
// pointer the kernel can store to / load from (the fused-exchange building block)?
// nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -I<nccl>/include nccl_window.cu -L<nccl>/lib -l:libnccl.so.2
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>
#include <cstdio>

__global__ void k(ncclWindow_t w, double *local, unsigned long long *out) {
    double *p = (double *)ncclGetPeerPointer(w, 64, 0);
    out[0] = (unsigned long long)p;
    out[1] = (unsigned long long)(local + 8);
    p[0] = 42.0;
    __threadfence_system();
    out[2] = (unsigned long long)(local[8] == 42.0);
}

int main() {
    ncclUniqueId id;
    ncclComm_t comm;
    if (ncclGetUniqueId(&id) || ncclCommInitRank(&comm, 1, id, 0)) { printf("init fail\n"); return 1; }
    void *buf = nullptr;
    ncclResult_t r = ncclMemAlloc(&buf, 1 << 20);
    printf("ncclMemAlloc %d %p\n", (int)r, buf);
    ncclWindow_t win = nullptr;
    r = ncclCommWindowRegister(comm, buf, 1 << 20, &win, NCCL_WIN_COLL_SYMMETRIC);
    printf("ncclCommWindowRegister(SYMMETRIC) %d %s win=%p\n", (int)r, ncclGetErrorString(r), (void *)win);
    ncclTeam_t lsa = ncclTeamLsa(comm);
    printf("lsa team nRanks=%d rank=%d stride=%d\n", lsa.nRanks, lsa.rank, lsa.stride);
    if (r) return 2;
    unsigned long long *out;
    cudaMallocManaged(&out, 64);
    k<<<1, 1>>>(win, (double *)buf, out);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel %s peer=%llx local=%llx same_data=%llu\n", cudaGetErrorString(e), out[0], out[1], out[2]);
    ncclCommWindowDeregister(comm, win);
    ncclMemFree(buf);
    ncclCommDestroy(comm);
    return 0;
}
