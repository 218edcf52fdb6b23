#include <cuda_runtime.h>
#include <cstdio>
__global__ void body(int *x, cudaGraphConditionalHandle h) {
    int v = ++(*x);
    cudaGraphSetConditional(h, v < 10 ? 1 : 0);
}
int main() {
    int *x; cudaMalloc(&x, 4); cudaMemset(x, 0, 4);
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    if (cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault)) { printf("handle fail\n"); return 1; }
    cudaGraphNodeParams cp = {};
    cp.type = cudaGraphNodeTypeConditional;
    cp.conditional.handle = h; cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
    cudaGraphNode_t node;
    if (cudaGraphAddNode(&node, g, nullptr, 0, &cp)) { printf("node fail\n"); return 1; }
    cudaGraph_t bodyg = cp.conditional.phGraph_out[0];
    cudaStream_t cs; cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking);
    cudaStreamBeginCaptureToGraph(cs, bodyg, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    body<<<1,1,0,cs>>>(x, h);
    cudaError_t e = cudaStreamEndCapture(cs, &bodyg);
    printf("capture %s\n", cudaGetErrorString(e));
    cudaGraphExec_t ge; e = cudaGraphInstantiate(&ge, g, 0); printf("inst %s\n", cudaGetErrorString(e));
    cudaGraphLaunch(ge, cs); cudaStreamSynchronize(cs);
    int hx; cudaMemcpy(&hx, x, 4, cudaMemcpyDeviceToHost); printf("x=%d (want 10) %s\n", hx, cudaGetErrorString(cudaGetLastError()));
}
