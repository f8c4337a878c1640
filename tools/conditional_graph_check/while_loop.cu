// minimal conditional-WHILE graph: does compute-sanitizer racecheck support it?
#include <cuda_runtime.h>
#include <stdio.h>
__global__ void body(int *cnt, cudaGraphConditionalHandle h) {
    __shared__ int s;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    atomicAdd(&s, 1);
    __syncthreads();
    if (threadIdx.x == 0) {
        int c = ++(*cnt);
        cudaGraphSetConditional(h, c < 5 ? 1u : 0u);
    }
}
int main() {
    int *cnt;
    cudaMalloc(&cnt, 4);
    cudaMemset(cnt, 0, 4);
    cudaStream_t st;
    cudaStreamCreate(&st);
    cudaGraph_t g;
    cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaError_t e = cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t n;
    if (!e) e = cudaGraphAddNode(&n, g, nullptr, 0, &p);
    if (!e) e = cudaStreamBeginCaptureToGraph(st, p.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    body<<<1, 64, 0, st>>>(cnt, h);
    cudaGraph_t out;
    if (!e) e = cudaStreamEndCapture(st, &out);
    cudaGraphExec_t ex;
    if (!e) e = cudaGraphInstantiate(&ex, g, 0);
    if (!e) e = cudaGraphLaunch(ex, st);
    if (!e) e = cudaStreamSynchronize(st);
    int c = -1;
    cudaMemcpy(&c, cnt, 4, cudaMemcpyDeviceToHost);
    printf("status %s count %d (expect 5)\n", cudaGetErrorString(e), c);
    return 0;
}
