// WHILE body = kernel A, then an IF node (added through the capture info) whose body = kernel B:
// the structure of the library's device loop.  Plain run vs compute-sanitizer.
#include <cuda_runtime.h>
#include <stdio.h>
__global__ void ka(int *cnt, cudaGraphConditionalHandle hi, cudaGraphConditionalHandle hw) {
    int c = ++cnt[0];
    cudaGraphSetConditional(hi, c < 9 ? 1u : 0u);
    if (c >= 9) cudaGraphSetConditional(hw, 0u);
}
__global__ void kb(int *cnt, cudaGraphConditionalHandle hw) {
    int c = ++cnt[0];
    cnt[1]++;
    cudaGraphSetConditional(hw, c < 9 ? 1u : 0u);
}
#define CKE(x) do { cudaError_t e_ = (x); if (e_) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); return 1; } } while (0)
int main() {
    int *cnt;
    CKE(cudaMalloc(&cnt, 8));
    CKE(cudaMemset(cnt, 0, 8));
    cudaStream_t st;
    CKE(cudaStreamCreate(&st));
    cudaGraph_t g;
    CKE(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hw, hi;
    CKE(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = hw;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t n;
    CKE(cudaGraphAddNode(&n, g, nullptr, 0, &p));
    cudaGraph_t BW = p.conditional.phGraph_out[0];
    CKE(cudaGraphConditionalHandleCreate(&hi, BW, 0, cudaGraphCondAssignDefault));
    CKE(cudaStreamBeginCaptureToGraph(st, BW, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    ka<<<1, 1, 0, st>>>(cnt, hi, hw);
    cudaStreamCaptureStatus cs;
    cudaGraph_t cg;
    const cudaGraphNode_t *deps;
    size_t nd;
    CKE(cudaStreamGetCaptureInfo(st, &cs, nullptr, &cg, &deps, &nd));
    cudaGraphNodeParams ip = {};
    ip.type = cudaGraphNodeTypeConditional;
    ip.conditional.handle = hi;
    ip.conditional.type = cudaGraphCondTypeIf;
    ip.conditional.size = 1;
    cudaGraphNode_t in;
    CKE(cudaGraphAddNode(&in, cg, deps, nd, &ip));
    CKE(cudaStreamUpdateCaptureDependencies(st, &in, 1, cudaStreamSetCaptureDependencies));
    cudaGraph_t out;
    CKE(cudaStreamEndCapture(st, &out));
    CKE(cudaStreamBeginCaptureToGraph(st, ip.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    kb<<<1, 1, 0, st>>>(cnt, hw);
    CKE(cudaStreamEndCapture(st, &out));
    cudaGraphExec_t ex;
    CKE(cudaGraphInstantiate(&ex, g, 0));
    CKE(cudaGraphLaunch(ex, st));
    CKE(cudaStreamSynchronize(st));
    int c[2] = {-1, -1};
    CKE(cudaMemcpy(c, cnt, 8, cudaMemcpyDeviceToHost));
    printf("count %d (expect 9), B ran %d (expect 4)\n", c[0], c[1]);
    return 0;
}
