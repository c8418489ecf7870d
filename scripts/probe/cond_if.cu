// Probe: WHILE node whose body holds IF nodes selected by a mode the body's
// kernels update (handles created on the body graph, no default assignment).
#include <cstdio>
#include <cuda_runtime.h>
struct St { int iter; int mode; int log[64]; };
__global__ void init_k(St* s, cudaGraphConditionalHandle h0, cudaGraphConditionalHandle h1) {
    cudaGraphSetConditional(h0, 0); cudaGraphSetConditional(h1, 1);
}
__global__ void work_k(St* s, int id, cudaGraphConditionalHandle hw, cudaGraphConditionalHandle h0,
                       cudaGraphConditionalHandle h1) {
    if (threadIdx.x || blockIdx.x) return;
    s->log[s->iter] = id;
    s->iter++;
    int next = s->iter >= 3 ? 0 : 1; // modes 1,1,1 then 0
    cudaGraphSetConditional(h0, next == 0); cudaGraphSetConditional(h1, next == 1);
    cudaGraphSetConditional(hw, s->iter < 6);
}
#define CK(x) do { cudaError_t e = (x); if (e) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)
int main() {
    St* s; CK(cudaMallocManaged(&s, sizeof(St)));
    cudaGraph_t g; CK(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle hw; CK(cudaGraphConditionalHandleCreate(&hw, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams cp = {}; cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = hw;
    cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
    // init node before the loop sets the mode handles (created on the body graph)
    cudaGraphNode_t wnode; CK(cudaGraphAddNode(&wnode, g, nullptr, 0, &cp));
    cudaGraph_t body = cp.conditional.phGraph_out[0];
    cudaGraphConditionalHandle h0, h1;
    CK(cudaGraphConditionalHandleCreate(&h0, body, 0, 0));
    CK(cudaGraphConditionalHandleCreate(&h1, body, 1, cudaGraphCondAssignDefault));
    cudaGraphNode_t prev = nullptr;
    cudaGraphConditionalHandle hs[2] = {h0, h1};
    for (int m = 0; m < 2; ++m) {
        cudaGraphNodeParams ip = {}; ip.type = cudaGraphNodeTypeConditional; ip.conditional.handle = hs[m];
        ip.conditional.type = cudaGraphCondTypeIf; ip.conditional.size = 1;
        cudaGraphNode_t in; CK(cudaGraphAddNode(&in, body, prev ? &prev : nullptr, prev ? 1 : 0, &ip));
        cudaGraph_t ib = ip.conditional.phGraph_out[0];
        cudaKernelNodeParams kp = {}; kp.func = (void*)work_k; kp.gridDim = dim3(1); kp.blockDim = dim3(32);
        int id = m; void* args[] = {&s, &id, &hw, &h0, &h1}; kp.kernelParams = args;
        cudaGraphNode_t kn; CK(cudaGraphAddKernelNode(&kn, ib, nullptr, 0, &kp));
        prev = in;
    }
    cudaGraphExec_t ex; CK(cudaGraphInstantiate(&ex, g, 0));
    for (int run = 0; run < 2; ++run) {
        s->iter = 0; for (int i = 0; i < 64; ++i) s->log[i] = -1;
        CK(cudaGraphLaunch(ex, 0)); CK(cudaDeviceSynchronize());
        printf("run %d iters %d:", run, s->iter); for (int i = 0; i < 8; ++i) printf(" %d", s->log[i]); printf("\n");
    }
    return 0;
}
