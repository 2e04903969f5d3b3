// Repro: compute-sanitizer --tool synccheck (CUDA 12.9) reports "Barrier error:
// divergent threads" and fails kernels launched inside a conditional WHILE
// graph body, even this trivially correct one; a plain run and memcheck are
// clean.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/ubench_cond_sync tools/ubench_cond_sync.cu
#include <cstdio>
#include <cuda_runtime.h>
__global__ void ka(unsigned* x, unsigned n) {  // 256 threads, early return, no barrier
    unsigned i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    atomicMin(&x[i % 64], i);
}
__global__ void __launch_bounds__(1024) kb(unsigned* x, unsigned* out) {  // 1024 threads, barriers
    __shared__ unsigned s[32];
    unsigned v = x[threadIdx.x % 64];
    if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
    __syncthreads();
    if (threadIdx.x == 0) { unsigned t = 0; for (int i = 0; i < 32; ++i) t += s[i]; out[blockIdx.x] = t; }
}
__global__ void kc(cudaGraphConditionalHandle h, unsigned* it) {
    unsigned t = ++*it;
    cudaGraphSetConditional(h, t < 3 ? 1u : 0u);
}
int main() {
    unsigned *x, *out, *it;
    cudaMalloc(&x, 4096); cudaMalloc(&out, 4096); cudaMalloc(&it, 4);
    cudaMemset(x, 0xFF, 4096); cudaMemset(it, 0, 4);
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h; cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams cp{}; cp.type = cudaGraphNodeTypeConditional; cp.conditional.handle = h;
    cp.conditional.type = cudaGraphCondTypeWhile; cp.conditional.size = 1;
    cudaGraphNode_t w; cudaGraphAddNode(&w, g, nullptr, 0, &cp);
    cudaStreamBeginCaptureToGraph(s, cp.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal);
    ka<<<2, 256, 0, s>>>(x, 300);
    kb<<<2, 1024, 0, s>>>(x, out);
    kc<<<1, 1, 0, s>>>(h, it);
    cudaGraph_t cap; cudaStreamEndCapture(s, &cap);
    cudaGraphExec_t e; cudaGraphInstantiate(&e, g, 0);
    cudaGraphLaunch(e, s);
    cudaError_t err = cudaStreamSynchronize(s);
    unsigned o; cudaMemcpy(&o, out, 4, cudaMemcpyDeviceToHost);
    printf("graph while: %s out %u\n", cudaGetErrorString(err), o);
    kb<<<2, 1024, 0, s>>>(x, out);  // the same kernel launched directly
    err = cudaStreamSynchronize(s);
    printf("direct: %s\n", cudaGetErrorString(err));
    return 0;
}
