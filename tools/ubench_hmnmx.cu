// ubench_hmnmx.cu -- which pipe does the packed binary16 max (max.f16x2 ->
// HMNMX2) issue on, and at what rate, next to the fp32 3-input max (FMNMX3,
// ALU pipe) that K3's epilogue tree is built from?  One CTA per SM, W warps,
// each lane running 8 independent dependency chains of the op under test;
// mode 2 interleaves both ops (if they use different pipes the mix runs at
// the slower of the two alone, not at their sum).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_hmnmx tools/ubench_hmnmx.cu
#include <cstdio>
#include <cuda_fp16.h>

__device__ __forceinline__ float fmax3(float a, float b, float c) {
    float d;
    asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ unsigned hmax2(unsigned a, unsigned b) {
    unsigned d;
    asm volatile("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}

template <int MODE>
__global__ void k(int iters, unsigned* out, unsigned long long* cyc) {
    float f[8];
    unsigned h[8];
    for (int i = 0; i < 8; ++i) {
        f[i] = 0.001f * (threadIdx.x + i);
        h[i] = 0x3c003c00u + threadIdx.x + i;
    }
    const float fx = 0.5f, fy = 0.25f;
    const unsigned hx = 0x38003800u, hy = 0x34003400u;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0 || MODE == 2) f[i] = fmax3(f[i], fx, fy);
            if (MODE == 1 || MODE == 2) h[i] = hmax2(h[i], hx ^ (unsigned)i);
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    unsigned s = 0;
    for (int i = 0; i < 8; ++i) s += __float_as_uint(f[i]) + h[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned* out;
    unsigned long long* cyc;
    cudaMalloc(&out, sms * 1024 * 4);
    cudaMalloc(&cyc, sms * 8);
    const int iters = 4096;
    const char* names[3] = {"FMNMX3 (max.f32 3-input)", "HMNMX2 (max.f16x2)", "both interleaved"};
    for (int mode = 0; mode < 3; ++mode)
        for (int w : {8, 16, 32}) {
            if (mode == 0) k<0><<<sms, w * 32>>>(iters, out, cyc);
            if (mode == 1) k<1><<<sms, w * 32>>>(iters, out, cyc);
            if (mode == 2) k<2><<<sms, w * 32>>>(iters, out, cyc);
            cudaDeviceSynchronize();
            unsigned long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            const double ops = (double)w * 32 * 8 * iters * (mode == 2 ? 2 : 1);
            printf("%-26s warps/SM %2d: %.1f thread-ops/clk/SM (%.0f cycles)\n", names[mode], w, ops / c, (double)c);
        }
    return 0;
}
