// ubench_ex2.cu -- MUFU.EX2 throughput per SM on this part (one CTA per SM,
// W warps, each lane running 8 independent ex2 chains), bare and inside the
// FlashMatch exp-pass instruction mix (FFMA -> EX2 -> FADD sum + F2FP pack).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_ex2 tools/ubench_ex2.cu
#include <cstdio>
#include <cuda_fp16.h>

__device__ __forceinline__ float ex2(float x) {
    float y;
    asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

template <int MIX>
__global__ void k(int iters, float* out, unsigned long long* cyc) {
    float v[8];
    for (int i = 0; i < 8; ++i) v[i] = 0.001f * (threadIdx.x + i);
    float acc = 0.f;
    unsigned pk = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MIX) {
                const float p = ex2(fmaf(v[i], 1.4427f, -0.5f));
                acc += p;
                v[i] = p * 0.25f;
            } else {
                v[i] = ex2(v[i]);
            }
        }
        if (MIX == 1) {
            __half2 h = __floats2half2_rn(v[0], v[1]);
            pk ^= *reinterpret_cast<unsigned*>(&h);
        }
        if (MIX == 2) {  // one binary16 pack per two exponentials, as the FlashMatch exp pass
#pragma unroll
            for (int i = 0; i < 8; i += 2) {
                __half2 h = __floats2half2_rn(v[i], v[i + 1]);
                pk ^= *reinterpret_cast<unsigned*>(&h);
            }
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    float s = acc + pk;
    for (int i = 0; i < 8; ++i) s += v[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    unsigned long long* cyc;
    cudaMalloc(&out, sms * 1024 * 4);
    cudaMalloc(&cyc, sms * 8);
    const int iters = 4096;
    for (int mix = 0; mix < 3; ++mix)
        for (int w : {4, 8, 16, 32}) {
            if (mix == 2) k<2><<<sms, w * 32>>>(iters, out, cyc);
            else if (mix == 1) k<1><<<sms, w * 32>>>(iters, out, cyc);
            else k<0><<<sms, w * 32>>>(iters, out, cyc);
            cudaDeviceSynchronize();
            unsigned long long c;
            cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
            printf("mix %d warps/SM %2d: %.2f ex2/clk/SM\n", mix, w, (double)w * 32 * 8 * iters / c);
        }
    return 0;
}
