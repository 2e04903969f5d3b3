// ubench_mufu.cu -- MUFU ex2 / FFMA throughput per SM on this B200.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mufu tools/ubench_mufu.cu
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
__device__ __forceinline__ uint32_t ex2h2(uint32_t x) { uint32_t y; asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(x)); return y; }
template <int MODE>
__global__ void bench(float* out, int iters, unsigned long long* cyc) {
    float v[8];
    for (int i = 0; i < 8; ++i) v[i] = -0.001f * (threadIdx.x + i);
    uint32_t h[8];
    for (int i = 0; i < 8; ++i) h[i] = 0x3c00bc00u + i;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            if (MODE == 0) v[i] = ex2(v[i]) - 1.0f;          // MUFU + FADD
            else if (MODE == 1) v[i] = fmaf(v[i], 0.999f, 0.001f);  // FFMA
            else h[i] = ex2h2(h[i]);                           // MUFU f16x2
        }
    }
    __syncthreads();
    unsigned long long t1 = clock64();
    float s = 0; for (int i = 0; i < 8; ++i) s += v[i] + (float)(h[i] & 1);
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
template <int MODE> void run(const char* name, int threads) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out; unsigned long long* cyc; cudaMalloc(&out, sms * threads * 4); cudaMalloc(&cyc, sms * 8);
    const int iters = 4096;
    bench<MODE><<<sms, threads>>>(out, iters, cyc); cudaDeviceSynchronize();
    bench<MODE><<<sms, threads>>>(out, iters, cyc); cudaDeviceSynchronize();
    unsigned long long h[1024]; cudaMemcpy(h, cyc, sms * 8, cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < sms; ++i) c += h[i]; c /= sms;
    printf("%-12s threads=%4d: %.2f ops/clk/SM\n", name, threads, (double)threads * iters * 8 / c);
}
int main() {
    for (int t : {128, 256, 512, 1024}) { run<0>("ex2.f32", t); run<1>("ffma", t); run<2>("ex2.f16x2", t); }
    return 0;
}
