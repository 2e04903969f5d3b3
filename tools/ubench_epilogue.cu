// ubench_epilogue.cu -- measures the ceilings of the K3 epilogue on this B200:
//   (1) tcgen05.ld (TMEM -> registers) bandwidth per SM for 4/8/16 warps and
//       .x32/.x64 shapes; (2) FMNMX3 and HMNMX2 issue throughput (pipe check).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench tools/ubench_epilogue.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int X>
__device__ __forceinline__ uint32_t ld_tmem(uint32_t taddr);

template <>
__device__ __forceinline__ uint32_t ld_tmem<32>(uint32_t taddr) {
    uint32_t r[32];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]),"=r"(r[1]),"=r"(r[2]),"=r"(r[3]),"=r"(r[4]),"=r"(r[5]),"=r"(r[6]),"=r"(r[7]),"=r"(r[8]),"=r"(r[9]),"=r"(r[10]),"=r"(r[11]),"=r"(r[12]),"=r"(r[13]),"=r"(r[14]),"=r"(r[15]),"=r"(r[16]),"=r"(r[17]),"=r"(r[18]),"=r"(r[19]),"=r"(r[20]),"=r"(r[21]),"=r"(r[22]),"=r"(r[23]),"=r"(r[24]),"=r"(r[25]),"=r"(r[26]),"=r"(r[27]),"=r"(r[28]),"=r"(r[29]),"=r"(r[30]),"=r"(r[31]) : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]),"+r"(r[31]) :: "memory");
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 32; ++i) x ^= r[i];
    return x;
}

template <int LOADS_IN_FLIGHT>
__global__ void tmem_bw(int iters, unsigned long long* cycles, uint32_t* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_addr(&slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = slot + (((warp & 3) * 32) << 16);
    uint32_t acc = 0;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        uint32_t col = ((i * LOADS_IN_FLIGHT + warp / 4) * 32) & 511;
        acc ^= ld_tmem<32>(tm + col);
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(slot), "r"(512));
}

__global__ void fmnmx3_tp(int iters, unsigned long long* cycles, float* sink) {
    float a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 0.001f + i;
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float d;
            asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a[i]), "f"(a[(i + 1) & 7]), "f"(a[(i + 3) & 7]));
            a[i] = d;
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void hmnmx2_tp(int iters, unsigned long long* cycles, float* sink) {
    __half2 a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __floats2half2_rn(threadIdx.x * 0.001f + i, i);
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = __hmax2(a[i], a[(i + 3) & 7]);
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    float s = 0; for (int i = 0; i < 8; ++i) s += __low2float(a[i]);
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// FMNMX3 and FFMA interleaved: if they share a pipe the time adds up
__global__ void mix_tp(int iters, unsigned long long* cycles, float* sink) {
    float a[8], b[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 0.001f + i; b[i] = i * 0.5f; }
    __syncthreads();
    const unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            float d;
            asm volatile("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a[i]), "f"(a[(i + 1) & 7]), "f"(a[(i + 3) & 7]));
            a[i] = d;
            b[i] = __fmaf_rn(b[i], 0.999f, 0.001f);
        }
    }
    __syncthreads();
    const unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + b[i];
    sink[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static double avg(unsigned long long* d, int n) {
    unsigned long long h[1024]; cudaMemcpy(h, d, n * 8, cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < n; ++i) s += h[i]; return s / n;
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* cyc; cudaMalloc(&cyc, 1024 * 8);
    uint32_t* sink; cudaMalloc(&sink, 1 << 24);
    const int iters = 4096;
    for (int warps : {4, 8, 16}) {
        tmem_bw<1><<<sms, warps * 32>>>(iters, cyc, sink);
        cudaDeviceSynchronize();
        double c = avg(cyc, sms);
        double bytes = (double)warps * iters * 32 * 32 * 4;
        printf("tcgen05.ld.32x32b.x32 + wait, %2d warps/SM: %.1f B/clk/SM (%.1f cyc per warp-load)\n", warps, bytes / c, c / iters);
    }
    for (int warps : {4, 8, 16, 32}) {
        fmnmx3_tp<<<sms, warps * 32>>>(iters, cyc, (float*)sink);
        cudaDeviceSynchronize();
        double c = avg(cyc, sms);
        printf("FMNMX3 %2d warps/SM: %.1f thread-ops/clk/SM\n", warps, (double)warps * 32 * iters * 8 / c);
        hmnmx2_tp<<<sms, warps * 32>>>(iters, cyc, (float*)sink);
        cudaDeviceSynchronize();
        c = avg(cyc, sms);
        printf("HMNMX2 %2d warps/SM: %.1f thread-ops/clk/SM\n", warps, (double)warps * 32 * iters * 8 / c);
        mix_tp<<<sms, warps * 32>>>(iters, cyc, (float*)sink);
        cudaDeviceSynchronize();
        c = avg(cyc, sms);
        printf("FMNMX3+FFMA pairs %2d warps/SM: %.1f pairs/clk/SM\n", warps, (double)warps * 32 * iters * 8 / c);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
