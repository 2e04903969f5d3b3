// ubench_f16acc.cu -- where does tcgen05.mma kind::f16 put a binary16
// accumulator (D format f16) in TMEM?  One M128 N128 K16 MMA of A = row index
// pattern, B = identity-like pattern; prints the raw 32-bit TMEM words of lane
// 0 / lane 5 for columns 0..7 and 64..71, with D in f32 and in f16.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_10017_b200/csrc
//          -o tools/ubench_f16acc tools/ubench_f16acc.cu
#include <cstdio>
#include <cstdint>
#include <cuda_fp16.h>
#include "tc_ptx.cuh"
using namespace fnl;

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {  // K-major, no swizzle, LBO 128, SBO 256 (K=16 rows of 32 B)
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(256u >> 4) << 32) |
           (1ull << 46);
}

__global__ void k(int f16d, uint32_t* out) {
    __shared__ __align__(1024) __half sA[128 * 16];
    __shared__ __align__(1024) __half sB[128 * 16];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // canonical no-swizzle K-major: core matrix (8 rows x 16 B): offset = (row/8)*256 + (k/8)*128 + (row%8)*16 + (k%8)*2
    for (uint32_t i = tid; i < 128 * 16; i += blockDim.x) {
        const uint32_t row = i / 16, kk = i % 16;
        const uint32_t off = (row / 8) * 128 + (kk / 8) * 64 + (row % 8) * 8 + (kk % 8);  // in halves
        sA[off] = __float2half(kk == 0 ? (float)(row + 1) : 0.0f);      // A[row][0] = row+1
        sB[off] = __float2half(kk == 0 ? (float)(row % 64 + 1) * 0.001f : 0.0f);  // B[n][0]
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) { mbar_init(&bar, 1); asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&slot)), "r"(256));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    if (tid == 0) {
        const uint32_t idesc = ((f16d ? 0u : 1u) << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
        tc_mma_f16(tmem, desc(smem_addr(sA)), desc(smem_addr(sB)), idesc, 0u);
        tc_commit(&bar);
    }
    mbar_wait(&bar, 0);
    tc_fence_after();
    if (warp == 0) {
        Frag f, g;
        frag_ld64(tmem, f, g);
        frag_wait2(f, g);
        if (lane == 0 || lane == 5)
            for (int c = 0; c < 8; ++c) {
                out[(lane ? 16 : 0) + c] = f.r[c];
                out[(lane ? 16 : 0) + 8 + c] = g.r[c];  // columns 32..39
            }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) { tc_fence_after(); asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256)); }
}

int main() {
    uint32_t* d; cudaMalloc(&d, 4 * 32);
    for (int f16d = 0; f16d < 2; ++f16d) {
        cudaMemset(d, 0, 128);
        k<<<1, 128>>>(f16d, d);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("err %s\n", cudaGetErrorString(e)); return 1; }
        uint32_t h[32]; cudaMemcpy(h, d, 128, cudaMemcpyDeviceToHost);
        printf("D %s:\n", f16d ? "f16" : "f32");
        for (int ln = 0; ln < 2; ++ln) {
            printf(" lane %d cols 0-7  :", ln ? 5 : 0);
            for (int c = 0; c < 8; ++c) {
                uint32_t w = h[ln * 16 + c];
                if (f16d) printf(" [%08x %.4f|%.4f]", w, __half2float(__ushort_as_half((unsigned short)(w & 0xffff))), __half2float(__ushort_as_half((unsigned short)(w >> 16))));
                else printf(" %.4f", *(float*)&w);
            }
            printf("\n lane %d cols 32-39:", ln ? 5 : 0);
            for (int c = 0; c < 8; ++c) {
                uint32_t w = h[ln * 16 + 8 + c];
                if (f16d) printf(" [%08x %.4f|%.4f]", w, __half2float(__ushort_as_half((unsigned short)(w & 0xffff))), __half2float(__ushort_as_half((unsigned short)(w >> 16))));
                else printf(" %.4f", *(float*)&w);
            }
            printf("\n");
        }
    }
    return 0;
}
