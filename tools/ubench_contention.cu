// ubench_contention.cu -- does tcgen05.mma (accumulating into TMEM) slow down
// concurrent tcgen05.ld traffic from other TMEM columns, and vice versa?
// The K3 round-trip analysis depends on it (K3 "What limits it").
//
// One CTA per SM, 512 TMEM columns.  Warp 0 issues M128 N<n> K16 MMAs
// (kind::f16, SS or A-from-TMEM) into columns [0, 256); warps 4..19 stream
// tcgen05.ld.32x32b.x64 from columns [256, 512).  mode 1 = MMA only, 2 = ld
// only, 3 = both.  Prints cycles per role and the implied rates.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_10017_b200/csrc
//          -o tools/ubench_contention tools/ubench_contention.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#include "tc_ptx.cuh"

using namespace fnl;

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(512u >> 4) << 32) |
           (1ull << 46);
}
// K-major operand descriptor of K step ks (16 elements) in layout `lay`:
// 0 = no swizzle (8x16 B core matrices, LBO 128 B, SBO 512 B, as K3 uses),
// 1 = SWIZZLE_64B (64 B rows = the whole K=32, SBO 512 B, K step = +32 B),
// 2 = SWIZZLE_32B (32 B rows per K=16 step, SBO 256 B, K step = next 4 KB block)
__device__ __forceinline__ uint64_t desc_k(uint32_t base, uint32_t ks, int lay) {
    if (lay == 0) return desc(base + ks * 256u);
    if (lay == 1)
        return (uint64_t)(((base + ks * 32u) >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(512u >> 4) << 32) |
               (1ull << 46) | (4ull << 61);
    return (uint64_t)(((base + ks * 4096u) >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(256u >> 4) << 32) |
           (1ull << 46) | (6ull << 61);
}

constexpr int kThreads = 20 * 32;

__global__ void __launch_bounds__(kThreads, 1)
contention(int mode, int n, int ts, int lay, int mma_iters, int ld_iters, unsigned long long* out, uint32_t* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (uint32_t i = threadIdx.x; i < (8192 + 16384) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u * ((i & 7) == 0);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t a_addr = (smem_addr(smem) + 1023u) & ~1023u, b_addr = a_addr + 8192;
    const uint32_t idesc = (1u << 4) | (((uint32_t)n >> 3) << 17) | ((128u >> 4) << 24);
    // A operand in TMEM (ts): columns 496..511 hold the query tile (ld readers only read them)
    if (ts && threadIdx.x == 0) {
        for (uint32_t ks = 0; ks < 2; ++ks) tc_cp_128x256b(tmem + 496u + ks * 8u, desc(a_addr + ks * 256u));
        tc_commit(&bar);
        mbar_wait(&bar, 0);
    }
    __syncthreads();
    unsigned long long t0 = clock64(), t1 = t0;
    uint32_t acc = 0;
    if (warp == 0 && (mode & 1)) {
        if (elect_one()) {
            const uint32_t span = 256u;
            uint32_t col = 0;
            for (int i = 0; i < mma_iters; ++i) {
                const uint32_t d = tmem + col;
                for (uint32_t ks = 0; ks < 2; ++ks) {
                    if (ts) tc_mma_f16_ts(d, tmem + 496u + ks * 8u, desc_k(b_addr, ks, lay), idesc, ks);
                    else tc_mma_f16(d, desc_k(a_addr, ks, lay), desc_k(b_addr, ks, lay), idesc, ks);
                }
                col += (uint32_t)n;
                if (col + (uint32_t)n > span) col = 0;
            }
            tc_commit(&bar);
            mbar_wait(&bar, ts ? 1 : 0);
            t1 = clock64();
        }
        __syncwarp();
    } else if (warp >= 4 && (mode & 2)) {
        const uint32_t g = (warp - 4) >> 2, quad = warp & 3u;
        const uint32_t base = tmem + ((quad * 32u) << 16) + 256u + g * 64u;
#pragma unroll 1
        for (int i = 0; i < ld_iters; ++i) {
            Frag f, h;
            frag_ld64(base, f, h);
            frag_wait2(f, h);
#pragma unroll
            for (int j = 0; j < 32; ++j) acc ^= f.r[j] + h.r[j];
        }
        t1 = clock64();
    }
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (lane == 0) out[blockIdx.x * 20 + warp] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

int main(int argc, char** argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = 8192 + 16384 + 2048;
    cudaFuncSetAttribute(contention, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* out;
    uint32_t* sink;
    cudaMalloc(&out, sms * 20 * 8);
    cudaMalloc(&sink, sms * kThreads * 4);
    const int mma_iters = argc > 1 ? atoi(argv[1]) : 20000;
    const int ld_iters = argc > 2 ? atoi(argv[2]) : 4000;
    printf("{\"sms\": %d, \"mma_iters\": %d, \"ld_iters\": %d, \"runs\": [\n", sms, mma_iters, ld_iters);
    bool first = true;
    for (int lay = 0; lay < 3; ++lay)
    for (int ts = 0; ts < 2; ++ts)
        for (int n : {64, 128, 256})
            for (int mode = 1; mode <= 3; ++mode) {
                if (mode != 1 && (lay != 0 || n == 64)) continue;
                contention<<<sms, kThreads, smem>>>(mode, n, ts, lay, mma_iters, ld_iters, out, sink);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("error %s\n", cudaGetErrorString(e));
                    return 1;
                }
                unsigned long long h[20];
                cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);  // CTA 0
                unsigned long long ldmax = 0;
                for (int w = 4; w < 20; ++w) ldmax = h[w] > ldmax ? h[w] : ldmax;
                const double mma_cyc = (mode & 1) ? (double)h[0] : 0, ld_cyc = (mode & 2) ? (double)ldmax : 0;
                // MMA: 128 x n x 32 MACs per iteration; ld: 16 warps x 32 lanes x 64 x 4 B per iteration
                printf("%s{\"layout\": %d, \"ts\": %d, \"n\": %d, \"mode\": %d, \"mma_cycles\": %.0f, \"mma_mac_per_clk\": %.1f, "
                       "\"ld_cycles\": %.0f, \"ld_bytes_per_clk\": %.1f}\n",
                       first ? "" : ",", lay, ts, n, mode, mma_cyc,
                       mma_cyc ? 128.0 * n * 32 * mma_iters / mma_cyc : 0.0, ld_cyc,
                       ld_cyc ? 16.0 * 32 * 64 * 4 * ld_iters / ld_cyc : 0.0);
                first = false;
            }
    printf("]}\n");
    return 0;
}
