// ubench_pair.cu -- does a CTA-pair MMA (tcgen05.mma.cta_group::2, M=256 over
// two SMs, each SM staging half of B) keep its rate while the epilogue warps of
// both SMs stream tcgen05.ld from other TMEM columns?  K3's accumulator chains
// use M128 N128 K16 MMAs, which tools/ubench_contention.cu measured at 93% of
// the tensor-pipe rate alone but 58% under concurrent TMEM loads (N=256: 100%
// either way); this decides whether a cta_group::2 K3 can escape that.
//
// Grid = #SMs CTAs in clusters of 2 (cg=2) or plain CTAs (cg=1).  Warp 0 of the
// leader (cg=2) or of every CTA (cg=1) issues M(128*cg) N<n> K16 kind::f16 MMAs
// from shared memory into TMEM columns [0, 256); warps 4..19 of every CTA
// stream tcgen05.ld.32x32b.x64 from columns [256, 512).  mode 1 = MMA only,
// 2 = ld only, 3 = both.  MAC rates are per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2503_10017_b200/csrc
//          -o tools/ubench_pair tools/ubench_pair.cu
#include <cstdio>
#include <cstdint>
#include <cstdlib>

#include "tc_ptx.cuh"

using namespace fnl;

__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(512u >> 4) << 32) |
           (1ull << 46);
}

constexpr int kThreads = 20 * 32;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int CG>
__device__ void body(int mode, int n, int mma_iters, int ld_iters, unsigned long long* out, uint32_t* sink) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = CG == 2 ? cluster_rank() : 0;
    for (uint32_t i = threadIdx.x; i < (8192 + 16384) / 4; i += blockDim.x)
        reinterpret_cast<uint32_t*>(smem)[i] = 0x3c003c00u * ((i & 7) == 0);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        if (CG == 2) {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&slot)),
                         "r"(512));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
        } else {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&slot)),
                         "r"(512));
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
        }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t a_addr = (smem_addr(smem) + 1023u) & ~1023u, b_addr = a_addr + 8192;
    const uint32_t idesc = (1u << 4) | (((uint32_t)n >> 3) << 17) | (((128u * CG) >> 4) << 24);
    unsigned long long t0 = clock64(), t1 = t0;
    uint32_t acc = 0;
    if (warp == 0 && (mode & 1) && rank == 0) {
        if (elect_one()) {
            uint32_t col = 0;
            for (int i = 0; i < mma_iters; ++i) {
                const uint32_t d = tmem + col;
                for (uint32_t ks = 0; ks < 2; ++ks) {
                    const uint64_t ad = desc(a_addr + ks * 256u), bd = desc(b_addr + ks * 256u);
                    if (CG == 2)
                        asm volatile(
                            "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, "
                            "%3, p; }" ::"r"(d),
                            "l"(ad), "l"(bd), "r"(idesc), "r"(ks));
                    else
                        tc_mma_f16(d, ad, bd, idesc, ks);
                }
                col += (uint32_t)n;
                if (col + (uint32_t)n > 256u) col = 0;
            }
            if (CG == 2)
                asm volatile(
                    "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], "
                    "%1;" ::"r"(smem_addr(&bar)),
                    "h"((uint16_t)3)
                    : "memory");
            else
                tc_commit(&bar);
            mbar_wait(&bar, 0);
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
    if (CG == 2 && (mode & 1) && rank == 1 && threadIdx.x == 0) mbar_wait(&bar, 0);  // peer's commit arrival
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (lane == 0) out[blockIdx.x * 20 + warp] = t1 - t0;
    tc_fence_before();
    if (CG == 2) cluster_sync_all(); else __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        if (CG == 2)
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
        else
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

__global__ void __launch_bounds__(kThreads, 1) k_cg1(int mode, int n, int mi, int li, unsigned long long* out,
                                                      uint32_t* sink) {
    body<1>(mode, n, mi, li, out, sink);
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads, 1)
    k_cg2(int mode, int n, int mi, int li, unsigned long long* out, uint32_t* sink) {
    body<2>(mode, n, mi, li, out, sink);
}

int main(int argc, char** argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    sms &= ~1;
    const int smem = 8192 + 16384 + 2048;
    cudaFuncSetAttribute(k_cg1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k_cg2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    unsigned long long* out;
    uint32_t* sink;
    cudaMalloc(&out, sms * 20 * 8);
    cudaMalloc(&sink, sms * kThreads * 4);
    const int mma_iters = argc > 1 ? atoi(argv[1]) : 20000;
    const int ld_iters = argc > 2 ? atoi(argv[2]) : 20000;
    printf("{\"sms\": %d, \"mma_iters\": %d, \"ld_iters\": %d, \"runs\": [\n", sms, mma_iters, ld_iters);
    bool first = true;
    for (int cg = 1; cg <= 2; ++cg)
        for (int n : {64, 128, 256})
            for (int mode = 1; mode <= 3; ++mode) {
                if (mode == 2 && n != 128) continue;
                if (cg == 1) k_cg1<<<sms, kThreads, smem>>>(mode, n, mma_iters, ld_iters, out, sink);
                else k_cg2<<<sms, kThreads, smem>>>(mode, n, mma_iters, ld_iters, out, sink);
                cudaError_t e = cudaDeviceSynchronize();
                if (e != cudaSuccess) {
                    printf("error cg %d n %d mode %d: %s\n", cg, n, mode, cudaGetErrorString(e));
                    return 1;
                }
                unsigned long long h[40];
                cudaMemcpy(h, out, sizeof(h), cudaMemcpyDeviceToHost);  // CTAs 0 and 1
                unsigned long long ldmax = 0;
                for (int c = 0; c < 2; ++c)
                    for (int w = 4; w < 20; ++w) ldmax = h[c * 20 + w] > ldmax ? h[c * 20 + w] : ldmax;
                const double mma_cyc = (mode & 1) ? (double)h[0] : 0, ld_cyc = (mode & 2) ? (double)ldmax : 0;
                // per SM: 128 rows x n x 32 MACs per iteration (cg=2: 256 rows over 2 SMs)
                printf("%s{\"cta_group\": %d, \"n\": %d, \"mode\": %d, \"mma_cycles\": %.0f, \"mma_mac_per_clk_per_sm\": %.1f, "
                       "\"ld_cycles\": %.0f, \"ld_bytes_per_clk\": %.1f}\n",
                       first ? "" : ",", cg, n, mode, mma_cyc, mma_cyc ? 128.0 * n * 32 * mma_iters / mma_cyc : 0.0,
                       ld_cyc, ld_cyc ? 16.0 * 32 * 64 * 4 * ld_iters / ld_cyc : 0.0);
                first = false;
            }
    printf("]}\n");
    return 0;
}
