// ubench_mma.cu -- cycles per tcgen05.mma.cta_group::1.kind::f16 on this B200
// for different issue styles (single diverged lane vs warp-uniform loop with
// elect.sync), N in {64,128,256}, SS vs TS operands.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_mma tools/ubench_mma.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(512u >> 4) << 32) | (1ull << 46);
}
__device__ __forceinline__ bool elect_one() {
    uint32_t pred = 0;
    asm volatile("{ .reg .pred p; elect.sync _|p, 0xffffffff; selp.u32 %0, 1, 0, p; }" : "=r"(pred));
    return pred != 0;
}
__device__ __forceinline__ void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }"
                 :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p; }"
                 :: "r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc));
}

// style 0: lane 0 only; style 1: whole warp 0, elect.sync per MMA; style 2: whole warp, elect once per 8 MMAs
template <int STYLE, int N, bool TS>
__global__ void mma_bench(int n_mma, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t slot;
    __shared__ uint64_t bar;
    const int warp = threadIdx.x / 32;
    for (int i = threadIdx.x; i < 65536 / 4; i += blockDim.x) ((uint32_t*)smem)[i] = 0;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_addr(&bar)), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" :: "r"(smem_addr(&slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = slot;
    const uint32_t a = smem_addr(smem), b = a + 16384;
    constexpr uint32_t idesc = (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((128u >> 4) << 24);
    const uint64_t ad = desc(a), bd = desc(b);
    unsigned long long t0 = clock64();
    if (STYLE == 0) {
        if (threadIdx.x == 0) {
            for (int i = 0; i < n_mma; i += 4) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t d = tm + (uint32_t)(j & 1) * N;
                    if (TS) mma_ts(d, tm + 448u, bd, idesc, j >> 1); else mma_ss(d, ad, bd, idesc, j >> 1);
                }
            }
        }
    } else if (STYLE >= 5) {
        // STYLE 5: style 4 + two tcgen05.commit per group; 6: + fence::after_thread_sync too;
        // 7: like 6 but commits/fence issued only by the elected lane inside the branch
        __shared__ uint64_t bars2[2];
        if (threadIdx.x == 0) { for (int q = 0; q < 2; ++q) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_addr(&bars2[q])), "r"(1 << 20)); }
        __syncwarp();
        if (warp == 0) {
            for (int i = 0; i < n_mma; i += 4) {
                const uint32_t k = (uint32_t)i >> 2;
                const uint32_t acc = k % 3u, s = k % 16u;
                const uint64_t bdk = desc(b + s * 1024u);
                if (STYLE >= 8) {  // 8: one, 9: two try_waits on an already-completed phase
                    for (int w = 0; w < (STYLE == 8 ? 1 : 2); ++w) {
                        uint32_t done = 0;
                        do asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(smem_addr(&bar)), "r"(1u)); while (!done);
                    }
                }
                if (STYLE >= 6) asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
                if (elect_one()) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t d = tm + acc * 128u + (uint32_t)(j & 1) * 64u;
                        if (TS) mma_ts(d, tm + 448u + (j >> 1) * 8u, bdk + (uint64_t)((j >> 1) * 16), idesc, j >> 1);
                        else mma_ss(d, ad, bdk, idesc, j >> 1);
                    }
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_addr(&bars2[0])));
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_addr(&bars2[1])));
                }
                __syncwarp();
            }
        }
    } else if (STYLE == 3 || STYLE == 4) {
        // runtime-computed accumulator slot (k % 3) and smem stage (k % 16) per MMA group,
        // as the production loop does; STYLE 3 lane 0 only, STYLE 4 warp-uniform + elect
        if ((STYLE == 3 && threadIdx.x == 0) || (STYLE == 4 && warp == 0)) {
            for (int i = 0; i < n_mma; i += 4) {
                const uint32_t k = (uint32_t)i >> 2;
                const uint32_t acc = k % 3u, s = k % 16u;
                const uint64_t bdk = desc(b + s * 1024u);
                const bool go = STYLE == 3 ? true : elect_one();
                if (go) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t d = tm + acc * 128u + (uint32_t)(j & 1) * 64u;
                        if (TS) mma_ts(d, tm + 448u + (j >> 1) * 8u, bdk + (uint64_t)((j >> 1) * 16), idesc, j >> 1);
                        else mma_ss(d, ad, bdk, idesc, j >> 1);
                    }
                }
                if (STYLE == 4) __syncwarp();
            }
        }
    } else if (warp == 0) {
        for (int i = 0; i < n_mma; i += 4) {
            if (STYLE == 1) {
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const uint32_t d = tm + (uint32_t)(j & 1) * N;
                    if (elect_one()) { if (TS) mma_ts(d, tm + 448u, bd, idesc, j >> 1); else mma_ss(d, ad, bd, idesc, j >> 1); }
                }
            } else {
                if (elect_one()) {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t d = tm + (uint32_t)(j & 1) * N;
                        if (TS) mma_ts(d, tm + 448u, bd, idesc, j >> 1); else mma_ss(d, ad, bd, idesc, j >> 1);
                    }
                }
                __syncwarp();
            }
        }
    }
    if (threadIdx.x == 0) {
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" :: "r"(smem_addr(&bar)));
        uint32_t done = 0;
        while (!done) asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }" : "=r"(done) : "r"(smem_addr(&bar)), "r"(0));
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tm), "r"(512));
}

template <int STYLE, int N, bool TS>
void run(int sms, unsigned long long* d) {
    cudaFuncSetAttribute(mma_bench<STYLE, N, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int n = 4096;
    mma_bench<STYLE, N, TS><<<sms, 128, 100 * 1024>>>(n, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[1024]; cudaMemcpy(h, d, sms * 8, cudaMemcpyDeviceToHost);
    double s = 0; for (int i = 0; i < sms; ++i) s += h[i]; s /= sms;
    const double cyc = s / n, macs = 128.0 * N * 16;
    printf("style=%d N=%3d %s: %6.1f cyc/mma  %6.0f MAC/clk/SM  (%s)\n", STYLE, N, TS ? "TS" : "SS", cyc, macs / cyc, cudaGetErrorString(e));
}

int main() {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    unsigned long long* d; cudaMalloc(&d, 1024 * 8);
    run<0, 64, false>(sms, d); run<0, 128, false>(sms, d); run<0, 256, false>(sms, d);
    run<1, 64, false>(sms, d); run<1, 128, false>(sms, d); run<1, 256, false>(sms, d);
    run<2, 64, false>(sms, d); run<2, 128, false>(sms, d); run<2, 256, false>(sms, d);
    run<1, 64, true>(sms, d); run<2, 64, true>(sms, d); run<2, 128, true>(sms, d); run<2, 256, true>(sms, d);
    run<3, 64, true>(sms, d); run<4, 64, true>(sms, d); run<3, 64, false>(sms, d); run<4, 64, false>(sms, d);
    run<5, 64, true>(sms, d); run<6, 64, true>(sms, d); run<5, 128, true>(sms, d); run<6, 128, true>(sms, d);
    run<8, 64, true>(sms, d); run<9, 64, true>(sms, d); run<8, 128, true>(sms, d); run<9, 128, true>(sms, d);
    return 0;
}
