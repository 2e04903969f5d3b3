// Pipe-overlap microbenchmark for the K3 epilogue (no MMA): 16 warps, one CTA
// per SM, each warp repeatedly drains 128 TMEM columns of its lane quadrant the
// way K3 does (tcgen05.ld x64, wait, reduce, tcgen05.ld x64, wait, reduce) and
// reduces each 64-score sub-tile by
//   mode 0: the K3 FMNMX3 tree over 64 scores (ALU pipe)            -- today
//   mode 1: FMNMX3 tree over 48 scores + sign count of the other 16 against
//           the row's threshold on the FMA pipe (8 FADD2 + 16 IMAD.HI)
//   mode 2: FMNMX3 tree over 40 scores + FMA-pipe sign count of 24
// Prints cycles per 128-column drain; if mode 1/2 < mode 0 the FMA pipe
// offload pays.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -Ipaper_2503_10017_b200/csrc -o tools/ubench_fma_offload tools/ubench_fma_offload.cu
#include <cstdint>
#include <cstdio>

#include "tc_ptx.cuh"

using namespace fnl;

__device__ __forceinline__ float mx3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ void sub2(float& dx, float& dy, float vx, float vy, float nb) {
    asm("{.reg .b64 a, c, d;\n mov.b64 a, {%2, %3};\n mov.b64 c, {%4, %4};\n add.rn.f32x2 d, a, c;\n mov.b64 {%0, %1}, d;}\n"
        : "=f"(dx), "=f"(dy) : "f"(vx), "f"(vy), "f"(nb));
}
__device__ __forceinline__ uint32_t sgn_acc(float d, uint32_t two, uint32_t acc) {
    uint32_t r;
    asm("mad.hi.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(__float_as_uint(d)), "r"(two), "r"(acc));
    return r;
}

// max of v[0..N): FMNMX3 tree, fully unrolled (compile-time indices only)
template <int N>
__device__ __forceinline__ float tree(const float* v) {
    if constexpr (N == 1) {
        return v[0];
    } else if constexpr (N == 2) {
        return fmaxf(v[0], v[1]);
    } else if constexpr (N == 3) {
        return mx3(v[0], v[1], v[2]);
    } else {
        constexpr int M = N / 3 + (N % 3 ? 1 : 0);
        float r[M];
#pragma unroll
        for (int i = 0; i < N / 3; ++i) r[i] = mx3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
        if constexpr (N % 3 == 1) r[M - 1] = v[N - 1];
        if constexpr (N % 3 == 2) r[M - 1] = fmaxf(v[N - 2], v[N - 1]);
        return tree<M>(r);
    }
}

template <int NFMA>
__device__ __forceinline__ float subtile(const Frag& f, const Frag& g, float b3, uint32_t two, uint32_t& cnt) {
    float v[64];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        v[j] = __uint_as_float(f.r[j]);
        v[32 + j] = __uint_as_float(g.r[j]);
    }
    const float m = tree<64 - NFMA>(v);
    if constexpr (NFMA > 0) {
        uint32_t c0 = 0, c1 = 0, c2 = 0, c3 = 0;
#pragma unroll
        for (int i = 64 - NFMA; i < 64; i += 4) {
            float a, b, c, d;
            sub2(a, b, v[i], v[i + 1], -b3);
            sub2(c, d, v[i + 2], v[i + 3], -b3);
            c0 = sgn_acc(a, two, c0);
            c1 = sgn_acc(b, two, c1);
            c2 = sgn_acc(c, two, c2);
            c3 = sgn_acc(d, two, c3);
        }
        cnt += c0 + c1 + c2 + c3;
    }
    return m;
}

template <int NFMA>
__global__ void __launch_bounds__(512, 1) k(uint32_t two, int iters, float* out, long long* cyc) {
    __shared__ uint32_t slot;
    const uint32_t warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&slot)), "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = slot;
    const uint32_t taddr = tmem + (((warp & 3u) * 32u) << 16) + (warp >> 2) * 128u;
    float b3 = -1e30f, acc = -1e30f;
    uint32_t cnt = 0;
    Frag f0, f1;
    __syncthreads();
    const long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < iters; ++it) {
        frag_ld64(taddr, f0, f1);
        frag_wait2(f0, f1);
        const float m0 = subtile<NFMA>(f0, f1, b3, two, cnt);
        frag_ld64(taddr + 64u, f0, f1);
        frag_wait2(f0, f1);
        const float m1 = subtile<NFMA>(f0, f1, b3, two, cnt);
        acc = fmaxf(acc, fmaxf(m0, m1));
        if (__any_sync(0xffffffffu, acc > b3 + 1e30f)) b3 = acc;  // never: keeps b3 a loop variable
    }
    const long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + (float)cnt;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    float* out;
    long long* cyc;
    cudaMalloc(&out, sms * 512 * sizeof(float));
    cudaMalloc(&cyc, sms * sizeof(long long));
    const int iters = 8192;
    printf("{\"sms\": %d, \"iters\": %d, \"warps\": 16, \"runs\": [\n", sms, iters);
    const int nf[3] = {0, 16, 24};
    for (int mode = 0; mode < 3; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            if (mode == 0) k<0><<<sms, 512>>>(2u, iters, out, cyc);
            if (mode == 1) k<16><<<sms, 512>>>(2u, iters, out, cyc);
            if (mode == 2) k<24><<<sms, 512>>>(2u, iters, out, cyc);
        }
        cudaDeviceSynchronize();
        long long c = 0;
        cudaMemcpy(&c, cyc, sizeof(long long), cudaMemcpyDeviceToHost);
        printf("%s{\"mode\": %d, \"fma_pipe_scores_per_64\": %d, \"cycles_per_128col_drain\": %.1f}\n", mode ? "," : "",
               mode, nf[mode], (double)c / iters);
    }
    printf("], \"err\": \"%s\"}\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
