// flashmatch.cu -- K7 FlashMatch: non-causal multi-head attention on the
// 5th-gen tensor cores (Speedy MASt3R's FlashMatch, which
// the reference only describes).
//
//   O = softmax(Q K^T * scale) V     per (batch, head), head_dim 64,
//   binary16 Q/K/V/O, fp32 scores, fp32 softmax statistics, fp32 accumulation
//   (HybridCast numerics).
//
// One CTA = 128 query rows of one (batch, head); 4 warps, thread r owns query
// row r (= TMEM lane r).  Per 128-key block j:
//   S_j = Q K_j^T        tcgen05.mma kind::f16 M128 N128 K16 x4 (SS) -> TMEM cols [0,128)
//   softmax              tcgen05.ld of the thread's 128 scores, online max /
//                        rescale / exp2 / row sum in registers, P_j (binary16)
//                        st.shared in the UMMA K-major layout
//   O_j = P_j V_j        tcgen05.mma M128 N64 K16 x8 (SS, V MN-major)  -> TMEM cols [128,192)
//   o = o * alpha + O_j  (registers; the final 1/l and binary16 cast in the epilogue)
// K/V blocks are double-buffered with cp.async (zero-filled past the ends), so
// block j+1 lands while block j is scored; two CTAs share an SM (112 KB smem,
// 256 TMEM columns each) so one CTA's softmax overlaps the other's MMAs.  The
// N x N score matrix never leaves the SM.
#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>

#include <string>

#include "fastnn_b200.h"
#include "fnl_common.cuh"
#include "fnl_internal.h"
#include "tc_ptx.cuh"

namespace fnl {

namespace {

constexpr uint32_t kFmThreads = 128;
constexpr uint32_t kHd = 64;         // head_dim
constexpr uint32_t kBlockQ = 128;    // query rows per CTA
constexpr uint32_t kBlockK = 128;    // keys per block
constexpr uint32_t kTileQK = kBlockQ * kHd * 2;   // 16 KB (Q, K blocks and V blocks alike)
constexpr uint32_t kTileP = kBlockQ * kBlockK * 2;  // 32 KB
constexpr uint32_t kSmemFm = kTileQK /*Q*/ + 2 * kTileQK /*K*/ + 2 * kTileQK /*V*/ + kTileP + 64;
constexpr uint32_t kTmemCols = 256;  // S [0,128) + O [128,192)

// UMMA shared-memory descriptor, no swizzle, version 1 (sm_100).
__device__ __forceinline__ uint64_t fm_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
           (1ull << 46);
}
// kind::f16 instruction descriptors: fp16 A/B, fp32 D.
//   S: M128 N128, A and B K-major.   PV: M128 N64, A K-major, B (V) MN-major.
constexpr uint32_t kIdescS = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdescPV = (1u << 4) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

// Layouts (bytes; all core matrices are 8 rows x 16 B = 128 B contiguous):
//   Q, K  [row][hd]   K-major:  (row/8)*1024 + (hd/8)*128 + (row%8)*16   LBO 128, SBO 1024
//   V     [key][hd]   MN-major: (hd/8)*2048 + (key/8)*128 + (key%8)*16   LBO 128 (key groups), SBO 2048 (hd groups)
//   P     [row][key]  K-major:  (row/8)*2048 + (key/8)*128 + (row%8)*16  LBO 128, SBO 2048
__device__ __forceinline__ uint32_t off_qk(uint32_t row, uint32_t chunk) {
    return (row >> 3) * 1024u + chunk * 128u + (row & 7u) * 16u;
}
__device__ __forceinline__ uint32_t off_v(uint32_t key, uint32_t chunk) {
    return chunk * 2048u + (key >> 3) * 128u + (key & 7u) * 16u;
}
__device__ __forceinline__ uint32_t off_p(uint32_t row, uint32_t chunk) {
    return (row >> 3) * 2048u + chunk * 128u + (row & 7u) * 16u;
}

__device__ __forceinline__ void cp_async16(uint32_t saddr, const void* g, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(saddr), "l"(g), "r"(valid ? 16u : 0u)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ uint32_t pack_half2_rn(float a, float b) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}
__device__ __forceinline__ float max3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}
__device__ __forceinline__ float ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

struct FmArgs {
    const __half* q;
    const __half* k;
    const __half* v;
    __half* o;
    uint32_t heads, nq, nkv;
    // element strides: batch, head, token (head_dim is contiguous)
    uint64_t q_sb, q_sh, q_sn;
    uint64_t k_sb, k_sh, k_sn;
    uint64_t v_sb, v_sh, v_sn;
    uint64_t o_sb, o_sh, o_sn;
    float scale_log2;  // softmax scale * log2(e)
};

// 128 rows x 64 hd of a [token][hd] operand into smem.  Warp lanes: row%8 and
// 4 consecutive 16 B chunks, so global reads are 64 B runs and every quarter
// warp writes one 128 B core matrix.
template <bool kV>
__device__ __forceinline__ void load_tile(uint32_t sbase, const __half* g, uint64_t sn, uint32_t nvalid) {
    const uint32_t lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
#pragma unroll
    for (uint32_t j = 0; j < 8; ++j) {
        const uint32_t combo = warp * 8u + j;
        const uint32_t chunk = (lane >> 3) + 4u * (combo & 1u);
        const uint32_t row = (combo >> 1) * 8u + (lane & 7u);
        const bool valid = row < nvalid;
        const __half* src = g + (valid ? (uint64_t)row * sn + chunk * 8u : 0);
        cp_async16(sbase + (kV ? off_v(row, chunk) : off_qk(row, chunk)), src, valid);
    }
}

__global__ void __launch_bounds__(kFmThreads, 2) flashmatch_kernel(FmArgs a) {
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t bar_s, bar_o;
    const uint32_t tid = threadIdx.x, warp = tid >> 5;
    const uint32_t q0 = blockIdx.x * kBlockQ, h = blockIdx.y, b = blockIdx.z;
    const uint32_t sQ = smem_addr(smem);
    const uint32_t sK = sQ + kTileQK, sV = sK + 2 * kTileQK, sP = sV + 2 * kTileQK;
    uint8_t* pP = smem + 5 * kTileQK;

    if (tid == 0) {
        mbar_init(&bar_s, 1);
        mbar_init(&bar_o, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_slot)),
                     "r"(kTmemCols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }

    const __half* gq = a.q + b * a.q_sb + h * a.q_sh + (uint64_t)q0 * a.q_sn;
    const __half* gk = a.k + b * a.k_sb + h * a.k_sh;
    const __half* gv = a.v + b * a.v_sb + h * a.v_sh;
    const uint32_t nblk = (a.nkv + kBlockK - 1) / kBlockK;
    // group 0: Q, K_0, V_0; group 1: K_1, V_1
    load_tile<false>(sQ, gq, a.q_sn, a.nq - q0);
    load_tile<false>(sK, gk, a.k_sn, a.nkv);
    load_tile<true>(sV, gv, a.v_sn, a.nkv);
    cp_async_commit();
    if (nblk > 1) {
        load_tile<false>(sK + kTileQK, gk + (uint64_t)kBlockK * a.k_sn, a.k_sn, a.nkv - kBlockK);
        load_tile<true>(sV + kTileQK, gv + (uint64_t)kBlockK * a.v_sn, a.v_sn, a.nkv - kBlockK);
    }
    cp_async_commit();

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    const uint32_t lane_base = (warp * 32u) << 16;

    float o[kHd];
#pragma unroll
    for (uint32_t i = 0; i < kHd; ++i) o[i] = 0.0f;
    float m = -INFINITY, l = 0.0f;
    const float sl2 = a.scale_log2;

    for (uint32_t j = 0; j < nblk; ++j) {
        const uint32_t buf = j & 1u;
        cp_async_wait<1>();  // this thread's copies of block j (and Q) have landed
        fence_async_smem();  // ... and are visible to the tensor core
        __syncthreads();
        if (warp == 0) {
            tc_fence_after();
            if (elect_one()) {
                const uint32_t kb = sK + buf * kTileQK;
#pragma unroll
                for (uint32_t ks = 0; ks < kHd / 16; ++ks)
                    tc_mma_f16(tmem, fm_desc(sQ + ks * 256u, 128u, 1024u), fm_desc(kb + ks * 256u, 128u, 1024u),
                               kIdescS, ks > 0 ? 1u : 0u);
                tc_commit(&bar_s);
            }
            __syncwarp();
        }
        mbar_wait(&bar_s, j & 1u);
        tc_fence_after();

        // ---- online softmax over this thread's 128 scores
        Frag f0, f1, f2, f3;
        frag_ld(tmem + lane_base + 0, f0);
        frag_ld(tmem + lane_base + 32, f1);
        frag_ld(tmem + lane_base + 64, f2);
        frag_ld(tmem + lane_base + 96, f3);
        frag_wait2(f0, f1);
        frag_wait2(f2, f3);
        float s[kBlockK];
#pragma unroll
        for (uint32_t i = 0; i < 32; ++i) {
            s[i] = __uint_as_float(f0.r[i]);
            s[32 + i] = __uint_as_float(f1.r[i]);
            s[64 + i] = __uint_as_float(f2.r[i]);
            s[96 + i] = __uint_as_float(f3.r[i]);
        }
        const uint32_t kvalid = a.nkv - j * kBlockK;
        if (kvalid < kBlockK) {
#pragma unroll
            for (uint32_t i = 0; i < kBlockK; ++i)
                if (i >= kvalid) s[i] = -INFINITY;
        }
        float mx = -INFINITY;
#pragma unroll
        for (uint32_t i = 0; i < kBlockK; i += 2) mx = max3(mx, s[i], s[i + 1]);
        const float m_new = fmaxf(m, mx * sl2);
        const float alpha = ex2(m - m_new);
        float sum = 0.0f;
#pragma unroll
        for (uint32_t c = 0; c < kBlockK / 8; ++c) {
            float p[8];
#pragma unroll
            for (uint32_t i = 0; i < 8; ++i) {
                p[i] = ex2(fmaf(s[c * 8 + i], sl2, -m_new));
                sum += p[i];
            }
            uint4 w;
            w.x = pack_half2_rn(p[0], p[1]);
            w.y = pack_half2_rn(p[2], p[3]);
            w.z = pack_half2_rn(p[4], p[5]);
            w.w = pack_half2_rn(p[6], p[7]);
            *reinterpret_cast<uint4*>(pP + off_p(tid, c)) = w;
        }
        l = l * alpha + sum;
        m = m_new;
        tc_fence_before();
        fence_async_smem();
        __syncthreads();  // P complete; every thread has drained S
        if (warp == 0) {
            tc_fence_after();
            if (elect_one()) {
                const uint32_t vb = sV + buf * kTileQK;
#pragma unroll
                for (uint32_t ks = 0; ks < kBlockK / 16; ++ks)
                    tc_mma_f16(tmem + 128u, fm_desc(sP + ks * 256u, 128u, 2048u), fm_desc(vb + ks * 256u, 128u, 2048u),
                               kIdescPV, ks > 0 ? 1u : 0u);
                tc_commit(&bar_o);
            }
            __syncwarp();
        }
        mbar_wait(&bar_o, j & 1u);
        tc_fence_after();
        Frag g0, g1;
        frag_ld(tmem + lane_base + 128u, g0);
        frag_ld(tmem + lane_base + 160u, g1);
        frag_wait2(g0, g1);
#pragma unroll
        for (uint32_t i = 0; i < 32; ++i) {
            o[i] = fmaf(o[i], alpha, __uint_as_float(g0.r[i]));
            o[32 + i] = fmaf(o[32 + i], alpha, __uint_as_float(g1.r[i]));
        }
        tc_fence_before();
        // K/V buffer `buf` is free (its MMAs retired): prefetch block j+2 into it
        if (j + 2 < nblk) {
            load_tile<false>(sK + buf * kTileQK, gk + (uint64_t)(j + 2) * kBlockK * a.k_sn, a.k_sn,
                             a.nkv - (j + 2) * kBlockK);
            load_tile<true>(sV + buf * kTileQK, gv + (uint64_t)(j + 2) * kBlockK * a.v_sn, a.v_sn,
                            a.nkv - (j + 2) * kBlockK);
        }
        cp_async_commit();
    }

    // ---- epilogue: normalise, binary16, one 128 B row per thread
    const uint32_t row = q0 + tid;
    if (row < a.nq) {
        const float inv = 1.0f / l;
        __half* go = a.o + b * a.o_sb + h * a.o_sh + (uint64_t)row * a.o_sn;
#pragma unroll
        for (uint32_t c = 0; c < kHd / 8; ++c) {
            uint4 w;
            w.x = pack_half2_rn(o[c * 8 + 0] * inv, o[c * 8 + 1] * inv);
            w.y = pack_half2_rn(o[c * 8 + 2] * inv, o[c * 8 + 3] * inv);
            w.z = pack_half2_rn(o[c * 8 + 4] * inv, o[c * 8 + 5] * inv);
            w.w = pack_half2_rn(o[c * 8 + 6] * inv, o[c * 8 + 7] * inv);
            *reinterpret_cast<uint4*>(go + c * 8) = w;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kTmemCols));
    }
}

bool fm_attr_done = false;

}  // namespace

int flashmatch_forward(fnl_context* ctx, const fnl_attention_desc& d) {
    if (d.head_dim != kHd)
        return fail(FNL_EINVAL, "flashmatch: head_dim " + std::to_string(d.head_dim) + " unsupported (64 only)");
    if (d.batch == 0 || d.heads == 0 || d.nq == 0 || d.nkv == 0) return FNL_OK;
    if (!d.q || !d.k || !d.v || !d.o) return fail(FNL_EINVAL, "flashmatch: null tensor pointer");
    const uint64_t strides[12] = {d.q_stride[0], d.q_stride[1], d.q_stride[2], d.k_stride[0],
                                  d.k_stride[1], d.k_stride[2], d.v_stride[0], d.v_stride[1],
                                  d.v_stride[2], d.o_stride[0], d.o_stride[1], d.o_stride[2]};
    for (uint64_t s : strides)
        if (s % 8) return fail(FNL_EINVAL, "flashmatch: strides must be multiples of 8 elements (16 B)");
    const uintptr_t ptrs[4] = {(uintptr_t)d.q, (uintptr_t)d.k, (uintptr_t)d.v, (uintptr_t)d.o};
    for (uintptr_t p : ptrs)
        if (p % 16) return fail(FNL_EINVAL, "flashmatch: tensors must be 16 B aligned");
    if (d.heads > 65535 || d.batch > 65535) return fail(FNL_EINVAL, "flashmatch: batch/heads exceed 65535");
    if (!fm_attr_done) {
        FNL_CUDA_TRY(cudaFuncSetAttribute(flashmatch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemFm));
        fm_attr_done = true;
    }
    FmArgs a{};
    a.q = static_cast<const __half*>(d.q);
    a.k = static_cast<const __half*>(d.k);
    a.v = static_cast<const __half*>(d.v);
    a.o = static_cast<__half*>(d.o);
    a.heads = d.heads;
    a.nq = d.nq;
    a.nkv = d.nkv;
    a.q_sb = d.q_stride[0]; a.q_sh = d.q_stride[1]; a.q_sn = d.q_stride[2];
    a.k_sb = d.k_stride[0]; a.k_sh = d.k_stride[1]; a.k_sn = d.k_stride[2];
    a.v_sb = d.v_stride[0]; a.v_sh = d.v_stride[1]; a.v_sn = d.v_stride[2];
    a.o_sb = d.o_stride[0]; a.o_sh = d.o_stride[1]; a.o_sn = d.o_stride[2];
    a.scale_log2 = d.scale * 1.4426950408889634f;
    dim3 grid((d.nq + kBlockQ - 1) / kBlockQ, d.heads, d.batch);
    cudaStream_t s = ctx_stream(ctx);
    ProfScope prof(ctx, FNL_KCLASS_ATTN);
    flashmatch_kernel<<<grid, kFmThreads, kSmemFm, s>>>(a);
    FNL_CUDA_TRY(cudaGetLastError());
    ctx_count_launches(ctx, 1);
    return FNL_OK;
}

}  // namespace fnl
