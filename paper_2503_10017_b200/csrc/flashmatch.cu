// flashmatch.cu -- K7 FlashMatch: non-causal multi-head attention on the
// 5th-gen tensor cores (Speedy MASt3R's FlashMatch, which
// the reference only describes).
//
//   O = softmax(Q K^T * scale) V     per (batch, head), head_dim 64,
//   binary16 Q/K/V/O, fp32 scores, fp32 softmax statistics, fp32 accumulation
//   (HybridCast numerics).
//
// Product kernel: flashmatch4_kernel (v4).  One CTA = one or two 128-row
// query tiles of one (batch, head), warp-specialised, mbarrier hand-offs only:
//   warps 0-15  softmax: warpgroup t (8 warps) owns query tile t, two threads
//               per row (TMEM lane quadrant w%4, key-column half (w/4)%2)
//   warp 16     MMA issuer: S_t(j) = Q_t K_j^T (M128 N128 K16 x4, SS) into
//               TMEM [256t, 256t+128) as soon as S_t(j-1) is in registers;
//               O_t += P_t(j) V_j (M128 N64 K16 x8, V MN-major) into
//               [256t+128, 256t+192) as soon as P_t(j) is published
//   warp 17     loader: one elected thread, TMA tensor-map boxes of 128 rows
//               x 64 channels (128B swizzle, zero fill past N) into a 3-stage
//               K/V ring
// Per block the softmax reads S once (tcgen05.ld.x64), releases it, takes
// the row max across the two half-row threads through shared memory, writes
// binary16 P = 2^(s*scale*log2e - m) to shared memory (UMMA K-major layout)
// and rescales O in TMEM only when the row max grew by more than 2^8 (lazy
// rescale; O and l carry the same stale max).  The N x N score matrix never
// leaves the SM.
// Measurements and the variants that lost: DESIGN.md section 7.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_fp16.h>
#include <math.h>
#include <stdint.h>

#include <stdlib.h>

#include <mutex>
#include <string>

#include "fastnn_b200.h"
#include "fnl_common.cuh"
#include "fnl_internal.h"
#include "tc_ptx.cuh"

namespace fnl {

namespace {

constexpr uint32_t kHd = 64;         // head_dim
constexpr uint32_t kBlockQ = 128;    // query rows per CTA
constexpr uint32_t kBlockK = 128;    // keys per block
constexpr uint32_t kTileQK = kBlockQ * kHd * 2;   // 16 KB (Q, K blocks and V blocks alike)
constexpr uint32_t kTileP = kBlockQ * kBlockK * 2;  // 32 KB

// UMMA shared-memory descriptor, no swizzle, version 1 (sm_100).
__device__ __forceinline__ uint64_t fm_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
           (1ull << 46);
}
// kind::f16 instruction descriptors: fp16 A/B, fp32 D.
//   S: M128 N128, A and B K-major.   PV: M128 N64, A K-major, B (V) MN-major.
constexpr uint32_t kIdescS = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);
constexpr uint32_t kIdescPV = (1u << 4) | (1u << 16) | ((64u >> 3) << 17) | ((128u >> 4) << 24);

// P [row][key] (written by the softmax threads), K-major, no swizzle, core
// matrices of 8 rows x 16 B: (row/8)*2048 + (key/8)*128 + (row%8)*16, LBO 128,
// SBO 2048.  Q, K and V arrive as TMA SWIZZLE_128B boxes (see K7 v4 below).
__device__ __forceinline__ uint32_t off_p(uint32_t row, uint32_t chunk) {
    return (row >> 3) * 2048u + chunk * 128u + (row & 7u) * 16u;
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

// profiling aid: per-phase clock64 stamps of CTA 0, thread 0 (FNL_FM_TRACE=1)
__device__ unsigned long long g_fm_trace[64];
#define FM_STAMP(i)                                                         \
    do {                                                                    \
        if (kTrace && a.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && \
            threadIdx.x == 0 && (i) < 64)                                   \
            g_fm_trace[(i)] = clock64();                                    \
    } while (0)

// same, from lane 0 of whichever warp executes it
#define FM_STAMP_L(i)                                                                              \
    do {                                                                                           \
        if (kTrace && a.trace && blockIdx.x == 0 && blockIdx.y == 0 && blockIdx.z == 0 && (threadIdx.x & 31) == 0) \
            g_fm_trace[(i)] = clock64();                                                           \
    } while (0)

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
    uint32_t tiles;    // query tiles per CTA (v4: 1 or 2)
    int trace;
};

// ---------------------------------------------------------------- K7 shared

__device__ __forceinline__ bool mbar_test(uint64_t* bar, uint32_t parity) {
    uint32_t done;
    asm volatile(
        "{ .reg .pred p; mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    return done != 0;
}

// ---------------------------------------------------------------- K7 helpers
// The softmax reads S_j once (tcgen05.ld.x64 into registers), hands the S
// buffer back at once so S_{j+1} runs on the tensor core under this block's
// exponentials, and keeps O in TMEM: PV_j accumulates into it, and O is
// rescaled (tcgen05.ld / st) only when a row max grows by more than
// kRescaleLog2 (P entries stay <= 2^kRescaleLog2, well inside binary16; l and O
// carry the same stale max, so O/l is exact).
constexpr float kRescaleLog2 = 8.0f;

__device__ __forceinline__ void frag_st(uint32_t taddr, const Frag& f) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr), "r"(f.r[0]),"r"(f.r[1]),"r"(f.r[2]),"r"(f.r[3]),"r"(f.r[4]),"r"(f.r[5]),"r"(f.r[6]),"r"(f.r[7]),"r"(f.r[8]),"r"(f.r[9]),"r"(f.r[10]),"r"(f.r[11]),"r"(f.r[12]),"r"(f.r[13]),"r"(f.r[14]),"r"(f.r[15]),"r"(f.r[16]),"r"(f.r[17]),"r"(f.r[18]),"r"(f.r[19]),"r"(f.r[20]),"r"(f.r[21]),"r"(f.r[22]),"r"(f.r[23]),"r"(f.r[24]),"r"(f.r[25]),"r"(f.r[26]),"r"(f.r[27]),"r"(f.r[28]),"r"(f.r[29]),"r"(f.r[30]),"r"(f.r[31]) : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// ---------------------------------------------------------------- K7 v4
// v3 with TMA: Q, K_j and V_j arrive by cp.async.bulk.tensor (one elected
// thread, 128B-swizzled boxes of 128 rows x 64 channels, zero fill past N)
// instead of 16-byte cp.async from three loader warps, which spent ~2.5k
// cycles just issuing the first Q tiles.  Operand descriptors switch to the
// SWIZZLE_128B canonical layouts: Q / K K-major (8-row atoms of 1 KB, K step
// = +32 B), V MN-major (hd contiguous, 8-key atoms 1 KB apart, K step of 16
// keys = +2 KB).  P keeps the no-swizzle layout the softmax writes.
constexpr uint32_t kKvStages4 = 3;
constexpr uint32_t kSmemFm4 = 2 * kTileQK + 2 * kKvStages4 * kTileQK + 2 * kTileP + 1024;  // + alignment slack

__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) |
           (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ void tma_load_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
        "[%6];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_addr(bar))
        : "memory");
}

// kH = threads per query row (2: 16 softmax warps, 64 key columns each, row
// max / sum halves meet in shared memory; 1: 8 softmax warps, a whole
// 128-column row per thread in 128 registers, no exchange).
// kTrace: the FNL_FM_TRACE clock stamps are compiled in (profiling only)
template <int kH, bool kTrace>
__global__ void __launch_bounds__((8 * kH + 2) * 32, 1)
    flashmatch4_kernel(FmArgs a, const __grid_constant__ CUtensorMap tq, const __grid_constant__ CUtensorMap tk,
                       const __grid_constant__ CUtensorMap tv) {
    constexpr uint32_t kSoftWarps = 8 * kH;          // both tiles
    constexpr uint32_t kTileWarps = 4 * kH;          // per tile
    constexpr uint32_t kCols = kBlockK / kH;         // key columns per thread
    constexpr uint32_t kSF = kCols / 32;             // 32-column S fragments per thread
    constexpr uint32_t kOF = kHd / kH / 32;          // 32-column O fragments per thread
    __shared__ float red[2][2][kBlockQ];  // [tile][column half][row] partial maxima / sums (kH = 2)
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ __align__(8) uint64_t s_full[2], s_free[2], p_full[2], o_full[2];
    __shared__ __align__(8) uint64_t kv_full[kKvStages4], kv_empty[kKvStages4];
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31u;
    const uint32_t ntile = a.tiles, q0 = blockIdx.x * ntile * kBlockQ, h = blockIdx.y, b = blockIdx.z;
    FM_STAMP(0);
    // SWIZZLE_128B operands need 1 KB aligned tiles
    const uint32_t base_pad = (1024u - (smem_addr(smem) & 1023u)) & 1023u;
    const uint32_t sQ = smem_addr(smem) + base_pad;
    const uint32_t sK = sQ + 2 * kTileQK, sV = sK + kKvStages4 * kTileQK, sP = sV + kKvStages4 * kTileQK;
    uint8_t* pP0 = smem + base_pad + (2 + 2 * kKvStages4) * kTileQK;
    const uint32_t nblk = (a.nkv + kBlockK - 1) / kBlockK;

    if (tid == 0) {
        for (int t = 0; t < 2; ++t) {
            mbar_init(&s_full[t], 1);
            mbar_init(&s_free[t], kTileWarps);
            mbar_init(&p_full[t], kTileWarps);
            mbar_init(&o_full[t], 1);
        }
        for (uint32_t st = 0; st < kKvStages4; ++st) {
            mbar_init(&kv_full[st], 1);   // the loader's expect_tx arrival; TMA completes the bytes
            mbar_init(&kv_empty[st], 1);  // one tcgen05.commit after the block's last PV
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        // the first boxes go out before the CTA-wide barrier / TMEM allocation
        const int hh = (int)h, bb = (int)b;
        mbar_expect_tx(&kv_full[0], (ntile + 2) * kTileQK);
        tma_load_4d(sQ, &tq, 0, (int)q0, hh, bb, &kv_full[0]);
        if (ntile == 2) tma_load_4d(sQ + kTileQK, &tq, 0, (int)(q0 + kBlockQ), hh, bb, &kv_full[0]);
        tma_load_4d(sK, &tk, 0, 0, hh, bb, &kv_full[0]);
        tma_load_4d(sV, &tv, 0, 0, hh, bb, &kv_full[0]);
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_slot)),
                     "r"(512u));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    FM_STAMP(34);

    if (warp == kSoftWarps + 1) {
        // ---------------- loader: one elected thread issues the remaining TMA boxes
        if (elect_one()) {
            const int hh = (int)h, bb = (int)b;
            for (uint32_t blk = 1; blk < nblk; ++blk) {
                const uint32_t st = blk % kKvStages4;
                mbar_wait(&kv_empty[st], ((blk / kKvStages4) & 1u) ^ 1u);
                mbar_expect_tx(&kv_full[st], 2 * kTileQK);
                tma_load_4d(sK + st * kTileQK, &tk, 0, (int)(blk * kBlockK), hh, bb, &kv_full[st]);
                tma_load_4d(sV + st * kTileQK, &tv, 0, (int)(blk * kBlockK), hh, bb, &kv_full[st]);
            }
        }
        __syncwarp();
    } else if (warp == kSoftWarps) {
        // ---------------- MMA warp: S_t(j+1) as soon as S_t(j) is drained,
        // PV_t(j) as soon as P_t(j) is published
        auto kv_ready = [&](uint32_t blk) {
            mbar_wait(&kv_full[blk % kKvStages4], (blk / kKvStages4) & 1u);
        };
        auto issue_s = [&](uint32_t t, uint32_t blk) {
            tc_fence_after();
            if (elect_one()) {
                const uint32_t kb = sK + (blk % kKvStages4) * kTileQK, qb = sQ + t * kTileQK;
#pragma unroll
                for (uint32_t ks = 0; ks < kHd / 16; ++ks)
                    tc_mma_f16(tmem + t * 256u, sw128_desc(qb + ks * 32u, 16u, 1024u),
                               sw128_desc(kb + ks * 32u, 16u, 1024u), kIdescS, ks > 0 ? 1u : 0u);
                tc_commit(&s_full[t]);
            }
            __syncwarp();
        };
        kv_ready(0);  // also covers Q (same barrier phase)
        issue_s(0, 0);
        if (ntile == 2) issue_s(1, 0);
        // a single-tile CTA never serves tile 1
        uint32_t js[2] = {1u, ntile == 2 ? 1u : nblk}, jp[2] = {0u, ntile == 2 ? 0u : nblk};
        while (jp[0] < nblk || jp[1] < nblk) {
#pragma unroll
            for (uint32_t t = 0; t < 2; ++t) {
                if (js[t] < nblk && mbar_test(&s_free[t], (js[t] - 1u) & 1u)) {
                    kv_ready(js[t]);  // the stage cannot have been refilled: its PVs are not issued yet
                    issue_s(t, js[t]);
                    ++js[t];
                }
                const uint32_t j = jp[t];
                if (j < nblk && mbar_test(&p_full[t], j & 1u)) {
                    tc_fence_after();
                    const bool last_reader = jp[t ^ 1u] > j;  // the other tile's PV_j is issued (or no other tile)
                    if (elect_one()) {
                        const uint32_t vb = sV + (j % kKvStages4) * kTileQK, pb = sP + t * kTileP;
#pragma unroll
                        for (uint32_t ks = 0; ks < kBlockK / 16; ++ks)
                            tc_mma_f16(tmem + t * 256u + 128u, fm_desc(pb + ks * 256u, 128u, 2048u),
                                       sw128_desc(vb + ks * 2048u, 1024u, 1024u), kIdescPV, (ks | j) > 0 ? 1u : 0u);
                        tc_commit(&o_full[t]);
                        if (last_reader) tc_commit(&kv_empty[j % kKvStages4]);
                    }
                    __syncwarp();
                    jp[t] = j + 1;
                }
            }
        }
    } else if (warp / kTileWarps < ntile) {
        // ---------------- softmax warpgroup t: warp w reads TMEM lane quadrant
        // w%4 and key-column part hf = (w/4)%kH
        const uint32_t t = warp / kTileWarps, hf = (warp >> 2) % kH, row = ((warp & 3u) << 5) | lane;
        const uint32_t lane_base = ((warp & 3u) * 32u) << 16;
        const uint32_t tS = tmem + lane_base + t * 256u + hf * kCols, tO = tmem + lane_base + t * 256u + 128u + hf * (kHd / kH);
        uint8_t* pP = pP0 + t * kTileP;
        float m = -INFINITY, l = 0.0f;
        const float sl2 = a.scale_log2;
        auto tile_sync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(1u + t), "r"(kTileWarps * 32) : "memory"); };
        for (uint32_t j = 0; j < nblk; ++j) {
            mbar_wait(&s_full[t], j & 1u);
            if (t == 0) FM_STAMP(3 + j);
            tc_fence_after();
            Frag f[kSF];
#pragma unroll
            for (uint32_t c = 0; c < kSF; c += 2) frag_ld64(tS + c * 32u, f[c], f[c + 1]);
#pragma unroll
            for (uint32_t c = 0; c < kSF; c += 2) frag_wait2(f[c], f[c + 1]);
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&s_free[t]);  // S_t(j) is in registers: S_t(j+1) may overwrite it
            const uint32_t kvalid = a.nkv - j * kBlockK;
            if (kvalid < kBlockK) {
#pragma unroll
                for (uint32_t c = 0; c < kSF; ++c)
#pragma unroll
                    for (uint32_t i = 0; i < 32; ++i)
                        if (hf * kCols + c * 32u + i >= kvalid) f[c].r[i] = __float_as_uint(-INFINITY);
            }
            float r4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
            for (uint32_t c = 0; c < kSF; ++c)
#pragma unroll
                for (uint32_t i = 0; i < 32; i += 8)
#pragma unroll
                    for (uint32_t u = 0; u < 4; ++u)
                        r4[u] = max3(r4[u], __uint_as_float(f[c].r[i + 2 * u]), __uint_as_float(f[c].r[i + 2 * u + 1]));
            float mx = fmaxf(fmaxf(r4[0], r4[1]), fmaxf(r4[2], r4[3]));
            if (kH == 2) {
                red[t][hf][row] = mx;
                tile_sync();
                mx = fmaxf(mx, red[t][hf ^ 1u][row]);
                tile_sync();  // both halves read before either writes the next value
            }
            // lazy rescale: keep the stale max unless the row max grew by more
            // than 2^kRescaleLog2 (the threads of a row decide identically)
            const float mc = mx * sl2;
            const bool grow = mc > m + kRescaleLog2;
            const float m_new = grow ? mc : m;
            const float alpha = (grow && j > 0) ? ex2(m - m_new) : 1.0f;
            if (t == 0 && j < 8) FM_STAMP(10 + j);
            // PV_t(j-1) must have retired before P is overwritten or O rescaled
            if (j > 0) {
                mbar_wait(&o_full[t], (j - 1) & 1u);
                tc_fence_after();
            }
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (uint32_t c = 0; c < kSF; ++c) {
                const uint32_t col0 = hf * kCols + c * 32u;
#pragma unroll
                for (uint32_t q = 0; q < 4; ++q) {
                    float p[8];
#pragma unroll
                    for (uint32_t i = 0; i < 8; ++i) p[i] = ex2(fmaf(__uint_as_float(f[c].r[q * 8 + i]), sl2, -m_new));
                    acc[q] += ((p[0] + p[1]) + (p[2] + p[3])) + ((p[4] + p[5]) + (p[6] + p[7]));
                    uint4 w;
                    w.x = pack_half2_rn(p[0], p[1]);
                    w.y = pack_half2_rn(p[2], p[3]);
                    w.z = pack_half2_rn(p[4], p[5]);
                    w.w = pack_half2_rn(p[6], p[7]);
                    *reinterpret_cast<uint4*>(pP + off_p(row, col0 / 8u + q)) = w;
                }
            }
            if (__any_sync(0xFFFFFFFFu, alpha != 1.0f)) {  // warp-collective TMEM round trip of O
#pragma unroll
                for (uint32_t c = 0; c < kOF; ++c) {
                    Frag o;
                    frag_ld(tO + c * 32u, o);
                    frag_wait1(o);
#pragma unroll
                    for (uint32_t i = 0; i < 32; ++i) o.r[i] = __float_as_uint(__uint_as_float(o.r[i]) * alpha);
                    frag_st(tO + c * 32u, o);
                }
                tmem_st_wait();
            }
            tc_fence_before();
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(&p_full[t]);  // P_t(j) written, O_t rescaled
            if (t == 0) FM_STAMP(20 + j);
            l = l * alpha + ((acc[0] + acc[1]) + (acc[2] + acc[3]));  // partial when kH = 2
            m = m_new;
        }
        mbar_wait(&o_full[t], (nblk - 1) & 1u);
        tc_fence_after();
        if (kH == 2) {
            red[t][hf][row] = l;
            tile_sync();
            l += red[t][hf ^ 1u][row];
        }
        const uint32_t grow_ = q0 + t * kBlockQ + row;
        const float inv = 1.0f / l;
#pragma unroll
        for (uint32_t c = 0; c < kOF; ++c) {
            Frag o;
            frag_ld(tO + c * 32u, o);
            frag_wait1(o);
            if (grow_ < a.nq) {
                __half* go = a.o + b * a.o_sb + h * a.o_sh + (uint64_t)grow_ * a.o_sn + hf * (kHd / kH) + c * 32u;
#pragma unroll
                for (uint32_t q = 0; q < 4; ++q) {
                    uint4 w;
                    w.x = pack_half2_rn(__uint_as_float(o.r[q * 8 + 0]) * inv, __uint_as_float(o.r[q * 8 + 1]) * inv);
                    w.y = pack_half2_rn(__uint_as_float(o.r[q * 8 + 2]) * inv, __uint_as_float(o.r[q * 8 + 3]) * inv);
                    w.z = pack_half2_rn(__uint_as_float(o.r[q * 8 + 4]) * inv, __uint_as_float(o.r[q * 8 + 5]) * inv);
                    w.w = pack_half2_rn(__uint_as_float(o.r[q * 8 + 6]) * inv, __uint_as_float(o.r[q * 8 + 7]) * inv);
                    *reinterpret_cast<uint4*>(go + q * 8) = w;
                }
            }
        }
    }
    FM_STAMP(63);
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512u));
    }
}

// cudaFuncSetAttribute applies to the current device only: one flag per device
std::mutex fm_attr_mu;
bool fm_attr_done[64] = {};

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
    {
        int dev = 0;
        FNL_CUDA_TRY(cudaGetDevice(&dev));
        std::lock_guard<std::mutex> lk(fm_attr_mu);
        if (dev < 0 || dev >= 64 || !fm_attr_done[dev]) {
            FNL_CUDA_TRY(cudaFuncSetAttribute(flashmatch4_kernel<1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemFm4));
            FNL_CUDA_TRY(cudaFuncSetAttribute(flashmatch4_kernel<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemFm4));
            FNL_CUDA_TRY(cudaFuncSetAttribute(flashmatch4_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemFm4));
            FNL_CUDA_TRY(cudaFuncSetAttribute(flashmatch4_kernel<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemFm4));
            if (dev >= 0 && dev < 64) fm_attr_done[dev] = true;
        }
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
    static const int trace = getenv("FNL_FM_TRACE") ? atoi(getenv("FNL_FM_TRACE")) : 0;
    a.trace = trace;
    cudaStream_t s = ctx_stream(ctx);
    ProfScope prof(ctx, FNL_KCLASS_ATTN);
    {
        // TMA tensor maps of Q, K, V viewed as [batch][heads][rows][64] binary16
        static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
        if (!encode) {
            void* fn = nullptr;
            cudaDriverEntryPointQueryResult qr{};
            FNL_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qr));
            if (!fn || qr != cudaDriverEntryPointSuccess)
                return fail(FNL_ERUNTIME, "flashmatch: cuTensorMapEncodeTiled unavailable");
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
        }
        auto make_map = [&](CUtensorMap* m, const void* ptr, uint32_t rows, const uint64_t* st) -> int {
            const cuuint64_t dims[4] = {kHd, rows, d.heads, d.batch};
            const cuuint64_t strides[3] = {st[2] * 2, st[1] * 2, st[0] * 2};
            const cuuint32_t box[4] = {kHd, kBlockQ, 1, 1}, es[4] = {1, 1, 1, 1};
            const CUresult r = encode(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 4, const_cast<void*>(ptr), dims, strides, box, es,
                                      CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                      CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS)
                return fail(FNL_EINVAL, "flashmatch: cuTensorMapEncodeTiled rejected the layout (error " +
                                            std::to_string((int)r) + ")");
            return FNL_OK;
        };
        CUtensorMap tq, tk, tv;
        int rc = make_map(&tq, d.q, d.nq, d.q_stride);
        if (rc == FNL_OK) rc = make_map(&tk, d.k, d.nkv, d.k_stride);
        if (rc == FNL_OK) rc = make_map(&tv, d.v, d.nkv, d.v_stride);
        if (rc != FNL_OK) return rc;
        // two query tiles per CTA share the SM's MUFU / tensor core; when one
        // tile per CTA still fits in a single wave, spread the tiles instead
        const uint64_t tiles1 = (uint64_t)((d.nq + kBlockQ - 1) / kBlockQ) * d.heads * d.batch;
        static const int force_tiles = getenv("FNL_FM_TILES") ? atoi(getenv("FNL_FM_TILES")) : 0;
        a.tiles = force_tiles == 1 || force_tiles == 2 ? (uint32_t)force_tiles
                                                       : (tiles1 <= (uint64_t)ctx_sm_count(ctx) ? 1u : 2u);
        // threads per query row: a whole row per thread when the CTA has one
        // tile (measured 11.2 vs 11.7 us per decoder launch), two otherwise
        // (15.2 vs 15.9 us per encoder launch)
        static const int force_rt = getenv("FNL_FM_ROW_THREADS") ? atoi(getenv("FNL_FM_ROW_THREADS")) : 0;
        const int row_threads = force_rt == 1 || force_rt == 2 ? force_rt : (a.tiles == 1 ? 1 : 2);
        const dim3 grid4((d.nq + a.tiles * kBlockQ - 1) / (a.tiles * kBlockQ), d.heads, d.batch);
        if (row_threads == 1)
            (a.trace ? flashmatch4_kernel<1, true> : flashmatch4_kernel<1, false>)<<<grid4, (8 * 1 + 2) * 32, kSmemFm4, s>>>(a, tq, tk, tv);
        else
            (a.trace ? flashmatch4_kernel<2, true> : flashmatch4_kernel<2, false>)<<<grid4, (8 * 2 + 2) * 32, kSmemFm4, s>>>(a, tq, tk, tv);
    }
    FNL_CUDA_TRY(cudaGetLastError());
    ctx_count_launches(ctx, 1);
    return FNL_OK;
}

int flashmatch_trace(unsigned long long* host64) {
    FNL_CUDA_TRY(cudaMemcpyFromSymbol(host64, g_fm_trace, sizeof(g_fm_trace)));
    return FNL_OK;
}

}  // namespace fnl
