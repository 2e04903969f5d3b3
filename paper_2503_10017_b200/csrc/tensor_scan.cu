// tensor_scan.cu -- the FastNN-Lite hot path on the 5th-gen tensor cores.
//
//   K1 pack     fp32 map -> binary16 rows (RNE + saturation, counted) in the UMMA
//               canonical K-major layout, row norms, per-map max norm.
//   K2 gather   active query rows -> contiguous 256-row query tile pairs, plus the
//               per-row certification margin.
//   K3 scan     one CTA = 256 queries x a range of 128-target tiles.  Warp 0
//               streams target tiles global->smem with cp.async.bulk through an
//               8-deep mbarrier ring; warp 1 (one thread) issues
//               tcgen05.mma.cta_group::1.kind::f16 (M=128, N=128, K=16, two
//               query tiles x two K steps per target tile) into a double-buffered
//               fp32 TMEM accumulator (4 x 128 columns = all 512); warps 2-9
//               drain TMEM with tcgen05.ld, free the buffer at once, and keep a
//               running (best, index, second) per query row in registers.  The
//               score matrix never leaves the SM.
//   K3b merge   per row over target splits; a row is certified when
//               best - second > margin, i.e. the fp32 tensor-core winner is
//               provably the reference FMA-chain winner.
//   K4' rescan  the uncertified rows (near ties, ~0.1%) re-run the reference FMA
//               chain over every target; lowest index on exact ties.
//
// Score convention: larger is better.  dot: s = q.t (dist = -s).  l2: the
// packed target carries -|t|^2/2 as two binary16 terms (hi + lo) in channels
// d, d+1 and the gathered query carries 1.0 there, so s = q.t - |t|^2/2 and
// dist = |q|^2 - 2 s.  Both are monotone in the reference distance, so argmax s
// == argmin dist up to rounding, which the margin covers.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "fastnn_b200.h"
#include "fnl_common.cuh"
#include "fnl_internal.h"
#include "tensor_scan.h"

namespace fnl {

namespace {

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    uint32_t done = 0;
    const uint32_t a = smem_addr(bar);
    do {
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(a), "r"(parity)
            : "memory");
    } while (!done);
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(bar))
        : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_addr(bar))
                 : "memory");
}
__device__ __forceinline__ void tc_mma_f16(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                           uint32_t accumulate) {
    asm volatile(
        "{ .reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p; }" ::"r"(
            d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}
// 32 consecutive fp32 columns of this thread's TMEM lane
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]),
          "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]),
          "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]),
          "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
__device__ __forceinline__ void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

__device__ __forceinline__ float max3(float a, float b, float c) {
    float d;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// Shared-memory matrix descriptor, K-major, no swizzle: LBO = 128 B between the
// two 8-channel chunks of one K=16 step, SBO = 512 B between 8-row groups,
// version 1 (sm_100), base offset 0.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(128u >> 4) << 16) | ((uint64_t)(512u >> 4) << 32) |
           (1ull << 46);
}
// kind::f16 instruction descriptor: A/B fp16, D fp32, both K-major, M=128, N=128.
constexpr uint32_t kIdescF16M128N128 = (1u << 4) | ((128u >> 3) << 17) | ((128u >> 4) << 24);

__host__ __device__ __forceinline__ uint64_t packed_offset(uint32_t row, uint32_t chunk) {
    return (uint64_t)(row >> 3) * 512u + chunk * 128u + (row & 7u) * 16u;
}

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// ---------------------------------------------------------------- K1 pack
// 4 threads per row (one 8-channel chunk each), 8 rows per warp = one group.
struct PackArgs {
    const float* src;
    uint8_t* dst;
    uint64_t pair_bytes;
    uint32_t rows;      // real rows per map
    uint32_t rows_pad;  // rows per map incl. padding (multiple of 128)
    uint32_t dim;
    bool l2;
    float* max_norm;                 // per pair, as non-negative float bits
    unsigned long long* bad;         // per pair first non-finite flat index
    unsigned long long* sat;         // per pair saturation count
};

__global__ void pack_kernel(PackArgs a) {
    const uint32_t pair = blockIdx.y;
    const uint32_t gthread = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t row = gthread >> 2, chunk = gthread & 3u;
    if (row >= a.rows_pad) return;  // whole groups of 4 lanes exit together
    const bool real = row < a.rows;
    const float* src = a.src + ((uint64_t)pair * a.rows + row) * a.dim;
    float v[8];
    uint32_t sat = 0;
    float ss = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        const uint32_t c = chunk * 8 + i;
        float x = 0.0f;
        if (real && c < a.dim) {
            x = src[c];
            if (!isfinite(x)) atomicMin(a.bad + pair, (unsigned long long)row * a.dim + c);
            x = half_round_sat(x, sat);
        }
        v[i] = x;
        ss = __fmaf_rn(x, x, ss);
    }
    // row norm^2 over the 4 chunk lanes (fixed order -> deterministic)
    ss += __shfl_xor_sync(0xFFFFFFFFu, ss, 1);
    ss += __shfl_xor_sync(0xFFFFFFFFu, ss, 2);
    if (a.l2 && real) {
        // -|t|^2/2 as hi + lo binary16 terms in channels dim, dim+1
        const float half_n2 = -0.5f * ss;
        const float hi = __half2float(__float2half_rn(half_n2));
        const float lo = __half2float(__float2half_rn(half_n2 - hi));
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t c = chunk * 8 + i;
            if (c == a.dim) v[i] = hi;
            if (c == a.dim + 1) v[i] = lo;
        }
    }
    uint4 out;
    out.x = pack_half2(v[0], v[1]);
    out.y = pack_half2(v[2], v[3]);
    out.z = pack_half2(v[4], v[5]);
    out.w = pack_half2(v[6], v[7]);
    *reinterpret_cast<uint4*>(a.dst + pair * a.pair_bytes + packed_offset(row, chunk)) = out;
    const uint32_t wsat = warp_sum(sat);
    if ((threadIdx.x & 31) == 0 && wsat) atomicAdd(a.sat + pair, (unsigned long long)wsat);
    if (real && chunk == 0)
        atomicMax(reinterpret_cast<unsigned int*>(a.max_norm) + pair, __float_as_uint(sqrtf(ss)));
}

// ---------------------------------------------------------------- K2 gather
struct GatherArgs {
    const uint8_t* qmap;  // packed query-side maps
    uint64_t qmap_pair_bytes;
    const uint32_t* ids;  // per pair query ids (cap stride), or null = identity
    uint32_t cap;
    const uint32_t* n_active;  // device per pair counts
    const uint32_t* slot_pair;  // gather slot -> pair (host-built, one per active pair)
    const uint32_t* slot_base;  // gather slot -> first row in qbuf
    uint8_t* qbuf;        // gathered query tiles (kQueryTilePair rows per tile pair)
    float* margin;        // per gathered row
    const float* tmax;    // per pair max target norm
    uint32_t dim;
    bool l2;
};

__global__ void gather_kernel(GatherArgs a) {
    const uint32_t slot = blockIdx.y;
    const uint32_t pair = a.slot_pair[slot];
    const uint32_t n = a.n_active[pair];
    const uint32_t npad = (n + kQueryTilePair - 1) / kQueryTilePair * kQueryTilePair;
    const uint32_t gthread = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t i = gthread >> 2, chunk = gthread & 3u;
    if (i >= npad) return;
    const uint32_t drow = a.slot_base[slot] + i;
    uint4 val = make_uint4(0, 0, 0, 0);
    float ss = 0.0f;
    if (i < n) {
        const uint32_t src_row = a.ids ? a.ids[(uint64_t)pair * a.cap + i] : i;
        val = *reinterpret_cast<const uint4*>(a.qmap + pair * a.qmap_pair_bytes + packed_offset(src_row, chunk));
        // query role: channels dim, dim+1 become 1.0 (l2) / 0 (dot)
        __half h[8];
        *reinterpret_cast<uint4*>(h) = val;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t c = chunk * 8 + k;
            if (c >= a.dim) h[k] = __float2half_rn((a.l2 && (c == a.dim || c == a.dim + 1)) ? 1.0f : 0.0f);
            const float x = __half2float(h[k]);
            if (c < a.dim) ss = __fmaf_rn(x, x, ss);
        }
        val = *reinterpret_cast<uint4*>(h);
    }
    ss += __shfl_xor_sync(0xFFFFFFFFu, ss, 1);
    ss += __shfl_xor_sync(0xFFFFFFFFu, ss, 2);
    *reinterpret_cast<uint4*>(a.qbuf + packed_offset(drow, chunk)) = val;
    if (chunk == 0) {
        // Certification margin (score units), see DESIGN.md "certified argmax":
        //   tensor-core accumulation error <= 2^-16 * sum|products| per score,
        //   reference FMA chain error <= (d+2) 2^-24 * sum|terms| per distance,
        //   l2 norm split / fp32 norm error <= 2^-20 |t|^2.
        const float qn = sqrtf(ss) * 1.0001f, tn = a.tmax[pair] * 1.0001f;
        const float d = (float)a.dim;
        float m;
        if (!a.l2) {
            const float A = qn * tn;
            m = 2.0f * ldexpf(A, -16) + 2.0f * (d + 2.0f) * ldexpf(A, -24);
        } else {
            const float A = qn * tn + tn * tn;
            const float S = (qn + tn) * (qn + tn);
            m = 2.0f * ldexpf(A, -16) + (d + 2.0f) * ldexpf(S, -24) + 2.0f * ldexpf(tn * tn, -20);
        }
        a.margin[drow] = 1.25f * m + 1e-30f;
    }
}

// ---------------------------------------------------------------- K3 scan
struct TcItem {
    uint32_t pair, qrow0, tile_begin, tile_end;  // qrow0: first gathered row (multiple of 256)
};

struct TcArgs {
    const uint8_t* qbuf;
    const float* margin;
    const uint8_t* tmap;
    uint64_t t_pair_bytes;
    uint32_t nt;
    const TcItem* items;
    float4* partial;  // [item][256] = (best, second, idx bits, 0)
};

constexpr int kStages = 8;
constexpr int kScanThreads = 320;  // warp 0 producer, warp 1 MMA, warps 2..9 epilogue
constexpr int kEpiWarps = 8;
constexpr uint32_t kSmemA = 2 * kTileBytes;                 // 16 KB: two query tiles
constexpr uint32_t kSmemB = kStages * kTileBytes;           // 64 KB ring
constexpr uint32_t kSmemBars = (2 * kStages + 2 + 2 + 1) * 8;
// Padded past half the SM's shared memory so a second CTA can never be
// co-resident and spin in tcgen05.alloc for the 512 TMEM columns.
constexpr uint32_t kSmemUsed = kSmemA + kSmemB + kSmemBars + 16;
constexpr uint32_t kSmemTotal = kSmemUsed > 120u * 1024u ? kSmemUsed : 120u * 1024u;

__device__ __forceinline__ float chunk_max(const float* v) {
    float r[11];
#pragma unroll
    for (int i = 0; i < 10; ++i) r[i] = max3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
    r[10] = fmaxf(v[30], v[31]);
    const float s0 = max3(r[0], r[1], r[2]), s1 = max3(r[3], r[4], r[5]), s2 = max3(r[6], r[7], r[8]);
    return max3(max3(s0, s1, s2), r[9], r[10]);
}

__global__ void __launch_bounds__(kScanThreads, 1) tc_scan_kernel(TcArgs a) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    uint8_t* sA = smem;
    uint8_t* sB = smem + kSmemA;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + kSmemA + kSmemB);
    uint64_t* full = bars;
    uint64_t* empty = bars + kStages;
    uint64_t* tfull = bars + 2 * kStages;
    uint64_t* tempty = bars + 2 * kStages + 2;
    uint64_t* afull = bars + 2 * kStages + 4;

    const TcItem item = a.items[blockIdx.x];
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t ntiles = item.tile_end - item.tile_begin;

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        for (int b = 0; b < 2; ++b) {
            mbar_init(&tfull[b], 1);
            mbar_init(&tempty[b], kEpiWarps);
        }
        mbar_init(afull, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // ---------------- producer: query tile pair once, then the target ring
            mbar_expect_tx(afull, kSmemA);
            bulk_g2s(sA, a.qbuf + (uint64_t)item.qrow0 * kPackRowBytes, kSmemA, afull);
            const uint8_t* tbase = a.tmap + (uint64_t)item.pair * a.t_pair_bytes;
            for (uint32_t k = 0; k < ntiles; ++k) {
                const uint32_t s = k % kStages, ph = (k / kStages) & 1u;
                mbar_wait(&empty[s], ph ^ 1u);
                mbar_expect_tx(&full[s], kTileBytes);
                bulk_g2s(sB + s * kTileBytes, tbase + (uint64_t)(item.tile_begin + k) * kTileBytes, kTileBytes,
                         &full[s]);
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            // ---------------- MMA issuer (single thread)
            mbar_wait(afull, 0);
            tc_fence_after();
            const uint32_t a_addr = smem_addr(sA), b_addr = smem_addr(sB);
            for (uint32_t k = 0; k < ntiles; ++k) {
                const uint32_t s = k % kStages, ph = (k / kStages) & 1u;
                const uint32_t acc = k & 1u, acc_ph = (k >> 1) & 1u;
                mbar_wait(&tempty[acc], acc_ph ^ 1u);
                mbar_wait(&full[s], ph);
                tc_fence_after();
#pragma unroll
                for (uint32_t qt = 0; qt < 2; ++qt) {
#pragma unroll
                    for (uint32_t ks = 0; ks < 2; ++ks) {
                        tc_mma_f16(tmem + acc * 256u + qt * 128u,
                                   umma_desc(a_addr + qt * kTileBytes + ks * 256u),
                                   umma_desc(b_addr + s * kTileBytes + ks * 256u), kIdescF16M128N128, ks);
                    }
                }
                tc_commit(&empty[s]);    // smem slot reusable once these MMAs retire
                tc_commit(&tfull[acc]);  // accumulator ready for the epilogue
            }
        }
    } else {
        // ---------------- epilogue: 8 warps, two per TMEM lane quadrant
        const uint32_t e = warp - 2, qt = e >> 2, quad = warp & 3u;
        const uint32_t row = qt * 128u + quad * 32u + lane;  // 0..255 within the tile pair
        const float margin = a.margin[item.qrow0 + row];
        float best = -INFINITY, second = -INFINITY, thr = -INFINITY;
        uint32_t bidx = 0xFFFFFFFFu;
        float v[128];
        for (uint32_t k = 0; k < ntiles; ++k) {
            const uint32_t acc = k & 1u, acc_ph = (k >> 1) & 1u;
            mbar_wait(&tfull[acc], acc_ph);
            tc_fence_after();
            const uint32_t taddr = tmem + ((quad * 32u) << 16) + acc * 256u + qt * 128u;
            tmem_ld32(taddr + 0, v + 0);
            tmem_ld32(taddr + 32, v + 32);
            tmem_ld32(taddr + 64, v + 64);
            tmem_ld32(taddr + 96, v + 96);
            tmem_ld_wait();
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);  // MMA may overwrite this buffer now
            const uint32_t col0 = (item.tile_begin + k) * kTileRows;
            if (col0 + kTileRows > a.nt) {  // last, partial tile: padded targets never win
#pragma unroll
                for (int j = 0; j < 128; ++j)
                    if (col0 + j >= a.nt) v[j] = -INFINITY;
            }
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float m = chunk_max(v + 32 * c);
                if (m >= thr) {  // rare after warm-up: this chunk may hold the best or a near tie
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        const float x = v[32 * c + j];
                        if (x > best) {
                            second = fmaxf(second, best);
                            best = x;
                            bidx = col0 + 32 * c + j;
                        } else {
                            second = fmaxf(second, x);
                        }
                    }
                    thr = best - margin;
                }
            }
        }
        a.partial[(uint64_t)blockIdx.x * kQueryTilePair + row] =
            make_float4(best, second, __uint_as_float(bidx), 0.0f);
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// ---------------------------------------------------------------- K3b merge
struct MergeArgs {
    const float4* partial;
    const uint32_t* tp_pair;   // tile pair -> pair
    const uint32_t* tp_row0;   // tile pair -> first gathered row
    const uint32_t* tp_qi0;    // tile pair -> first query index within the pair
    uint32_t splits;
    const uint32_t* n_active;
    const float* margin;
    uint32_t* out;
    uint32_t out_stride;
    uint32_t* rescan;           // (gathered row, pair, qi) triples
    unsigned int* rescan_count;
    unsigned long long* near_ties;  // per pair
};

__global__ void merge_kernel(MergeArgs a) {
    const uint32_t tp = blockIdx.x, r = threadIdx.x;
    const uint32_t pair = a.tp_pair[tp];
    const uint32_t qi = a.tp_qi0[tp] + r;
    if (qi >= a.n_active[pair]) return;
    float best = -INFINITY, second = -INFINITY;
    uint32_t idx = 0;
    for (uint32_t s = 0; s < a.splits; ++s) {
        const float4 p = a.partial[((uint64_t)tp * a.splits + s) * kQueryTilePair + r];
        if (p.x > best) {
            second = fmaxf(second, best);
            best = p.x;
            idx = __float_as_uint(p.z);
        } else {
            second = fmaxf(second, p.x);
        }
        second = fmaxf(second, p.y);
    }
    const uint32_t grow = a.tp_row0[tp] + r;
    if (best - second > a.margin[grow]) {
        a.out[(uint64_t)pair * a.out_stride + qi] = idx;
    } else {
        const uint32_t k = atomicAdd(a.rescan_count, 1u);
        a.rescan[3 * k] = grow;
        a.rescan[3 * k + 1] = pair;
        a.rescan[3 * k + 2] = qi;
        atomicAdd(a.near_ties + pair, 1ull);
    }
}

// ---------------------------------------------------------------- K4' rescan
// Reference FMA chain on binary16 values (packed layout), channels < dim only.
template <bool kL2>
__device__ __forceinline__ float packed_chain(const float* q, const uint8_t* map, uint32_t row, uint32_t dim) {
    float acc = 0.0f;
    for (uint32_t c0 = 0; c0 < dim; c0 += 8) {
        const uint4 raw = *reinterpret_cast<const uint4*>(map + packed_offset(row, c0 >> 3));
        const __half* h = reinterpret_cast<const __half*>(&raw);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            if (c0 + k < dim) {
                const float t = __half2float(h[k]);
                if constexpr (kL2) {
                    const float d = __fsub_rn(q[c0 + k], t);
                    acc = __fmaf_rn(d, d, acc);
                } else {
                    acc = __fmaf_rn(q[c0 + k], t, acc);
                }
            }
        }
    }
    return kL2 ? acc : -acc;
}

__device__ __forceinline__ void load_query(const uint8_t* qbuf, uint32_t grow, uint32_t dim, float* q) {
    for (uint32_t c0 = 0; c0 < dim; c0 += 8) {
        const uint4 raw = *reinterpret_cast<const uint4*>(qbuf + packed_offset(grow, c0 >> 3));
        const __half* h = reinterpret_cast<const __half*>(&raw);
#pragma unroll
        for (int k = 0; k < 8; ++k) q[c0 + k] = __half2float(h[k]);
    }
}

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) {
    return a < b ? a : b;
}

struct RescanArgs {
    const uint32_t* rescan;
    const unsigned int* rescan_count;
    const uint8_t* qbuf;
    const uint8_t* tmap;
    uint64_t t_pair_bytes;
    uint32_t nt;
    uint32_t dim;
    uint32_t chunk;                 // targets per work unit
    unsigned long long* keys;       // per rescan entry
    bool l2;
};

constexpr int kRescanThreads = 256;

template <bool kL2>
__global__ void __launch_bounds__(kRescanThreads) rescan_kernel(RescanArgs a) {
    const uint32_t count = *a.rescan_count;
    const uint32_t nchunks = (a.nt + a.chunk - 1) / a.chunk;
    __shared__ unsigned long long red[kRescanThreads / 32];
    float q[kPackK];
    for (uint32_t unit = blockIdx.x; unit < count * nchunks; unit += gridDim.x) {
        const uint32_t k = unit / nchunks, ch = unit % nchunks;
        const uint32_t grow = a.rescan[3 * k], pair = a.rescan[3 * k + 1];
        load_query(a.qbuf, grow, a.dim, q);
        const uint8_t* tm = a.tmap + pair * a.t_pair_bytes;
        const uint32_t t0 = ch * a.chunk, t1 = min(a.nt, t0 + a.chunk);
        unsigned long long key = ~0ull;
        for (uint32_t t = t0 + threadIdx.x; t < t1; t += kRescanThreads)
            key = umin64(key, (unsigned long long)pack_key(packed_chain<kL2>(q, tm, t, a.dim), t));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) key = umin64(key, __shfl_xor_sync(0xFFFFFFFFu, key, o));
        if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = key;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long m = red[0];
            for (int w = 1; w < kRescanThreads / 32; ++w) m = umin64(m, red[w]);
            atomicMin(a.keys + k, m);
        }
        __syncthreads();
    }
}

__global__ void rescan_finish_kernel(const uint32_t* rescan, const unsigned int* count,
                                     unsigned long long* keys, uint32_t* out, uint32_t out_stride) {
    const uint32_t n = *count;
    for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        out[(uint64_t)rescan[3 * k + 1] * out_stride + rescan[3 * k + 2]] = (uint32_t)(keys[k] & 0xFFFFFFFFull);
        keys[k] = ~0ull;
    }
}

// Exact reference distance of each winner (dense API).
template <bool kL2>
__global__ void winner_dist_kernel(const uint8_t* qbuf, const uint8_t* tmap, uint32_t nq, uint32_t dim,
                                   const uint32_t* nearest, float* min_dist) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nq) return;
    float q[kPackK];
    load_query(qbuf, i, dim, q);
    min_dist[i] = packed_chain<kL2>(q, tmap, nearest[i], dim);
}

// Raw scores of one tile pair x one target tile (UMMA layout self-test).
__global__ void __launch_bounds__(kScanThreads, 1) selftest_kernel(const uint8_t* qbuf, const uint8_t* tmap,
                                                                    float* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    __shared__ uint64_t bar_ld, bar_mma;
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        mbar_init(&bar_ld, 1);
        mbar_init(&bar_mma, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {
        mbar_expect_tx(&bar_ld, kSmemA + kTileBytes);
        bulk_g2s(smem, qbuf, kSmemA, &bar_ld);
        bulk_g2s(smem + kSmemA, tmap, kTileBytes, &bar_ld);
        mbar_wait(&bar_ld, 0);
        tc_fence_after();
        const uint32_t a_addr = smem_addr(smem), b_addr = a_addr + kSmemA;
        for (uint32_t qt = 0; qt < 2; ++qt)
            for (uint32_t ks = 0; ks < 2; ++ks)
                tc_mma_f16(tmem + qt * 128u, umma_desc(a_addr + qt * kTileBytes + ks * 256u),
                           umma_desc(b_addr + ks * 256u), kIdescF16M128N128, ks);
        tc_commit(&bar_mma);
    }
    if (warp >= 2) {
        mbar_wait(&bar_mma, 0);
        tc_fence_after();
        const uint32_t e = warp - 2, qt = e >> 2, quad = warp & 3u;
        const uint32_t row = qt * 128u + quad * 32u + lane;
        float v[32];
        for (int c = 0; c < 4; ++c) {
            tmem_ld32(tmem + ((quad * 32u) << 16) + qt * 128u + 32u * c, v);
            tmem_ld_wait();
            for (int j = 0; j < 32; ++j) out[row * 128 + 32 * c + j] = v[j];
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

uint32_t ceil_div_u(uint32_t a, uint32_t b) { return (a + b - 1) / b; }

#define TRY(x)                         \
    do {                               \
        int _st = (x);                 \
        if (_st != FNL_OK) return _st; \
    } while (0)

bool attr_done = false;

int ensure_attrs() {
    if (attr_done) return FNL_OK;
    FNL_CUDA_TRY(cudaFuncSetAttribute(tc_scan_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemTotal));
    FNL_CUDA_TRY(cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemTotal));
    attr_done = true;
    return FNL_OK;
}

}  // namespace

// ====================================================================== host
int tensor_pack(fnl_context* ctx, const char* tag, const float* d_src, uint32_t npairs, uint32_t rows,
                uint32_t dim, bool l2, unsigned long long* d_bad, unsigned long long* d_sat, PackedMaps* out) {
    if (dim == 0 || dim + (l2 ? 2u : 0u) > kPackK)
        return fail(FNL_EINVAL, "tensor backend: descriptor dim " + std::to_string(dim) + " exceeds " +
                                    std::to_string(l2 ? kPackK - 2 : kPackK) + " (" + (l2 ? "l2" : "dot") +
                                    " metric); use the exact backends");
    const uint32_t rows_pad = ceil_div_u(rows, kTileRows) * kTileRows;
    const uint64_t pair_bytes = (uint64_t)rows_pad * kPackRowBytes;
    std::string t(tag);
    TRY(ws_arr(ctx, (t + ".packed").c_str(), (size_t)npairs * pair_bytes, &out->data));
    TRY(ws_arr(ctx, (t + ".maxnorm").c_str(), npairs, &out->max_norm));
    cudaStream_t s = ctx_stream(ctx);
    FNL_CUDA_TRY(cudaMemsetAsync(out->max_norm, 0, npairs * sizeof(float), s));
    out->pair_bytes = pair_bytes;
    out->rows = rows;
    out->npairs = npairs;
    PackArgs a{d_src, out->data, pair_bytes, rows, rows_pad, dim, l2, out->max_norm, d_bad, d_sat};
    const uint32_t threads = rows_pad * 4;
    dim3 grid(ceil_div_u(threads, 256), npairs);
    pack_kernel<<<grid, 256, 0, s>>>(a);
    FNL_CUDA_TRY(cudaGetLastError());
    ctx_count_launches(ctx, 1);
    return FNL_OK;
}

int tensor_nn_pass(fnl_context* ctx, uint32_t npairs, const PackedMaps& Q, const uint32_t* ids, uint32_t cap,
                   const uint32_t* h_active, const uint8_t* h_done, const PackedMaps& T, uint32_t dim, bool l2,
                   uint32_t* out, uint32_t out_stride, float* min_dist, unsigned long long* d_near_ties) {
    TRY(ensure_attrs());
    cudaStream_t s = ctx_stream(ctx);
    const uint32_t nt = T.rows;
    const uint32_t ntiles = ceil_div_u(nt, kTileRows);

    // ---- host work list: gather slots (one per active pair) and tile pairs
    std::vector<uint32_t> slot_pair, slot_base, tp_pair, tp_row0, tp_qi0;
    uint32_t rows_total = 0;
    for (uint32_t p = 0; p < npairs; ++p) {
        if (h_active[p] == 0 || (h_done && h_done[p])) continue;
        slot_pair.push_back(p);
        slot_base.push_back(rows_total);
        const uint32_t ntp = ceil_div_u(h_active[p], kQueryTilePair);
        for (uint32_t j = 0; j < ntp; ++j) {
            tp_pair.push_back(p);
            tp_row0.push_back(rows_total + j * kQueryTilePair);
            tp_qi0.push_back(j * kQueryTilePair);
        }
        rows_total += ntp * kQueryTilePair;
    }
    if (slot_pair.empty()) return FNL_OK;
    const uint32_t ntp = (uint32_t)tp_pair.size();
    // Target splits: pick the split count that minimises the modelled makespan
    // (waves of one CTA per SM x (tiles per CTA + fixed prologue cost)).
    const uint32_t sms = (uint32_t)ctx_sm_count(ctx);
    uint32_t best_s = 1;
    double best_cost = 1e300;
    for (uint32_t sp = 1; sp <= std::min<uint32_t>(ntiles, 64); ++sp) {
        const double waves = std::ceil((double)ntp * sp / sms);
        const double cost = waves * (std::ceil((double)ntiles / sp) + 24.0);
        if (cost < best_cost - 1e-9) {
            best_cost = cost;
            best_s = sp;
        }
    }
    const uint32_t per = ceil_div_u(ntiles, best_s);
    const uint32_t splits = ceil_div_u(ntiles, per);
    std::vector<TcItem> items;
    items.reserve((size_t)ntp * splits);
    for (uint32_t j = 0; j < ntp; ++j)
        for (uint32_t sp = 0; sp < splits; ++sp)
            items.push_back({tp_pair[j], tp_row0[j], sp * per, std::min(ntiles, (sp + 1) * per)});
    const uint32_t nitems = (uint32_t)items.size();
    const uint32_t nslots = (uint32_t)slot_pair.size();

    // ---- stage the lists (pinned, alternating halves so an in-flight copy of
    // the previous pass is never overwritten)
    static thread_local int flip = 0;
    flip ^= 1;
    const size_t words = 2 * (size_t)nslots + 3 * (size_t)ntp + 4 * (size_t)nitems;
    uint32_t* pin = nullptr;
    uint32_t* dlist = nullptr;
    TRY(ws_pinned(ctx, flip ? "tc.list.pin1" : "tc.list.pin0", words * 4, (void**)&pin));
    TRY(ws_arr(ctx, flip ? "tc.list1" : "tc.list0", words, &dlist));
    uint32_t* w = pin;
    std::copy(slot_pair.begin(), slot_pair.end(), w);
    std::copy(slot_base.begin(), slot_base.end(), w + nslots);
    std::copy(tp_pair.begin(), tp_pair.end(), w + 2 * nslots);
    std::copy(tp_row0.begin(), tp_row0.end(), w + 2 * nslots + ntp);
    std::copy(tp_qi0.begin(), tp_qi0.end(), w + 2 * nslots + 2 * ntp);
    memcpy(w + 2 * nslots + 3 * ntp, items.data(), items.size() * sizeof(TcItem));
    FNL_CUDA_TRY(cudaMemcpyAsync(dlist, pin, words * 4, cudaMemcpyHostToDevice, s));
    const uint32_t* d_slot_pair = dlist;
    const uint32_t* d_slot_base = dlist + nslots;
    const uint32_t* d_tp_pair = dlist + 2 * nslots;
    const uint32_t* d_tp_row0 = d_tp_pair + ntp;
    const uint32_t* d_tp_qi0 = d_tp_row0 + ntp;
    const TcItem* d_items = reinterpret_cast<const TcItem*>(d_tp_qi0 + ntp);

    // ---- device scratch
    uint8_t* qbuf;
    float* margin;
    float4* partial;
    uint32_t* rescan;
    unsigned int* rcount;
    unsigned long long* keys;
    uint32_t* d_active;
    TRY(ws_arr(ctx, "tc.qbuf", (size_t)rows_total * kPackRowBytes, &qbuf));
    TRY(ws_arr(ctx, "tc.margin", rows_total, &margin));
    TRY(ws_arr(ctx, "tc.partial", (size_t)nitems * kQueryTilePair, &partial));
    TRY(ws_arr(ctx, "tc.rescan", (size_t)3 * rows_total, &rescan));
    TRY(ws_arr(ctx, "tc.rcount", 1, &rcount));
    TRY(ws_arr(ctx, "tc.keys", rows_total, &keys));
    TRY(ws_arr(ctx, "tc.active", npairs, &d_active));
    // active counts as the host saw them (the pass must use exactly these)
    uint32_t* pin_act = nullptr;
    TRY(ws_pinned(ctx, flip ? "tc.act.pin1" : "tc.act.pin0", npairs * 4, (void**)&pin_act));
    memcpy(pin_act, h_active, npairs * 4);
    FNL_CUDA_TRY(cudaMemcpyAsync(d_active, pin_act, npairs * 4, cudaMemcpyHostToDevice, s));
    FNL_CUDA_TRY(cudaMemsetAsync(rcount, 0, 4, s));
    FNL_CUDA_TRY(cudaMemsetAsync(keys, 0xFF, (size_t)rows_total * 8, s));

    // ---- K2 gather
    {
        GatherArgs g{Q.data, Q.pair_bytes, ids, cap, d_active, d_slot_pair, d_slot_base, qbuf, margin,
                     T.max_norm, dim, l2};
        uint32_t max_rows = 0;
        for (uint32_t p : slot_pair) max_rows = std::max(max_rows, ceil_div_u(h_active[p], kQueryTilePair) * kQueryTilePair);
        dim3 grid(ceil_div_u(max_rows * 4, 256), nslots);
        gather_kernel<<<grid, 256, 0, s>>>(g);
        FNL_CUDA_TRY(cudaGetLastError());
    }
    // ---- K3 tensor-core scan (the dominant kernel; timed)
    {
        TcArgs t{qbuf, margin, T.data, T.pair_bytes, nt, d_items, partial};
        cudaEvent_t end_ev;
        ctx_score_begin(ctx, &end_ev);
        tc_scan_kernel<<<nitems, kScanThreads, kSmemTotal, s>>>(t);
        ctx_score_end(ctx, end_ev);
        FNL_CUDA_TRY(cudaGetLastError());
    }
    // ---- K3b merge + certification
    {
        MergeArgs m{partial, d_tp_pair, d_tp_row0, d_tp_qi0, splits, d_active, margin, out, out_stride,
                    rescan, rcount, d_near_ties};
        merge_kernel<<<ntp, kQueryTilePair, 0, s>>>(m);
        FNL_CUDA_TRY(cudaGetLastError());
    }
    // ---- K4' exact re-decision of near ties (grid-stride over a device count)
    {
        RescanArgs r{rescan, rcount, qbuf, T.data, T.pair_bytes, nt, dim, 4096u, keys, l2};
        const uint32_t grid = 2 * (uint32_t)ctx_sm_count(ctx);
        if (l2) rescan_kernel<true><<<grid, kRescanThreads, 0, s>>>(r);
        else rescan_kernel<false><<<grid, kRescanThreads, 0, s>>>(r);
        FNL_CUDA_TRY(cudaGetLastError());
        rescan_finish_kernel<<<4, 256, 0, s>>>(rescan, rcount, keys, out, out_stride);
        FNL_CUDA_TRY(cudaGetLastError());
    }
    if (min_dist) {  // dense API only: single slot, identity rows
        const uint32_t nq = h_active[slot_pair[0]];
        if (l2) winner_dist_kernel<true><<<ceil_div_u(nq, 256), 256, 0, s>>>(qbuf, T.data, nq, dim, out, min_dist);
        else winner_dist_kernel<false><<<ceil_div_u(nq, 256), 256, 0, s>>>(qbuf, T.data, nq, dim, out, min_dist);
        FNL_CUDA_TRY(cudaGetLastError());
    }
    ctx_count_launches(ctx, 5 + (min_dist ? 1 : 0));
    return FNL_OK;
}

int tensor_nn_dense(fnl_context* ctx, const float* d_q, uint32_t nq, const float* d_t, uint32_t nt,
                    uint32_t dim, bool l2, uint32_t* d_nearest, float* d_min_dist) {
    unsigned long long* scratch;
    TRY(ws_arr(ctx, "tc.dense.scratch", 4, &scratch));
    cudaStream_t s = ctx_stream(ctx);
    FNL_CUDA_TRY(cudaMemsetAsync(scratch, 0xFF, 16, s));
    FNL_CUDA_TRY(cudaMemsetAsync(scratch + 2, 0, 16, s));
    PackedMaps Q, T;
    TRY(tensor_pack(ctx, "tc.dense.q", d_q, 1, nq, dim, l2, scratch, scratch + 2, &Q));
    TRY(tensor_pack(ctx, "tc.dense.t", d_t, 1, nt, dim, l2, scratch + 1, scratch + 3, &T));
    unsigned long long* ties;
    TRY(ws_arr(ctx, "tc.dense.ties", 1, &ties));
    FNL_CUDA_TRY(cudaMemsetAsync(ties, 0, 8, s));
    const uint8_t done = 0;
    return tensor_nn_pass(ctx, 1, Q, nullptr, nq, &nq, &done, T, dim, l2, d_nearest, nq, d_min_dist, ties);
}

int tensor_selftest_scores(fnl_context* ctx, const float* d_q, const float* d_t, uint32_t dim, bool l2,
                           float* d_out) {
    TRY(ensure_attrs());
    unsigned long long* scratch;
    TRY(ws_arr(ctx, "tc.st.scratch", 4, &scratch));
    cudaStream_t s = ctx_stream(ctx);
    FNL_CUDA_TRY(cudaMemsetAsync(scratch, 0xFF, 16, s));
    FNL_CUDA_TRY(cudaMemsetAsync(scratch + 2, 0, 16, s));
    PackedMaps Q, T;
    TRY(tensor_pack(ctx, "tc.st.q", d_q, 1, kQueryTilePair, dim, l2, scratch, scratch + 2, &Q));
    TRY(tensor_pack(ctx, "tc.st.t", d_t, 1, kTileRows, dim, l2, scratch + 1, scratch + 3, &T));
    // query role of the l2 channels, as the gather writes it
    uint8_t* qbuf;
    float* margin;
    uint32_t *act, *lists;
    TRY(ws_arr(ctx, "tc.st.qbuf", (size_t)kQueryTilePair * kPackRowBytes, &qbuf));
    TRY(ws_arr(ctx, "tc.st.margin", kQueryTilePair, &margin));
    TRY(ws_arr(ctx, "tc.st.act", 1, &act));
    TRY(ws_arr(ctx, "tc.st.lists", 2, &lists));
    const uint32_t host[2] = {0, 0};
    const uint32_t n = kQueryTilePair;
    FNL_CUDA_TRY(cudaMemcpyAsync(act, &n, 4, cudaMemcpyHostToDevice, s));
    FNL_CUDA_TRY(cudaMemcpyAsync(lists, host, 8, cudaMemcpyHostToDevice, s));
    GatherArgs g{Q.data, Q.pair_bytes, nullptr, n, act, lists, lists + 1, qbuf, margin, T.max_norm, dim, l2};
    gather_kernel<<<dim3(4, 1), 256, 0, s>>>(g);
    FNL_CUDA_TRY(cudaGetLastError());
    selftest_kernel<<<1, kScanThreads, kSmemTotal, s>>>(qbuf, T.data, d_out);
    FNL_CUDA_TRY(cudaGetLastError());
    FNL_CUDA_TRY(cudaStreamSynchronize(s));
    return FNL_OK;
}

}  // namespace fnl
