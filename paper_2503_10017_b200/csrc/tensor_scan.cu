// tensor_scan.cu -- the FastNN-Lite hot path on the 5th-gen tensor cores.
//
//   K1 pack     fp32 map -> binary16 rows (RNE + saturation, counted) in the UMMA
//               canonical K-major layout, row norms, per-map max norm.
//   K2p plan    per-pass work lists from the device state (no host round trip).
//   K2 gather   active query rows -> contiguous 256-row query tile pairs, plus the
//               per-row one-sided certification margin of the resolve mode.
//   K3 scan     persistent, one CTA per SM: 256 queries x a range of 256-target
//               tiles.  Warp 0 streams target tiles global->smem with
//               cp.async.bulk through a 4-deep mbarrier ring; warps 1-2 (one
//               per query tile) issue tcgen05.mma.cta_group::1.kind::f16 (M128
//               N128 K16, two K steps) into four 128-column fp32 TMEM
//               accumulator chains (query tile x 128-target half = all 512
//               columns); 16 epilogue warps drain TMEM with tcgen05.ld and keep,
//               per query row, the top-4 maxima of 64-target sub-tiles (with the
//               first three sub-tile ids) in registers.  The score matrix never
//               leaves the SM.
//   K3b merge   per row over target splits: resolve the best sub-tile with the
//               reference FMA chain in the mode's arithmetic, close the row when
//               the exact winner beats the next bound by the margin, else the
//               second and third sub-tiles.
//   K4' rescan  rows still open (four sub-tiles inside the margin) re-run the
//               exact chain over every target; lowest index on exact ties.
//
// Score convention: larger is better.  dot: s = q.t (dist = -s).  l2: the
// packed target carries -|t|^2/2 as two binary16 terms (hi + lo) in channels
// d, d+1 and the gathered query carries 1.0 there, so s = q.t - |t|^2/2 and
// dist = |q|^2 - 2 s.  Both are monotone in the reference distance, so argmax s
// == argmin dist up to rounding, which the margin covers.
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <mutex>
#include <string>
#include <vector>

#include "fastnn_b200.h"
#include "fnl_common.cuh"
#include "fnl_internal.h"
#include "tensor_scan.h"
#include "tc_ptx.cuh"

namespace fnl {

namespace {

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

// gathered query tiles (qbuf, K3's A operand): row-group-major, 512 B per 8 rows
__host__ __device__ __forceinline__ uint64_t packed_offset(uint32_t row, uint32_t chunk) {
    return (uint64_t)(row >> 3) * 512u + chunk * 128u + (row & 7u) * 16u;
}
// packed maps (K3's B operand): chunk-major per 256-row tile, cpr chunks stored
__host__ __device__ __forceinline__ uint64_t map_offset(uint32_t row, uint32_t chunk, uint32_t cpr) {
    return (uint64_t)(row >> 8) * cpr * kChunkBytes + chunk * kChunkBytes + ((row >> 3) & 31u) * 128u +
           (row & 7u) * 16u;
}
// B-operand descriptor of the chunk-major layout: LBO 4 KB (next chunk), SBO
// 128 B (next 8-row group)
__device__ __forceinline__ uint64_t umma_desc_b(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFFu) | ((uint64_t)(kChunkBytes >> 4) << 16) | ((uint64_t)(128u >> 4) << 32) |
           (1ull << 46);
}

__device__ __forceinline__ uint32_t pack_half2(float a, float b) {
    const __half2 h = __floats2half2_rn(a, b);
    return *reinterpret_cast<const uint32_t*>(&h);
}

// ---------------------------------------------------------------- K1 pack
// HBM-bound stream: 4 lanes per row (one 8-channel chunk each), so a warp
// covers one 8-row group = 768 B of fp32 in and 512 B of binary16 out, both
// fully coalesced.  Blocks are persistent per pair (grid-stride over the
// pair's row groups, two groups in flight per warp), and the per-pair max
// norm / saturation count are reduced in the block, so a map costs a handful
// of atomics instead of one per warp.
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
    float* max_norm_hi;              // per pair: max norm over packed channels 16..31
    uint32_t cpr;                    // stored chunks per row
};

constexpr int kPackThreads = 256;

__device__ __forceinline__ void pack_load(const PackArgs& a, const float* src, uint32_t row, uint32_t chunk,
                                          float (&v)[8]) {
    const bool real = row < a.rows;
    const bool vec = (a.dim & 7u) == 0 && chunk * 8 < a.dim;  // whole 8-channel chunk, 32 B aligned
    if (real && vec) {
        const float4 lo = __ldcs(reinterpret_cast<const float4*>(src + (uint64_t)row * a.dim + chunk * 8));
        const float4 hi = __ldcs(reinterpret_cast<const float4*>(src + (uint64_t)row * a.dim + chunk * 8 + 4));
        v[0] = lo.x; v[1] = lo.y; v[2] = lo.z; v[3] = lo.w;
        v[4] = hi.x; v[5] = hi.y; v[6] = hi.z; v[7] = hi.w;
    } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const uint32_t c = chunk * 8 + i;
            v[i] = (real && c < a.dim) ? src[(uint64_t)row * a.dim + c] : 0.0f;
        }
    }
}

// rounds one row chunk, writes it, returns the row's squared norm (0 for padding rows)
__device__ __forceinline__ float pack_store(const PackArgs& a, uint8_t* dst, uint32_t pair, uint32_t row,
                                            uint32_t chunk, float (&v)[8], uint32_t& sat, float& nmax_hi) {
    const bool real = row < a.rows;
    float ss = 0.0f;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        float x = v[i];
        if (!isfinite(x)) atomicMin(a.bad + pair, (unsigned long long)row * a.dim + chunk * 8 + i);
        x = half_round_sat(x, sat);
        v[i] = x;
        ss = __fmaf_rn(x, x, ss);
    }
    // row norm^2 over the 4 chunk lanes (fixed order -> deterministic); after
    // the first step lanes 2-3 hold the norm^2 of channels 16..31.  Maxima are
    // kept squared (one sqrt per flush)
    ss += __shfl_xor_sync(0xFFFFFFFFu, ss, 1);
    if (real && chunk >= 2) nmax_hi = fmaxf(nmax_hi, ss);
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
    if (chunk < a.cpr) {  // chunks past cpr hold no data (zero for this map)
        uint4 out;
        out.x = pack_half2(v[0], v[1]);
        out.y = pack_half2(v[2], v[3]);
        out.z = pack_half2(v[4], v[5]);
        out.w = pack_half2(v[6], v[7]);
        *reinterpret_cast<uint4*>(dst + map_offset(row, chunk, a.cpr)) = out;
    }
    return real ? ss : 0.0f;
}

__device__ __forceinline__ void pack_flush(const PackArgs& a, uint32_t pair, uint32_t& sat, float& nmax,
                                           float& nmax_hi) {
    sat = warp_sum(sat);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nmax = fmaxf(nmax, __shfl_xor_sync(0xFFFFFFFFu, nmax, o));
        nmax_hi = fmaxf(nmax_hi, __shfl_xor_sync(0xFFFFFFFFu, nmax_hi, o));
    }
    if ((threadIdx.x & 31u) == 0) {
        if (sat) atomicAdd(a.sat + pair, (unsigned long long)sat);
        // non-negative floats order like their bits (maxima of squared norms)
        nmax = sqrtf(nmax);
        nmax_hi = sqrtf(nmax_hi);
        if (nmax > 0.0f) atomicMax(reinterpret_cast<unsigned int*>(a.max_norm) + pair, __float_as_uint(nmax));
        if (nmax_hi > 0.0f)
            atomicMax(reinterpret_cast<unsigned int*>(a.max_norm_hi) + pair, __float_as_uint(nmax_hi));
    }
    sat = 0;
    nmax = 0.0f;
    nmax_hi = 0.0f;
}

// Flat over (pair, 8-row group): warp w owns a contiguous range of groups of
// the whole batch (exactly one wave of warps, no tail), two groups in flight;
// counters are flushed once per pair the warp touches.
__global__ void __launch_bounds__(kPackThreads) pack_kernel(PackArgs a, uint32_t npairs) {
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t chunk = lane & 3u, sub = lane >> 2;
    const uint32_t groups = a.rows_pad >> 3;
    const uint64_t total = (uint64_t)npairs * groups;
    const uint64_t nwarps = (uint64_t)gridDim.x * (kPackThreads / 32);
    const uint64_t w = (uint64_t)blockIdx.x * (kPackThreads / 32) + (threadIdx.x >> 5);
    uint64_t g = total * w / nwarps;
    const uint64_t end = total * (w + 1) / nwarps;
    if (g >= end) return;
    uint32_t pair = (uint32_t)(g / groups);
    uint32_t sat = 0;
    float nmax = 0.0f, nmax_hi = 0.0f;
    while (g < end) {
        const uint32_t gi = (uint32_t)(g - (uint64_t)pair * groups);
        const float* src = a.src + (uint64_t)pair * a.rows * a.dim;
        uint8_t* dst = a.dst + pair * a.pair_bytes;
        // groups of this pair left in this warp's range, two at a time
        const uint64_t left = end - g;
        const uint32_t n = left < (uint64_t)(groups - gi) ? (uint32_t)left : groups - gi;
        uint32_t j = 0;
        for (; j + 3 < n; j += 4) {  // four row groups (3 KB of fp32) in flight per warp
            float v[4][8];
            const uint32_t r0 = (gi + j) * 8 + sub;
#pragma unroll
            for (int q = 0; q < 4; ++q) pack_load(a, src, r0 + 8 * q, chunk, v[q]);
#pragma unroll
            for (int q = 0; q < 4; ++q) nmax = fmaxf(nmax, pack_store(a, dst, pair, r0 + 8 * q, chunk, v[q], sat, nmax_hi));
        }
        for (; j + 1 < n; j += 2) {
            float v0[8], v1[8];
            const uint32_t r0 = (gi + j) * 8 + sub, r1 = r0 + 8;
            pack_load(a, src, r0, chunk, v0);
            pack_load(a, src, r1, chunk, v1);
            nmax = fmaxf(nmax, pack_store(a, dst, pair, r0, chunk, v0, sat, nmax_hi));
            nmax = fmaxf(nmax, pack_store(a, dst, pair, r1, chunk, v1, sat, nmax_hi));
        }
        if (j < n) {
            float v0[8];
            const uint32_t r0 = (gi + j) * 8 + sub;
            pack_load(a, src, r0, chunk, v0);
            nmax = fmaxf(nmax, pack_store(a, dst, pair, r0, chunk, v0, sat, nmax_hi));
        }
        pack_flush(a, pair, sat, nmax, nmax_hi);
        g += n;
        ++pair;
    }
}

// K1 v2 (TMA-staged): one thread per target row.  A 256-row target tile of
// fp32 rows is one contiguous block (256 x dim x 4 B, 24 KB at d = 24), so a
// single cp.async.bulk stages it into shared memory; persistent blocks keep
// kPackStages tiles in flight (the copy engine, not warps, holds the bytes in
// flight), each thread rounds its own row (no idle lane for d = 24, no norm
// shuffles) and writes the row's cpr chunks, which are contiguous across the
// threads of a warp in the chunk-major layout.  Same outputs, bit for bit, as
// pack_kernel (norm^2 summed per 8-channel chunk, then (s0 + s1) + (s2 + s3)).
// Needs rows x dim to be a multiple of 4 (16-byte tile sizes); else K1 v1.
constexpr int kPackStages = 3;
constexpr uint32_t kPackTileRows = 256;

__device__ __forceinline__ void pack2_flush(const PackArgs& a, uint32_t pair, uint32_t& sat, float& nmax,
                                            float& nmax_hi) {
    sat = warp_sum(sat);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        nmax = fmaxf(nmax, __shfl_xor_sync(0xFFFFFFFFu, nmax, o));
        nmax_hi = fmaxf(nmax_hi, __shfl_xor_sync(0xFFFFFFFFu, nmax_hi, o));
    }
    if ((threadIdx.x & 31u) == 0) {
        if (sat) atomicAdd(a.sat + pair, (unsigned long long)sat);
        nmax = sqrtf(nmax);
        nmax_hi = sqrtf(nmax_hi);
        if (nmax > 0.0f) atomicMax(reinterpret_cast<unsigned int*>(a.max_norm) + pair, __float_as_uint(nmax));
        if (nmax_hi > 0.0f)
            atomicMax(reinterpret_cast<unsigned int*>(a.max_norm_hi) + pair, __float_as_uint(nmax_hi));
    }
    sat = 0;
    nmax = 0.0f;
    nmax_hi = 0.0f;
}

__global__ void __launch_bounds__(kPackTileRows) pack_tma_kernel(PackArgs a, uint32_t npairs) {
    extern __shared__ __align__(128) uint8_t psm[];
    __shared__ __align__(8) uint64_t full[kPackStages];
    const uint32_t tid = threadIdx.x;
    const uint32_t tiles_per_pair = a.rows_pad / kPackTileRows;
    const uint64_t total = (uint64_t)npairs * tiles_per_pair;
    const uint32_t stage_bytes = kPackTileRows * a.dim * 4u;
    const uint64_t i0 = total * blockIdx.x / gridDim.x, i1 = total * (blockIdx.x + 1) / gridDim.x;
    if (i0 >= i1) return;
    auto issue = [&](uint64_t i, uint32_t st) {
        const uint32_t pair = (uint32_t)(i / tiles_per_pair);
        const uint32_t r0 = (uint32_t)(i - (uint64_t)pair * tiles_per_pair) * kPackTileRows;
        const uint32_t nrows = r0 < a.rows ? min(kPackTileRows, a.rows - r0) : 0u;
        if (nrows == 0) {
            mbar_arrive(&full[st]);  // an all-padding tile: nothing to stage
            return;
        }
        const uint32_t bytes = nrows * a.dim * 4u;
        mbar_expect_tx(&full[st], bytes);
        bulk_g2s(psm + st * stage_bytes, a.src + ((uint64_t)pair * a.rows + r0) * a.dim, bytes, &full[st]);
    };
    if (tid == 0) {
        for (int st = 0; st < kPackStages; ++st) mbar_init(&full[st], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (uint32_t st = 0; st < kPackStages && i0 + st < i1; ++st) issue(i0 + st, st);
    }
    __syncthreads();
    uint32_t cur = (uint32_t)(i0 / tiles_per_pair);
    uint32_t sat = 0;
    float nmax = 0.0f, nmax_hi = 0.0f;
    for (uint64_t i = i0; i < i1; ++i) {
        const uint32_t k = (uint32_t)(i - i0), st = k % kPackStages;
        const uint32_t pair = (uint32_t)(i / tiles_per_pair);
        if (pair != cur) {  // block-uniform
            pack2_flush(a, cur, sat, nmax, nmax_hi);
            cur = pair;
        }
        const uint32_t r0 = (uint32_t)(i - (uint64_t)pair * tiles_per_pair) * kPackTileRows;
        const uint32_t row = r0 + tid;
        const bool real = row < a.rows;
        mbar_wait(&full[st], (k / kPackStages) & 1u);
        float v[kPackK];
        const float* srow = reinterpret_cast<const float*>(psm + st * stage_bytes) + tid * a.dim;
        if ((a.dim & 3u) == 0) {
#pragma unroll
            for (uint32_t c = 0; c < kPackK; c += 4) {
                float4 x = make_float4(0.0f, 0.0f, 0.0f, 0.0f);
                if (real && c < a.dim) x = *reinterpret_cast<const float4*>(srow + c);
                v[c] = x.x, v[c + 1] = x.y, v[c + 2] = x.z, v[c + 3] = x.w;
            }
        } else {
#pragma unroll
            for (uint32_t c = 0; c < kPackK; ++c) v[c] = (real && c < a.dim) ? srow[c] : 0.0f;
        }
        __syncthreads();  // every row of the stage is in registers: refill it
        if (tid == 0 && i + kPackStages < i1) issue(i + kPackStages, st);
        float s4[4];
#pragma unroll
        for (int ch = 0; ch < 4; ++ch) {
            float ss = 0.0f;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const int c = ch * 8 + j;
                float x = v[c];
                if (!isfinite(x)) atomicMin(a.bad + pair, (unsigned long long)row * a.dim + c);
                x = half_round_sat(x, sat);
                v[c] = x;
                ss = __fmaf_rn(x, x, ss);
            }
            s4[ch] = ss;
        }
        const float hi2 = s4[2] + s4[3];
        const float n2 = (s4[0] + s4[1]) + hi2;
        if (real) {
            nmax = fmaxf(nmax, n2);
            nmax_hi = fmaxf(nmax_hi, hi2);
            if (a.l2) {
                const float half_n2 = -0.5f * n2;
                const float h = __half2float(__float2half_rn(half_n2));
                const float l = __half2float(__float2half_rn(half_n2 - h));
#pragma unroll
                for (uint32_t c = 0; c < kPackK; ++c) {
                    if (c == a.dim) v[c] = h;
                    if (c == a.dim + 1) v[c] = l;
                }
            }
        }
        uint8_t* dst = a.dst + (uint64_t)pair * a.pair_bytes;
#pragma unroll
        for (uint32_t ch = 0; ch < 4; ++ch) {
            if (ch < a.cpr) {
                uint4 out;
                out.x = pack_half2(v[8 * ch], v[8 * ch + 1]);
                out.y = pack_half2(v[8 * ch + 2], v[8 * ch + 3]);
                out.z = pack_half2(v[8 * ch + 4], v[8 * ch + 5]);
                out.w = pack_half2(v[8 * ch + 6], v[8 * ch + 7]);
                *reinterpret_cast<uint4*>(dst + map_offset(row, ch, a.cpr)) = out;
            }
        }
    }
    pack2_flush(a, cur, sat, nmax, nmax_hi);
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
    const uint32_t* nslots;  // device slot count (plan header), or null = gridDim.y
    int mode;                // ResolveMode the margin is for
    // the original fp32 query-side maps (pair stride in floats), or null: a
    // query row is then read as dim contiguous floats (96 B at d = 24) and
    // rounded like K1, instead of as four 16-byte chunks spread over four
    // 128-byte lines of the packed layout (3.9x DRAM over-fetch, round 1)
    const float* q32;
    uint64_t q32_pair_stride;
    bool acc16;  // K3 accumulates in binary16: add its first rounding to the margin
    const float* tmax_hi;  // per pair max target norm over channels 16..31 (acc16)
    uint32_t qcpr;         // stored chunks per row of qmap
};

__global__ void gather_kernel(GatherArgs a) {
    const uint32_t slot = blockIdx.y;
    if (a.nslots && slot >= *a.nslots) return;
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
        __half h[8];
        if (a.q32) {
            const float* row = a.q32 + pair * a.q32_pair_stride + (uint64_t)src_row * a.dim;
            float v[8];
            if ((a.dim & 3u) == 0 && chunk * 8 + 8 <= a.dim) {
                const float4 lo = __ldg(reinterpret_cast<const float4*>(row + chunk * 8));
                const float4 hi = __ldg(reinterpret_cast<const float4*>(row + chunk * 8 + 4));
                v[0] = lo.x; v[1] = lo.y; v[2] = lo.z; v[3] = lo.w;
                v[4] = hi.x; v[5] = hi.y; v[6] = hi.z; v[7] = hi.w;
            } else {
#pragma unroll
                for (int k = 0; k < 8; ++k) v[k] = chunk * 8 + k < a.dim ? __ldg(row + chunk * 8 + k) : 0.0f;
            }
            uint32_t sat = 0;  // counted by K1
#pragma unroll
            for (int k = 0; k < 8; ++k) h[k] = __float2half_rn(half_round_sat(v[k], sat));
        } else {
            val = chunk < a.qcpr ? *reinterpret_cast<const uint4*>(a.qmap + pair * a.qmap_pair_bytes +
                                                                   map_offset(src_row, chunk, a.qcpr))
                                 : make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(h) = val;
        }
        // query role: channels dim, dim+1 become 1.0 (l2) / 0 (dot)
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t c = chunk * 8 + k;
            if (c >= a.dim) h[k] = __float2half_rn((a.l2 && (c == a.dim || c == a.dim + 1)) ? 1.0f : 0.0f);
            const float x = __half2float(h[k]);
            if (c < a.dim) ss = __fmaf_rn(x, x, ss);
        }
        val = *reinterpret_cast<uint4*>(h);
    }
    float sh = chunk >= 2 ? ss : 0.0f;  // channels 16..31: the binary16 accumulator's first K step
    ss += __shfl_xor_sync(0xFFFFFFFFu, ss, 1);
    ss += __shfl_xor_sync(0xFFFFFFFFu, ss, 2);
    sh += __shfl_xor_sync(0xFFFFFFFFu, sh, 1);
    sh += __shfl_xor_sync(0xFFFFFFFFu, sh, 2);
    *reinterpret_cast<uint4*>(a.qbuf + packed_offset(drow, chunk)) = val;
    if (chunk == 0) {
        // One-sided certification margin M (score units, larger is better):
        // for EVERY target t, the score the resolve mode's exact arithmetic
        // gives t is <= tc_score(t) + M, so a target whose tensor-core score
        // bound B satisfies exact_winner > B + M provably loses (DESIGN.md
        // "certified argmax").  Terms, with |q| <= qn and |t| <= tn:
        //   tensor-core accumulation          2^-15 (qn tn + tn^2 [l2])
        //   reference FMA chain rounding      (d+2) 2^-24 qn tn            (dot)
        //                                     (d+2) 2^-25 (qn + tn)^2      (l2, half a distance)
        //   l2: -|t|^2/2 as binary16 hi + lo  2^-20 tn^2, query |q|^2 chain (d+2) 2^-25 qn^2
        //   kResolveFull: binary16 input rounding of q and t (u = 2^-11, subnormal step 2^-24)
        //                                     2^-10 qn tn + 2^-24 sqrt(d) (qn + tn) (+ 2^-11 tn^2 l2)
        // The norms are of the binary16 rows; the fp32 rows differ by <= u
        // relative plus 2^-25 per channel, covered by the 1.001 / additive
        // inflation.
        const float d = (float)a.dim, sd = sqrtf(d);
        const float qn = sqrtf(ss) * 1.001f + ldexpf(sd, -24);
        const float tn = a.tmax[pair] * 1.001f + ldexpf(sd, -24);
        const bool full = a.mode == kResolveFull;
        float m;
        if (!a.l2) {
            const float A = qn * tn;
            m = ldexpf(A, -15) + (d + 2.0f) * ldexpf(A, -24);
            if (full) m += ldexpf(A, -10) + ldexpf(sd * (qn + tn), -24);
            // binary16 accumulator (K3 issues channels 16..31 first): the first
            // K step's partial sum, |.| <= |q_hi| |t_hi| by Cauchy-Schwarz, is
            // rounded to binary16 once (2^-11 relative, 2^-25 absolute below the
            // normal range); the final rounding, 2^-11 of the score itself, is
            // added by the merge from the bound it compares against
            if (a.acc16) {
                const float qh = sqrtf(sh) * 1.001f + ldexpf(sd, -24);
                const float th = a.tmax_hi[pair] * 1.001f + ldexpf(sd, -24);
                m += 1.001f * ldexpf(qh * th, -11) + ldexpf(1.0f, -23);
            }
        } else {
            const float A = qn * tn + tn * tn;
            const float S = (qn + tn) * (qn + tn);
            m = ldexpf(A, -15) + (d + 2.0f) * ldexpf(S, -25) + ldexpf(tn * tn, -20) + (d + 2.0f) * ldexpf(qn * qn, -25);
            if (full) m += ldexpf(qn * tn, -10) + ldexpf(tn * tn, -11) + ldexpf(sd * (qn + tn), -24);
            // binary16 accumulator: the first K step (channels 16..31) also holds
            // the -|t|^2/2 terms when dim >= 14: |partial| <= |q_hi| |t_hi| + |t|^2/2
            if (a.acc16) {
                const float qh = sqrtf(sh) * 1.001f + ldexpf(sd, -24);
                const float th = a.tmax_hi[pair] * 1.001f + ldexpf(sd, -24);
                m += 1.001f * ldexpf(qh * th + 0.501f * tn * tn, -11) + ldexpf(1.0f, -23);
            }
        }
        a.margin[drow] = 1.25f * m + 1e-30f;
    }
}

// ---------------------------------------------------------------- K3 scan
// A work unit = one query tile pair (256 gathered rows) x a contiguous range of
// 256-target tiles.  The kernel is persistent: CTA b runs units b, b+G, b+2G...
// (static round robin over equal-sized units), so TMEM allocation, barrier
// setup and the pipeline prologue are paid once per SM, and the query tile of
// the next unit is fetched into the second A buffer while the current unit is
// still being scored.
struct TcItem {
    uint32_t pair, qrow0, tile_begin, tile_end;  // qrow0: first gathered row (multiple of 256)
    uint32_t nvalid;                             // real query rows in the tile pair (<= 256)
    uint32_t dual;  // nvalid <= 128: both query tiles score the same 128 rows, query tile 0
                    // over the first half of the tile range, query tile 1 over the second
    uint32_t pad1, pad2;
};
// a tile pair runs in dual mode when its second query tile would be all padding
__host__ __device__ __forceinline__ bool tp_dual(uint32_t nvalid) { return nvalid <= kTileRows; }
// dual mode: steps of a unit, and the first tile of query tile 1
__device__ __forceinline__ uint32_t unit_steps(const TcItem& it) {
    const uint32_t n = it.tile_end - it.tile_begin;
    return it.dual ? (n + 1) / 2 : n;
}
__device__ __forceinline__ uint32_t unit_mid(const TcItem& it) {
    return it.tile_begin + (it.tile_end - it.tile_begin + 1) / 2;
}

struct TcArgs {
    const uint8_t* qbuf;
    const uint8_t* tmap;
    uint64_t t_pair_bytes;
    uint32_t cpr;  // 16-B K chunks stored per target row (chunk-major tiles)
    uint32_t nt;
    const TcItem* items;
    const uint32_t* nitems;  // device item count (plan header)
    float4* partial;  // [item][col half][256][3] = (b1..b4), (b5, b6, t1, t2), (t3, t4, t5 bits, 0)
    int debug;        // profiling only: 1 = epilogue releases buffers unread, 16 = clock trace of CTA 0
    unsigned long long* trace;  // [7][4096] clock64 stamps of CTA 0 (debug & 16, tools/tc_trace.py)
};

// K3 structure (v11; measured on this B200 with the clock traces of
// FNL_TC_DEBUG=16):
//  * a target tile is 256 targets (16 KB, one cp.async.bulk) in a 4-stage ring;
//  * query tile qt (128 rows) owns TMEM columns [256 qt, 256 qt + 256), split
//    into two 128-target halves that are independent accumulator chains; its
//    issuer warp (1 + qt) waits "B landed" and "this half drained", then issues
//    two M128 N128 K16 MMAs (the 24 channels + norm terms padded to K = 32)
//    and one commit per half, so every mbarrier has one producer chain and one
//    consumer chain;
//  * 16 epilogue warps = (query tile, half, TMEM lane quadrant w%4): warps 3-10
//    drain query tile 0, warps 11-18 query tile 1, so one tile's TMEM loads
//    overlap the other tile's compares.
constexpr uint32_t kBTileRows = kTargetTileRows;                // 256 targets per B tile
constexpr uint32_t kBTileBytes = kBTileRows * kPackRowBytes;  // 16 KB
constexpr int kStages = 4;
// warps: 0 loader, 1-2 MMA issuers (query tile 0 / 1), 3..18 epilogue
// (column quarter = (w-3)/4, TMEM lane quadrant = w%4)
constexpr uint32_t kSubPerTile = 4;  // 64-target sub-tiles per 256-target tile
constexpr int kPartialSplit = 2;     // partial states per (work unit, row): one per 128-column half
constexpr int kPartialF4 = 3;        // float4s per partial state: b1..b6, t1..t5
constexpr int kEpiWarps = 16;
constexpr int kFirstEpiWarp = 3;
constexpr int kScanThreads = (kFirstEpiWarp + kEpiWarps) * 32;
constexpr uint32_t kSmemA = 2 * kTileBytes;                  // 16 KB: two query tiles
constexpr uint32_t kStageBytes = 2 * kBTileBytes;            // a stage holds two B tiles (dual mode)
constexpr uint32_t kSmemB = kStages * kStageBytes;           // 128 KB ring
constexpr uint32_t kSmemBars = (2 * kStages + 8 + 2 + 2) * 8;
// A double buffered (next unit's queries load under the current unit); padded
// past half the SM's shared memory so no second CTA co-resides and spins in
// tcgen05.alloc for the 512 TMEM columns.
constexpr uint32_t kSmemUsed = 2 * kSmemA + kSmemB + kSmemBars + 16;
constexpr uint32_t kSmemTotal = kSmemUsed > 120u * 1024u ? kSmemUsed : 120u * 1024u;
constexpr uint32_t kSubTile = 64;  // winner granularity handed to the merge

// Per query row and 64-target sub-tile: m = max of the 64 fp32 scores
// (3-input-max tree, ~0.5 ALU op per score, no data-dependent branch), then a
// branch-free insert of (m, sub-tile) into the row's top-kTopSub of sub-tile maxima:
// b1 >= ... >= b6 with the sub-tiles t1..t5 of the first five.  The merge
// resolves t1, t2, ... with the exact reference chain and closes the row as
// soon as the exact winner beats the next bound by the certification margin;
// only rows with six sub-tiles inside the margin are re-scanned (with binary16
// accumulators the margin is ~2^-11 |q| |t|, and a top-4 state sent ~230 rows
// per 128-pair step to the full rescan).
constexpr int kTopSub = 6;  // <= 6 (partial state: 3 float4)
struct RowState {
    float b[kTopSub];
    uint32_t t[kTopSub - 1];
};
__device__ __forceinline__ RowState row_state_init() {
    RowState st;
#pragma unroll
    for (int i = 0; i < kTopSub; ++i) st.b[i] = -INFINITY;
#pragma unroll
    for (int i = 0; i < kTopSub - 1; ++i) st.t[i] = 0xFFFFFFFFu;
    return st;
}

// Binary16-accumulator path: a sub-tile maximum is an exact binary16 value, so
// as an fp32 its 13 low mantissa bits are zero; they carry the sub-tile index
// relative to the work unit's first tile (< 8192: the plan caps a unit at 2048
// tiles).  Keys of different maxima order like the maxima (the index moves a
// value by less than one binary16 ulp), so the row's top-6 is a plain
// min/max network over keys -- no index selects.
constexpr uint32_t kKeyBits = 13;
constexpr uint32_t kKeyMask = (1u << kKeyBits) - 1u;
constexpr uint32_t kMaxUnitTiles = (1u << kKeyBits) / kSubPerTile;  // 2048
__device__ __forceinline__ float key_of(float m, uint32_t rel) {
    m = fmaxf(m, -0x1p126f);  // -inf (all padding) -> a finite floor, so the index bits stay a number
    return __uint_as_float((__float_as_uint(m) & ~kKeyMask) | rel);
}
__device__ __forceinline__ float key_value(float k) { return __uint_as_float(__float_as_uint(k) & ~kKeyMask); }
__device__ __forceinline__ uint32_t key_rel(float k) { return __float_as_uint(k) & kKeyMask; }
// both keys of a tile half at once: the i-th largest of the union of the
// sorted top-6 and the sorted pair (hi, lo) is max(b_i, min(b_{i-1}, hi),
// min(b_{i-2}, lo)) -- one FMNMX3 and two FMNMX per level, evaluated bottom-up
// on the old values (17 instructions instead of two 12-instruction inserts)
__device__ __forceinline__ void key_insert2(float (&kb)[kTopSub], float k0, float k1) {
    const float hi = fmaxf(k0, k1), lo = fminf(k0, k1);
#pragma unroll
    for (int i = kTopSub - 1; i >= 2; --i) kb[i] = max3(kb[i], fminf(kb[i - 1], hi), fminf(kb[i - 2], lo));
    kb[1] = max3(kb[1], fminf(kb[0], hi), lo);
    kb[0] = fmaxf(kb[0], hi);
}

__device__ __forceinline__ float tile_max64(const float* v) {
    float r[22];
#pragma unroll
    for (int i = 0; i < 21; ++i) r[i] = max3(v[3 * i], v[3 * i + 1], v[3 * i + 2]);
    r[21] = v[63];
    float q[8];
#pragma unroll
    for (int i = 0; i < 7; ++i) q[i] = max3(r[3 * i], r[3 * i + 1], r[3 * i + 2]);
    q[7] = r[21];
    return max3(max3(q[0], q[1], q[2]), max3(q[3], q[4], q[5]), fmaxf(q[6], q[7]));
}

__device__ __forceinline__ void tile_update(RowState& st, float m, uint32_t tile) {
    bool gt[kTopSub - 1];
#pragma unroll
    for (int i = 0; i < kTopSub - 1; ++i) gt[i] = m > st.b[i];
    st.b[kTopSub - 1] = fmaxf(st.b[kTopSub - 1], fminf(st.b[kTopSub - 2], m));
#pragma unroll
    for (int i = kTopSub - 2; i >= 1; --i) {
        st.t[i] = gt[i - 1] ? st.t[i - 1] : (gt[i] ? tile : st.t[i]);
        st.b[i] = fmaxf(st.b[i], fminf(st.b[i - 1], m));
    }
    st.t[0] = gt[0] ? tile : st.t[0];
    st.b[0] = fmaxf(st.b[0], m);
}

// 64 consecutive scores of one row -> sub-tile update (padding masked)
__device__ __forceinline__ void subtile_scan(RowState& st, const Frag& f, const Frag& g, uint32_t sub,
                                             uint32_t nt) {
    float v[64];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
        v[j] = __uint_as_float(f.r[j]);
        v[32 + j] = __uint_as_float(g.r[j]);
    }
    if ((sub + 1) * kSubTile > nt) {  // last, partial sub-tile: padding never wins
#pragma unroll
        for (int j = 0; j < 64; ++j)
            if (sub * kSubTile + j >= nt) v[j] = -INFINITY;
    }
    // most sub-tile maxima fall below the row's third-best (record-breaking
    // statistics: ~3 ln(#sub-tiles) updates per row over a whole scan), so the
    // branch-free top-3 insert runs only when some lane of the warp needs it
    const float m = tile_max64(v);
    if (__any_sync(0xFFFFFFFFu, m > st.b[kTopSub - 1])) tile_update(st, m, sub);
}

// binary16 accumulator variant: 64 scores of one row as 32 packed f16x2
// registers (tcgen05.ld .pack::16b) -> their max (max.f16x2 tree), padding
// columns past nt masked to -inf
__device__ __forceinline__ uint32_t hmax2(uint32_t a, uint32_t b) {
    uint32_t d;
    asm("max.f16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
    return d;
}
__device__ __forceinline__ float tile_max64_h(const Frag& f, uint32_t sub, uint32_t nt) {
    uint32_t v[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) v[j] = f.r[j];
    if ((sub + 1) * kSubTile > nt) {
#pragma unroll
        for (int j = 0; j < 32; ++j) {
            const uint32_t c = sub * kSubTile + 2u * j;
            if (c >= nt) v[j] = (v[j] & 0xFFFF0000u) | 0xFC00u;
            if (c + 1 >= nt) v[j] = (v[j] & 0x0000FFFFu) | 0xFC000000u;
        }
    }
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1)
#pragma unroll
        for (int j = 0; j < w; ++j) v[j] = hmax2(v[j], v[j + w]);
    const float lo = __half2float(__ushort_as_half((unsigned short)(v[0] & 0xFFFFu)));
    const float hi = __half2float(__ushort_as_half((unsigned short)(v[0] >> 16)));
    return fmaxf(lo, hi);
}

// kF16: the accumulators are binary16 (instruction descriptor D format f16,
// dot metric only, margin widened in K2): a warp reads its 128 columns with
// ONE packed tcgen05.ld (64 registers), releases the accumulator at once and
// reduces afterwards with max.f16x2 trees.
// kDebug: the profiling aids of TcArgs::debug (clock trace, unread release)
// are compiled in; the production instantiation carries none of them.
template <bool kF16, bool kDebug>
__global__ void __launch_bounds__(kScanThreads, 1) tc_scan_kernel(TcArgs a) {
    constexpr uint32_t kIdesc = kF16 ? (kIdescF16M128N128 & ~(1u << 4)) : kIdescF16M128N128;
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint32_t tmem_slot;
    uint8_t* sA = smem;                  // [2][16 KB]
    uint8_t* sB = smem + 2 * kSmemA;     // [kStages][2][16 KB]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + 2 * kSmemA + kSmemB);
    uint64_t* full = bars;                     // [kStages]  B tile landed
    uint64_t* empty = bars + kStages;          // [kStages]  both query tiles' MMAs on the slot retired
    uint64_t* tfull = bars + 2 * kStages;      // [2 qt][2 halves]  accumulator half ready
    uint64_t* accfree = tfull + 4;             // [2 qt][2 halves]  accumulator half drained
    uint64_t* afull = accfree + 4;             // [2]
    uint64_t* afree = afull + 2;               // [2]

    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t G = gridDim.x;
    const bool trace = kDebug && (a.debug & 16) && blockIdx.x == 0;
    const uint32_t nitems = *a.nitems;
    if (blockIdx.x >= nitems) return;  // CTA-uniform, before any barrier or TMEM allocation

    if (threadIdx.x == 0) {
        for (int s = 0; s < kStages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 2);  // one commit per issuer
        }
        for (int q = 0; q < 4; ++q) {
            mbar_init(&tfull[q], 1);
            mbar_init(&accfree[q], kEpiWarps / 4);  // the four warps of that query tile and half
        }
        for (int q = 0; q < 2; ++q) {
            mbar_init(&afull[q], 1);
            mbar_init(&afree[q], 2);  // both MMA issuers
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_addr(&tmem_slot)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    // chunks [cpr, 4) of every ring slot are K padding the loads never write:
    // zero them once, visible to the async proxy before the first MMA
    if (a.cpr < 4u) {
        const uint32_t pad = (4u - a.cpr) * kChunkBytes / 16u;  // uint4 per slot
        for (uint32_t i = threadIdx.x; i < 2u * kStages * pad; i += blockDim.x) {
            const uint32_t slot = i / pad;
            reinterpret_cast<uint4*>(sB + slot * kBTileBytes + a.cpr * kChunkBytes)[i - slot * pad] =
                make_uint4(0u, 0u, 0u, 0u);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;

    if (warp == 0) {
        // ---------------- loader: query tile pair per unit, then the target ring
        uint32_t k = 0, i = 0;
        for (uint32_t u = blockIdx.x; u < nitems; u += G, ++i) {
            const TcItem item = a.items[u];
            const uint32_t ab = i & 1u;
            mbar_wait(&afree[ab], ((i >> 1) & 1u) ^ 1u);
            if (elect_one()) {
                mbar_expect_tx(&afull[ab], kSmemA);
                bulk_g2s(sA + ab * kSmemA, a.qbuf + (uint64_t)item.qrow0 * kPackRowBytes, kSmemA, &afull[ab]);
            }
            __syncwarp();
            const uint8_t* tbase = a.tmap + (uint64_t)item.pair * a.t_pair_bytes;
            const uint32_t tb = a.cpr * kChunkBytes;  // stored bytes of one target tile
            const uint32_t steps = unit_steps(item), tmid = unit_mid(item);
            for (uint32_t st = 0; st < steps; ++st, ++k) {
                const uint32_t s = k % kStages;
                const uint32_t t0 = item.tile_begin + st, t1 = tmid + st;
                const bool two = item.dual && t1 < item.tile_end;
                mbar_wait(&empty[s], ((k / kStages) & 1u) ^ 1u);
                if (trace && lane == 0 && k < 4096) a.trace[k] = clock64();
                if (elect_one()) {
                    mbar_expect_tx(&full[s], two ? 2 * tb : tb);
                    bulk_g2s(sB + s * kStageBytes, tbase + (uint64_t)t0 * tb, tb, &full[s]);
                    if (two) bulk_g2s(sB + s * kStageBytes + kBTileBytes, tbase + (uint64_t)t1 * tb, tb, &full[s]);
                }
                __syncwarp();
            }
        }
    } else if (warp == 1 || warp == 2) {
        // ---------------- MMA issuer of query tile qt = warp - 1: per target
        // tile, wait "B landed" and "my accumulator drained", two MMAs
        // (K-steps) M128 N256 into TMEM columns [256 qt, 256 qt + 256)
        const uint32_t qt = warp - 1;
        const uint32_t b_addr = smem_addr(sB);
        const uint32_t d = tmem + qt * 256u;
        uint32_t k = 0, i = 0, kq = 0;  // kq: tiles this query tile's chains were issued for
        for (uint32_t u = blockIdx.x; u < nitems; u += G, ++i) {
            const TcItem item = a.items[u];
            const uint32_t nt_unit = unit_steps(item);
            const uint32_t ab = i & 1u;
            mbar_wait(&afull[ab], (i >> 1) & 1u);
            tc_fence_after();
            if (qt * 128u >= item.nvalid && !item.dual) {
                // an all-padding query tile (the last tile pair of a pass with
                // n % 256 <= 128 live rows): no MMAs, so its chains do not
                // compete for the tensor pipe; the B slots and the query buffer
                // are handed back as soon as they are this unit's
                for (uint32_t t = 0; t < nt_unit; ++t, ++k) {
                    const uint32_t s = k % kStages;
                    mbar_wait(&full[s], (k / kStages) & 1u);
                    if (elect_one()) mbar_arrive(&empty[s]);
                    __syncwarp();
                }
                if (elect_one()) mbar_arrive(&afree[ab]);
                __syncwarp();
                continue;
            }
            // dual mode: query tile 1 scores query tile 0's rows against the stage's
            // second B tile (the second half of the unit's tile range)
            const bool q1dual = item.dual && qt == 1;
            const uint64_t ad = umma_desc(smem_addr(sA + ab * kSmemA + (item.dual ? 0u : qt * kTileBytes)));
            const uint32_t tmid = unit_mid(item);
            for (uint32_t t = 0; t < nt_unit; ++t, ++k) {
                const uint32_t s = k % kStages;
                if (trace && qt == 0 && lane == 0 && k < 4096) a.trace[4096 + k] = clock64();
                mbar_wait(&full[s], (k / kStages) & 1u);
                if (q1dual && tmid + t >= item.tile_end) {  // odd range: no second tile on the last step
                    if (elect_one()) mbar_arrive(&empty[s]);
                    __syncwarp();
                    continue;
                }
                const uint64_t bd = umma_desc_b(b_addr + s * kStageBytes + (q1dual ? kBTileBytes : 0u));
#pragma unroll
                for (uint32_t h = 0; h < 2; ++h) {
                    // each 128-target half of the tile is its own accumulator chain,
                    // refilled as soon as its four epilogue warps drained it
                    mbar_spin(&accfree[qt * 2 + h], (kq & 1u) ^ 1u);
                    if (trace && qt == 0 && lane == 0 && k < 4096) a.trace[8192 + h * 4096 + k] = clock64();
                    tc_fence_after();
                    if (elect_one()) {
                        // half h starts 16 row groups (2 KB) further; K-step 1 starts two
                        // chunks (8 KB) further in B and 256 B further in A
                        const uint64_t bh = bd + (uint64_t)h * (2048u >> 4);
                        constexpr uint64_t kB1 = (2u * kChunkBytes) >> 4;
                        if (kF16) {  // channels 16..31 first: the rounded partial sum is the smaller one
                            tc_mma_f16(d + h * 128u, ad + 16u, bh + kB1, kIdesc, 0u);
                            tc_mma_f16(d + h * 128u, ad, bh, kIdesc, 1u);
                        } else {
                            tc_mma_f16(d + h * 128u, ad, bh, kIdesc, 0u);
                            tc_mma_f16(d + h * 128u, ad + 16u, bh + kB1, kIdesc, 1u);
                        }
                        tc_commit(&tfull[qt * 2 + h]);
                        if (h == 1) tc_commit(&empty[s]);
                    }
                    __syncwarp();
                }
                ++kq;
            }
            if (elect_one()) tc_commit(&afree[ab]);  // this issuer no longer reads this unit's query tile
            __syncwarp();
        }
    } else {
        // ---------------- epilogue: 16 warps; warps 3..10 drain query tile 0,
        // warps 11..18 query tile 1 (warp = (query tile, 128-column half h,
        // TMEM lane quadrant w%4)), so while one tile's warps load, the other
        // tile's warps compare.  Per tile a warp loads its two 64-target
        // sub-tiles one after the other (the first is reduced before the
        // second is loaded, keeping 64 fragment registers), then releases.
        const uint32_t e = warp - kFirstEpiWarp, quad = warp & 3u;
        const uint32_t qt = e >> 3, h = (e >> 2) & 1u;
        const uint32_t lane_base = (quad * 32u) << 16;
        uint32_t k = 0;  // tiles of this query tile's chains (all-padding units skipped, as the issuer)
        Frag f0, f1;
        for (uint32_t u = blockIdx.x; u < nitems; u += G) {
            const TcItem item = a.items[u];
            RowState st = row_state_init();
            float kb[kTopSub];  // kF16: top-6 keys
#pragma unroll
            for (int i = 0; i < kTopSub; ++i) kb[i] = key_of(-INFINITY, 0);
            // dual mode: query tile 1 holds query tile 0's rows and the second
            // half of the unit's targets
            const bool q1dual = item.dual && qt == 1;
            const uint32_t qrow_base = item.dual ? 0u : qt * 128u;
            const bool warp_real = qrow_base + quad * 32u < item.nvalid;  // else all rows padding
            const bool tile_live = qrow_base < item.nvalid;                // else no MMAs were issued
            const uint32_t t_first = q1dual ? unit_mid(item) : item.tile_begin;
            const uint32_t t_last = item.dual && qt == 0 ? unit_mid(item) : item.tile_end;
            for (uint32_t t = t_first; t < t_last && tile_live; ++t, ++k) {
                mbar_wait(&tfull[qt * 2 + h], k & 1u);
                const bool tw = trace && warp == kFirstEpiWarp && k < 4096;
                // chain (qt 0, half 0): every quadrant's wake and release (k < 1024)
                const bool tq = kF16 && trace && e < 4 && k < 1024;  // (binary16 path only: registers)
                if (tq && lane == 0) a.trace[16384 + quad * 1024 + k] = clock64();
                if (!warp_real || (kDebug && (a.debug & 1))) {  // nothing to score: hand the buffer straight back
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&accfree[qt * 2 + h]);
                    continue;
                }
                tc_fence_after();
                const uint32_t taddr = tmem + lane_base + qt * 256u + h * 128u;
                const uint32_t sub0 = t * kSubPerTile + 2u * h;
                if constexpr (kF16) {
                    frag_ld128_p16(taddr, f0, f1);
                    frag_wait2(f0, f1);
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&accfree[qt * 2 + h]);  // all 128 columns read
                    if (tq && lane == 0) a.trace[20480 + quad * 1024 + k] = clock64();
                    const uint32_t rel = (t - item.tile_begin) * kSubPerTile + 2u * h;
                    const float k0 = key_of(tile_max64_h(f0, sub0, a.nt), rel);
                    const float k1 = key_of(tile_max64_h(f1, sub0 + 1, a.nt), rel + 1);
                    if (__any_sync(0xFFFFFFFFu, fmaxf(k0, k1) > kb[kTopSub - 1])) {
                        key_insert2(kb, k0, k1);
                    }
                    if (tw) {
                        __syncwarp();
                        if (lane == 0) a.trace[24576 + k] = clock64() + (kb[0] > 1e30f ? 1 : 0);
                    }
                    continue;
                }
                frag_ld64(taddr, f0, f1);
                frag_wait2(f0, f1);
                float m0;
                {
                    float v[64];
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        v[j] = __uint_as_float(f0.r[j]);
                        v[32 + j] = __uint_as_float(f1.r[j]);
                    }
                    if ((sub0 + 1) * kSubTile > a.nt) {
#pragma unroll
                        for (int j = 0; j < 64; ++j)
                            if (sub0 * kSubTile + j >= a.nt) v[j] = -INFINITY;
                    }
                    m0 = tile_max64(v);
                }
                frag_ld64(taddr + 64u, f0, f1);
                frag_wait2(f0, f1);
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&accfree[qt * 2 + h]);  // this warp's 128 columns drained
                if (tq && lane == 0) a.trace[20480 + quad * 1024 + k] = clock64();
                if (__any_sync(0xFFFFFFFFu, m0 > st.b[kTopSub - 1])) tile_update(st, m0, sub0);
                subtile_scan(st, f0, f1, sub0 + 1, a.nt);
                if (tw) {
                    __syncwarp();
                    if (lane == 0) a.trace[24576 + k] = clock64() + (st.b[0] > 1e30f ? 1 : 0);
                }
            }
            const uint32_t row = qt * 128u + quad * 32u + lane;  // 0..255 within the tile pair
            float4* po = a.partial + (((uint64_t)u * kPartialSplit + h) * kQueryTilePair + row) * kPartialF4;
            if constexpr (kF16) {  // keys -> (bound, absolute sub-tile) state
#pragma unroll
                for (int i = 0; i < kTopSub; ++i) st.b[i] = key_value(kb[i]);
#pragma unroll
                for (int i = 0; i < kTopSub - 1; ++i) st.t[i] = item.tile_begin * kSubPerTile + key_rel(kb[i]);
            }
            // 12 slots: b[0..kTopSub) then t[0..kTopSub-1) at slot 6
            float w[4 * kPartialF4];
#pragma unroll
            for (int i = 0; i < 4 * kPartialF4; ++i) w[i] = 0.0f;
#pragma unroll
            for (int i = 0; i < kTopSub; ++i) w[i] = st.b[i];
#pragma unroll
            for (int i = 0; i < kTopSub - 1; ++i) w[6 + i] = __uint_as_float(st.t[i]);
#pragma unroll
            for (int i = 0; i < kPartialF4; ++i) po[i] = make_float4(w[4 * i], w[4 * i + 1], w[4 * i + 2], w[4 * i + 3]);
        }
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
    const uint32_t* hdr;       // plan header: [1] tile pairs, [3] target splits
    const uint32_t* n_active;
    const float* margin;
    const uint8_t* qbuf;
    const uint8_t* tmap;
    uint64_t t_pair_bytes;
    uint32_t tcpr;
    uint32_t nt;
    uint32_t dim;
    uint32_t* out;
    float* min_dist;            // may be null
    uint32_t out_stride;
    uint32_t* rescan;           // (gathered row, pair, qi) triples
    unsigned int* rescan_count;
    unsigned long long* near_ties;  // [p] rows not closed by T1, [npairs + p] rows sent to the rescan
    uint32_t npairs;
    long long* shard_keys;      // sharded mode: signed winner keys instead of out/min_dist
    ShardPeers peers;           // sharded mode over peer memory (peers.n > 0)
    const uint32_t* ids;        // query ids of the pass (null = identity), pair stride cap
    uint32_t cap;
    ResolveSrc rs;              // kResolveFull: original fp32 rows
    bool acc16;                 // K3 scores are binary16 accumulations: + 2^-11 |bound|
    bool prefilter;             // kResolveFull: binary16 prefilter before the fp32 rows
};

// sharded mode: this rank's winner key of output slot o -- a local store, or
// a system-scope atomicMin into every rank's key buffer (peer memory)
__device__ __forceinline__ void shard_emit(long long* local, const ShardPeers& p, uint64_t o, long long key) {
    if (p.n == 0) {
        local[o] = key;
        return;
    }
    for (uint32_t r = 0; r < p.n; ++r) atomicMin_system(p.keys[r] + o, key);
}

// Reference FMA chain over channels < dim of binary16 values (packed layout).
// DIM > 0: dim is the compile-time constant DIM (query fully in registers);
// DIM == 0: runtime dim <= kPackK (all loops unrolled to kPackK, predicated).
template <bool kL2, int DIM>
__device__ __forceinline__ float packed_chain(const float (&q)[kPackK], const uint8_t* map, uint32_t row,
                                              uint32_t dim, uint32_t cpr) {
    float acc = 0.0f;
#pragma unroll
    for (uint32_t c0 = 0; c0 < kPackK; c0 += 8) {
        if (DIM > 0 ? c0 < (uint32_t)DIM : c0 < dim) {  // (dim <= 8 cpr: these chunks are stored)
            const uint4 raw = *reinterpret_cast<const uint4*>(map + map_offset(row, c0 >> 3, cpr));
            const __half* h = reinterpret_cast<const __half*>(&raw);
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                if (DIM > 0 ? c0 + k < (uint32_t)DIM : c0 + k < dim) {
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
    }
    return kL2 ? acc : -acc;
}

// The same chain over an original fp32 row (kResolveFull), 16 B loads when
// the row is a whole number of float4s.
template <bool kL2, int DIM>
__device__ __forceinline__ float f32_chain(const float (&q)[kPackK], const float* row, uint32_t dim) {
    float acc = 0.0f;
    if constexpr (DIM > 0 && DIM % 4 == 0) {
#pragma unroll
        for (int c0 = 0; c0 < DIM; c0 += 4) {
            const float4 v = __ldg(reinterpret_cast<const float4*>(row + c0));
            const float t[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                if constexpr (kL2) {
                    const float d = __fsub_rn(q[c0 + k], t[k]);
                    acc = __fmaf_rn(d, d, acc);
                } else {
                    acc = __fmaf_rn(q[c0 + k], t[k], acc);
                }
            }
        }
    } else {
#pragma unroll
        for (uint32_t c = 0; c < kPackK; ++c) {
            if (DIM > 0 ? c < (uint32_t)DIM : c < dim) {
                const float t = __ldg(row + c);
                if constexpr (kL2) {
                    const float d = __fsub_rn(q[c], t);
                    acc = __fmaf_rn(d, d, acc);
                } else {
                    acc = __fmaf_rn(q[c], t, acc);
                }
            }
        }
    }
    return kL2 ? acc : -acc;
}

__device__ __forceinline__ void load_query(const uint8_t* qbuf, uint32_t grow, float (&q)[kPackK]) {
#pragma unroll
    for (uint32_t c0 = 0; c0 < kPackK; c0 += 8) {
        const uint4 raw = *reinterpret_cast<const uint4*>(qbuf + packed_offset(grow, c0 >> 3));
        const __half* h = reinterpret_cast<const __half*>(&raw);
#pragma unroll
        for (int k = 0; k < 8; ++k) q[c0 + k] = __half2float(h[k]);
    }
}
// fp32 query row: 16-byte loads when the row is 16-byte aligned (dim a
// multiple of 4 and an aligned map), else scalar
__device__ __forceinline__ void load_query32(const float* row, uint32_t dim, float (&q)[kPackK]) {
    if ((dim & 3u) == 0 && (reinterpret_cast<uintptr_t>(row) & 15u) == 0) {
#pragma unroll
        for (uint32_t c = 0; c < kPackK; c += 4) {
            const float4 v = c < dim ? __ldg(reinterpret_cast<const float4*>(row + c)) : make_float4(0.f, 0.f, 0.f, 0.f);
            q[c] = v.x, q[c + 1] = v.y, q[c + 2] = v.z, q[c + 3] = v.w;
        }
        return;
    }
#pragma unroll
    for (uint32_t c = 0; c < kPackK; ++c) q[c] = c < dim ? __ldg(row + c) : 0.0f;
}

// Query row in the resolve mode's arithmetic: the original fp32 row
// (kResolveFull) or the gathered binary16 row.
template <int MODE>
__device__ __forceinline__ void mode_query(const uint8_t* qbuf, uint32_t grow, const ResolveSrc& rs,
                                           const uint32_t* ids, uint32_t cap, uint32_t pair, uint32_t qi,
                                           uint32_t dim, float (&q)[kPackK]) {
    if constexpr (MODE == kResolveFull) {
        const uint32_t id = ids ? ids[(uint64_t)pair * cap + qi] : qi;
        load_query32(rs.q32 + pair * rs.q32_pair_stride + (uint64_t)id * dim, dim, q);
    } else {
        load_query(qbuf, grow, q);
    }
}

// Exact reference distance of target t, and the value the reference compares
// (hybrid: the distance cast to binary16, src/kernels.cpp:162-170; routing
// guarantees no saturation on this path).
template <bool kL2, int DIM, int MODE>
__device__ __forceinline__ float mode_chain(const float (&q)[kPackK], const uint8_t* tm, const float* t32,
                                            uint32_t t, uint32_t dim, uint32_t cpr) {
    if constexpr (MODE == kResolveFull) return f32_chain<kL2, DIM>(q, t32 + (uint64_t)t * dim, dim);
    else return packed_chain<kL2, DIM>(q, tm, t, dim, cpr);
}
template <int MODE>
__device__ __forceinline__ float mode_cmp(float d) {
    if constexpr (MODE == kResolveHybrid) return half_round_nosat(d);
    else return d;
}

// binary16 unit in the last place of |x| (normal binade, else the subnormal
// step 2^-24): two values whose binary16 roundings coincide differ by less
// than 2 ulp16 of either
__device__ __forceinline__ float ulp16(float x) {
    const int e = (int)((__float_as_uint(x) >> 23) & 0xFFu) - 127;
    return ldexpf(1.0f, max(e - 10, -24));
}

__device__ __forceinline__ unsigned long long umin64(unsigned long long a, unsigned long long b) {
    return a < b ? a : b;
}

// One CTA per 64-row slice of a tile pair: phase 2 is a chain of dependent
// L2/HBM loads per row, so the kernel is latency bound and wants many rows in
// flight -- four slices per tile pair give each warp 8 rows instead of 32
// (measured: 1.07 -> 0.74 ms per 128-pair step; 32-row slices: 0.84 ms).
// Passes with few tile pairs (one pair's passes) use 16-row slices instead:
// 16 times the CTAs, and phase 1 spreads a row's up to 256 split entries over
// 16 threads.
constexpr uint32_t kMergeThreads = 256;
constexpr uint32_t kNoTile = 0xFFFFFFFFu;

template <bool kL2, int DIM, int MODE, uint32_t kMergeRows>
__global__ void __launch_bounds__(kMergeThreads, 4) merge_kernel(MergeArgs a) {
    constexpr uint32_t kMergeSlices = kQueryTilePair / kMergeRows;
    constexpr uint32_t kMergeParts = kMergeThreads / kMergeRows;  // phase-1 threads per row
    // phase 1 (four threads per row): global top-6 of sub-tile maxima over
    //   the target splits / column halves -> candidates T1..T5 and the bounds
    //   B2..B6 on everything not yet resolved after 1..5 of them
    // phase 2 (16 lanes per row, two rows per warp): resolve T1 with the exact
    //   chain (four targets per lane, (cmp, index) key min), close the row if
    //   the exact winner beats B2 by the margin, else resolve T2 against B3,
    //   and so on; rows still open after T5 go to the full rescan
    __shared__ uint32_t s_t[kMergeRows][kTopSub - 1];
    __shared__ float s_b[kMergeRows][kTopSub - 1];
    // phase 1 partial lists handed down the fold tree (top-5 and the bound on the rest)
    __shared__ float s_pb[kMergeParts / 2][kMergeRows][kTopSub];
    __shared__ uint32_t s_pt[kMergeParts / 2][kMergeRows][kTopSub - 1];
    const uint32_t tp = blockIdx.x / kMergeSlices, slice = blockIdx.x % kMergeSlices;
    if (tp >= a.hdr[1]) return;
    const uint32_t splits = a.hdr[3];
    const uint32_t pair = a.tp_pair[tp];
    const uint32_t tp_rows = min(kQueryTilePair, a.n_active[pair] - a.tp_qi0[tp]);
    if (slice * kMergeRows >= tp_rows) return;  // CTA-uniform
    const uint32_t nrows = min(kMergeRows, tp_rows - slice * kMergeRows);
    const uint32_t row0 = a.tp_row0[tp] + slice * kMergeRows;  // first gathered row of the slice
    const uint32_t qi0 = a.tp_qi0[tp] + slice * kMergeRows;     // its query index within the pair
    const uint32_t r = threadIdx.x;
    // global top-6 over the splits: B[0..5] with sub-tiles T[0..4]; B[5]
    // bounds everything below the fifth.  The (split, half, source) entries
    // of a row are spread over kMergeParts threads (a single pair's passes
    // split the targets up to 64 ways), whose lists part 0 then folds
    const uint32_t pr = r % kMergeRows, part = r / kMergeRows;
    float B[kTopSub];
    uint32_t T[kTopSub - 1];
#pragma unroll
    for (int i = 0; i < kTopSub; ++i) B[i] = -INFINITY;
#pragma unroll
    for (int i = 0; i < kTopSub - 1; ++i) T[i] = kNoTile;
    auto insert = [&](float v, uint32_t t) {
        // sorted insert into the first five (branch-free shifts); what falls
        // off the fifth only raises the bound B[5]
        B[kTopSub - 1] = fmaxf(B[kTopSub - 1], fminf(B[kTopSub - 2], v));
#pragma unroll
        for (int i = kTopSub - 2; i >= 1; --i) {
            const bool gp = v > B[i - 1], gi = v > B[i];
            T[i] = gp ? T[i - 1] : (gi ? t : T[i]);
            B[i] = gp ? B[i - 1] : (gi ? v : B[i]);
        }
        if (v > B[0]) T[0] = t, B[0] = v;
    };
    if (pr < nrows) {
        // dual tile pairs (<= 128 rows): query tile 1 scored the same rows over
        // the second half of each unit's targets, in partial rows 128..255
        const uint32_t nsrc = tp_dual(tp_rows) ? 2u : 1u;
#pragma unroll 4
        for (uint32_t s = part; s < splits * kPartialSplit * nsrc; s += kMergeParts) {
            const uint32_t sp = s % (splits * kPartialSplit), hi = s / (splits * kPartialSplit);
            const float4* pp = a.partial + (((uint64_t)tp * splits * kPartialSplit + sp) * kQueryTilePair +
                                            hi * kTileRows + slice * kMergeRows + pr) * kPartialF4;
            float w[4 * kPartialF4];
#pragma unroll
            for (int i = 0; i < kPartialF4; ++i) {
                const float4 v = pp[i];
                w[4 * i] = v.x, w[4 * i + 1] = v.y, w[4 * i + 2] = v.z, w[4 * i + 3] = v.w;
            }
#pragma unroll
            for (int i = 0; i < kTopSub - 1; ++i) insert(w[i], __float_as_uint(w[6 + i]));
            B[kTopSub - 1] = fmaxf(B[kTopSub - 1], w[kTopSub - 1]);
        }
    }
    // fold the parts' lists pairwise: log2(kMergeParts) rounds
#pragma unroll
    for (uint32_t h = kMergeParts / 2; h >= 1; h >>= 1) {
        if (part >= h && part < 2 * h) {
#pragma unroll
            for (int i = 0; i < kTopSub; ++i) s_pb[part - h][pr][i] = B[i];
#pragma unroll
            for (int i = 0; i < kTopSub - 1; ++i) s_pt[part - h][pr][i] = T[i];
        }
        __syncthreads();
        if (part < h) {
#pragma unroll
            for (int i = 0; i < kTopSub - 1; ++i) insert(s_pb[part][pr][i], s_pt[part][pr][i]);
            B[kTopSub - 1] = fmaxf(B[kTopSub - 1], s_pb[part][pr][kTopSub - 1]);
        }
        __syncthreads();
    }
    if (part == 0 && pr < nrows) {
#pragma unroll
        for (int c = 0; c < kTopSub - 1; ++c) {
            s_t[pr][c] = T[c];
            s_b[pr][c] = B[c + 1];
        }
    }
    __syncthreads();
    const uint32_t warp = r >> 5, lane = r & 31;
    const uint8_t* tm = a.tmap + pair * a.t_pair_bytes;
    const float* t32 = MODE == kResolveFull ? a.rs.t32 + pair * a.rs.t32_pair_stride : nullptr;
    const uint32_t half = lane >> 4, hl = lane & 15u;
    for (uint32_t rb = warp; rb < nrows; rb += 2 * (kMergeThreads / 32)) {
        const uint32_t row = rb + half * (kMergeThreads / 32);
        const bool valid = row < nrows;
        float q[kPackK];
        float qq = 0.0f, M = 0.0f;
        if (valid) {
            mode_query<MODE>(a.qbuf, row0 + row, a.rs, a.ids, a.cap, pair, qi0 + row, a.dim, q);
            M = a.margin[row0 + row];
            if constexpr (kL2) {
#pragma unroll
                for (uint32_t c = 0; c < kPackK; ++c)
                    if (DIM > 0 ? c < (uint32_t)DIM : c < a.dim) qq = __fmaf_rn(q[c], q[c], qq);
            }
        }
        unsigned long long key = ~0ull;
        float dmin = INFINITY;
        bool done = !valid;
#pragma unroll 1
        for (int c = 0; c < kTopSub - 1; ++c) {
            const uint32_t st = done ? kNoTile : s_t[row][c];
            if (MODE == kResolveFull && a.prefilter) {
                // Full precision: a binary16 prefilter (the chain over the packed
                // rows, 48 of 96 bytes per target) keeps only targets within 4E of
                // the sub-tile's best approximation -- E bounds the input rounding
                // and both chains and is inside the certification margin -- and
                // only those read their fp32 rows
                float da[kSubTile / 16];
                float dam = INFINITY;
#pragma unroll
                for (uint32_t h = 0; h < kSubTile / 16; ++h) {
                    const uint32_t t = st * kSubTile + h * 16 + hl;
                    da[h] = (st != kNoTile && t < a.nt) ? packed_chain<kL2, DIM>(q, tm, t, a.dim, a.tcpr) : INFINITY;
                    dam = fminf(dam, da[h]);
                }
#pragma unroll
                for (int o = 8; o > 0; o >>= 1) dam = fminf(dam, __shfl_xor_sync(0xFFFFFFFFu, dam, o));
                const float thr = dam + 4.0f * (kL2 ? 2.0f * M : M);
#pragma unroll
                for (uint32_t h = 0; h < kSubTile / 16; ++h) {
                    const uint32_t t = st * kSubTile + h * 16 + hl;
                    if (st != kNoTile && t < a.nt && da[h] <= thr) {
                        const float d = f32_chain<kL2, DIM>(q, t32 + (uint64_t)t * a.dim, a.dim);
                        key = umin64(key, pack_key(d, t));
                        dmin = fminf(dmin, d);
                    }
                }
            } else if (st != kNoTile) {
#pragma unroll
                for (uint32_t h = 0; h < kSubTile; h += 16) {
                    const uint32_t t = st * kSubTile + h + hl;
                    if (t < a.nt) {
                        const float d = mode_chain<kL2, DIM, MODE>(q, tm, t32, t, a.dim, a.tcpr);
                        key = umin64(key, pack_key(mode_cmp<MODE>(d), t));
                        dmin = fminf(dmin, d);
                    }
                }
            }
#pragma unroll
            for (int o = 8; o > 0; o >>= 1) {  // within each 16-lane half
                key = umin64(key, __shfl_xor_sync(0xFFFFFFFFu, key, o));
                dmin = fminf(dmin, __shfl_xor_sync(0xFFFFFFFFu, dmin, o));
            }
            if (!done) {
                bool closed = true;  // no candidate left: every target resolved
                if (st != kNoTile) {
                    const float Bn = s_b[row][c];
                    // binary16 accumulator: its final rounding moves a score by at most
                    // 2^-11 of itself, and score + 2^-11 |score| grows with the score
                    const float Mf = a.acc16 ? M + 1.001f * ldexpf(fabsf(Bn), -11) : M;
                    const float lb = kL2 ? qq - 2.0f * (Bn + Mf) : -(Bn + Mf);  // bound on every other distance
                    const float dref = MODE == kResolveHybrid ? dmin + 2.0f * ulp16(fabsf(dmin)) : dmin;
                    closed = dref < lb;
                }
                if (c == 0 && !closed && hl == 0) atomicAdd(a.near_ties + pair, 1ull);
                if (closed) {
                    done = true;
                    if (hl == 0) {
                        const uint64_t o = (uint64_t)pair * a.out_stride + qi0 + row;
                        if (a.shard_keys) {
                            shard_emit(a.shard_keys, a.peers, o, (long long)(key ^ 0x8000000000000000ull));
                        } else {
                            a.out[o] = (uint32_t)(key & 0xFFFFFFFFull);
                            if (a.min_dist) {
                                float d = from_orderable((uint32_t)(key >> 32));
                                if (d == 0.0f)  // keys merge +-0: the winner's own zero (hybrid cast) or canonical
                                    d = MODE == kResolveHybrid
                                            ? mode_cmp<MODE>(mode_chain<kL2, DIM, MODE>(
                                                  q, tm, t32, (uint32_t)(key & 0xFFFFFFFFull), a.dim, a.tcpr))
                                            : (kL2 ? 0.0f : -0.0f);
                                a.min_dist[o] = d;
                            }
                        }
                    }
                }
            }
            if (!__any_sync(0xFFFFFFFFu, !done)) break;
        }
        if (!done && hl == 0) {
            atomicAdd(a.near_ties + a.npairs + pair, 1ull);
            const uint32_t k = atomicAdd(a.rescan_count, 1u);
            a.rescan[3 * k] = row0 + row;
            a.rescan[3 * k + 1] = pair;
            a.rescan[3 * k + 2] = qi0 + row;
        }
    }
}

// ---------------------------------------------------------------- K4' rescan
// Rows with four sub-tiles inside the margin: the resolve mode's exact chain
// over every target of the scanned range, lowest index on exact ties.
struct RescanArgs {
    const uint32_t* rescan;
    const unsigned int* rescan_count;
    const uint8_t* qbuf;
    const uint8_t* tmap;
    uint64_t t_pair_bytes;
    uint32_t tcpr;
    uint32_t t_begin, nt;           // scanned target range [t_begin, nt)
    uint32_t dim;
    uint32_t chunk;                 // targets per work unit
    unsigned long long* keys;       // per rescan entry
    bool l2;
    const uint32_t* ids;
    uint32_t cap;
    ResolveSrc rs;
    // finish (the last CTA to retire): winners into out / min_dist, or signed
    // keys into the shard buffers
    unsigned int* done_ctr;  // zeroed with the row count before each pass
    uint32_t* out;
    float* min_dist;
    uint32_t out_stride;
    long long* shard_keys;
    ShardPeers peers;
};

constexpr int kRescanThreads = 256;

// rows resolved by the scan below: winners out (one CTA)
template <bool kL2, int DIM, int MODE>
__device__ void rescan_finish(const RescanArgs& a, uint32_t n) {
    for (uint32_t k = threadIdx.x; k < n; k += blockDim.x) {
        const uint32_t pair = a.rescan[3 * k + 1], qi = a.rescan[3 * k + 2];
        const uint64_t o = (uint64_t)pair * a.out_stride + qi;
        const unsigned long long key = a.keys[k];
        if (a.shard_keys) {
            shard_emit(a.shard_keys, a.peers, o, (long long)(key ^ 0x8000000000000000ull));
            a.keys[k] = ~0ull;
            continue;
        }
        const uint32_t idx = (uint32_t)(key & 0xFFFFFFFFull);
        a.out[o] = idx;
        if (a.min_dist) {
            float d = from_orderable((uint32_t)(key >> 32));
            if (d == 0.0f) {
                if constexpr (MODE == kResolveHybrid) {  // the winner's own signed zero
                    float q[kPackK];
                    mode_query<MODE>(a.qbuf, a.rescan[3 * k], a.rs, a.ids, a.cap, pair, qi, a.dim, q);
                    d = mode_cmp<MODE>(mode_chain<kL2, DIM, MODE>(q, a.tmap + pair * a.t_pair_bytes, nullptr, idx,
                                                                    a.dim, a.tcpr));
                } else {
                    d = kL2 ? 0.0f : -0.0f;  // canonical sign of an exact zero
                }
            }
            a.min_dist[o] = d;
        }
        a.keys[k] = ~0ull;
    }
}

// Grid-stride over (row, target chunk) units; the last CTA to retire (a
// counter, zeroed with the row count before the pass) writes the winners,
// so a pass with no open rows costs one short launch.
template <bool kL2, int DIM, int MODE>
__global__ void __launch_bounds__(kRescanThreads) rescan_kernel(RescanArgs a) {
    const uint64_t count = *a.rescan_count;
    if (count == 0) return;  // the usual case: nothing to scan, nothing to finish
    const uint64_t nchunks = (a.nt - a.t_begin + a.chunk - 1) / a.chunk;
    __shared__ unsigned long long red[kRescanThreads / 32];
    __shared__ bool last;
    float q[kPackK];
    for (uint64_t unit = blockIdx.x; unit < count * nchunks; unit += gridDim.x) {
        const uint64_t k = unit / nchunks, ch = unit % nchunks;
        const uint32_t grow = a.rescan[3 * k], pair = a.rescan[3 * k + 1], qi = a.rescan[3 * k + 2];
        mode_query<MODE>(a.qbuf, grow, a.rs, a.ids, a.cap, pair, qi, a.dim, q);
        const uint8_t* tm = a.tmap + pair * a.t_pair_bytes;
        const float* t32 = MODE == kResolveFull ? a.rs.t32 + pair * a.rs.t32_pair_stride : nullptr;
        const uint32_t t0 = a.t_begin + (uint32_t)ch * a.chunk, t1 = min(a.nt, t0 + a.chunk);
        unsigned long long key = ~0ull;
        for (uint32_t t = t0 + threadIdx.x; t < t1; t += kRescanThreads)
            key = umin64(key, pack_key(mode_cmp<MODE>(mode_chain<kL2, DIM, MODE>(q, tm, t32, t, a.dim, a.tcpr)), t));
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
    if (threadIdx.x == 0) {
        __threadfence();  // this CTA's key minima before its retirement
        last = atomicAdd(a.done_ctr, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (!last) return;
    __threadfence();
    rescan_finish<kL2, DIM, MODE>(a, (uint32_t)count);
}

__global__ void shard_finalize_kernel(const long long* keys, uint32_t stride, const uint32_t* n_active,
                                      const uint8_t* done, uint32_t* out) {
    const uint32_t p = blockIdx.y;
    if (done && done[p]) return;
    const uint32_t n = n_active[p];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint64_t o = (uint64_t)p * stride + i;
        out[o] = (uint32_t)(((unsigned long long)keys[o] ^ 0x8000000000000000ull) & 0xFFFFFFFFull);
    }
}

struct PeerFlags {
    unsigned int* flags[kMaxShardPeers];
    uint32_t n;
};

__global__ void shard_barrier_kernel(PeerFlags f, unsigned int* own, unsigned int target, unsigned int* err) {
    __threadfence_system();  // this rank's key pushes (earlier kernels) before the arrivals
    for (uint32_t r = 0; r < f.n; ++r) atomicAdd_system(f.flags[r], 1u);
    // an earlier barrier of this run already timed out: the run fails anyway,
    // so do not stall another 20 s here (the arrivals above still let peers on)
    if (*reinterpret_cast<volatile unsigned int*>(err)) return;
    unsigned long long t0, t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    for (;;) {
        unsigned int v;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(own) : "memory");
        if ((int)(v - target) >= 0) break;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        if (t - t0 > 20000000000ull) {  // a peer never arrived: report instead of hanging the GPU
            atomicExch(err, 1u);
            break;
        }
        __nanosleep(256);
    }
    __threadfence_system();
}

__global__ void shard_reset_kernel(long long* keys, uint64_t n) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        keys[i] = kShardKeyNone;
}

// Raw scores of one tile pair x one target tile (UMMA layout self-test).
constexpr int kSelftestThreads = 320;
constexpr uint32_t kTmemA = 384;  // self-test: query tiles copied into TMEM columns 384..415
__global__ void __launch_bounds__(kSelftestThreads, 1) selftest_kernel(const uint8_t* qbuf, const uint8_t* tmap,
                                                                    uint32_t cpr, float* out, int mode) {
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
    // the chunks the map does not store are zero K padding
    for (uint32_t i = cpr * kChunkBytes / 16u + threadIdx.x; i < kBTileBytes / 16u; i += blockDim.x)
        reinterpret_cast<uint4*>(smem + kSmemA)[i] = make_uint4(0u, 0u, 0u, 0u);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_slot;
    if (threadIdx.x == 0) {
        mbar_expect_tx(&bar_ld, kSmemA + cpr * kChunkBytes);
        bulk_g2s(smem, qbuf, kSmemA, &bar_ld);
        bulk_g2s(smem + kSmemA, tmap, cpr * kChunkBytes, &bar_ld);
        mbar_wait(&bar_ld, 0);
        tc_fence_after();
        const uint32_t a_addr = smem_addr(smem), b_addr = a_addr + kSmemA;
        if (mode == 0) {  // both operands from shared memory
            for (uint32_t qt = 0; qt < 2; ++qt)
                for (uint32_t ks = 0; ks < 2; ++ks)
                    tc_mma_f16(tmem + qt * 128u, umma_desc(a_addr + qt * kTileBytes + ks * 256u),
                               umma_desc_b(b_addr + ks * 2u * kChunkBytes), kIdescF16M128N128, ks);
        } else {  // production path: query tiles copied into TMEM, TS MMA
            for (uint32_t qt = 0; qt < 2; ++qt)
                for (uint32_t ks = 0; ks < 2; ++ks)
                    tc_cp_128x256b(tmem + kTmemA + qt * 16u + ks * 8u, umma_desc(a_addr + qt * kTileBytes + ks * 256u));
            for (uint32_t qt = 0; qt < 2; ++qt)
                for (uint32_t ks = 0; ks < 2; ++ks)
                    tc_mma_f16_ts(tmem + qt * 128u, tmem + kTmemA + qt * 16u + ks * 8u,
                                  umma_desc_b(b_addr + ks * 2u * kChunkBytes), kIdescF16M128N128, ks);
        }
        tc_commit(&bar_mma);
    }
    if (warp >= 2) {
        mbar_wait(&bar_mma, 0);
        tc_fence_after();
        const uint32_t e = warp - 2, qt = e >> 2, quad = warp & 3u;
        const uint32_t row = qt * 128u + quad * 32u + lane;
        Frag f, g;
        for (int c = 0; c < 4; c += 2) {
            frag_ld(tmem + ((quad * 32u) << 16) + qt * 128u + 32u * c, f);
            frag_ld(tmem + ((quad * 32u) << 16) + qt * 128u + 32u * (c + 1), g);
            frag_wait2(f, g);
            for (int j = 0; j < 32; ++j) {
                out[row * 128 + 32 * c + j] = __uint_as_float(f.r[j]);
                out[row * 128 + 32 * (c + 1) + j] = __uint_as_float(g.r[j]);
            }
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

// cudaFuncSetAttribute applies to the current device only: one flag per
// device, set under a lock (threads may drive different GPUs)
std::mutex attr_mu;
bool attr_done[64] = {};

int ensure_attrs() {
    int dev = 0;
    FNL_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(attr_mu);
    if (dev >= 0 && dev < 64 && attr_done[dev]) return FNL_OK;
    FNL_CUDA_TRY(cudaFuncSetAttribute(tc_scan_kernel<false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemTotal));
    FNL_CUDA_TRY(cudaFuncSetAttribute(tc_scan_kernel<true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemTotal));
    FNL_CUDA_TRY(cudaFuncSetAttribute(tc_scan_kernel<false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemTotal));
    FNL_CUDA_TRY(cudaFuncSetAttribute(tc_scan_kernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemTotal));
    FNL_CUDA_TRY(cudaFuncSetAttribute(selftest_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemTotal));
    FNL_CUDA_TRY(cudaFuncSetAttribute(pack_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      kPackStages * kPackTileRows * kPackK * 4));
    if (dev >= 0 && dev < 64) attr_done[dev] = true;
    return FNL_OK;
}

template <bool kL2, int DIM>
void launch_merge_rows(int mode, uint32_t grid, const MergeArgs& m, cudaStream_t s, bool small) {
    if (small) {
        grid *= kQueryTilePair / 16;
        if (mode == kResolveFull) merge_kernel<kL2, DIM, kResolveFull, 16><<<grid, kMergeThreads, 0, s>>>(m);
        else if (mode == kResolveHybrid) merge_kernel<kL2, DIM, kResolveHybrid, 16><<<grid, kMergeThreads, 0, s>>>(m);
        else merge_kernel<kL2, DIM, kResolveRounded, 16><<<grid, kMergeThreads, 0, s>>>(m);
        return;
    }
    grid *= kQueryTilePair / 64;
    if (mode == kResolveFull) merge_kernel<kL2, DIM, kResolveFull, 64><<<grid, kMergeThreads, 0, s>>>(m);
    else if (mode == kResolveHybrid) merge_kernel<kL2, DIM, kResolveHybrid, 64><<<grid, kMergeThreads, 0, s>>>(m);
    else merge_kernel<kL2, DIM, kResolveRounded, 64><<<grid, kMergeThreads, 0, s>>>(m);
}
template <bool kL2, int DIM>
void launch_merge_mode(int mode, uint32_t tp_max, uint32_t sms, const MergeArgs& m, cudaStream_t s) {
    // 64-row slices (4 per tile pair) fill the GPU once there are >= one tile
    // pair per SM; below that (a single pair's passes) 16-row slices
    static const int env = getenv("FNL_MERGE_SMALL") ? atoi(getenv("FNL_MERGE_SMALL")) : -1;
    const bool small = env >= 0 ? env != 0 : tp_max < sms;
    launch_merge_rows<kL2, DIM>(mode, tp_max, m, s, small);
}
template <bool kL2, int DIM, int MODE>
void launch_rescan_t(uint32_t grid, const RescanArgs& r, cudaStream_t s) {
    rescan_kernel<kL2, DIM, MODE><<<grid, kRescanThreads, 0, s>>>(r);
}
template <bool kL2, int DIM>
void launch_rescan_mode(int mode, uint32_t grid, const RescanArgs& r, cudaStream_t s) {
    if (mode == kResolveFull) launch_rescan_t<kL2, DIM, kResolveFull>(grid, r, s);
    else if (mode == kResolveHybrid) launch_rescan_t<kL2, DIM, kResolveHybrid>(grid, r, s);
    else launch_rescan_t<kL2, DIM, kResolveRounded>(grid, r, s);
}

}  // namespace

// profiling aid: with FNL_TC_DEBUG & 16 the last tc_scan launch's clock trace
// of CTA 0 is written to $FNL_TC_TRACE (default /tmp/fnl_tc_trace.bin)
static bool debug_mode_trace_dump(fnl_context* ctx, cudaStream_t s) {
    static const int debug_mode = getenv("FNL_TC_DEBUG") ? atoi(getenv("FNL_TC_DEBUG")) : 0;
    if (!(debug_mode & 16)) return false;
    unsigned long long* trace = nullptr;
    if (ws_arr(ctx, "tc.trace", 7 * 4096, &trace) != FNL_OK) return false;
    static unsigned long long host[7 * 4096];
    cudaMemcpyAsync(host, trace, sizeof(host), cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
    const char* path = getenv("FNL_TC_TRACE") ? getenv("FNL_TC_TRACE") : "/tmp/fnl_tc_trace.bin";
    if (FILE* f = fopen(path, "wb")) {
        fwrite(host, 1, sizeof(host), f);
        fclose(f);
    }
    return true;
}

// ---------------------------------------------------------------- K2p plan
// One block builds the pass's work lists from the DEVICE per-pair state
// (n_active, done), so the reciprocal loop never waits on the host between
// passes: gather slots (one per live pair), 256-query tile pairs, the target
// split count (the modelled makespan of the persistent K3 grid: waves x
// (tiles per unit + switch cost)) and the K3 work units.  Consumers read the
// counts from the header and early-exit past them (grids are upper bounds).
struct PlanArgs {
    uint32_t npairs;
    const uint32_t* n_active;
    const uint8_t* done;  // may be null
    uint32_t tile_begin, ntiles;
    uint32_t sms;
    uint32_t nitems_cap;
    uint32_t switch_cost;  // modelled cost of starting a work unit, in target tiles
    uint32_t* hdr;  // [0] slots [1] tile pairs [2] items [3] splits [4] tiles per split
    uint32_t* slot_pair;
    uint32_t* slot_base;
    uint32_t* tp_pair;
    uint32_t* tp_row0;
    uint32_t* tp_qi0;
    TcItem* items;
    unsigned int* rescan_ctr;  // [2] open-row count and retired rescan CTAs, zeroed here
};

constexpr int kPlanThreads = 1024;

__global__ void __launch_bounds__(kPlanThreads) plan_kernel(PlanArgs a) {
    __shared__ uint32_t s_warp[2][32];
    __shared__ uint32_t s_carry[2];
    __shared__ uint32_t s_split[2];
    const uint32_t tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0) {
        s_carry[0] = s_carry[1] = 0;
        a.rescan_ctr[0] = a.rescan_ctr[1] = 0u;  // the pass's merge / rescan counters
    }
    __syncthreads();
    for (uint32_t base = 0; base < a.npairs; base += kPlanThreads) {
        const uint32_t p = base + tid;
        uint32_t act = p < a.npairs ? a.n_active[p] : 0u;
        if (p < a.npairs && a.done && a.done[p]) act = 0;
        const uint32_t has = act ? 1u : 0u;
        const uint32_t ntp = (act + kQueryTilePair - 1) / kQueryTilePair;
        // block exclusive scan of (has, ntp)
        uint32_t ih = has, it = ntp;
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t h = __shfl_up_sync(0xffffffffu, ih, o), t = __shfl_up_sync(0xffffffffu, it, o);
            if (lane >= (uint32_t)o) ih += h, it += t;
        }
        if (lane == 31) s_warp[0][warp] = ih, s_warp[1][warp] = it;
        __syncthreads();
        if (warp == 0) {
            uint32_t wh = s_warp[0][lane], wt = s_warp[1][lane];
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t h = __shfl_up_sync(0xffffffffu, wh, o), t = __shfl_up_sync(0xffffffffu, wt, o);
                if (lane >= (uint32_t)o) wh += h, wt += t;
            }
            s_warp[0][lane] = wh - s_warp[0][lane];  // exclusive warp offsets
            s_warp[1][lane] = wt - s_warp[1][lane];
        }
        __syncthreads();
        const uint32_t slot = s_carry[0] + s_warp[0][warp] + ih - has;
        const uint32_t tp0 = s_carry[1] + s_warp[1][warp] + it - ntp;
        if (has) {
            a.slot_pair[slot] = p;
            a.slot_base[slot] = tp0 * kQueryTilePair;
            for (uint32_t j = 0; j < ntp; ++j) {
                a.tp_pair[tp0 + j] = p;
                a.tp_row0[tp0 + j] = (tp0 + j) * kQueryTilePair;
                a.tp_qi0[tp0 + j] = j * kQueryTilePair;
            }
        }
        __syncthreads();
        if (tid == kPlanThreads - 1) s_carry[0] = slot + has, s_carry[1] = tp0 + ntp;
        __syncthreads();
    }
    const uint32_t nslots = s_carry[0], ntp = s_carry[1];
    if (warp == 0) {
        // the split count with the smallest modelled makespan (first minimum,
        // i.e. the fewest splits on ties), one candidate per lane
        const uint32_t smax = min(min(a.ntiles, 64u), ntp ? max(1u, a.nitems_cap / ntp) : 1u);
        // a unit spans at most kMaxUnitTiles target tiles (K3's sub-tile keys)
        const uint32_t sp_min = (a.ntiles + kMaxUnitTiles - 1) / kMaxUnitTiles;
        uint32_t best = sp_min;
        float best_cost = 3.0e38f;
        for (uint32_t sp = sp_min + lane; sp <= smax; sp += 32) {
            const float waves = (float)((ntp * sp + a.sms - 1) / a.sms);
            const float cost = waves * (float)((a.ntiles + sp - 1) / sp + a.switch_cost);
            if (cost < best_cost) best_cost = cost, best = sp;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const float oc = __shfl_xor_sync(0xFFFFFFFFu, best_cost, o);
            const uint32_t os = __shfl_xor_sync(0xFFFFFFFFu, best, o);
            if (oc < best_cost || (oc == best_cost && os < best)) best_cost = oc, best = os;
        }
        if (lane == 0) {
            const uint32_t per = (a.ntiles + best - 1) / best;
            const uint32_t splits = (a.ntiles + per - 1) / per;
            s_split[0] = splits;
            s_split[1] = per;
            a.hdr[0] = nslots;
            a.hdr[1] = ntp;
            a.hdr[2] = ntp * splits;
            a.hdr[3] = splits;
            a.hdr[4] = per;
        }
    }
    __syncthreads();
    const uint32_t splits = s_split[0], per = s_split[1];
    for (uint32_t u = tid; u < ntp * splits; u += kPlanThreads) {
        const uint32_t j = u / splits, sp = u - j * splits;
        const uint32_t pair = a.tp_pair[j], qi0 = a.tp_qi0[j];
        TcItem it;
        it.pair = pair;
        it.qrow0 = a.tp_row0[j];
        it.tile_begin = a.tile_begin + sp * per;
        it.tile_end = a.tile_begin + min(a.ntiles, (sp + 1) * per);
        it.nvalid = min(kQueryTilePair, a.n_active[pair] - qi0);
        it.dual = tp_dual(it.nvalid) ? 1u : 0u;
        it.pad1 = it.pad2 = 0;
        a.items[u] = it;
    }
}

// ====================================================================== host
int tensor_pack(fnl_context* ctx, const char* tag, const float* d_src, uint32_t npairs, uint32_t rows,
                uint32_t dim, bool l2, unsigned long long* d_bad, unsigned long long* d_sat, PackedMaps* out,
                float* d_max_norm) {
    if (dim == 0 || dim + (l2 ? 2u : 0u) > kPackK)
        return fail(FNL_EINVAL, "tensor backend: descriptor dim " + std::to_string(dim) + " exceeds " +
                                    std::to_string(l2 ? kPackK - 2 : kPackK) + " (" + (l2 ? "l2" : "dot") +
                                    " metric); use the exact backends");
    // padded to whole 256-target B tiles (also a whole number of 128-row operand tiles)
    const uint32_t rows_pad = ceil_div_u(rows, kTargetTileRows) * kTargetTileRows;
    const uint32_t cpr = ceil_div_u(dim + (l2 ? 2u : 0u), 8);  // chunks that carry data
    const uint64_t pair_bytes = (uint64_t)(rows_pad / kTargetTileRows) * cpr * kChunkBytes;
    std::string t(tag);
    TRY(ws_arr(ctx, (t + ".packed").c_str(), (size_t)npairs * pair_bytes, &out->data));
    cudaStream_t s = ctx_stream(ctx);
    if (d_max_norm) {
        out->max_norm = d_max_norm;  // [2 npairs], zeroed by the caller
    } else {
        TRY(ws_arr(ctx, (t + ".maxnorm").c_str(), 2 * (size_t)npairs, &out->max_norm));
        FNL_CUDA_TRY(cudaMemsetAsync(out->max_norm, 0, 2 * (size_t)npairs * sizeof(float), s));
    }
    out->max_norm_hi = out->max_norm + npairs;
    out->pair_bytes = pair_bytes;
    out->cpr = cpr;
    out->rows = rows;
    out->npairs = npairs;
    PackArgs a{d_src, out->data, pair_bytes, rows, rows_pad, dim, l2, out->max_norm, d_bad, d_sat, out->max_norm_hi,
               cpr};
    // K1 v2 (TMA-staged, one thread per row) whenever every 256-row tile is a
    // whole number of 16-byte units: 1.26 vs 1.56 ms per 128 C2 pairs for v1
    // (FNL_PACK_V=1; 3 blocks per SM for v2 measured no faster).  v1: 8 blocks
    // per SM, 4 lanes per row, any dim / row count.
    ProfScope prof(ctx, FNL_KCLASS_PACK);
    static const int pack_v = getenv("FNL_PACK_V") ? atoi(getenv("FNL_PACK_V")) : 2;
    if (pack_v == 2 && ((uint64_t)rows * dim) % 4 == 0) {
        // K1 v2: 2 resident blocks per SM, kPackStages staged tiles each
        const uint32_t smem = kPackStages * kPackTileRows * dim * 4u;
        TRY(ensure_attrs());
        static const uint32_t bps = getenv("FNL_PACK_BPS") ? (uint32_t)atoi(getenv("FNL_PACK_BPS")) : 2u;
        const uint32_t grid = std::max(1u, bps) * (uint32_t)ctx_sm_count(ctx);
        pack_tma_kernel<<<grid, kPackTileRows, smem, s>>>(a, npairs);
    } else {
        const uint32_t grid = 8u * (uint32_t)ctx_sm_count(ctx);
        pack_kernel<<<grid, kPackThreads, 0, s>>>(a, npairs);
    }
    FNL_CUDA_TRY(cudaGetLastError());
    ctx_count_launches(ctx, 1);
    return FNL_OK;
}

// full-precision merge resolves through a binary16 prefilter (FNL_MERGE_PREFILTER=0: off)
static bool merge_prefilter() {
    static const bool on = !(getenv("FNL_MERGE_PREFILTER") && atoi(getenv("FNL_MERGE_PREFILTER")) == 0);
    return on;
}

int tensor_nn_pass(fnl_context* ctx, uint32_t npairs, const PackedMaps& Q, const uint32_t* ids, uint32_t cap,
                   const uint32_t* d_active, const uint8_t* d_done, const PackedMaps& T, uint32_t dim, bool l2,
                   uint32_t* out, uint32_t out_stride, float* min_dist, unsigned long long* d_near_ties,
                   uint32_t tile_begin, uint32_t tile_end, long long* shard_keys, const ShardPeers* peers,
                   const ResolveSrc* resolve) {
    const ShardPeers no_peers{};
    const ShardPeers& pp = peers ? *peers : no_peers;
    const ResolveSrc rs = resolve ? *resolve : ResolveSrc{};
    if (rs.mode == kResolveFull && (!rs.q32 || !rs.t32))
        return fail(FNL_EINVAL, "tensor_nn_pass: full-precision resolution needs the fp32 maps");
    TRY(ensure_attrs());
    cudaStream_t s = ctx_stream(ctx);
    const uint32_t nt = T.rows;
    const uint32_t all_tiles = ceil_div_u(nt, kBTileRows);
    if (tile_end == 0 || tile_end > all_tiles) tile_end = all_tiles;
    if (tile_begin >= tile_end) return fail(FNL_EINVAL, "tensor_nn_pass: empty target tile range");
    if (npairs == 0 || cap == 0) return FNL_OK;
    const uint32_t ntiles = tile_end - tile_begin;  // tiles of this shard
    const uint32_t sms = (uint32_t)ctx_sm_count(ctx);

    // ---- upper bounds: every pair live with all `cap` queries.  The actual
    // lists are built on the device (K2p) from n_active / done, so no pass
    // waits for the host.
    const uint32_t tp_per_pair = ceil_div_u(cap, kQueryTilePair);
    const uint32_t tp_max = npairs * tp_per_pair;
    const uint32_t rows_max = tp_max * kQueryTilePair;
    const uint32_t nitems_cap = std::max<uint32_t>(std::max<uint32_t>(2 * tp_max, tp_max * ceil_div_u(ntiles, kMaxUnitTiles)),
                                                   std::min<uint32_t>(64 * tp_max, 64 * sms));
    const size_t item_off = (8 + 2 * (size_t)npairs + 3 * (size_t)tp_max + 3) & ~(size_t)3;
    const size_t words = item_off + 8 * (size_t)nitems_cap;
    uint32_t* dlist = nullptr;
    TRY(ws_arr(ctx, "tc.plan", words, &dlist));
    uint32_t* d_hdr = dlist;
    uint32_t* d_slot_pair = dlist + 8;
    uint32_t* d_slot_base = d_slot_pair + npairs;
    uint32_t* d_tp_pair = d_slot_base + npairs;
    uint32_t* d_tp_row0 = d_tp_pair + tp_max;
    uint32_t* d_tp_qi0 = d_tp_row0 + tp_max;
    TcItem* d_items = reinterpret_cast<TcItem*>(dlist + item_off);

    // ---- device scratch
    uint8_t* qbuf;
    float* margin;
    float4* partial;
    uint32_t* rescan;
    unsigned int* rcount;
    unsigned long long* keys;
    TRY(ws_arr(ctx, "tc.qbuf", (size_t)rows_max * kPackRowBytes, &qbuf));
    TRY(ws_arr(ctx, "tc.margin", rows_max, &margin));
    TRY(ws_arr(ctx, "tc.partial", (size_t)nitems_cap * kPartialSplit * kQueryTilePair * kPartialF4, &partial));
    TRY(ws_arr(ctx, "tc.rescan", (size_t)3 * rows_max, &rescan));
    TRY(ws_arr(ctx, "tc.rcount", 2, &rcount));  // [0] open rows, [1] rescan CTAs retired
    TRY(ws_arr(ctx, "tc.keys", rows_max, &keys));
    // the rescan's finish hands every key it used back as ~0, so the key
    // slots need their initialisation only once per allocation
    if (ws_fresh(ctx, "tc.keys", keys, (size_t)rows_max * 8))
        FNL_CUDA_TRY(cudaMemsetAsync(keys, 0xFF, (size_t)rows_max * 8, s));

    // ---- K2p plan
    {
        static const uint32_t switch_cost =
            getenv("FNL_PLAN_SWITCH") ? (uint32_t)atoi(getenv("FNL_PLAN_SWITCH")) : 3u;
        PlanArgs pa{npairs, d_active, d_done, tile_begin, ntiles, sms, nitems_cap, switch_cost, d_hdr,
                    d_slot_pair, d_slot_base, d_tp_pair, d_tp_row0, d_tp_qi0, d_items, rcount};
        ProfScope prof(ctx, FNL_KCLASS_GATHER);
        plan_kernel<<<1, kPlanThreads, 0, s>>>(pa);
        FNL_CUDA_TRY(cudaGetLastError());
    }
    // binary16 accumulators in K3 when the caller established they are safe
    const bool acc16 = rs.acc16 != 0;
    // ---- K2 gather
    {
        GatherArgs g{Q.data, Q.pair_bytes, ids, cap, d_active, d_slot_pair, d_slot_base, qbuf, margin,
                     T.max_norm, dim, l2, d_hdr, rs.mode, rs.q32, rs.q32_pair_stride, acc16, T.max_norm_hi, Q.cpr};
        dim3 grid(ceil_div_u(tp_per_pair * kQueryTilePair * 4, 256), npairs);
        ProfScope prof(ctx, FNL_KCLASS_GATHER);
        gather_kernel<<<grid, 256, 0, s>>>(g);
        FNL_CUDA_TRY(cudaGetLastError());
    }
    // ---- K3 tensor-core scan (the dominant kernel; timed)
    {
        static const int debug_mode = getenv("FNL_TC_DEBUG") ? atoi(getenv("FNL_TC_DEBUG")) : 0;
        unsigned long long* trace = nullptr;
        if (debug_mode & 16) {
            TRY(ws_arr(ctx, "tc.trace", 7 * 4096, &trace));
            FNL_CUDA_TRY(cudaMemsetAsync(trace, 0, 7 * 4096 * 8, s));
        }
        TcArgs t{qbuf, T.data, T.pair_bytes, T.cpr, nt, d_items, d_hdr + 2, partial, debug_mode, trace};
        const uint32_t grid = std::min<uint32_t>(nitems_cap, sms);
        cudaEvent_t end_ev;
        ctx_score_begin(ctx, &end_ev);
        if (debug_mode) {
            if (acc16) tc_scan_kernel<true, true><<<grid, kScanThreads, kSmemTotal, s>>>(t);
            else tc_scan_kernel<false, true><<<grid, kScanThreads, kSmemTotal, s>>>(t);
        } else {
            if (acc16) tc_scan_kernel<true, false><<<grid, kScanThreads, kSmemTotal, s>>>(t);
            else tc_scan_kernel<false, false><<<grid, kScanThreads, kSmemTotal, s>>>(t);
        }
        ctx_score_end(ctx, end_ev);
        FNL_CUDA_TRY(cudaGetLastError());
    }
    // ---- K3b merge + certification
    {
        MergeArgs m{partial, d_tp_pair, d_tp_row0, d_tp_qi0, d_hdr, d_active, margin, qbuf, T.data,
                    T.pair_bytes, T.cpr, nt, dim, out, min_dist, out_stride, rescan, rcount, d_near_ties, npairs, shard_keys,
                    pp, ids, cap, rs, acc16, merge_prefilter()};
        ProfScope prof(ctx, FNL_KCLASS_MERGE);
        const uint32_t sms_u = (uint32_t)ctx_sm_count(ctx);
        if (dim == 24) {
            if (l2) launch_merge_mode<true, 24>(rs.mode, tp_max, sms_u, m, s);
            else launch_merge_mode<false, 24>(rs.mode, tp_max, sms_u, m, s);
        } else {
            if (l2) launch_merge_mode<true, 0>(rs.mode, tp_max, sms_u, m, s);
            else launch_merge_mode<false, 0>(rs.mode, tp_max, sms_u, m, s);
        }
        FNL_CUDA_TRY(cudaGetLastError());
    }
    // ---- K4' exact re-decision of rows left open (grid-stride over a device count)
    {
        RescanArgs r{rescan, rcount, qbuf, T.data, T.pair_bytes, T.cpr, tile_begin * kBTileRows,
                     std::min(nt, tile_end * kBTileRows), dim, 4096u, keys, l2, ids, cap, rs,
                     rcount + 1, out, min_dist, out_stride, shard_keys, pp};
        const uint32_t grid = 2 * (uint32_t)ctx_sm_count(ctx);
        ProfScope prof(ctx, FNL_KCLASS_RESCAN);
        if (dim == 24) {
            if (l2) launch_rescan_mode<true, 24>(rs.mode, grid, r, s);
            else launch_rescan_mode<false, 24>(rs.mode, grid, r, s);
        } else {
            if (l2) launch_rescan_mode<true, 0>(rs.mode, grid, r, s);
            else launch_rescan_mode<false, 0>(rs.mode, grid, r, s);
        }
        FNL_CUDA_TRY(cudaGetLastError());
    }
    if (debug_mode_trace_dump(ctx, s)) {}
    ctx_count_launches(ctx, 5);
    return FNL_OK;
}

int tensor_shard_finalize(fnl_context* ctx, uint32_t npairs, const long long* keys, uint32_t stride,
                          const uint32_t* d_n_active, const uint8_t* d_done, uint32_t* out) {
    cudaStream_t s = ctx_stream(ctx);
    ProfScope prof(ctx, FNL_KCLASS_OTHER);
    shard_finalize_kernel<<<dim3(ceil_div_u(stride, 256), npairs), 256, 0, s>>>(keys, stride, d_n_active, d_done, out);
    FNL_CUDA_TRY(cudaGetLastError());
    ctx_count_launches(ctx, 1);
    return FNL_OK;
}

int tensor_shard_barrier(fnl_context* ctx, unsigned int* const* flags, uint32_t n, unsigned int* own,
                         unsigned int target, unsigned int* d_err) {
    if (n > (uint32_t)kMaxShardPeers) return fail(FNL_EINVAL, "shard barrier: at most 8 ranks");
    PeerFlags f{};
    for (uint32_t r = 0; r < n; ++r) f.flags[r] = flags[r];
    f.n = n;
    shard_barrier_kernel<<<1, 1, 0, ctx_stream(ctx)>>>(f, own, target, d_err);
    FNL_CUDA_TRY(cudaGetLastError());
    ctx_count_launches(ctx, 1);
    return FNL_OK;
}

int tensor_shard_reset(fnl_context* ctx, long long* keys, uint64_t n) {
    cudaStream_t s = ctx_stream(ctx);
    shard_reset_kernel<<<(uint32_t)std::min<uint64_t>(1024, (n + 255) / 256), 256, 0, s>>>(keys, n);
    FNL_CUDA_TRY(cudaGetLastError());
    ctx_count_launches(ctx, 1);
    return FNL_OK;
}

bool tensor_route_ok(int mode, bool l2, uint32_t dim, float qmax_norm, float tmax_norm,
                     unsigned long long sat, unsigned long long bad) {
    if (dim == 0 || dim + (l2 ? 2u : 0u) > kPackK) return false;
    if (bad != ~0ull) return false;  // non-finite input: the exact kernels decide it
    const double q = (double)qmax_norm * 1.001, t = (double)tmax_norm * 1.001;
    // -|t|^2/2 (both maps serve as targets) must stay a finite binary16 hi term
    if (l2 && std::max(q, t) * std::max(q, t) / 2.0 >= 65504.0) return false;
    if (mode == kResolveRounded) return true;  // its contract is the binary16 rows, saturated or not
    if (sat != 0) return false;                // saturated inputs: relative rounding bound does not hold
    if (mode == kResolveHybrid) {
        // every distance must round to binary16 without saturating (so the
        // reference's distance-saturation count is 0): |d| <= |q||t| (dot),
        // (|q| + |t|)^2 (l2), with the chain's own rounding
        const double dmax = l2 ? (q + t) * (q + t) : q * t;
        if (dmax * 1.01 >= 65504.0) return false;
    }
    return true;
}

bool acc16_ok(bool l2, float qmax_norm, float tmax_norm) {
    static const bool off = getenv("FNL_TC_F16ACC") && atoi(getenv("FNL_TC_F16ACC")) == 0;
    if (off) return false;
    // every score / partial sum stays below 2^14, far inside binary16 (max
    // 65504): dot |q.t| <= |q| |t|; l2 |q.t - |t|^2/2| <= |q| |t| + |t|^2/2,
    // with either map as the target side
    const double q = (double)qmax_norm * 1.001, t = (double)tmax_norm * 1.001;
    if (!l2) return q * t < 16384.0;
    const double m = std::max(q, t);
    return 1.5 * m * m < 16384.0;
}

int tensor_nn_dense(fnl_context* ctx, const float* d_q, uint32_t nq, const float* d_t, uint32_t nt,
                    uint32_t dim, bool l2, uint32_t* d_nearest, float* d_min_dist, int mode, bool* routed) {
    if (routed) {
        *routed = false;
        if (dim == 0 || dim + (l2 ? 2u : 0u) > kPackK) return FNL_OK;
    }
    unsigned long long* scratch;
    TRY(ws_arr(ctx, "tc.dense.scratch", 4, &scratch));
    cudaStream_t s = ctx_stream(ctx);
    FNL_CUDA_TRY(cudaMemsetAsync(scratch, 0xFF, 16, s));
    FNL_CUDA_TRY(cudaMemsetAsync(scratch + 2, 0, 16, s));
    PackedMaps Q, T;
    bool acc16 = false;  // binary16 accumulators only once the norms are known
    TRY(tensor_pack(ctx, "tc.dense.q", d_q, 1, nq, dim, l2, scratch, scratch + 2, &Q));
    TRY(tensor_pack(ctx, "tc.dense.t", d_t, 1, nt, dim, l2, scratch + 1, scratch + 3, &T));
    if (routed) {
        // one host round trip: the pack's norms / saturations / finiteness
        // decide whether this call may take the tensor route
        unsigned long long h[4];
        float n[2];
        FNL_CUDA_TRY(cudaMemcpyAsync(h, scratch, 32, cudaMemcpyDeviceToHost, s));
        FNL_CUDA_TRY(cudaMemcpyAsync(&n[0], Q.max_norm, 4, cudaMemcpyDeviceToHost, s));
        FNL_CUDA_TRY(cudaMemcpyAsync(&n[1], T.max_norm, 4, cudaMemcpyDeviceToHost, s));
        FNL_CUDA_TRY(cudaStreamSynchronize(s));
        const unsigned long long bad = std::min(h[0], h[1]);
        if (!tensor_route_ok(mode, l2, dim, n[0], n[1], h[2] + h[3], bad)) return FNL_OK;
        *routed = true;
        acc16 = acc16_ok(l2, n[0], n[1]);
    }
    unsigned long long* ties;
    TRY(ws_arr(ctx, "tc.dense.ties", 2, &ties));
    FNL_CUDA_TRY(cudaMemsetAsync(ties, 0, 16, s));
    uint32_t* d_nq;
    TRY(ws_arr(ctx, "tc.dense.nq", 1, &d_nq));
    FNL_CUDA_TRY(cudaMemcpyAsync(d_nq, &nq, 4, cudaMemcpyHostToDevice, s));  // pageable: staged before return
    ResolveSrc rs;
    rs.mode = mode;
    rs.acc16 = acc16;
    rs.q32 = d_q;
    rs.q32_pair_stride = (uint64_t)nq * dim;
    rs.t32 = d_t;
    rs.t32_pair_stride = (uint64_t)nt * dim;
    return tensor_nn_pass(ctx, 1, Q, nullptr, nq, d_nq, nullptr, T, dim, l2, d_nearest, nq, d_min_dist, ties, 0, 0,
                          nullptr, nullptr, &rs);
}

int tensor_mutual_dense(fnl_context* ctx, const float* d1, uint32_t p1, const float* d2, uint32_t p2, uint32_t dim,
                        bool l2, int mode, uint32_t* d_fwd, uint32_t* d_bwd, bool* routed,
                        unsigned long long* bad_out) {
    *routed = false;
    if (dim == 0 || dim + (l2 ? 2u : 0u) > kPackK) return FNL_OK;
    unsigned long long* scratch;
    TRY(ws_arr(ctx, "tc.mu.scratch", 4, &scratch));
    cudaStream_t s = ctx_stream(ctx);
    FNL_CUDA_TRY(cudaMemsetAsync(scratch, 0xFF, 16, s));
    FNL_CUDA_TRY(cudaMemsetAsync(scratch + 2, 0, 16, s));
    // each map is packed ONCE and serves as query side in one direction and
    // target side in the other (the gather rewrites the norm channels)
    PackedMaps M1, M2;
    TRY(tensor_pack(ctx, "tc.mu.1", d1, 1, p1, dim, l2, scratch, scratch + 2, &M1));
    TRY(tensor_pack(ctx, "tc.mu.2", d2, 1, p2, dim, l2, scratch + 1, scratch + 3, &M2));
    unsigned long long h[4];
    float n[2];
    FNL_CUDA_TRY(cudaMemcpyAsync(h, scratch, 32, cudaMemcpyDeviceToHost, s));
    FNL_CUDA_TRY(cudaMemcpyAsync(&n[0], M1.max_norm, 4, cudaMemcpyDeviceToHost, s));
    FNL_CUDA_TRY(cudaMemcpyAsync(&n[1], M2.max_norm, 4, cudaMemcpyDeviceToHost, s));
    FNL_CUDA_TRY(cudaStreamSynchronize(s));
    if (bad_out) bad_out[0] = h[0], bad_out[1] = h[1];
    if (!tensor_route_ok(mode, l2, dim, n[0], n[1], h[2] + h[3], std::min(h[0], h[1]))) return FNL_OK;
    *routed = true;
    unsigned long long* ties;
    uint32_t* d_n;
    TRY(ws_arr(ctx, "tc.mu.ties", 2, &ties));
    TRY(ws_arr(ctx, "tc.mu.n", 2, &d_n));
    FNL_CUDA_TRY(cudaMemsetAsync(ties, 0, 16, s));
    const uint32_t hn[2] = {p1, p2};
    FNL_CUDA_TRY(cudaMemcpyAsync(d_n, hn, 8, cudaMemcpyHostToDevice, s));
    FNL_CUDA_TRY(cudaStreamSynchronize(s));  // hn is pageable stack memory
    ResolveSrc f;
    f.mode = mode;
    f.acc16 = acc16_ok(l2, n[0], n[1]);
    f.q32 = d1;
    f.q32_pair_stride = (uint64_t)p1 * dim;
    f.t32 = d2;
    f.t32_pair_stride = (uint64_t)p2 * dim;
    ResolveSrc b = f;
    b.q32 = d2;
    b.q32_pair_stride = (uint64_t)p2 * dim;
    b.t32 = d1;
    b.t32_pair_stride = (uint64_t)p1 * dim;
    TRY(tensor_nn_pass(ctx, 1, M1, nullptr, p1, d_n, nullptr, M2, dim, l2, d_fwd, p1, nullptr, ties, 0, 0, nullptr,
                       nullptr, &f));
    return tensor_nn_pass(ctx, 1, M2, nullptr, p2, d_n + 1, nullptr, M1, dim, l2, d_bwd, p2, nullptr, ties, 0, 0,
                          nullptr, nullptr, &b);
}

int tensor_selftest_scores(fnl_context* ctx, const float* d_q, const float* d_t, uint32_t dim, bool l2,
                           int mode, float* d_out) {
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
    g.qcpr = Q.cpr;
    gather_kernel<<<dim3(4, 1), 256, 0, s>>>(g);
    FNL_CUDA_TRY(cudaGetLastError());
    selftest_kernel<<<1, kSelftestThreads, kSmemTotal, s>>>(qbuf, T.data, T.cpr, d_out, mode);
    FNL_CUDA_TRY(cudaGetLastError());
    FNL_CUDA_TRY(cudaStreamSynchronize(s));
    return FNL_OK;
}

}  // namespace fnl
