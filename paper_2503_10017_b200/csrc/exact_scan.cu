// exact_scan.cu -- K1 prepare, K4 exact fused score+argmin, block scorer.
//
// K4 is the bit-faithful CUDA-core path behind the reference backends
// (bruteforce / double / single / hybrid): every distance is the reference
// FMA chain in channel order (src/kernels.cpp:31-43), hybrid rounds inputs and
// each distance to binary16 with saturation counting (src/kernels.cpp:64-89,
// :117-125, :165), and the argmin keeps the lowest index on exact ties
// (src/kernels.cpp:202-229).  Layout: one thread owns one query row in
// registers; targets stream through shared memory in chunks that every thread
// of the CTA reads by broadcast; gridDim.y splits the target range and the
// split results merge through a 64-bit atomicMin on packed keys, which is
// order independent, so the answer never depends on the split or schedule.
//
// Roofline: FMA-pipe bound, dim FFMA (dot) or dim FADD + dim FFMA (l2) per
// score; target traffic is L2-resident (every CTA re-reads its split).
#include <math.h>

#include "fnl_common.cuh"
#include "fnl_internal.h"

namespace fnl {

// ---------------------------------------------------------------- K1 prepare
__global__ void prepare_kernel(PrepareArgs a) {
    const uint64_t row = blockIdx.x * (uint64_t)blockDim.y + threadIdx.y;
    uint32_t sat = 0;
    if (row < a.rows) {
        const float* src = a.src + row * a.dim;
        for (uint32_t c = threadIdx.x; c < a.dim; c += blockDim.x) {
            const float v = src[c];
            if (!isfinite(v)) atomicMin(a.bad_index, (unsigned long long)(row * a.dim + c));
            if (a.rounded) {
                uint32_t s = 0;
                a.rounded[row * a.dim + c] = half_round_sat(v, s);
                sat += s;
            }
        }
    }
    if (a.rounded) {
        // blockDim.x == 32: one warp per row
        const uint32_t row_total = warp_sum(sat);
        if (threadIdx.x == 0 && row < a.rows) {
            if (a.row_sat) a.row_sat[row] = (uint8_t)min(row_total, 255u);
            if (row_total) atomicAdd(a.total_sat, (unsigned long long)row_total);
        }
    }
}

cudaError_t launch_prepare(const PrepareArgs& a, cudaStream_t s) {
    if (a.rows == 0) return cudaSuccess;
    dim3 block(32, 8);
    dim3 grid((unsigned)((a.rows + 7) / 8));
    prepare_kernel<<<grid, block, 0, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- K4 exact scan
constexpr int kScanThreads = 128;

template <int DMAX>
struct QueryRegs {
    float v[DMAX];
};

// Distance of the register-resident query against one smem target row.
template <bool kL2, int DMAX, bool kExactDim>
__device__ __forceinline__ float reg_chain(const QueryRegs<DMAX>& q, const float* __restrict__ t,
                                           uint32_t dim) {
    float acc = 0.0f;
#pragma unroll
    for (int c = 0; c < DMAX; ++c) {
        if (kExactDim || (uint32_t)c < dim) {
            if constexpr (kL2) {
                const float d = __fsub_rn(q.v[c], t[c]);
                acc = __fmaf_rn(d, d, acc);
            } else {
                acc = __fmaf_rn(q.v[c], t[c], acc);
            }
        }
    }
    return kL2 ? acc : -acc;
}

// DMAX > 0: queries in registers (dim <= DMAX; kExactDim when dim == DMAX).
// DMAX == 0: generic dim, query re-read from global memory (L1 resident).
// Each thread scores QB queries (q, q + kScanThreads, ...) against every
// staged target, so one broadcast shared-memory read of a target channel feeds
// QB independent FMA chains (the scan is otherwise bound by LDS issue).
// Queries per thread: 4, or 2 when a query row of up to 64 channels lives in
// registers (4 x 64 would spill).  dim 33..64 are the DMAX = 64 kernels.
constexpr int kQB = 4;
// (1 for the hybrid kernels of dim 33..63, whose predicated channel loop
// would otherwise spill inside the scan loop).
__host__ __device__ constexpr int qb_for(int dmax, bool hyb, bool exact_dim) {
    return dmax > 32 ? (hyb && !exact_dim ? 1 : 2) : kQB;
}
__host__ __device__ constexpr int qb_for_dim(uint32_t dim, bool hyb) {
    return dim > 32 && dim <= 64 ? (hyb && dim != 64 ? 1 : 2) : kQB;
}

template <bool kL2, bool kHyb, int DMAX, bool kExactDim>
__global__ void __launch_bounds__(kScanThreads) exact_scan_kernel(ScanArgs a, uint32_t chunk) {
    constexpr int QB = qb_for(DMAX, kHyb, kExactDim);
    extern __shared__ float4 smem4[];
    float* tile = reinterpret_cast<float*>(smem4);
    const uint32_t pair = blockIdx.z;
    if (a.pair_done && a.pair_done[pair]) return;
    const uint32_t nq = a.qcount ? a.qcount[pair] : a.qcount_const;
    if (blockIdx.x * kScanThreads * QB >= nq) return;
    const uint32_t t0 = blockIdx.y * a.split_len;
    if (t0 >= a.nt) return;
    const uint32_t t1 = min(a.nt, t0 + a.split_len);
    const uint32_t dim = a.dim;

    uint32_t qi[QB], row[QB];
    bool active[QB];
    const float* qsrc[QB];
    QueryRegs<(DMAX > 0 ? DMAX : 1)> qr[QB];
#pragma unroll
    for (int b = 0; b < QB; ++b) {
        qi[b] = blockIdx.x * kScanThreads * QB + b * kScanThreads + threadIdx.x;
        active[b] = qi[b] < nq;
        row[b] = 0;
        if (active[b]) row[b] = a.qids ? a.qids[(size_t)pair * a.qids_pair_stride + qi[b]] : qi[b];
        qsrc[b] = a.qmap + pair * a.qmap_pair_stride + (size_t)row[b] * dim;
        if constexpr (DMAX > 0) {
#pragma unroll
            for (int c = 0; c < DMAX; ++c)
                qr[b].v[c] = (active[b] && (kExactDim || (uint32_t)c < dim)) ? qsrc[b][c] : 0.0f;
        }
    }
    const bool any_active = active[0];

    const float* T = a.tmap + pair * a.tmap_pair_stride;
    float best[QB];
    uint32_t bidx[QB];
#pragma unroll
    for (int b = 0; b < QB; ++b) {
        best[b] = INFINITY;
        bidx[b] = t0;
    }
    uint32_t dsat = 0;

    for (uint32_t c0 = t0; c0 < t1; c0 += chunk) {
        const uint32_t n = min(chunk, t1 - c0);
        __syncthreads();
        const float* src = T + (size_t)c0 * dim;
        const uint32_t total = n * dim;
        // float4 staging needs a 16 B aligned source (rows of dim % 4 != 0
        // floats start at 8 B boundaries) and a whole number of float4s
        if ((reinterpret_cast<uintptr_t>(src) & 15u) == 0 && (total & 3u) == 0) {
            const float4* s4 = reinterpret_cast<const float4*>(src);
            for (uint32_t i = threadIdx.x; i < total / 4; i += kScanThreads) smem4[i] = __ldg(s4 + i);
        } else {
            for (uint32_t i = threadIdx.x; i < total; i += kScanThreads) tile[i] = __ldg(src + i);
        }
        __syncthreads();
        if (any_active) {
#pragma unroll 2
            for (uint32_t j = 0; j < n; ++j) {
                const float* t = tile + (size_t)j * dim;
#pragma unroll
                for (int b = 0; b < QB; ++b) {
                    float d;
                    if constexpr (DMAX > 0) {
                        d = reg_chain<kL2, DMAX, kExactDim>(qr[b], t, dim);
                    } else {
                        d = chain<kL2>(qsrc[b], t, dim);
                    }
                    if constexpr (kHyb) {
                        uint32_t sb = 0;
                        d = half_round_sat(d, sb);
                        if (active[b]) dsat += sb;
                    }
                    if (d < best[b]) {  // strict: earlier index keeps a tie; NaN never wins
                        best[b] = d;
                        bidx[b] = c0 + j;
                    }
                }
            }
        }
    }
#pragma unroll
    for (int b = 0; b < QB; ++b)
        if (active[b]) atomicMin(a.keys + (size_t)pair * a.keys_pair_stride + qi[b], pack_key(best[b], bidx[b]));

    if constexpr (kHyb) {
        uint32_t qsat = 0;
        if (blockIdx.y == 0 && a.q_row_sat) {
#pragma unroll
            for (int b = 0; b < QB; ++b)
                if (active[b]) qsat += a.q_row_sat[pair * a.q_row_sat_pair_stride + row[b]];
        }
        const uint32_t ws = warp_sum(dsat), wq = warp_sum(qsat);
        if ((threadIdx.x & 31) == 0) {
            if (wq) atomicAdd(a.counters + 2 * pair + 0, (unsigned long long)wq);
            if (ws) atomicAdd(a.counters + 2 * pair + 1, (unsigned long long)ws);
        }
    }
}

template <bool kL2, bool kHyb>
static cudaError_t dispatch_dim(const ScanArgs& a, dim3 grid, uint32_t chunk, size_t smem,
                                cudaStream_t s) {
    switch (a.dim) {
        case 24: exact_scan_kernel<kL2, kHyb, 24, true><<<grid, kScanThreads, smem, s>>>(a, chunk); break;
        case 16: exact_scan_kernel<kL2, kHyb, 16, true><<<grid, kScanThreads, smem, s>>>(a, chunk); break;
        case 32: exact_scan_kernel<kL2, kHyb, 32, true><<<grid, kScanThreads, smem, s>>>(a, chunk); break;
        case 64: exact_scan_kernel<kL2, kHyb, 64, true><<<grid, kScanThreads, smem, s>>>(a, chunk); break;
        default:
            if (a.dim <= 8)
                exact_scan_kernel<kL2, kHyb, 8, false><<<grid, kScanThreads, smem, s>>>(a, chunk);
            else if (a.dim <= 32)
                exact_scan_kernel<kL2, kHyb, 32, false><<<grid, kScanThreads, smem, s>>>(a, chunk);
            else if (a.dim <= 64)
                exact_scan_kernel<kL2, kHyb, 64, false><<<grid, kScanThreads, smem, s>>>(a, chunk);
            else
                exact_scan_kernel<kL2, kHyb, 0, false><<<grid, kScanThreads, smem, s>>>(a, chunk);
    }
    return cudaGetLastError();
}

cudaError_t launch_exact_scan(const ScanArgs& a, uint32_t max_q, uint32_t npairs, bool l2,
                              bool hybrid, cudaStream_t s) {
    if (max_q == 0 || npairs == 0 || a.nt == 0) return cudaSuccess;
    // chunk of targets staged per smem round (<= 32 KB)
    uint32_t chunk = 8192u / a.dim;
    chunk = chunk < 1 ? 1 : (chunk > 256 ? 256 : chunk);
    const size_t smem = (size_t)chunk * a.dim * sizeof(float);
    const uint32_t qb = (uint32_t)qb_for_dim(a.dim, hybrid);
    const uint32_t gx = (max_q + kScanThreads * qb - 1) / (kScanThreads * qb);
    // Split targets so that the grid covers the machine several times over.
    const uint32_t want_ctas = 148u * 8u;
    uint32_t splits = (want_ctas + gx * npairs - 1) / (gx * npairs);
    const uint32_t max_splits = (a.nt + chunk - 1) / chunk;
    splits = splits < 1 ? 1 : (splits > max_splits ? max_splits : splits);
    if (splits > 65535) splits = 65535;
    ScanArgs b = a;
    b.split_len = (a.nt + splits - 1) / splits;
    splits = (a.nt + b.split_len - 1) / b.split_len;
    dim3 grid(gx, splits, npairs);
    if (l2) return hybrid ? dispatch_dim<true, true>(b, grid, chunk, smem, s)
                          : dispatch_dim<true, false>(b, grid, chunk, smem, s);
    return hybrid ? dispatch_dim<false, true>(b, grid, chunk, smem, s)
                  : dispatch_dim<false, false>(b, grid, chunk, smem, s);
}

// ---------------------------------------------------------------- finalize
__global__ void finalize_kernel(FinalizeArgs a) {
    const uint32_t pair = blockIdx.y;
    if (a.pair_done && a.pair_done[pair]) return;
    const uint32_t nq = a.qcount ? a.qcount[pair] : a.qcount_const;
    const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nq) return;
    unsigned long long* kp = a.keys + (size_t)pair * a.keys_pair_stride + q;
    const unsigned long long key = *kp;
    *kp = ~0ull;
    a.nearest[(size_t)pair * a.nearest_pair_stride + q] = (uint32_t)(key & 0xFFFFFFFFull);
    if (a.min_dist) {
        float d = from_orderable((uint32_t)(key >> 32));
        if (d == 0.0f) {
            if (a.hybrid && a.qmap) {  // the winner's own signed zero
                const uint32_t idx = (uint32_t)(key & 0xFFFFFFFFull);
                const float* qr = a.qmap + (size_t)q * a.dim;
                const float* tr = a.tmap + (size_t)idx * a.dim;
                d = half_round_nosat(a.dot ? chain<false>(qr, tr, a.dim) : chain<true>(qr, tr, a.dim));
            } else {
                d = a.dot ? -0.0f : 0.0f;  // canonical sign of an exact zero (fp32 chain)
            }
        }
        a.min_dist[(size_t)pair * a.nearest_pair_stride + q] = d;
    }
}

cudaError_t launch_finalize(const FinalizeArgs& a, uint32_t max_q, uint32_t npairs, cudaStream_t s) {
    if (max_q == 0 || npairs == 0) return cudaSuccess;
    dim3 grid((max_q + 255) / 256, npairs);
    finalize_kernel<<<grid, 256, 0, s>>>(a);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- block scorer
template <bool kL2, bool kHyb>
__global__ void block_distances_kernel(const float* __restrict__ q, uint32_t nq,
                                       const float* __restrict__ t, uint32_t nt, uint32_t dim,
                                       float* __restrict__ out, unsigned long long* sat) {
    const uint32_t col = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t r = blockIdx.y;
    uint32_t s = 0;
    if (col < nt) {
        float d = chain<kL2>(q + (size_t)r * dim, t + (size_t)col * dim, dim);
        if constexpr (kHyb) d = half_round_sat(d, s);
        out[(size_t)r * nt + col] = d;
    }
    if constexpr (kHyb) {
        const uint32_t w = warp_sum(s);
        if ((threadIdx.x & 31) == 0 && w) atomicAdd(sat, (unsigned long long)w);
    }
}

cudaError_t launch_block_distances(const float* q, uint32_t nq, const float* t, uint32_t nt,
                                   uint32_t dim, bool l2, bool hybrid, float* out,
                                   unsigned long long* dist_sat, cudaStream_t s) {
    if (nq == 0 || nt == 0) return cudaSuccess;
    for (uint32_t r0 = 0; r0 < nq; r0 += 65535) {
        const uint32_t rows = min(65535u, nq - r0);
        dim3 grid((nt + 127) / 128, rows);
        const float* qq = q + (size_t)r0 * dim;
        float* oo = out + (size_t)r0 * nt;
        if (l2) {
            if (hybrid) block_distances_kernel<true, true><<<grid, 128, 0, s>>>(qq, rows, t, nt, dim, oo, dist_sat);
            else block_distances_kernel<true, false><<<grid, 128, 0, s>>>(qq, rows, t, nt, dim, oo, dist_sat);
        } else {
            if (hybrid) block_distances_kernel<false, true><<<grid, 128, 0, s>>>(qq, rows, t, nt, dim, oo, dist_sat);
            else block_distances_kernel<false, false><<<grid, 128, 0, s>>>(qq, rows, t, nt, dim, oo, dist_sat);
        }
    }
    return cudaGetLastError();
}

}  // namespace fnl
