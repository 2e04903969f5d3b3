// match_loop.cu -- K5 harvest/compaction, K6 convergence, grid init, mutual filter.
//
// The iterative reciprocal matcher of src/reciprocal.cpp:97-206 kept entirely on
// the device, batched over pairs (one CTA per pair per launch):
//   init     : U^0 = row-major centred grid (src/reciprocal.cpp:12-23, :64-80)
//   harvest  : cycle check back[s] == U[s]; converged entries counted (duplicates
//              included); the first (u, v) in sample order is emitted unless u or
//              v was already used; survivors are compacted in order with U <- back
//              (src/reciprocal.cpp:154-179); history push and termination test
//              (src/reciprocal.cpp:180-185) set the pair's done flag.
// Emission order is (iteration, sample position), deterministic: block-wide
// exclusive scans, not atomics, assign every output slot.
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>

#include "fnl_common.cuh"
#include "fnl_internal.h"

namespace fnl {

__device__ __forceinline__ uint32_t axis_position(uint32_t extent, uint32_t stride, uint32_t i,
                                                  uint32_t n) {
    if (n == 1) return extent / 2;
    return min(stride / 2 + i * stride, extent - 1);
}

__global__ void match_init_kernel(MatchState m) {
    const uint32_t p = blockIdx.y;
    const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t nr = (m.h1 + m.grid_stride - 1) / m.grid_stride;
    const uint32_t nc = (m.w1 + m.grid_stride - 1) / m.grid_stride;
    if (s < m.samples) {
        const uint32_t r = s / nc, c = s % nc;
        m.active_u[(size_t)p * m.cap + s] =
            axis_position(m.h1, m.grid_stride, r, nr) * m.w1 + axis_position(m.w1, m.grid_stride, c, nc);
    }
    if (s == 0) {
        m.n_active[p] = m.samples;
        m.n_pairs[p] = 0;
        m.done[p] = m.samples == 0 ? 1 : 0;
        uint32_t* st = m.stats + (size_t)p * kStatWords;
        for (int i = 0; i < kStatWords; ++i) st[i] = 0;
        if (m.samples == 0) atomicAdd(m.n_done, 1u);
    }
}

cudaError_t launch_match_init(const MatchState& m, cudaStream_t s) {
    const uint32_t n = m.samples > 0 ? m.samples : 1;
    dim3 grid((n + 255) / 256, m.npairs);
    match_init_kernel<<<grid, 256, 0, s>>>(m);
    return cudaGetLastError();
}

constexpr int kHarvestThreads = 1024;
constexpr int kHashSlots = 2048;  // >= 2 * kHarvestThreads, power of two

// Block-wide exclusive scan of a 0/1 flag; returns this thread's offset and the total.
__device__ __forceinline__ uint32_t block_scan(uint32_t flag, uint32_t* warp_tot, uint32_t& total) {
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ballot = __ballot_sync(0xFFFFFFFFu, flag);
    const uint32_t in_warp = __popc(ballot & ((1u << lane) - 1u));
    if (lane == 0) warp_tot[warp] = __popc(ballot);
    __syncthreads();
    if (warp == 0) {
        const uint32_t v = warp_tot[lane];  // blockDim == 1024 -> 32 warps
        uint32_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xFFFFFFFFu, x, o);
            if (lane >= (uint32_t)o) x += y;
        }
        warp_tot[lane] = x - v;        // exclusive prefix of warp totals
        if (lane == 31) warp_tot[32] = x;
    }
    __syncthreads();
    const uint32_t off = warp_tot[warp] + in_warp;
    total = warp_tot[32];
    __syncthreads();
    return off;
}

__global__ void __launch_bounds__(kHarvestThreads) harvest_kernel(MatchState m, uint32_t t_arg) {
    const uint32_t p = blockIdx.x;
    if (m.done[p]) return;
    const uint32_t t = m.iter ? *m.iter + 1 : t_arg;  // graph replay: the device counter
    __shared__ uint32_t hkey[kHashSlots];
    __shared__ uint32_t hpos[kHashSlots];
    __shared__ uint32_t warp_tot[33];

    const uint32_t n = m.n_active[p];
    uint32_t* U = m.active_u + (size_t)p * m.cap;
    uint32_t* V = m.active_v + (size_t)p * m.cap;
    const uint32_t* B = m.back + (size_t)p * m.cap;
    uint32_t* used_i = m.used_i + (size_t)p * m.words_i;
    uint32_t* used_j = m.used_j + (size_t)p * m.words_j;
    uint32_t* out = m.pairs + (size_t)p * 3 * m.cap;
    uint32_t* st = m.stats + (size_t)p * kStatWords;

    uint32_t kept = 0, emitted = m.n_pairs[p], conv_total = 0, dup_total = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += kHarvestThreads) {
        const uint32_t s = c0 + threadIdx.x;
        const bool valid = s < n;
        const uint32_t u = valid ? U[s] : 0u, v = valid ? V[s] : 0u, b = valid ? B[s] : 0u;
        const bool conv = valid && b == u;

        // first converged occurrence of u inside this chunk (min sample position)
        for (uint32_t i = threadIdx.x; i < kHashSlots; i += kHarvestThreads) {
            hkey[i] = 0xFFFFFFFFu;
            hpos[i] = 0xFFFFFFFFu;
        }
        __syncthreads();
        uint32_t slot = 0;
        if (conv) {
            slot = (u * 2654435761u) & (kHashSlots - 1);
            while (true) {
                const uint32_t prev = atomicCAS(&hkey[slot], 0xFFFFFFFFu, u);
                if (prev == 0xFFFFFFFFu || prev == u) break;
                slot = (slot + 1) & (kHashSlots - 1);
            }
            atomicMin(&hpos[slot], s);
        }
        __syncthreads();
        const bool first = conv && hpos[slot] == s;
        const bool emit = first && !((used_i[u >> 5] >> (u & 31)) & 1u) &&
                          !((used_j[v >> 5] >> (v & 31)) & 1u);
        const bool surv = valid && !conv;

        uint32_t n_emit, n_surv, n_conv;
        const uint32_t epos = block_scan(emit ? 1u : 0u, warp_tot, n_emit);
        const uint32_t spos = block_scan(surv ? 1u : 0u, warp_tot, n_surv);
        block_scan(conv ? 1u : 0u, warp_tot, n_conv);

        if (surv) {  // in place: kept + spos <= s, positions already read
            U[kept + spos] = b;
            V[kept + spos] = v;
        }
        if (emit) {
            uint32_t* o = out + 3u * (emitted + epos);
            o[0] = u;
            o[1] = v;
            o[2] = t;
            atomicOr(&used_i[u >> 5], 1u << (u & 31));
            atomicOr(&used_j[v >> 5], 1u << (v & 31));
        }
        kept += n_surv;
        emitted += n_emit;
        conv_total += n_conv;
        dup_total += n_conv - n_emit;
        __syncthreads();
    }

    if (threadIdx.x == 0) {
        m.n_active[p] = kept;
        m.n_pairs[p] = emitted;
        const uint32_t converged = st[kStatConverged] + conv_total;
        st[kStatConverged] = converged;
        st[kStatDups] += dup_total;
        st[kStatIters] = t;
        const uint32_t hl = st[kStatHistLen];
        if (hl < 64) st[kStatHist + hl] = kept;
        st[kStatHistLen] = hl + 1;
        const double frac = (double)converged / (double)m.samples;
        if (frac >= m.convergence || t == m.max_iters || kept == 0) {
            m.done[p] = 1;
            atomicAdd(m.n_done, 1u);
        }
    }
}

cudaError_t launch_harvest(const MatchState& m, uint32_t iteration, cudaStream_t s) {
    harvest_kernel<<<m.npairs, kHarvestThreads, 0, s>>>(m, iteration);
    return cudaGetLastError();
}

__global__ void loop_cond_kernel(MatchState m, cudaGraphConditionalHandle h) {
    const uint32_t t = *m.iter + 1;  // the iteration just harvested
    *m.iter = t;
    cudaGraphSetConditional(h, (*m.n_done < m.npairs && t < m.max_iters) ? 1u : 0u);
}

cudaError_t launch_loop_cond(const MatchState& m, cudaGraphConditionalHandle h, cudaStream_t s) {
    loop_cond_kernel<<<1, 1, 0, s>>>(m, h);
    return cudaGetLastError();
}

// ---------------------------------------------------------------- mutual filter
struct MutualPred {
    const uint32_t* fwd;
    const uint32_t* bwd;
    __device__ bool operator()(uint32_t i) const { return bwd[fwd[i]] == i; }
};

__global__ void expand_pairs_kernel(const uint32_t* idx, const uint32_t* count, const uint32_t* fwd,
                                    uint32_t* pairs) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k < *count) {
        const uint32_t i = idx[k];
        pairs[2 * k] = i;
        pairs[2 * k + 1] = fwd[i];
    }
}

// Confidence-thresholded correspondence compaction (north-star extension; the
// reference has no threshold): per pair, keep the matches (i, j, iter) whose
// reference distance dist_scalar(D1[i], D2[j]) (src/kernels.cpp:277-285, the
// FMA chain in channel order on the maps as given) is <= max_dist.  Keep
// flags are counted per warp with ballot/popc and the warp offsets are scanned
// in warp order, so the compaction is in place and stable (the MatchSet keeps
// the reference emission order).
__global__ void __launch_bounds__(kHarvestThreads) confidence_compact_kernel(ConfArgs a) {
    __shared__ uint32_t warp_tot[33];
    const uint32_t p = blockIdx.x;
    const uint32_t n = a.n_pairs[p];
    uint32_t* P = a.pairs + (size_t)p * 3 * a.cap;
    const float* D1 = a.d1 + (size_t)p * a.map1_stride;
    const float* D2 = a.d2 + (size_t)p * a.map2_stride;
    uint32_t kept = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += kHarvestThreads) {
        const uint32_t s = c0 + threadIdx.x;
        const bool valid = s < n;
        uint32_t i = 0, j = 0, it = 0;
        bool keep = false;
        if (valid) {
            i = P[3 * s];
            j = P[3 * s + 1];
            it = P[3 * s + 2];
            const float d = a.l2 ? chain<true>(D1 + (size_t)i * a.dim, D2 + (size_t)j * a.dim, a.dim)
                                 : chain<false>(D1 + (size_t)i * a.dim, D2 + (size_t)j * a.dim, a.dim);
            keep = d <= a.max_dist;  // NaN is never kept
        }
        uint32_t nk;
        const uint32_t pos = block_scan(keep ? 1u : 0u, warp_tot, nk);
        if (keep) {  // kept + pos <= s: every source entry of this chunk is already in registers
            uint32_t* o = P + 3 * (kept + pos);
            o[0] = i;
            o[1] = j;
            o[2] = it;
        }
        kept += nk;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        a.n_pairs[p] = kept;
        if (a.dropped) a.dropped[p] = n - kept;
    }
}

// ---------------------------------------------------------------- reverse-NN memo
// rev_cache[j]: the NN of map-2 pixel j once known (< 2^31), kRevUnknown, or
// 2^31 | i while active entry i is the lowest one asking for j in this pass.
// Lookup: known pixels answer back[i] at once; unknown ones take the minimum
// claimant by atomicMin.  Compaction: the claimants, in entry order (block
// scans, so every rank of a sharded run builds the same list), form the pass's
// query list.  Fill: results into the memo, back[i] for every active entry.
constexpr uint32_t kRevClaim = 0x80000000u;

__global__ void rev_claim_kernel(MatchState m) {
    const uint32_t p = blockIdx.y;
    if (m.done[p]) return;
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= m.n_active[p]) return;
    const uint32_t j = m.active_v[(size_t)p * m.cap + i];
    uint32_t* cache = m.rev_cache + (size_t)p * m.p2;
    const uint32_t c = cache[j];
    if (c < kRevClaim) m.back[(size_t)p * m.cap + i] = c;
    else atomicMin(&cache[j], kRevClaim | i);
}

__global__ void __launch_bounds__(kHarvestThreads) rev_compact_kernel(MatchState m) {
    __shared__ uint32_t warp_tot[33];
    __shared__ uint32_t s_n;
    const uint32_t p = blockIdx.x;
    if (threadIdx.x == 0) s_n = m.done[p] ? 0xFFFFFFFFu : m.n_active[p];
    __syncthreads();
    const uint32_t n = s_n;  // one read per block: the loop below is CTA-uniform
    if (n == 0xFFFFFFFFu) return;
    const uint32_t* V = m.active_v + (size_t)p * m.cap;
    const uint32_t* cache = m.rev_cache + (size_t)p * m.p2;
    uint32_t* L = m.rev_list + (size_t)p * m.cap;
    uint32_t kept = 0;
    for (uint32_t c0 = 0; c0 < n; c0 += kHarvestThreads) {
        const uint32_t i = c0 + threadIdx.x;
        const uint32_t j = i < n ? V[i] : 0u;
        const bool claim = i < n && cache[j] == (kRevClaim | i);
        uint32_t total;
        const uint32_t off = block_scan(claim ? 1u : 0u, warp_tot, total);
        if (claim) L[kept + off] = j;
        kept += total;
    }
    if (threadIdx.x == 0) m.rev_n[p] = kept;
}

__global__ void __launch_bounds__(kHarvestThreads) rev_fill_kernel(MatchState m) {
    const uint32_t p = blockIdx.x;
    if (m.done[p]) return;
    const uint32_t nl = m.rev_n[p], n = m.n_active[p];
    uint32_t* cache = m.rev_cache + (size_t)p * m.p2;
    const uint32_t* L = m.rev_list + (size_t)p * m.cap;
    const uint32_t* R = m.rev_out + (size_t)p * m.cap;
    for (uint32_t k = threadIdx.x; k < nl; k += blockDim.x) cache[L[k]] = R[k];
    __syncthreads();
    const uint32_t* V = m.active_v + (size_t)p * m.cap;
    uint32_t* B = m.back + (size_t)p * m.cap;
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) B[i] = cache[V[i]];
    if (threadIdx.x == 0) m.stats[(size_t)p * kStatWords + kStatRevComputed] += nl;
}

cudaError_t launch_rev_lookup(const MatchState& m, cudaStream_t s) {
    const uint32_t n = m.cap > 0 ? m.cap : 1;
    rev_claim_kernel<<<dim3((n + 255) / 256, m.npairs), 256, 0, s>>>(m);
    rev_compact_kernel<<<m.npairs, kHarvestThreads, 0, s>>>(m);
    return cudaGetLastError();
}
cudaError_t launch_rev_fill(const MatchState& m, cudaStream_t s) {
    rev_fill_kernel<<<m.npairs, kHarvestThreads, 0, s>>>(m);
    return cudaGetLastError();
}

cudaError_t launch_confidence_compact(const ConfArgs& a, uint32_t npairs, cudaStream_t s) {
    if (npairs == 0) return cudaSuccess;
    confidence_compact_kernel<<<npairs, kHarvestThreads, 0, s>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_mutual_filter(const uint32_t* fwd, const uint32_t* bwd, uint32_t n,
                                 uint32_t* pairs, uint32_t* count, cudaStream_t s) {
    // pairs doubles as scratch: selected indices land in its upper half first.
    uint32_t* idx = pairs + n;
    thrust::counting_iterator<uint32_t> it(0);
    size_t temp = 0;
    cudaError_t e = cub::DeviceSelect::If(nullptr, temp, it, idx, count, (int)n, MutualPred{fwd, bwd}, s);
    if (e != cudaSuccess) return e;
    void* tmp = nullptr;
    e = cudaMallocAsync(&tmp, temp, s);
    if (e != cudaSuccess) return e;
    e = cub::DeviceSelect::If(tmp, temp, it, idx, count, (int)n, MutualPred{fwd, bwd}, s);
    cudaFreeAsync(tmp, s);
    if (e != cudaSuccess) return e;
    // expand in place (k-th output pair at 2k, 2k+1 never overtakes idx[k] at n+k
    // within one thread, but different threads race) -> use a separate pass.
    uint32_t* tmp_idx = nullptr;
    e = cudaMallocAsync(&tmp_idx, (size_t)n * 4, s);
    if (e != cudaSuccess) return e;
    cudaMemcpyAsync(tmp_idx, idx, (size_t)n * 4, cudaMemcpyDeviceToDevice, s);
    expand_pairs_kernel<<<(n + 255) / 256, 256, 0, s>>>(tmp_idx, count, fwd, pairs);
    cudaFreeAsync(tmp_idx, s);
    return cudaGetLastError();
}

}  // namespace fnl
