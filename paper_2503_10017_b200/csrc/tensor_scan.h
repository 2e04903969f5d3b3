// tensor_scan.h -- K1 pack, K2 gather, K3 tcgen05 HybridCast score + certified
// argmax, K3b merge, K4' exact re-decision of near ties (tensor_scan.cu).
//
// Numeric contract: descriptors are cast to binary16 once (RNE, +-65504
// saturation) and scored on the 5th-gen tensor cores with fp32 accumulation
// (Alg. 3, HybridCast).  The tensor-core scores only ever NOMINATE
// candidates: the winner is decided by the reference FMA chain in the
// arithmetic of the requested backend (ResolveMode), and a row is closed only
// when every target outside the resolved 64-target sub-tiles provably loses
// (its tensor-core score plus a rigorous error bound stays below the exact
// winner).  So the nearest indices and min_dist are bit-identical to the
// reference backend the mode names.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

struct fnl_context;

namespace fnl {

constexpr uint32_t kPackK = 32;            // binary16 channels per packed row
constexpr uint32_t kPackRowBytes = 64;     // 32 x 2 B
constexpr uint32_t kTileRows = 128;        // rows per UMMA operand tile
constexpr uint32_t kTileBytes = kTileRows * kPackRowBytes;  // 8 KB
constexpr uint32_t kQueryTilePair = 256;   // query rows per CTA (two M=128 tiles)

// Packed maps, chunk-major per 256-row tile (a UMMA canonical K-major
// no-swizzle operand with LBO = 4 KB between channel chunks, SBO = 128 B
// between 8-row groups): tile T at T * cpr * 4 KB, channel chunk c (8 halves,
// 16 B per row) at c * 4 KB inside it, row group g at g * 128, row r%8 at
// (r%8) * 16.  Only the cpr = ceil((dim + 2 l2) / 8) chunks that carry data are
// stored (3 for dot at d = 24: 48 of 64 bytes per row); K3 keeps the missing
// chunks zero in shared memory, so one cp.async.bulk of cpr * 4 KB stages a
// 256-target tile.
constexpr uint32_t kChunkBytes = 256 * 16;  // one 8-channel chunk of a 256-row tile
struct PackedMaps {
    uint8_t* data = nullptr;
    uint32_t cpr = 4;         // stored channel chunks per row
    uint64_t pair_bytes = 0;  // bytes per pair's map (rows padded to 256)
    uint32_t rows = 0;        // real rows per map
    uint32_t npairs = 0;
    float* max_norm = nullptr;  // per pair: max L2 norm of a binary16 row (device)
    // per pair: max norm of a row's packed channels 16..31, the first K step of
    // the binary16-accumulator MMA (bounds the partial sum it rounds)
    float* max_norm_hi = nullptr;
};

// K1: fp32 maps (npairs x rows x dim, device) -> packed binary16.  Role
// "target" stores -|t|^2/2 split over channels dim, dim+1 for the l2 metric.
// Non-finite values: first flat index per map into d_bad[pair] (init ~0).
// Saturations per pair added into d_sat[pair].
int tensor_pack(fnl_context* ctx, const char* tag, const float* d_src, uint32_t npairs, uint32_t rows,
                uint32_t dim, bool l2, unsigned long long* d_bad, unsigned long long* d_sat,
                PackedMaps* out, float* d_max_norm = nullptr);

// One NN pass of gathered query rows against target maps, batched over pairs.
// Query rows of pair p: ids[p*cap + i] (or i when ids is null), i < d_active[p];
// pairs with d_active[p] == 0 or d_done[p] (d_done may be null) are skipped.  Both
// are DEVICE arrays: the work lists are planned on the device, so consecutive
// passes are enqueued without a host round trip.  Winner indices land in
// out[p*out_stride + i]; if min_dist is non-null the exact reference distance of
// the winner is written beside it.  d_near_ties[p] counts rows the first
// candidate sub-tile did not settle, d_near_ties[npairs + p] rows that needed
// the full rescan (2 * npairs entries).
//
// Target sharding (config C5): only target tiles [tile_begin, tile_end) of T
// (kTargetTileRows = 256 targets per tile; tile_end = 0 means all) are scanned, and with
// shard_keys non-null the exact per-query winner of that range is written as a
// signed 64-bit key  ((orderable(dist) << 32 | index) ^ 2^63)  into
// shard_keys[p*out_stride + i] instead of out/min_dist, so a MIN all-reduce of
// the keys over the shards (NCCL / gloo int64 MIN) yields the global winner
// with the reference's lowest-index tie rule; tensor_shard_finalize decodes.
// Peer-memory key exchange (config C5 without NCCL): with n > 0 the pass
// pushes every winner key into all n ranks' key buffers (keys[r], mapped into
// this process by CUDA IPC / NVLink peer access) with a system-scope
// atomicMin from the merge / rescan epilogues themselves, so the "all-reduce"
// is fused into the kernels that produce the keys.
constexpr int kMaxShardPeers = 8;

// The arithmetic a pass's winner is decided in (the reference backend it is
// bit-identical to):
enum ResolveMode : int {
    // tensor backend (Alg. 3): reference FMA chain on the binary16-rounded
    // rows, fp32 compare == ref `single` on to_half_round(D)
    kResolveRounded = 0,
    // ref `hybrid` / HybridCast (src/kernels.cpp:117-170): chain on the
    // binary16 rows, each distance cast to binary16, lowest index on ties
    kResolveHybrid = 1,
    // ref `single` / `double` / `bruteforce`, full precision
    // (src/kernels.cpp:31-43): chain on the ORIGINAL fp32 rows
    kResolveFull = 2,
};
// Where kResolveFull reads the original fp32 rows: query map rows (indexed by
// the pass's query ids) and target map rows, npairs stacked maps each.
struct ResolveSrc {
    int mode = kResolveRounded;
    // K3 may accumulate in binary16 (norms small enough that no partial sum
    // saturates; see acc16_ok): certified with a wider margin
    int acc16 = 0;
    const float* q32 = nullptr;
    uint64_t q32_pair_stride = 0;  // floats
    const float* t32 = nullptr;
    uint64_t t32_pair_stride = 0;
};
// Host-side eligibility of the tensor route for one map pair (max row norm of
// the binary16 rows, binary16 saturations, first non-finite index): the packed
// l2 norm term -|t|^2/2 must stay inside binary16, no input may saturate
// (kResolveFull / kResolveHybrid), and hybrid distances must not saturate.
bool tensor_route_ok(int mode, bool l2, uint32_t dim, float qmax_norm, float tmax_norm,
                     unsigned long long sat, unsigned long long bad);
// binary16 accumulators are safe when every score / partial sum stays far
// inside binary16 range: max|q| max|t| < 2^14 (dot), 1.5 max(|q|,|t|)^2 < 2^14
// (l2); FNL_TC_F16ACC=0 turns them off
bool acc16_ok(bool l2, float qmax_norm, float tmax_norm);
struct ShardPeers {
    long long* keys[kMaxShardPeers];
    uint32_t n;
};

int tensor_nn_pass(fnl_context* ctx, uint32_t npairs, const PackedMaps& Q, const uint32_t* ids,
                   uint32_t cap, const uint32_t* d_active, const uint8_t* d_done,
                   const PackedMaps& T, uint32_t dim, bool l2, uint32_t* out, uint32_t out_stride,
                   float* min_dist, unsigned long long* d_near_ties, uint32_t tile_begin = 0,
                   uint32_t tile_end = 0, long long* shard_keys = nullptr, const ShardPeers* peers = nullptr,
                   const ResolveSrc* resolve = nullptr);

// shard keys -> nearest indices for the active queries of every pair
int tensor_shard_finalize(fnl_context* ctx, uint32_t npairs, const long long* keys, uint32_t stride,
                          const uint32_t* d_n_active, const uint8_t* d_done, uint32_t* out);
int tensor_shard_reset(fnl_context* ctx, long long* keys, uint64_t n);
// Cross-GPU barrier over peer memory: increments every rank's counter
// (flags[r], system scope, after a system fence that publishes this rank's
// key pushes), then waits until its own counter reaches `target` (wrapping
// compare).  Gives up after ~20 s and raises *d_err instead of hanging.
int tensor_shard_barrier(fnl_context* ctx, unsigned int* const* flags, uint32_t n, unsigned int* own,
                         unsigned int target, unsigned int* d_err);
// value every shard key starts from (no candidate in this shard)
constexpr long long kShardKeyNone = 0x7FFFFFFFFFFFFFFFll;
constexpr uint32_t kTargetTileRows = 256;  // targets per K3 B tile (shard granularity)

// Dense convenience (fnl_nn_query / mutual NN): all rows of d_q against d_t,
// resolved in the arithmetic of `mode` (ResolveSrc::mode; the fp32 originals
// are d_q / d_t themselves).  With `routed` non-null the pack's norms and
// saturation counts are read back first and the pass runs only if
// tensor_route_ok holds (*routed says whether it did).
int tensor_nn_dense(fnl_context* ctx, const float* d_q, uint32_t nq, const float* d_t, uint32_t nt,
                    uint32_t dim, bool l2, uint32_t* d_nearest, float* d_min_dist, int mode = 0,
                    bool* routed = nullptr);

// Dense mutual NN on the device: each map packed once,
// NN of every D1 pixel in D2 (d_fwd) and of every D2 pixel in D1 (d_bwd),
// back to back with no host round trip, resolved in `mode`'s arithmetic.
// *routed = false (nothing computed) when tensor_route_ok refuses the maps.
// bad_out (optional, 2 entries): first non-finite flat index of D1 / D2 (~0 = none).
int tensor_mutual_dense(fnl_context* ctx, const float* d1, uint32_t p1, const float* d2, uint32_t p2, uint32_t dim,
                        bool l2, int mode, uint32_t* d_fwd, uint32_t* d_bwd, bool* routed,
                        unsigned long long* bad_out = nullptr);

// Self-test: raw tensor-core scores of a packed query tile pair (256 rows)
// against one packed target tile (128 rows) -> out[256][128] fp32.
// mode 0: both operands from shared memory; mode 1: query tiles copied to TMEM
// with tcgen05.cp and a TS MMA (the production path).
int tensor_selftest_scores(fnl_context* ctx, const float* d_q, const float* d_t, uint32_t dim,
                           bool l2, int mode, float* d_out);

}  // namespace fnl
