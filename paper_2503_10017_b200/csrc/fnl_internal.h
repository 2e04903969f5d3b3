// fnl_internal.h -- launchers shared by the .cu translation units of
// libfastnn_b200.so.  Not part of the public ABI (include/fastnn_b200.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

namespace fnl {

// thread-local error plumbing (capi.cu)
int fail(int status, const std::string& msg);
int fail_cuda(cudaError_t e, const char* expr, const char* file, int line);

// context services (capi.cu) for the other translation units
}  // namespace fnl
struct fnl_context;
namespace fnl {
cudaStream_t ctx_stream(fnl_context* ctx);
int ctx_sm_count(fnl_context* ctx);
// grow-only named device / pinned-host workspace slots
int ws_device(fnl_context* ctx, const char* name, size_t bytes, void** out);
int ws_pinned(fnl_context* ctx, const char* name, size_t bytes, void** out);
// true the first time workspace slot `name` is seen at address p with this
// size (its contents still need their one-time initialisation)
bool ws_fresh(fnl_context* ctx, const char* name, const void* p, size_t bytes);
template <typename T>
int ws_arr(fnl_context* ctx, const char* name, size_t count, T** out) {
    void* p = nullptr;
    const int st = ws_device(ctx, name, count * sizeof(T), &p);
    *out = static_cast<T*>(p);
    return st;
}
// brackets one launch of the dominant scoring kernel (CUDA events)
void ctx_score_begin(fnl_context* ctx, cudaEvent_t* end_event);
void ctx_score_end(fnl_context* ctx, cudaEvent_t end_event);
void ctx_count_launches(fnl_context* ctx, int n);
// brackets one launch of kernel class cls (FNL_KCLASS_*); no-op unless profiling
void ctx_prof_begin(fnl_context* ctx, int cls, cudaEvent_t* end_event);
void ctx_prof_end(fnl_context* ctx, int cls, cudaEvent_t end_event);
struct ProfScope {
    fnl_context* ctx;
    int cls;
    cudaEvent_t end = nullptr;
    ProfScope(fnl_context* c, int k) : ctx(c), cls(k) { ctx_prof_begin(ctx, cls, &end); }
    ~ProfScope() { ctx_prof_end(ctx, cls, end); }
};

// ---------------------------------------------------------------- K7 FlashMatch
int flashmatch_forward(fnl_context* ctx, const struct fnl_attention_desc& d);
// native NCCL (comm.cu)
int comm_allreduce_min_i64(struct fnl_comm* comm, long long* d_keys, uint64_t count, cudaStream_t stream);
int comm_size(const struct fnl_comm* comm, int* nranks, int* rank);
int flashmatch_trace(unsigned long long* host64);  // profiling aid (FNL_FM_TRACE=1)

// ---------------------------------------------------------------- K1 prepare
// Validates finiteness (first offending flat index into *bad_index, which the
// caller initialises to UINT64_MAX), and for hybrid writes the binary16-rounded
// copy `rounded` plus per-row saturation counts `row_sat` and the map total.
struct PrepareArgs {
    const float* src;
    float* rounded;              // may be null (full precision)
    uint8_t* row_sat;            // may be null; one byte per row (saturating channels, <=255 kept)
    unsigned long long* total_sat;
    unsigned long long* bad_index;
    uint64_t rows;
    uint32_t dim;
};
cudaError_t launch_prepare(const PrepareArgs& a, cudaStream_t s);

// ---------------------------------------------------------------- K4 exact scan
// Fused score + lowest-index argmin of gathered query rows against a target
// map, bit-identical to src/kernels.cpp:137-233.  Batched over pairs
// (gridDim.z), split over target ranges (gridDim.y) and merged with a 64-bit
// atomicMin on packed (orderable dist, index) keys.
struct ScanArgs {
    const float* qmap;            // query map rows (fp32, rounded for hybrid)
    uint64_t qmap_pair_stride;    // floats between consecutive pairs' maps
    const uint32_t* qids;         // per pair query pixel ids, or null = identity
    uint32_t qids_pair_stride;
    const uint32_t* qcount;       // per pair active query count, or null
    uint32_t qcount_const;        // used when qcount is null
    const uint8_t* pair_done;     // per pair skip flag, or null
    const uint8_t* q_row_sat;     // hybrid: saturations of each query-map row, or null
    uint64_t q_row_sat_pair_stride;
    const float* tmap;            // target map rows (fp32, rounded for hybrid)
    uint64_t tmap_pair_stride;
    uint32_t nt;
    uint32_t dim;
    uint32_t split_len;           // targets per gridDim.y slice
    unsigned long long* keys;     // per pair x query packed keys (init ~0)
    uint32_t keys_pair_stride;
    unsigned long long* counters; // [0] query-row saturations, [1] distance saturations
};
// max_q: upper bound of queries per pair (sizes gridDim.x)
cudaError_t launch_exact_scan(const ScanArgs& a, uint32_t max_q, uint32_t npairs, bool l2,
                              bool hybrid, cudaStream_t s);

// keys -> nearest / min_dist; resets keys to ~0 for the next call.
struct FinalizeArgs {
    unsigned long long* keys;
    uint32_t keys_pair_stride;
    const uint32_t* qcount;
    uint32_t qcount_const;
    const uint8_t* pair_done;
    uint32_t* nearest;            // per pair x query
    uint32_t nearest_pair_stride;
    float* min_dist;              // may be null
    bool dot;                     // exact zero distance is -0.0f under NegativeDot
    // hybrid min_dist: a binary16-cast distance that rounds to zero keeps the
    // winner's sign (h(-acc) is -0 for tiny positive acc, +0 for negative), so
    // a zero is re-evaluated from the (rounded) rows; dense queries only
    bool hybrid;
    const float* qmap;
    const float* tmap;
    uint32_t dim;
};
cudaError_t launch_finalize(const FinalizeArgs& a, uint32_t max_q, uint32_t npairs, cudaStream_t s);

// Materialising scorer (src/kernels.cpp:235-273, block_distances :377-400).
cudaError_t launch_block_distances(const float* q, uint32_t nq, const float* t, uint32_t nt,
                                   uint32_t dim, bool l2, bool hybrid, float* out,
                                   unsigned long long* dist_sat, cudaStream_t s);

// ---------------------------------------------------------------- K5/K6 matcher
struct MatchState {
    uint32_t npairs;
    uint32_t cap;                 // samples per pair (capacity of the active arrays)
    uint32_t samples;
    uint32_t h1, w1, p1, p2;
    uint32_t grid_stride;         // effective (derived when cfg.k > 0)
    uint32_t max_iters;
    double convergence;
    uint32_t* active_u;           // [npairs][cap]
    uint32_t* active_v;           // [npairs][cap]
    uint32_t* back;               // [npairs][cap]
    uint32_t* n_active;           // [npairs]
    uint8_t* done;                // [npairs]
    uint32_t* used_i;             // [npairs][ceil(p1/32)]
    uint32_t* used_j;             // [npairs][ceil(p2/32)]
    uint32_t words_i, words_j;
    uint32_t* pairs;              // [npairs][3*cap]
    uint32_t* n_pairs;            // [npairs]
    uint32_t* stats;              // [npairs][kStatWords] (see below)
    unsigned int* n_done;         // scalar
    // reverse-NN memo (tensor route): NN in map 1 of every map-2 pixel already
    // queried in this run, so a reverse pass only computes pixels it has not
    // seen (the chains u -> v -> u' that have not converged mostly come back
    // to a v of an earlier iteration)
    uint32_t* rev_cache;          // [npairs][p2]: NN, kRevUnknown, or 2^31 | claiming entry
    uint32_t* rev_list;           // [npairs][cap]: pixels this reverse pass computes
    uint32_t* rev_n;              // [npairs]
    uint32_t* rev_out;            // [npairs][cap]: their NN
    // graph-replayed loop: iterations harvested so far (device counter, the
    // harvest and loop-condition kernels read it); null when the host drives
    // the loop and passes the iteration by value
    uint32_t* iter;
};
constexpr uint32_t kRevUnknown = 0xFFFFFFFFu;
// stats words per pair: converged, duplicates, iterations, history_len,
// history[FNL_MAX_ITERS], reverse rows actually computed
constexpr int kStatConverged = 0, kStatDups = 1, kStatIters = 2, kStatHistLen = 3, kStatHist = 4;
constexpr int kStatRevComputed = 4 + 64;
constexpr int kStatWords = 4 + 64 + 1;

cudaError_t launch_match_init(const MatchState& m, cudaStream_t s);
cudaError_t launch_harvest(const MatchState& m, uint32_t iteration, cudaStream_t s);
// graph-replayed loop: after harvest, advance *m.iter and set the WHILE
// node's condition (more iterations: some pair not done and t < max_iters)
cudaError_t launch_loop_cond(const MatchState& m, cudaGraphConditionalHandle h, cudaStream_t s);
// reverse-NN memo: back[i] from the memo where known; unseen pixels claimed
// (once each, by their lowest entry) into rev_list / rev_n in entry order for
// the pass; then memo <- pass results and back[i] <- memo for every active i
cudaError_t launch_rev_lookup(const MatchState& m, cudaStream_t s);
cudaError_t launch_rev_fill(const MatchState& m, cudaStream_t s);

// confidence-thresholded compaction of finished MatchSets (in place, stable)
struct ConfArgs {
    const float* d1;
    const float* d2;
    uint64_t map1_stride, map2_stride;  // floats between consecutive pairs' maps
    uint32_t dim;
    bool l2;
    float max_dist;
    uint32_t* pairs;      // [npairs][3*cap]
    uint32_t* n_pairs;    // [npairs], updated
    uint32_t cap;
    uint32_t* dropped;    // [npairs] or null
};
cudaError_t launch_confidence_compact(const ConfArgs& a, uint32_t npairs, cudaStream_t s);

// exhaustive mutual filter: i kept iff bwd[fwd[i]] == i, in ascending i
cudaError_t launch_mutual_filter(const uint32_t* fwd, const uint32_t* bwd, uint32_t n,
                                 uint32_t* pairs, uint32_t* count, cudaStream_t s);

}  // namespace fnl
