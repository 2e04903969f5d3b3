/*
 * fastnn_b200.h -- C-ABI of the B200-native FastNN-Lite matching path.
 *
 * This is the drop-in boundary: plain pointers, sizes and enums, no C++ or
 * torch types.  The reference (/root/reference/proj) is a C++ library whose
 * hot path is reached through the functions cited on each entry point; the
 * host C++ wrapper (paper_2503_10017_b200/csrc/host/) keeps those C++
 * signatures intact and forwards here, and INTEGRATION.md shows the binding a
 * maintainer adds on the reference side.
 *
 * Conventions
 *  - Every entry point returns FNL_OK (0) or an error class; the message of the
 *    last failure on the calling thread is fnl_last_error().  FNL_EINVAL maps to
 *    std::invalid_argument (ValueError in Python), FNL_ERUNTIME to
 *    std::runtime_error (RuntimeError), exactly as the reference throws.
 *  - Pointers named h_* are host memory (pageable or pinned); d_* are device
 *    memory on the context's GPU.  Work is ordered on the context's stream;
 *    calls taking host outputs synchronise before returning.
 *  - There is no CPU fallback: without a usable sm_100 device every compute
 *    entry point returns FNL_ERUNTIME.
 */
#ifndef FASTNN_B200_H
#define FASTNN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FNL_ABI_VERSION 1

enum fnl_status { FNL_OK = 0, FNL_EINVAL = 1, FNL_ERUNTIME = 2 };

/* include/fastnn/core.hpp:75-88 (DistanceMetric / PrecisionMode) */
enum fnl_metric { FNL_METRIC_L2 = 0, FNL_METRIC_DOT = 1 };
enum fnl_precision { FNL_PREC_FULL = 0, FNL_PREC_HYBRID = 1 };

/* include/fastnn/nn.hpp:20 (NnBackend) plus the tensor-core HybridCast path.
 * FNL_BACKEND_TENSOR: binary16 cast-in, tcgen05 fp32 accumulate, fp32 compare
 * (Alg. 3); near ties are re-decided by the exact FMA chain, so the
 * result equals the reference `single` backend run on binary16-rounded maps.
 * The reference backends keep their own arithmetic bit for bit: they take the
 * same tensor route (tcgen05 scores nominate 64-target sub-tiles, the winner is
 * decided by the reference chain on the fp32 rows -- or, for hybrid, on the
 * binary16 rows with the binary16 distance cast) whenever dim <= 32 (dot) /
 * 30 (l2), the inputs are finite and nothing saturates in binary16, and run on
 * the CUDA-core exact scan otherwise (or with FNL_EXACT_KERNEL=cuda_core). */
enum fnl_backend {
    FNL_BACKEND_BRUTEFORCE = 0,
    FNL_BACKEND_DOUBLE = 1,
    FNL_BACKEND_SINGLE = 2,
    FNL_BACKEND_HYBRIDCAST = 3,
    FNL_BACKEND_TENSOR = 4
};

/* include/fastnn/core.hpp:92-103 (MatchConfig), field for field. */
typedef struct {
    uint32_t k;
    uint32_t grid_stride;
    uint32_t max_iters;
    double convergence_fraction;
    int32_t metric;    /* enum fnl_metric */
    int32_t precision; /* enum fnl_precision */
    uint32_t block_size;
} fnl_match_config;

/* Device-side counters of one reciprocal run, from which the host rebuilds the
 * reference RunReport (include/fastnn/instrument.hpp:44-77) exactly. */
#define FNL_MAX_ITERS 64
typedef struct {
    uint32_t samples;
    uint32_t iterations;
    uint32_t converged;
    uint32_t duplicates_dropped;
    uint32_t matches;
    uint32_t history_len;
    uint32_t active_history[FNL_MAX_ITERS];
    uint64_t a_block_fetches;
    uint64_t b_block_fetches;
    uint64_t half_saturation_events;
    /* tensor route only: rows whose first candidate sub-tile did not settle
     * the winner (tensor-core top-2 gap inside the certified error band) */
    uint64_t near_tie_rows;
    uint64_t query_rows; /* total NN query rows issued (forward + reverse) */
    /* device time of each phase (CUDA events on the context stream), shared by
     * all pairs of one batched launch; RunReport *_us fields */
    double subsample_us, forward_nn_us, reverse_nn_us, harvest_us;
    /* tensor route only: rows whose three candidate sub-tiles did not settle
     * the winner and were re-decided over every target (K4' rescan) */
    uint64_t rescan_rows;
    /* 1 when the run took the tensor route (K1 pack + tcgen05 K3 + certified
     * resolution), 0 when it ran on the CUDA-core exact scan K4 */
    uint32_t tensor_route;
    /* NN query rows actually computed: query_rows minus the reverse queries
     * answered from the run's reverse-NN memo (tensor route) */
    uint64_t computed_query_rows;
} fnl_run_stats;

typedef struct fnl_context fnl_context;

/* ---- lifetime ---------------------------------------------------------- */
int fnl_abi_version(void);
const char* fnl_last_error(void);
int fnl_device_count(int* count);
/* One context = one GPU + one stream + a grow-only workspace.  A context is
 * single-owner (one matcher state per pair, single owner);
 * concurrent callers use one context each. */
int fnl_context_create(int device, fnl_context** out);
int fnl_context_destroy(fnl_context* ctx);
/* Replace the context's stream (a cudaStream_t / CUstream handle); NULL
 * restores the context's own stream. */
int fnl_context_set_stream(fnl_context* ctx, void* stream);
int fnl_context_synchronize(fnl_context* ctx);

/* ---- L1: materialising block scorer --------------------------------------
 * src/kernels.cpp:377-400 block_distances (kernels.hpp:72-74): writes the
 * nq x nt distance matrix row-major to h_out with the reference per-pair FMA
 * chain; hybrid rounds inputs and outputs to binary16 (saturations counted). */
int fnl_block_distances(fnl_context* ctx, const float* h_queries, uint32_t nq,
                        const float* h_targets, uint32_t nt, uint32_t dim, int metric,
                        int precision, float* h_out, uint64_t* saturation_events);

/* ---- L2: nearest-neighbour query -----------------------------------------
 * src/nn.cpp:65-164 nn_query_{bruteforce,double_loop,single_loop}
 * (nn.hpp:54-63) and the FeatureMap wrappers nn.cpp:166-187.  One fused
 * score+argmin pass over all targets.  q_blocks / t_blocks are the block
 * counts of the caller's query / target partitions (ceil(n / block_size) for
 * make_partition); they only drive the reference's logical counters:
 * single/hybrid a = b = q_blocks, double a = q_blocks, b = q_blocks * t_blocks,
 * bruteforce none; hybrid saturations follow src/nn.cpp:143-161 (single) and
 * src/kernels.cpp:387-398 per block pair (double). */
int fnl_nn_query(fnl_context* ctx, const float* h_queries, uint32_t nq, const float* h_targets,
                 uint32_t nt, uint32_t dim, int metric, int precision, int backend,
                 uint32_t q_blocks, uint32_t t_blocks, uint32_t* h_nearest, float* h_min_dist,
                 uint64_t* a_fetches, uint64_t* b_fetches, uint64_t* saturation_events);

/* ---- L3: reciprocal matching ----------------------------------------------
 * src/reciprocal.cpp:97-206 reciprocal_match (reciprocal.hpp:50-51).  Maps are
 * H x W x dim fp32 row-major host arrays; non-finite values are rejected with
 * the reference's message (src/core.cpp:19-25).  h_pairs receives
 * (i, j, iteration) triples in harvest order; capacity = 3 * samples. */
int fnl_reciprocal_match(fnl_context* ctx, const float* h_d1, uint32_t h1, uint32_t w1,
                         const float* h_d2, uint32_t h2, uint32_t w2, uint32_t dim,
                         const fnl_match_config* cfg, int backend, uint32_t* h_pairs,
                         uint32_t* n_pairs, fnl_run_stats* stats);

/* Batched form: npairs independent pairs of identical shape, all matched in
 * lock-step on one GPU.  h_d1/h_d2 point at npairs
 * contiguous maps each; host->device copies are pipelined with compute.
 * h_pairs holds npairs * 3 * samples u32, n_pairs npairs counts, stats npairs
 * entries (NULL allowed). */
int fnl_reciprocal_match_batch(fnl_context* ctx, uint32_t npairs, const float* h_d1,
                               const float* h_d2, uint32_t h, uint32_t w, uint32_t dim,
                               const fnl_match_config* cfg, int backend, uint32_t* h_pairs,
                               uint32_t* n_pairs, fnl_run_stats* stats);

/* Same, with the maps already resident in device memory (d_d1/d_d2: npairs
 * contiguous H x W x dim fp32 maps).  Outputs stay on the device:
 * d_pairs npairs * 3 * samples u32, d_n_pairs npairs u32.  Asynchronous on the
 * context stream except for one small convergence read per iteration.  For
 * speed, non-finite inputs are not rejected here (the host-buffer entry points
 * validate like the reference); they still take the route that keeps the
 * results identical to the reference's arithmetic on those values.  The maps
 * must be 16-byte aligned (FNL_EINVAL otherwise).  With h_stats == NULL and
 * npairs <= 64 the second call with the same buffers and configuration
 * captures the reciprocal loop as one CUDA graph (a WHILE node whose
 * condition the device sets) and later calls replay it: no per-iteration
 * host read, one graph launch after the pack's route read-back
 * (FNL_LOOP_GRAPH=0 disables it). */
int fnl_reciprocal_match_batch_device(fnl_context* ctx, uint32_t npairs, const float* d_d1,
                                      const float* d_d2, uint32_t h, uint32_t w, uint32_t dim,
                                      const fnl_match_config* cfg, int backend,
                                      uint32_t* d_pairs, uint32_t* d_n_pairs,
                                      fnl_run_stats* h_stats);

/* Confidence-thresholded correspondence compaction (extension; the reference
 * has no threshold, so it is off unless called): for each of npairs finished
 * MatchSets in device memory (d_pairs[p*3*cap ..], d_n_pairs[p], as written by
 * fnl_reciprocal_match_batch_device), keep the matches (i, j, iter) whose
 * reference distance dist_scalar(D1[i], D2[j]) on the device maps d_d1 / d_d2
 * (npairs stacked h*w*dim fp32 maps) is <= max_distance, in place and in
 * emission order.  d_dropped (optional) receives the per-pair drop count. */
int fnl_confidence_compact_device(fnl_context* ctx, uint32_t npairs, const float* d_d1, const float* d_d2,
                                  uint32_t h, uint32_t w, uint32_t dim, int metric, float max_distance,
                                  uint32_t* d_pairs, uint32_t* d_n_pairs, uint32_t cap,
                                  uint32_t* d_dropped);

/* src/reciprocal.cpp:82-95 mutual_nn_exact (reciprocal.hpp:26): exhaustive
 * mutual NN, full precision, lowest-index ties; h_pairs capacity 2*h1*w1. */
int fnl_mutual_nn(fnl_context* ctx, const float* h_d1, uint32_t h1, uint32_t w1,
                  const float* h_d2, uint32_t h2, uint32_t w2, uint32_t dim, int metric,
                  uint32_t* h_pairs, uint32_t* n_pairs);

/* Dense mutual NN on the tensor cores (binary16 in, fp32 accumulate, certified
 * exact resolution): equals fnl_mutual_nn on binary16-rounded maps.  Same
 * arguments and output layout as fnl_mutual_nn. */
int fnl_mutual_nn_tensor(fnl_context* ctx, const float* h_d1, uint32_t h1, uint32_t w1,
                         const float* h_d2, uint32_t h2, uint32_t w2, uint32_t dim, int metric,
                         uint32_t* h_pairs, uint32_t* n_pairs);

/* ---- target-sharded matching (config C5: one oversized pair over N GPUs) -----
 * Every process holds both maps; for each NN pass, shard `rank` of `count`
 * scans only its contiguous range of 256-target tiles of the target map (image
 * B's pixels in the forward pass, image A's in the reverse pass) and writes
 * each query's exact winner in that range as a signed 64-bit key
 *   ((orderable(dist) << 32) | index) ^ 2^63     (INT64_MAX = no candidate)
 * into the caller-owned device buffer d_keys[pair * samples + i].  The
 * library then calls reduce(user, d_keys, n, stream): the caller must perform
 * an in-place MIN all-reduce of d_keys[0, n) over the `count` processes,
 * ordered on `stream` (e.g. torch.distributed.all_reduce(op=MIN) on NCCL).
 * The reduced key is the global reference winner (lowest index on exact
 * ties), so every process continues with identical state and the MatchSet is
 * bit-identical to the unsharded run.  Any backend on the tensor route (the
 * winner keys carry the backend's own distances; inputs the route refuses are
 * rejected with FNL_EINVAL).  Replaces nothing
 * in the reference (it has no distributed code); the entry point mirrors
 * fnl_reciprocal_match_batch_device. */
typedef int (*fnl_key_reduce_fn)(void* user, int64_t* d_keys, uint64_t count, void* stream);
typedef struct fnl_shard_spec {
    uint32_t rank, count;
    int64_t* d_keys;          /* device, >= npairs * samples entries (peer mode: 2x, see below) */
    uint64_t keys_capacity;
    fnl_key_reduce_fn reduce; /* returns 0 on success */
    void* user;
    /* Optional peer-memory transport (replaces `reduce` when peer_keys != NULL;
     * count <= 8): peer_keys[r] / peer_flags[r] are rank r's key buffer
     * (2 * npairs * samples entries: one half per NN-pass parity, all
     * INT64_MAX when the call starts; left that way on return) and barrier
     * counter, mapped into this process (fnl_ipc_open; entry `rank` is this
     * rank's own d_keys / flag).  The merge and rescan epilogues push every
     * winner key into all ranks' buffers with a system-scope atomicMin over
     * NVLink and a peer-memory barrier replaces the all-reduce.
     * *barrier_seq (host, in/out) counts the barriers completed on these
     * counters by earlier calls; all ranks must pass the same value. */
    int64_t* const* peer_keys;
    uint32_t* const* peer_flags;
    uint64_t* barrier_seq;
    /* Optional native NCCL communicator (fnl_comm_create; used when
     * peer_keys is NULL): the library all-reduces the keys itself with
     * ncclAllReduce(int64, ncclMin) on the context stream and `reduce` may be
     * NULL.  rank / count must equal the communicator's. */
    struct fnl_comm* comm;
} fnl_shard_spec;

/* Native NCCL communicator for the C5 key reduction.  libnccl.so.2 is
 * opened at first use (dlopen: the copy already loaded in the process, e.g.
 * torch's, else the system one), so the library has no link-time NCCL
 * dependency.  Rank 0 calls fnl_nccl_unique_id and hands the 128 bytes to the
 * other ranks out of band; every rank then calls fnl_comm_create (collective,
 * one GPU per rank: the context's device). */
typedef struct fnl_comm fnl_comm;
int fnl_nccl_unique_id(unsigned char id[128]);
int fnl_comm_create(fnl_context* ctx, const unsigned char id[128], int nranks, int rank, fnl_comm** out);
int fnl_comm_destroy(fnl_comm* comm);
int fnl_comm_info(const fnl_comm* comm, int* nranks, int* rank, int* nccl_version);

/* Config C5 from host buffers with a native communicator: every rank passes
 * the same two maps; the target columns of each NN pass are split over the
 * communicator's ranks and the winner keys are MIN-all-reduced with NCCL.
 * Every rank receives the MatchSet of the unsharded run (same arguments and
 * outputs as fnl_reciprocal_match). */
int fnl_reciprocal_match_sharded(fnl_context* ctx, fnl_comm* comm, const float* h_d1, uint32_t h1,
                                 uint32_t w1, const float* h_d2, uint32_t h2, uint32_t w2, uint32_t dim,
                                 const fnl_match_config* cfg, int backend, uint32_t* h_pairs,
                                 uint32_t* n_pairs, fnl_run_stats* stats);

/* Peer-memory buffers for fnl_shard_spec's peer transport: device allocations
 * of their own (so CUDA IPC handles cover exactly them), filled with INT64_MAX
 * (fill_key_none != 0, bytes a multiple of 8) or zero. */
int fnl_p2p_alloc(fnl_context* ctx, uint64_t bytes, int fill_key_none, void** d_ptr);
int fnl_p2p_free(void* d_ptr);
/* CUDA IPC: 64-byte handle of a fnl_p2p_alloc buffer; open / close a peer's. */
int fnl_ipc_handle(const void* d_ptr, unsigned char handle[64]);
int fnl_ipc_open(fnl_context* ctx, const unsigned char handle[64], void** d_ptr);
int fnl_ipc_close(void* d_ptr);
int fnl_reciprocal_match_sharded_device(fnl_context* ctx, uint32_t npairs, const float* d_d1,
                                        const float* d_d2, uint32_t h, uint32_t w, uint32_t dim,
                                        const fnl_match_config* cfg, int backend,
                                        const fnl_shard_spec* shard, uint32_t* d_pairs,
                                        uint32_t* d_n_pairs, fnl_run_stats* h_stats);

/* ---- K7 FlashMatch attention (no reference code) --------------
 * O = softmax(Q K^T * scale) V per (batch, head), non-causal, binary16 Q/K/V/O
 * (device pointers, 16 B aligned), fp32 scores / softmax statistics /
 * accumulation on the tcgen05 tensor cores.  head_dim must be 64.  Strides are
 * in elements (multiples of 8) for [batch][head][token]; head_dim is
 * contiguous, so e.g. a fused QKV projection [B][N][3][H][64] is read in place
 * (q/k/v = base + {0,1,2}*H*64, strides {N*3*H*64, 64, 3*H*64}).  Runs on the
 * context stream; asynchronous. */
typedef struct fnl_attention_desc {
    const void* q;
    const void* k;
    const void* v;
    void* o;
    uint32_t batch, heads, nq, nkv, head_dim;
    float scale;              /* softmax scale, usually 1/sqrt(head_dim) */
    uint64_t q_stride[3];     /* batch, head, token */
    uint64_t k_stride[3];
    uint64_t v_stride[3];
    uint64_t o_stride[3];
} fnl_attention_desc;
int fnl_flashmatch_fwd(fnl_context* ctx, const fnl_attention_desc* desc);
/* profiling aid: the 64 clock64 stamps of CTA 0 of the last traced launch
 * (set FNL_FM_TRACE=1 before the first launch) */
int fnl_flashmatch_trace(fnl_context* ctx, unsigned long long* stamps64);

/* ---- diagnostics -------------------------------------------------------------
 * Raw tensor-core scores (fp32 TMEM accumulators) of 256 query rows against 128
 * target rows after the binary16 pack: h_scores[256][128].  dot: q.t;
 * l2: q.t - |t|^2/2.  Used by the tests to pin the UMMA operand layout and to
 * measure the accumulation error the certification margin must cover.
 * mode 0: A and B from shared memory; mode 1: A copied into tensor memory with
 * tcgen05.cp and consumed by a TS MMA (the production K3 path). */
int fnl_tensor_selftest(fnl_context* ctx, const float* h_queries, const float* h_targets,
                        uint32_t dim, int metric, int mode, float* h_scores);

/* ---- instrumentation -------------------------------------------------------
 * Device time (ms, CUDA events on the context stream) of the dominant scoring
 * kernel summed since the last reset, and its launch count. */
int fnl_kernel_timing(fnl_context* ctx, int reset, double* score_ms, uint64_t* score_launches,
                      uint64_t* total_launches);

/* Per-kernel-class device time (CUDA events around every launch of the class,
 * on the context stream) since the last reset.  enable = 1 turns the
 * non-score classes on, 0 off, -1 leaves the setting; class_ms and
 * class_launches (may be null) receive FNL_KCLASS_COUNT entries.  The score
 * class is always timed (same numbers as fnl_kernel_timing). */
enum {
    FNL_KCLASS_SCORE = 0,   /* K3 tcgen05 score + running argmax / K4 exact scan  */
    FNL_KCLASS_PACK = 1,    /* K1 fp32 -> binary16 pack (tensor) / prepare (exact) */
    FNL_KCLASS_GATHER = 2,  /* K2 query gather + certification margin              */
    FNL_KCLASS_MERGE = 3,   /* K3b split merge + certification + sub-tile resolve  */
    FNL_KCLASS_RESCAN = 4,  /* K4' exact re-decision of uncertified rows           */
    FNL_KCLASS_HARVEST = 5, /* K5 harvest / compaction / convergence, K6 init      */
    FNL_KCLASS_ATTN = 6,    /* K7 FlashMatch attention                             */
    FNL_KCLASS_OTHER = 7,
    FNL_KCLASS_COUNT = 8
};
int fnl_kernel_profile(fnl_context* ctx, int enable, int reset, double* class_ms,
                       uint64_t* class_launches);

/* Largest batch (pairs per call) whose reciprocal loop is captured and
 * replayed as a CUDA graph (see fnl_reciprocal_match_batch_device); 0 turns
 * the graph off for this context.  Kernels inside a replayed graph are not
 * bracketed by the fnl_kernel_timing / fnl_kernel_profile events, so a
 * caller that times the dominant kernel keeps its batches host-driven.
 * max_pairs < 0 only queries; *previous (may be NULL) receives the value in
 * force before the call (default 64, or FNL_LOOP_GRAPH_MAX). */
int fnl_loop_graph_max_pairs(fnl_context* ctx, int max_pairs, int* previous);

#ifdef __cplusplus
}
#endif
#endif
