// capi.cu -- the extern "C" boundary of libfastnn_b200.so (include/fastnn_b200.h).
//
// Owns contexts (device + stream + grow-only workspace), argument checking with
// the reference's error classes, host<->device staging, the per-backend fetch
// and saturation accounting of the reference (src/nn.cpp:143-161, :101-130;
// src/kernels.cpp:387-398), and the host side of the device-resident matcher
// loop (src/reciprocal.cpp:97-206).  All scoring runs in the kernels of
// exact_scan.cu / tensor_scan.cu; there is no host compute path.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <condition_variable>
#include <mutex>
#include <thread>
#include <string>
#include <vector>

#include "fastnn_b200.h"
#include "fnl_common.cuh"
#include "fnl_internal.h"
#include "tensor_scan.h"

namespace fnl {

static thread_local std::string g_last_error;

int fail(int status, const std::string& msg) {
    g_last_error = msg;
    return status;
}

int fail_cuda(cudaError_t e, const char* expr, const char* file, int line) {
    return fail(FNL_ERUNTIME, std::string("CUDA error ") + cudaGetErrorName(e) + " (" +
                                  cudaGetErrorString(e) + ") at " + file + ":" +
                                  std::to_string(line) + ": " + expr);
}

}  // namespace fnl

using fnl::fail;

struct fnl_context {
    int device = 0;
    int sm_count = 148;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t copy_stream = nullptr;
    struct Buf {
        void* p = nullptr;
        size_t bytes = 0;
    };
    std::map<std::string, Buf> dev;
    std::map<std::string, Buf> pinned;
    std::map<std::string, std::pair<const void*, size_t>> initialised;  // ws_fresh
    // instrumentation of the dominant scoring kernel
    bool timing = true;
    bool profile_all = false;  // per-kernel-class breakdown (fnl_kernel_profile)
    struct Mark {
        int cls;
        cudaEvent_t a, b;
    };
    std::vector<Mark> ev_used;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_free;
    double score_ms = 0.0;
    uint64_t score_launches = 0, total_launches = 0;
    double class_ms[FNL_KCLASS_COUNT] = {};
    uint64_t class_launches[FNL_KCLASS_COUNT] = {};
    cudaEvent_t lag[2] = {nullptr, nullptr};  // lagged convergence check of the reciprocal loop
    // graph replay of the reciprocal loop for small batches (run_match)
    uint64_t ws_gen = 0;  // bumped on every workspace (re)allocation
    struct LoopGraph {
        std::vector<uint64_t> key;
        cudaGraph_t graph = nullptr;
        cudaGraphExec_t exec = nullptr;
        uint64_t launches = 0;  // kernels per loop iteration
    };
    std::vector<LoopGraph> graphs;
    std::vector<uint64_t> last_key;  // loop key of the previous host-driven run
    std::vector<uint64_t> failed_key;  // a configuration whose capture failed (not retried)
    int loop_graph_max = -1;           // fnl_loop_graph_max_pairs (-1: the default)
    cudaStream_t cap_stream = nullptr;
    cudaEvent_t route_ev = nullptr;  // the pack's route read-back landed (speculative replay)
};

namespace {

using fnl::fail_cuda;

// batches up to this many pairs replay the reciprocal loop as a CUDA graph
// (FNL_LOOP_GRAPH_MAX, or fnl_loop_graph_max_pairs per context)
uint32_t loop_graph_max_pairs(const fnl_context* ctx) {
    static const uint32_t v =
        getenv("FNL_LOOP_GRAPH_MAX") ? (uint32_t)atoi(getenv("FNL_LOOP_GRAPH_MAX")) : 64u;
    return ctx && ctx->loop_graph_max >= 0 ? (uint32_t)ctx->loop_graph_max : v;
}

int check_device(fnl_context* ctx) {
    if (!ctx) return fail(FNL_EINVAL, "fastnn_b200: null context");
    cudaError_t e = cudaSetDevice(ctx->device);
    if (e != cudaSuccess) return fnl::fail_cuda(e, "cudaSetDevice", __FILE__, __LINE__);
    return FNL_OK;
}

int lag_events(fnl_context* ctx, cudaEvent_t** out) {
    for (auto& e : ctx->lag)
        if (!e) FNL_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    *out = ctx->lag;
    return FNL_OK;
}

// Grow-only device workspace slot.
int dev_buf(fnl_context* ctx, const char* name, size_t bytes, void** out) {
    auto& b = ctx->dev[name];
    if (b.bytes < bytes) {
        if (b.p) cudaFree(b.p);
        b.p = nullptr;
        b.bytes = 0;
        const size_t want = std::max<size_t>(bytes, 256);
        ++ctx->ws_gen;  // captured loop graphs hold the old pointers
        cudaError_t e = cudaMalloc(&b.p, want);
        if (e != cudaSuccess) return fnl::fail_cuda(e, name, __FILE__, __LINE__);
        b.bytes = want;
    }
    *out = b.p;
    return FNL_OK;
}

template <typename T>
int dev_arr(fnl_context* ctx, const char* name, size_t count, T** out) {
    void* p = nullptr;
    int st = dev_buf(ctx, name, count * sizeof(T), &p);
    *out = static_cast<T*>(p);
    return st;
}

#define TRY(x)                          \
    do {                                \
        int _st = (x);                  \
        if (_st != FNL_OK) return _st;  \
    } while (0)

uint64_t ceil_div(uint64_t a, uint64_t b) { return (a + b - 1) / b; }

// Kernel timing: events bracket every dominant-kernel launch (class
// FNL_KCLASS_SCORE) and, when profiling is on, every other kernel class.
void timing_begin(fnl_context* ctx, cudaEvent_t* a, cudaEvent_t* b, int cls = FNL_KCLASS_SCORE) {
    *a = *b = nullptr;
    if (!ctx->timing) return;
    if (cls != FNL_KCLASS_SCORE && !ctx->profile_all) return;
    std::pair<cudaEvent_t, cudaEvent_t> ev;
    if (!ctx->ev_free.empty()) {
        ev = ctx->ev_free.back();
        ctx->ev_free.pop_back();
    } else {
        cudaEventCreate(&ev.first);
        cudaEventCreate(&ev.second);
    }
    cudaEventRecord(ev.first, ctx->stream);
    ctx->ev_used.push_back({cls, ev.first, ev.second});
    *a = ev.first;
    *b = ev.second;
}
void timing_end(fnl_context* ctx, cudaEvent_t b, int cls = FNL_KCLASS_SCORE) {
    if (cls == FNL_KCLASS_SCORE) ctx->score_launches++;
    ctx->class_launches[cls]++;
    if (b) cudaEventRecord(b, ctx->stream);
}
void timing_harvest(fnl_context* ctx) {
    // consumes the marks whose end event has completed (all of them when the
    // caller synchronised the stream); later marks wait for the next harvest
    size_t done = 0;
    for (auto& m : ctx->ev_used) {
        if (cudaEventQuery(m.b) != cudaSuccess) break;
        float ms = 0.0f;
        if (cudaEventElapsedTime(&ms, m.a, m.b) == cudaSuccess) {
            if (m.cls == FNL_KCLASS_SCORE) ctx->score_ms += ms;
            ctx->class_ms[m.cls] += ms;
        }
        ctx->ev_free.push_back({m.a, m.b});
        ++done;
    }
    ctx->ev_used.erase(ctx->ev_used.begin(), ctx->ev_used.begin() + done);
}

// Phase timers for the RunReport *_us fields (device time, microseconds).
struct PhaseTimer {
    fnl_context* ctx;
    bool enabled = true;  // off when the caller asked for no stats (no event churn)
    std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> marks;
    cudaEvent_t open = nullptr;
    int open_phase = -1;
    void begin(int phase) {
        if (!enabled) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, ctx->stream);
        open = e;
        open_phase = phase;
    }
    void end() {
        if (!enabled) return;
        cudaEvent_t e;
        cudaEventCreate(&e);
        cudaEventRecord(e, ctx->stream);
        marks.push_back({open_phase, {open, e}});
        open = nullptr;
    }
    // caller synchronised the stream
    void collect(double us[4]) {
        for (auto& m : marks) {
            float ms = 0.0f;
            if (cudaEventElapsedTime(&ms, m.second.first, m.second.second) == cudaSuccess)
                us[m.first] += 1000.0 * ms;
            cudaEventDestroy(m.second.first);
            cudaEventDestroy(m.second.second);
        }
        marks.clear();
    }
    ~PhaseTimer() {
        for (auto& m : marks) {
            cudaEventDestroy(m.second.first);
            cudaEventDestroy(m.second.second);
        }
        if (open) cudaEventDestroy(open);
    }
};
enum { kPhaseSubsample = 0, kPhaseForward = 1, kPhaseReverse = 2, kPhaseHarvest = 3 };

bool valid_metric(int m) { return m == FNL_METRIC_L2 || m == FNL_METRIC_DOT; }
bool valid_prec(int p) { return p == FNL_PREC_FULL || p == FNL_PREC_HYBRID; }
bool valid_backend(int b) { return b >= FNL_BACKEND_BRUTEFORCE && b <= FNL_BACKEND_TENSOR; }

// Effective precision of a backend (src/reciprocal.cpp:105-107, nn.cpp:184-187).
bool backend_hybrid(int backend, int precision) {
    if (backend == FNL_BACKEND_BRUTEFORCE) return false;
    if (backend == FNL_BACKEND_HYBRIDCAST) return true;
    if (backend == FNL_BACKEND_TENSOR) return false;  // tensor path keeps fp32 distances
    return precision == FNL_PREC_HYBRID;
}

// FNL_EXACT_KERNEL=cuda_core keeps the reference backends on the CUDA-core
// exact scan K4 (tests pin both kernels); read per call so a test can flip it
bool force_cuda_core() {
    const char* e = getenv("FNL_EXACT_KERNEL");
    return e && strcmp(e, "cuda_core") == 0;
}

std::string nonfinite_msg(uint64_t idx) {
    return "FeatureMap: non-finite value at flat index " + std::to_string(idx);
}

// Uploads (if host) and prepares a stack of maps: finiteness check, optional
// binary16 copy with per-row saturation counts and per-map totals.
struct Prepared {
    const float* data = nullptr;   // what the scorer reads
    uint8_t* row_sat = nullptr;
    unsigned long long* map_sat = nullptr;  // per map totals (device)
};

int prepare_maps(fnl_context* ctx, const char* tag, const float* d_src, uint32_t nmaps,
                 uint64_t rows_per_map, uint32_t dim, bool hybrid, bool validate,
                 Prepared* out, unsigned long long* d_bad) {
    const uint64_t rows = rows_per_map * nmaps;
    out->data = d_src;
    out->row_sat = nullptr;
    std::string t(tag);
    TRY(dev_arr(ctx, (t + ".mapsat").c_str(), nmaps, &out->map_sat));
    FNL_CUDA_TRY(cudaMemsetAsync(out->map_sat, 0, nmaps * sizeof(unsigned long long), ctx->stream));
    if (!hybrid && !validate) return FNL_OK;
    fnl::PrepareArgs a{};
    a.src = d_src;
    a.rows = rows;
    a.dim = dim;
    a.bad_index = d_bad;
    a.total_sat = out->map_sat;
    if (hybrid) {
        float* r = nullptr;
        TRY(dev_arr(ctx, (t + ".half").c_str(), rows * dim, &r));
        TRY(dev_arr(ctx, (t + ".rowsat").c_str(), rows, &out->row_sat));
        a.rounded = r;
        a.row_sat = out->row_sat;
        out->data = r;
    }
    fnl::ProfScope prof(ctx, FNL_KCLASS_PACK);
    if (nmaps == 1) {
        FNL_CUDA_TRY(fnl::launch_prepare(a, ctx->stream));
    } else {
        // per-map totals: one launch per map keeps the kernel simple
        for (uint32_t m = 0; m < nmaps; ++m) {
            fnl::PrepareArgs b = a;
            b.src = d_src + (size_t)m * rows_per_map * dim;
            b.rows = rows_per_map;
            if (hybrid) {
                b.rounded = a.rounded + (size_t)m * rows_per_map * dim;
                b.row_sat = a.row_sat + (size_t)m * rows_per_map;
            }
            b.total_sat = out->map_sat + m;
            FNL_CUDA_TRY(fnl::launch_prepare(b, ctx->stream));
        }
    }
    return FNL_OK;
}

// One exact NN pass (K4 + finalize) over the current query set of every pair.
int exact_nn(fnl_context* ctx, const fnl::ScanArgs& sa, uint32_t max_q, uint32_t npairs, bool l2,
             bool hybrid, const fnl::FinalizeArgs& fa) {
    cudaEvent_t e0, e1;
    timing_begin(ctx, &e0, &e1);
    FNL_CUDA_TRY(fnl::launch_exact_scan(sa, max_q, npairs, l2, hybrid, ctx->stream));
    timing_end(ctx, e1);
    {
        fnl::ProfScope prof(ctx, FNL_KCLASS_OTHER);
        FNL_CUDA_TRY(fnl::launch_finalize(fa, max_q, npairs, ctx->stream));
    }
    ctx->total_launches += 2;
    return FNL_OK;
}

}  // namespace

// ============================================================== services
namespace fnl {
cudaStream_t ctx_stream(fnl_context* ctx) { return ctx->stream; }
int ctx_sm_count(fnl_context* ctx) { return ctx->sm_count; }
int ws_device(fnl_context* ctx, const char* name, size_t bytes, void** out) {
    return dev_buf(ctx, name, bytes, out);
}
bool ws_fresh(fnl_context* ctx, const char* name, const void* p, size_t bytes) {
    auto& seen = ctx->initialised[name];
    if (seen.first == p && seen.second == bytes) return false;
    seen = {p, bytes};
    return true;
}
int ws_pinned(fnl_context* ctx, const char* name, size_t bytes, void** out) {
    auto& b = ctx->pinned[name];
    if (b.bytes < bytes) {
        if (b.p) cudaFreeHost(b.p);
        b.p = nullptr;
        b.bytes = 0;
        const size_t want = std::max<size_t>(bytes, 256);
        cudaError_t e = cudaMallocHost(&b.p, want);
        if (e != cudaSuccess) return fail_cuda(e, name, __FILE__, __LINE__);
        b.bytes = want;
    }
    *out = b.p;
    return FNL_OK;
}
void ctx_score_begin(fnl_context* ctx, cudaEvent_t* end_event) {
    cudaEvent_t a;
    timing_begin(ctx, &a, end_event);
}
void ctx_score_end(fnl_context* ctx, cudaEvent_t end_event) { timing_end(ctx, end_event); }
void ctx_prof_begin(fnl_context* ctx, int cls, cudaEvent_t* end_event) {
    cudaEvent_t a;
    timing_begin(ctx, &a, end_event, cls);
}
void ctx_prof_end(fnl_context* ctx, int cls, cudaEvent_t end_event) { timing_end(ctx, end_event, cls); }
void ctx_count_launches(fnl_context* ctx, int n) { ctx->total_launches += n; }
}  // namespace fnl

// ============================================================== lifetime
extern "C" int fnl_abi_version(void) { return FNL_ABI_VERSION; }

extern "C" const char* fnl_last_error(void) { return fnl::g_last_error.c_str(); }

extern "C" int fnl_device_count(int* count) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (count) *count = e == cudaSuccess ? n : 0;
    if (e != cudaSuccess) return fnl::fail_cuda(e, "cudaGetDeviceCount", __FILE__, __LINE__);
    return FNL_OK;
}

extern "C" int fnl_context_create(int device, fnl_context** out) {
    if (!out) return fail(FNL_EINVAL, "fnl_context_create: null out");
    *out = nullptr;
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0)
        return fail(FNL_ERUNTIME, std::string("fastnn_b200: no CUDA device available (") +
                                      (e == cudaSuccess ? "0 devices" : cudaGetErrorString(e)) +
                                      "); this library has no CPU fallback");
    if (device < 0 || device >= n)
        return fail(FNL_EINVAL, "fnl_context_create: device " + std::to_string(device) +
                                    " out of range (" + std::to_string(n) + " devices)");
    cudaDeviceProp prop{};
    FNL_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(FNL_ERUNTIME, std::string("fastnn_b200: device '") + prop.name +
                                      "' is sm_" + std::to_string(prop.major) +
                                      std::to_string(prop.minor) + "; kernels are built for sm_100a");
    FNL_CUDA_TRY(cudaSetDevice(device));
    auto* ctx = new fnl_context();
    ctx->device = device;
    ctx->sm_count = prop.multiProcessorCount;
    cudaError_t e1 = cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
    cudaError_t e2 = cudaStreamCreateWithFlags(&ctx->copy_stream, cudaStreamNonBlocking);
    if (e1 != cudaSuccess || e2 != cudaSuccess) {
        delete ctx;
        return fnl::fail_cuda(e1 != cudaSuccess ? e1 : e2, "cudaStreamCreate", __FILE__, __LINE__);
    }
    ctx->stream = ctx->own_stream;
    *out = ctx;
    return FNL_OK;
}

extern "C" int fnl_context_destroy(fnl_context* ctx) {
    if (!ctx) return FNL_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& kv : ctx->dev) cudaFree(kv.second.p);
    for (auto& kv : ctx->pinned) cudaFreeHost(kv.second.p);
    for (auto& m : ctx->ev_used) { cudaEventDestroy(m.a); cudaEventDestroy(m.b); }
    for (auto& ev : ctx->ev_free) { cudaEventDestroy(ev.first); cudaEventDestroy(ev.second); }
    for (auto& e : ctx->lag)
        if (e) cudaEventDestroy(e);
    for (auto& g : ctx->graphs) {
        cudaGraphExecDestroy(g.exec);
        cudaGraphDestroy(g.graph);
    }
    if (ctx->cap_stream) cudaStreamDestroy(ctx->cap_stream);
    if (ctx->route_ev) cudaEventDestroy(ctx->route_ev);
    cudaStreamDestroy(ctx->own_stream);
    cudaStreamDestroy(ctx->copy_stream);
    delete ctx;
    return FNL_OK;
}

extern "C" int fnl_context_set_stream(fnl_context* ctx, void* stream) {
    TRY(check_device(ctx));
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own_stream;
    return FNL_OK;
}

extern "C" int fnl_context_synchronize(fnl_context* ctx) {
    TRY(check_device(ctx));
    FNL_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    timing_harvest(ctx);
    return FNL_OK;
}

extern "C" int fnl_kernel_timing(fnl_context* ctx, int reset, double* score_ms,
                                 uint64_t* score_launches, uint64_t* total_launches) {
    TRY(check_device(ctx));
    FNL_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    timing_harvest(ctx);
    if (score_ms) *score_ms = ctx->score_ms;
    if (score_launches) *score_launches = ctx->score_launches;
    if (total_launches) *total_launches = ctx->total_launches;
    if (reset) {
        ctx->score_ms = 0.0;
        ctx->score_launches = 0;
        ctx->total_launches = 0;
    }
    return FNL_OK;
}

extern "C" int fnl_loop_graph_max_pairs(fnl_context* ctx, int max_pairs, int* previous) {
    if (!ctx) return fail(FNL_EINVAL, "fastnn_b200: null context");
    if (previous) *previous = (int)loop_graph_max_pairs(ctx);
    if (max_pairs >= 0) ctx->loop_graph_max = max_pairs;
    return FNL_OK;
}

extern "C" int fnl_kernel_profile(fnl_context* ctx, int enable, int reset, double* class_ms,
                                  uint64_t* class_launches) {
    TRY(check_device(ctx));
    FNL_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    timing_harvest(ctx);
    for (int c = 0; c < FNL_KCLASS_COUNT; ++c) {
        if (class_ms) class_ms[c] = ctx->class_ms[c];
        if (class_launches) class_launches[c] = ctx->class_launches[c];
        if (reset) {
            ctx->class_ms[c] = 0.0;
            ctx->class_launches[c] = 0;
        }
    }
    if (enable >= 0) ctx->profile_all = enable != 0;
    return FNL_OK;
}

extern "C" int fnl_flashmatch_fwd(fnl_context* ctx, const fnl_attention_desc* desc) {
    TRY(check_device(ctx));
    if (!desc) return fail(FNL_EINVAL, "fnl_flashmatch_fwd: null descriptor");
    return fnl::flashmatch_forward(ctx, *desc);
}

extern "C" int fnl_flashmatch_trace(fnl_context* ctx, unsigned long long* stamps64) {
    TRY(check_device(ctx));
    if (!stamps64) return fail(FNL_EINVAL, "fnl_flashmatch_trace: null output");
    return fnl::flashmatch_trace(stamps64);
}

// ============================================================== L1 block scorer
extern "C" int fnl_block_distances(fnl_context* ctx, const float* h_q, uint32_t nq,
                                   const float* h_t, uint32_t nt, uint32_t dim, int metric,
                                   int precision, float* h_out, uint64_t* sat_out) {
    TRY(check_device(ctx));
    if (!valid_metric(metric) || !valid_prec(precision))
        return fail(FNL_EINVAL, "fnl_block_distances: bad metric/precision");
    if (nq == 0 || nt == 0) return fail(FNL_EINVAL, "block_distances: empty block");
    if (dim == 0) return fail(FNL_EINVAL, "block_distances: zero dim");
    const bool hyb = precision == FNL_PREC_HYBRID;
    float *dq, *dt, *dout;
    unsigned long long* cnt;
    TRY(dev_arr(ctx, "bd.q", (size_t)nq * dim, &dq));
    TRY(dev_arr(ctx, "bd.t", (size_t)nt * dim, &dt));
    TRY(dev_arr(ctx, "bd.out", (size_t)nq * nt, &dout));
    TRY(dev_arr(ctx, "bd.cnt", 8, &cnt));
    FNL_CUDA_TRY(cudaMemsetAsync(cnt, 0, 8 * sizeof(unsigned long long), ctx->stream));
    FNL_CUDA_TRY(cudaMemcpyAsync(dq, h_q, (size_t)nq * dim * 4, cudaMemcpyHostToDevice, ctx->stream));
    FNL_CUDA_TRY(cudaMemcpyAsync(dt, h_t, (size_t)nt * dim * 4, cudaMemcpyHostToDevice, ctx->stream));
    Prepared pq, pt;
    unsigned long long* bad;
    TRY(dev_arr(ctx, "bd.bad", 1, &bad));
    FNL_CUDA_TRY(cudaMemsetAsync(bad, 0xFF, 8, ctx->stream));
    TRY(prepare_maps(ctx, "bd.pq", dq, 1, nq, dim, hyb, false, &pq, bad));
    TRY(prepare_maps(ctx, "bd.pt", dt, 1, nt, dim, hyb, false, &pt, bad));
    cudaEvent_t e0, e1;
    timing_begin(ctx, &e0, &e1);
    FNL_CUDA_TRY(fnl::launch_block_distances(pq.data, nq, pt.data, nt, dim, metric == FNL_METRIC_L2,
                                             hyb, dout, cnt + 1, ctx->stream));
    timing_end(ctx, e1);
    FNL_CUDA_TRY(cudaMemcpyAsync(h_out, dout, (size_t)nq * nt * 4, cudaMemcpyDeviceToHost, ctx->stream));
    unsigned long long h_cnt[3] = {0, 0, 0};
    FNL_CUDA_TRY(cudaMemcpyAsync(h_cnt, cnt + 1, 8, cudaMemcpyDeviceToHost, ctx->stream));
    unsigned long long h_ms[2] = {0, 0};
    FNL_CUDA_TRY(cudaMemcpyAsync(&h_ms[0], pq.map_sat, 8, cudaMemcpyDeviceToHost, ctx->stream));
    FNL_CUDA_TRY(cudaMemcpyAsync(&h_ms[1], pt.map_sat, 8, cudaMemcpyDeviceToHost, ctx->stream));
    FNL_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    timing_harvest(ctx);
    ctx->total_launches += 1;
    // src/kernels.cpp:387-398: targets rounded once, every query row once, every distance
    if (sat_out) *sat_out = hyb ? (h_ms[0] + h_ms[1] + h_cnt[0]) : 0;
    return FNL_OK;
}

// ============================================================== L2 NN query
extern "C" int fnl_nn_query(fnl_context* ctx, const float* h_q, uint32_t nq, const float* h_t,
                            uint32_t nt, uint32_t dim, int metric, int precision, int backend,
                            uint32_t q_blocks, uint32_t t_blocks, uint32_t* h_nearest, float* h_min_dist,
                            uint64_t* a_fetches, uint64_t* b_fetches, uint64_t* sat_out) {
    TRY(check_device(ctx));
    if (!valid_metric(metric) || !valid_prec(precision) || !valid_backend(backend))
        return fail(FNL_EINVAL, "fnl_nn_query: bad metric/precision/backend");
    if (nt == 0) return fail(FNL_EINVAL, "nn: no target pixels");
    if (dim == 0) return fail(FNL_EINVAL, "nn: zero dim");
    const bool hyb = backend_hybrid(backend, precision);
    const bool l2 = metric == FNL_METRIC_L2;
    if (a_fetches) *a_fetches = 0;
    if (b_fetches) *b_fetches = 0;
    if (sat_out) *sat_out = 0;
    if (nq == 0) return FNL_OK;

    float *dq, *dt, *dmd;
    uint32_t* dnear;
    unsigned long long *keys, *cnt, *bad;
    TRY(dev_arr(ctx, "nn.q", (size_t)nq * dim, &dq));
    TRY(dev_arr(ctx, "nn.t", (size_t)nt * dim, &dt));
    TRY(dev_arr(ctx, "nn.keys", nq, &keys));
    TRY(dev_arr(ctx, "nn.near", nq, &dnear));
    TRY(dev_arr(ctx, "nn.md", nq, &dmd));
    TRY(dev_arr(ctx, "nn.cnt", 2, &cnt));
    TRY(dev_arr(ctx, "nn.bad", 1, &bad));
    FNL_CUDA_TRY(cudaMemcpyAsync(dq, h_q, (size_t)nq * dim * 4, cudaMemcpyHostToDevice, ctx->stream));
    FNL_CUDA_TRY(cudaMemcpyAsync(dt, h_t, (size_t)nt * dim * 4, cudaMemcpyHostToDevice, ctx->stream));
    FNL_CUDA_TRY(cudaMemsetAsync(keys, 0xFF, (size_t)nq * 8, ctx->stream));
    FNL_CUDA_TRY(cudaMemsetAsync(cnt, 0, 16, ctx->stream));

    // Tensor route (K1 pack + K3 tcgen05 scores + certified exact resolution
    // in the backend's own arithmetic) whenever the inputs allow it; else the
    // CUDA-core exact scan K4.  Both are bit-identical to the reference.
    const int mode = backend == FNL_BACKEND_TENSOR ? fnl::kResolveRounded
                                                   : (hyb ? fnl::kResolveHybrid : fnl::kResolveFull);
    bool routed = false;
    if (backend == FNL_BACKEND_TENSOR || !force_cuda_core())
        TRY(fnl::tensor_nn_dense(ctx, dq, nq, dt, nt, dim, l2, dnear, dmd, mode, &routed));
    unsigned long long h_cnt[2] = {0, 0}, h_ms[2] = {0, 0};
    if (!routed) {
        // the tensor backend's contract is ref single on binary16-rounded
        // rows: K4 on the rounded rows, fp32 compare
        const bool round_in = hyb || backend == FNL_BACKEND_TENSOR;
        Prepared pq, pt;
        TRY(prepare_maps(ctx, "nn.pq", dq, 1, nq, dim, round_in, false, &pq, bad));
        TRY(prepare_maps(ctx, "nn.pt", dt, 1, nt, dim, round_in, false, &pt, bad));
        fnl::ScanArgs sa{};
        sa.qmap = pq.data;
        sa.qcount_const = nq;
        sa.q_row_sat = pq.row_sat;
        sa.tmap = pt.data;
        sa.nt = nt;
        sa.dim = dim;
        sa.keys = keys;
        sa.keys_pair_stride = nq;
        sa.counters = cnt;
        fnl::FinalizeArgs fa{};
        fa.keys = keys;
        fa.keys_pair_stride = nq;
        fa.qcount_const = nq;
        fa.nearest = dnear;
        fa.nearest_pair_stride = nq;
        fa.min_dist = dmd;
        fa.dot = !l2;
        fa.hybrid = hyb;
        fa.qmap = pq.data;
        fa.tmap = pt.data;
        fa.dim = dim;
        TRY(exact_nn(ctx, sa, nq, 1, l2, hyb, fa));
        FNL_CUDA_TRY(cudaMemcpyAsync(h_cnt, cnt, 16, cudaMemcpyDeviceToHost, ctx->stream));
        FNL_CUDA_TRY(cudaMemcpyAsync(&h_ms[0], pq.map_sat, 8, cudaMemcpyDeviceToHost, ctx->stream));
        FNL_CUDA_TRY(cudaMemcpyAsync(&h_ms[1], pt.map_sat, 8, cudaMemcpyDeviceToHost, ctx->stream));
    }
    // (routed: no input or distance saturates -- tensor_route_ok -- so the
    // reference's hybrid saturation count is 0)
    FNL_CUDA_TRY(cudaMemcpyAsync(h_nearest, dnear, (size_t)nq * 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (h_min_dist)
        FNL_CUDA_TRY(cudaMemcpyAsync(h_min_dist, dmd, (size_t)nq * 4, cudaMemcpyDeviceToHost, ctx->stream));
    FNL_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    timing_harvest(ctx);

    // logical fetch law + saturation law of the chosen backend
    const uint64_t nqb = backend == FNL_BACKEND_BRUTEFORCE ? 0 : q_blocks;
    const uint64_t ntb = backend == FNL_BACKEND_BRUTEFORCE ? 0 : t_blocks;
    uint64_t a = 0, b = 0, sat = 0;
    if (backend == FNL_BACKEND_DOUBLE) {
        a = nqb;
        b = nqb * ntb;
        if (hyb) sat = nqb * h_ms[1] + ntb * h_cnt[0] + h_cnt[1];
    } else if (backend != FNL_BACKEND_BRUTEFORCE) {
        a = nqb;
        b = nqb;
        if (hyb) sat = h_ms[1] + h_cnt[0] + h_cnt[1];
    }
    if (a_fetches) *a_fetches = a;
    if (b_fetches) *b_fetches = b;
    if (sat_out) *sat_out = sat;
    return FNL_OK;
}

// ============================================================== L3 matcher
namespace {

uint32_t derived_stride(uint32_t h, uint32_t w, uint32_t k, uint32_t stride) {
    if (stride != 0) return stride;
    const double cells = (double)h * (double)w / (double)k;
    const long s = lround(sqrt(cells));
    return s < 1 ? 1u : (uint32_t)s;
}

int check_cfg(const fnl_match_config* cfg) {
    if (!cfg) return fail(FNL_EINVAL, "MatchConfig: null");
    if (cfg->grid_stride == 0 && cfg->k == 0)
        return fail(FNL_EINVAL, "MatchConfig: one of k or grid_stride must be >= 1");
    if (cfg->max_iters == 0) return fail(FNL_EINVAL, "MatchConfig: max_iters must be >= 1");
    if (!(cfg->convergence_fraction > 0.0) || cfg->convergence_fraction > 1.0)
        return fail(FNL_EINVAL, "MatchConfig: convergence_fraction must be in (0, 1]");
    if (cfg->block_size == 0) return fail(FNL_EINVAL, "MatchConfig: block_size must be >= 1");
    if (!valid_metric(cfg->metric) || !valid_prec(cfg->precision))
        return fail(FNL_EINVAL, "MatchConfig: bad metric/precision");
    if (cfg->max_iters > FNL_MAX_ITERS)
        return fail(FNL_EINVAL, "MatchConfig: max_iters above " + std::to_string(FNL_MAX_ITERS) +
                                    " is not supported by this build");
    return FNL_OK;
}



// The device-resident matcher over npairs stacked pairs.  d_d1 / d_d2 are raw
// fp32 maps on the device.  Results stay on the device in the MatchState.
int run_match(fnl_context* ctx, uint32_t npairs, const float* d_d1, uint32_t h1, uint32_t w1,
              const float* d_d2, uint32_t h2, uint32_t w2, uint32_t dim,
              const fnl_match_config* cfg, int backend, uint32_t* d_pairs_out,
              uint32_t* d_npairs_out, fnl_run_stats* h_stats, bool validate,
              const fnl_shard_spec* shard = nullptr) {
    TRY(check_cfg(cfg));
    if (!valid_backend(backend)) return fail(FNL_EINVAL, "reciprocal_match: unknown backend");
    // the kernels read map rows with 16-byte vector loads
    if ((reinterpret_cast<uintptr_t>(d_d1) | reinterpret_cast<uintptr_t>(d_d2)) & 15u)
        return fail(FNL_EINVAL, "reciprocal_match: device maps must be 16-byte aligned");
    if (dim == 0 || h1 == 0 || w1 == 0 || h2 == 0 || w2 == 0)
        return fail(FNL_EINVAL, "FeatureMap: height, width and dim must all be >= 1");
    const bool hyb = backend_hybrid(backend, cfg->precision);
    const bool l2 = cfg->metric == FNL_METRIC_L2;
    const uint32_t p1 = h1 * w1, p2 = h2 * w2;
    const uint32_t stride = derived_stride(h1, w1, cfg->k, cfg->grid_stride);
    const uint32_t samples = ((h1 + stride - 1) / stride) * ((w1 + stride - 1) / stride);
    const uint32_t cap = std::max<uint32_t>(samples, 1);
    const uint32_t T = cfg->max_iters;

    // ---- workspace
    fnl::MatchState m{};
    m.npairs = npairs;
    m.cap = cap;
    m.samples = samples;
    m.h1 = h1;
    m.w1 = w1;
    m.p1 = p1;
    m.p2 = p2;
    m.grid_stride = stride;
    m.max_iters = T;
    m.convergence = cfg->convergence_fraction;
    m.words_i = (p1 + 31) / 32;
    m.words_j = (p2 + 31) / 32;
    const size_t pc = (size_t)npairs * cap;
    TRY(dev_arr(ctx, "m.u", pc, &m.active_u));
    TRY(dev_arr(ctx, "m.v", pc, &m.active_v));
    TRY(dev_arr(ctx, "m.back", pc, &m.back));
    TRY(dev_arr(ctx, "m.nact", npairs, &m.n_active));
    TRY(dev_arr(ctx, "m.done", npairs, &m.done));
    TRY(dev_arr(ctx, "m.usedi", (size_t)npairs * m.words_i, &m.used_i));
    TRY(dev_arr(ctx, "m.usedj", (size_t)npairs * m.words_j, &m.used_j));
    m.pairs = d_pairs_out;
    m.n_pairs = d_npairs_out;
    TRY(dev_arr(ctx, "m.stats", (size_t)npairs * fnl::kStatWords, &m.stats));
    TRY(dev_arr(ctx, "m.ndone", 1, &m.n_done));
    unsigned long long *keys, *bad, *counters;
    TRY(dev_arr(ctx, "m.keys", pc, &keys));
    TRY(dev_arr(ctx, "m.bad", 2, &bad));
    const uint32_t max_calls = 2 * T + 1;
    TRY(dev_arr(ctx, "m.counters", (size_t)max_calls * npairs * 2, &counters));
    cudaStream_t s = ctx->stream;

    // ---- K1: binary16 pack for the tensor route, or validate + (hybrid)
    // round for the CUDA-core exact scan.  Every backend takes the tensor
    // route (K3 scores + certified resolution in the backend's arithmetic,
    // bit-identical to the reference) when the inputs allow it.
    const bool tensor = backend == FNL_BACKEND_TENSOR;
    // (a native communicator takes the key path even with one rank, so the
    // NCCL reduction is exercised wherever the run happens)
    const bool sharded = shard && (shard->count > 1 || (shard->comm && !shard->peer_keys));
    if (shard) {
        if (shard->count == 0 || shard->rank >= shard->count)
            return fail(FNL_EINVAL, "sharded reciprocal_match: rank must be < count");
        const bool peer = sharded && shard->peer_keys;
        if (sharded && !peer &&
            (!shard->d_keys || (!shard->reduce && !shard->comm) || shard->keys_capacity < (uint64_t)npairs * cap))
            return fail(FNL_EINVAL, "sharded reciprocal_match: key buffer (npairs * samples) and a reduce callback "
                                    "or NCCL communicator required");
        if (shard->comm && !peer) {
            int nr = 0, rk = 0;
            fnl::comm_size(shard->comm, &nr, &rk);
            if ((uint32_t)nr != shard->count || (uint32_t)rk != shard->rank)
                return fail(FNL_EINVAL, "sharded reciprocal_match: rank / count differ from the communicator's");
        }
        if (peer && (shard->count > (uint32_t)fnl::kMaxShardPeers || !shard->peer_flags || !shard->barrier_seq ||
                     !shard->d_keys || shard->keys_capacity < 2ull * npairs * cap))
            return fail(FNL_EINVAL, "sharded reciprocal_match (peer memory): at most 8 ranks, key buffers of "
                                    "2 * npairs * samples, flags and barrier_seq required");
    }
    const int mode = tensor ? fnl::kResolveRounded : (hyb ? fnl::kResolveHybrid : fnl::kResolveFull);
    bool tc = false;  // tensor route taken
    bool acc16 = false;  // K3 may accumulate in binary16 (every pair's norms allow it)
    Prepared P1, P2;
    fnl::PackedMaps T1, T2;
    unsigned long long *near_ties = nullptr, *tsat = nullptr;
    TRY(dev_arr(ctx, "m.neartie", 2 * (size_t)npairs, &near_ties));
    // the pack's per-pair outputs in one region, read back by one copy:
    // [first non-finite index: 2n u64 (~0)][saturations: 2n u64 (0)]
    // [norm maxima of map 1: 2n f32 (0)][of map 2: 2n f32 (0)]
    unsigned long long* route = nullptr;
    const size_t route_bytes = (size_t)npairs * 48;
    TRY(dev_arr(ctx, "m.route", (size_t)npairs * 6, &route));
    tsat = route + 2 * (size_t)npairs;
    float* maxn = reinterpret_cast<float*>(route + 4 * (size_t)npairs);
    FNL_CUDA_TRY(cudaMemsetAsync(tsat, 0, (size_t)npairs * 32, s));
    // loop-graph keys (see the graph block below); the replay can start right
    // behind the pack's route read-back when the configuration already has a
    // graph for the route it took last time (speculation: a different route
    // re-runs the call from scratch behind it)
    static const bool memo_env = !(getenv("FNL_REV_MEMO") && atoi(getenv("FNL_REV_MEMO")) == 0);
    static const bool graph_env = !(getenv("FNL_LOOP_GRAPH") && atoi(getenv("FNL_LOOP_GRAPH")) == 0);
    auto make_key = [&](bool k_acc16, bool k_memo) {
        return std::vector<uint64_t>{npairs, (uint64_t)(uintptr_t)d_d1, (uint64_t)(uintptr_t)d_d2, h1, w1, h2, w2,
                                     dim, cfg->k, cfg->grid_stride, T,
                                     (uint64_t)(cfg->convergence_fraction * 1e15), (uint64_t)cfg->metric,
                                     (uint64_t)cfg->precision, cfg->block_size, (uint64_t)backend,
                                     (uint64_t)(uintptr_t)d_pairs_out, (uint64_t)(uintptr_t)d_npairs_out,
                                     (uint64_t)k_acc16, (uint64_t)mode, (uint64_t)k_memo, ctx->ws_gen};
    };
    fnl_context::LoopGraph* spec = nullptr;  // replay launched ahead of the route decision
    const bool fits = dim + (l2 ? 2u : 0u) <= fnl::kPackK;
    if ((tensor && fits) || (!tensor && fits && !force_cuda_core())) {
        unsigned long long* tbad = route;
        FNL_CUDA_TRY(cudaMemsetAsync(tbad, 0xFF, (size_t)npairs * 16, s));
        TRY(fnl::tensor_pack(ctx, "m.t1", d_d1, npairs, p1, dim, l2, tbad, tsat, &T1, maxn));
        TRY(fnl::tensor_pack(ctx, "m.t2", d_d2, npairs, p2, dim, l2, tbad + npairs, tsat + npairs, &T2,
                             maxn + 2 * (size_t)npairs));
        tc = true;
        // The host reads the pack's per-pair finiteness / norms / saturations
        // (one small round trip): to validate like the reference FeatureMap
        // (host-buffer entry points), to check the route, and to choose the
        // K3 accumulator (binary16 when every pair's norms allow it).
        {
            // one pinned copy of the whole region behind the packs; the host
            // waits once (pageable copies each block)
            void* pin = nullptr;
            TRY(fnl::ws_pinned(ctx, "m.route", route_bytes, &pin));
            unsigned long long* hb = static_cast<unsigned long long*>(pin);
            unsigned long long* hs = hb + 2 * (size_t)npairs;
            const float* hn1 = reinterpret_cast<const float*>(hs + 2 * (size_t)npairs);  // map 1 maxima
            const float* hn2 = hn1 + 2 * (size_t)npairs;                                    // map 2 maxima
            FNL_CUDA_TRY(cudaMemcpyAsync(hb, route, route_bytes, cudaMemcpyDeviceToHost, s));
            if (graph_env && !validate && !shard && !h_stats && !ctx->profile_all && samples > 0 &&
                npairs <= loop_graph_max_pairs(ctx) && !ctx->graphs.empty()) {
                const std::vector<uint64_t> k = make_key(true, memo_env);
                for (auto& g : ctx->graphs)
                    if (g.key == k) spec = &g;
            }
            if (spec) {
                if (!ctx->route_ev) FNL_CUDA_TRY(cudaEventCreateWithFlags(&ctx->route_ev, cudaEventDisableTiming));
                FNL_CUDA_TRY(cudaEventRecord(ctx->route_ev, s));
                FNL_CUDA_TRY(cudaGraphLaunch(spec->exec, s));
                FNL_CUDA_TRY(cudaEventSynchronize(ctx->route_ev));
            } else {
                FNL_CUDA_TRY(cudaStreamSynchronize(s));
            }
            if (validate) {
                // D1 is checked before D2, as the reference converts D1 first
                // (bindings/module.cpp:232-233); indices are flat within one map
                for (uint32_t p = 0; p < npairs; ++p)
                    if (hb[p] != ~0ull) return fail(FNL_EINVAL, nonfinite_msg(hb[p]));
                for (uint32_t p = 0; p < npairs; ++p)
                    if (hb[npairs + p] != ~0ull) return fail(FNL_EINVAL, nonfinite_msg(hb[npairs + p]));
            }
            for (uint32_t p = 0; p < npairs && tc; ++p)
                tc = fnl::tensor_route_ok(mode, l2, dim, hn1[p], hn2[p], hs[p] + hs[npairs + p],
                                          std::min(hb[p], hb[npairs + p]));
            acc16 = tc;
            for (uint32_t p = 0; p < npairs && acc16; ++p) acc16 = fnl::acc16_ok(l2, hn1[p], hn2[p]);
        }
    }
    if (shard && !tc)
        return fail(FNL_EINVAL, "sharded reciprocal_match: needs the tensor route (descriptor dim <= 32 for dot, "
                                "<= 30 for l2; finite inputs without binary16 saturation)");
    if (!tc) {
        // the tensor backend's contract is ref single on binary16-rounded
        // rows: K4 on the rounded rows, fp32 compare
        FNL_CUDA_TRY(cudaMemsetAsync(bad, 0xFF, 16, s));
        TRY(prepare_maps(ctx, "m.p1", d_d1, npairs, p1, dim, hyb || tensor, validate, &P1, bad));
        TRY(prepare_maps(ctx, "m.p2", d_d2, npairs, p2, dim, hyb || tensor, validate, &P2, bad + 1));
        if (validate) {
            unsigned long long hb[2] = {~0ull, ~0ull};
            FNL_CUDA_TRY(cudaMemcpyAsync(hb, bad, 16, cudaMemcpyDeviceToHost, s));
            FNL_CUDA_TRY(cudaStreamSynchronize(s));
            if (hb[0] != ~0ull) return fail(FNL_EINVAL, nonfinite_msg(hb[0] % ((uint64_t)p1 * dim)));
            if (hb[1] != ~0ull) return fail(FNL_EINVAL, nonfinite_msg(hb[1] % ((uint64_t)p2 * dim)));
        }
    }
    PhaseTimer timer{ctx};
    timer.enabled = h_stats != nullptr;

    // ---- NN pass helper: queries = rows of qmap at ids, targets = tmap
    uint32_t call = 0;
    const bool peer = sharded && shard->peer_keys;
    unsigned int* barrier_err = nullptr;
    if (peer) {
        TRY(dev_arr(ctx, "m.p2perr", 1, &barrier_err));
        FNL_CUDA_TRY(cudaMemsetAsync(barrier_err, 0, 4, s));
    }
    uint32_t peer_pass = 0;
    // d_count: per-pair query counts of the pass (default: the active counts)
    auto nn_pass = [&](const Prepared& Q, uint32_t qrows, const uint32_t* ids, const Prepared& Tm,
                       uint32_t nt, uint32_t* out, const uint32_t* d_count = nullptr) -> int {
        if (!d_count) d_count = m.n_active;
        if (tc) {
            const bool fwd = qrows == p1 && ids == m.active_u;
            const fnl::PackedMaps& TQ = fwd ? T1 : T2;
            const fnl::PackedMaps& TT = fwd ? T2 : T1;
            fnl::ResolveSrc rs;
            rs.mode = mode;
            rs.acc16 = acc16;
            rs.q32 = fwd ? d_d1 : d_d2;
            rs.q32_pair_stride = (uint64_t)(fwd ? p1 : p2) * dim;
            rs.t32 = fwd ? d_d2 : d_d1;
            rs.t32_pair_stride = (uint64_t)(fwd ? p2 : p1) * dim;
            ++call;
            if (!sharded)
                return fnl::tensor_nn_pass(ctx, npairs, TQ, ids, cap, d_count, m.done, TT, dim, l2, out, cap,
                                           nullptr, near_ties, 0, 0, nullptr, nullptr, &rs);            // target shard of this rank: contiguous 256-target tiles
            const uint64_t tiles = ceil_div(nt, fnl::kTargetTileRows);
            const uint32_t tb = (uint32_t)(tiles * shard->rank / shard->count);
            const uint32_t te = (uint32_t)(tiles * (shard->rank + 1) / shard->count);
            const uint64_t nkeys = (uint64_t)npairs * cap;
            if (peer) {
                // keys go straight into every rank's buffer (half `par`) from the
                // merge / rescan epilogues; a peer-memory barrier replaces the
                // all-reduce; the half is reset after decoding, before this rank
                // can take part in the next barrier (the earliest a peer pushes
                // into it again)
                const uint32_t par = peer_pass++ & 1u;
                fnl::ShardPeers pp{};
                pp.n = shard->count;
                for (uint32_t r = 0; r < shard->count; ++r)
                    pp.keys[r] = reinterpret_cast<long long*>(shard->peer_keys[r]) + par * nkeys;
                long long* own = reinterpret_cast<long long*>(shard->d_keys) + par * nkeys;
                if (te > tb)
                    TRY(fnl::tensor_nn_pass(ctx, npairs, TQ, ids, cap, d_count, m.done, TT, dim, l2, out, cap,
                                            nullptr, near_ties, tb, te, own, &pp, &rs));
                const uint64_t seq = ++*shard->barrier_seq;
                TRY(fnl::tensor_shard_barrier(ctx, reinterpret_cast<unsigned int* const*>(shard->peer_flags),
                                              shard->count,
                                              reinterpret_cast<unsigned int*>(shard->peer_flags[shard->rank]),
                                              (unsigned int)(seq * shard->count), barrier_err));
                TRY(fnl::tensor_shard_finalize(ctx, npairs, own, cap, d_count, m.done, out));
                return fnl::tensor_shard_reset(ctx, own, nkeys);
            }
            TRY(fnl::tensor_shard_reset(ctx, reinterpret_cast<long long*>(shard->d_keys), nkeys));
            if (te > tb)
                TRY(fnl::tensor_nn_pass(ctx, npairs, TQ, ids, cap, d_count, m.done, TT, dim, l2, out, cap,
                                        nullptr, near_ties, tb, te,
                                        reinterpret_cast<long long*>(shard->d_keys), nullptr, &rs));
            if (shard->comm) {
                TRY(fnl::comm_allreduce_min_i64(shard->comm, reinterpret_cast<long long*>(shard->d_keys), nkeys,
                                                ctx->stream));
            } else if (shard->reduce(shard->user, shard->d_keys, nkeys, ctx->stream) != 0) {
                return fail(FNL_ERUNTIME, "sharded reciprocal_match: key reduction callback failed");
            }
            return fnl::tensor_shard_finalize(ctx, npairs, reinterpret_cast<const long long*>(shard->d_keys), cap,
                                              d_count, m.done, out);
        }
        fnl::ScanArgs sa{};
        sa.qmap = Q.data;
        sa.qmap_pair_stride = (uint64_t)qrows * dim;
        sa.qids = ids;
        sa.qids_pair_stride = cap;
        sa.qcount = m.n_active;
        sa.pair_done = m.done;
        sa.q_row_sat = Q.row_sat;
        sa.q_row_sat_pair_stride = qrows;
        sa.tmap = Tm.data;
        sa.tmap_pair_stride = (uint64_t)nt * dim;
        sa.nt = nt;
        sa.dim = dim;
        sa.keys = keys;
        sa.keys_pair_stride = cap;
        sa.counters = counters + (size_t)call * npairs * 2;
        fnl::FinalizeArgs fa{};
        fa.keys = keys;
        fa.keys_pair_stride = cap;
        fa.qcount = m.n_active;
        fa.pair_done = m.done;
        fa.nearest = out;
        fa.nearest_pair_stride = cap;
        fa.dot = !l2;
        ++call;
        return exact_nn(ctx, sa, cap, npairs, l2, hyb, fa);
    };

    // reverse-NN memo (tensor route, one process; FNL_REV_MEMO=0 turns it off)
    // (the claimant lists are built in entry order, so every rank of a
    // sharded run queries the same rows in the same slots)
    const bool memo = tc && memo_env && samples > 0;
    if (memo) {
        TRY(dev_arr(ctx, "m.revcache", (size_t)npairs * p2, &m.rev_cache));
        TRY(dev_arr(ctx, "m.revlist", pc, &m.rev_list));
        TRY(dev_arr(ctx, "m.revout", pc, &m.rev_out));
        TRY(dev_arr(ctx, "m.revn", npairs, &m.rev_n));
    }
    auto reverse_pass = [&]() -> int {
        if (!memo) return nn_pass(P2, p2, m.active_v, P1, p1, m.back);
        // (rev_compact writes rev_n of every pair still running; a finished
        // pair's count is never read, so no reset is needed)
        FNL_CUDA_TRY(fnl::launch_rev_lookup(m, s));
        TRY(nn_pass(P2, p2, m.rev_list, P1, p1, m.rev_out, m.rev_n));
        FNL_CUDA_TRY(fnl::launch_rev_fill(m, s));
        ctx->total_launches += 3;  // claim, compact, fill
        return FNL_OK;
    };
    unsigned int* lag_done = nullptr;  // pinned [2]: n_done after iterations t-1, t
    cudaEvent_t* lag_ev = nullptr;
    if (tc) {
        TRY(fnl::ws_pinned(ctx, "m.lagdone", 8, (void**)&lag_done));
        TRY(lag_events(ctx, &lag_ev));
    }
    // sampling, the memo reset and the first forward pass (src/reciprocal.cpp:128-139)
    auto prefix = [&]() -> int {
        // loop state (inside the loop graph when it replays)
        FNL_CUDA_TRY(cudaMemsetAsync(m.used_i, 0, (size_t)npairs * m.words_i * 4, s));
        FNL_CUDA_TRY(cudaMemsetAsync(m.used_j, 0, (size_t)npairs * m.words_j * 4, s));
        FNL_CUDA_TRY(cudaMemsetAsync(m.n_done, 0, 4, s));
        // CUDA-core path state, and counters only the RunReport reads
        if (!tc) FNL_CUDA_TRY(cudaMemsetAsync(keys, 0xFF, pc * 8, s));
        if (!tc || h_stats) FNL_CUDA_TRY(cudaMemsetAsync(counters, 0, (size_t)max_calls * npairs * 16, s));
        if (h_stats) FNL_CUDA_TRY(cudaMemsetAsync(near_ties, 0, (size_t)npairs * 16, s));
        timer.begin(kPhaseSubsample);
        {
            fnl::ProfScope prof(ctx, FNL_KCLASS_HARVEST);
            FNL_CUDA_TRY(fnl::launch_match_init(m, s));
            ctx->total_launches += 1;
        }
        timer.end();
        if (memo) FNL_CUDA_TRY(cudaMemsetAsync(m.rev_cache, 0xFF, (size_t)npairs * p2 * 4, s));
        if (samples > 0) {
            timer.begin(kPhaseForward);
            TRY(nn_pass(P1, p1, m.active_u, P2, p2, m.active_v));
            timer.end();
        }
        return FNL_OK;
    };
    // ---- batches up to loop_graph_max_pairs (64): a small batch's loop is
    // launch-bound (a pass is a few tens of microseconds of GPU work behind
    // ~40 us of host launch cost), so it runs as ONE CUDA graph: the prefix
    // (state reset, sampling, memo reset, first forward pass), then a WHILE
    // node whose body is an iteration (reverse pass, harvest, condition
    // kernel, forward pass) and whose condition the device sets (some pair not
    // done and t < T).  Captured on the second run with an identical
    // configuration (same buffers, shapes, route and workspace), replayed
    // afterwards (speculatively, right behind the pack, when the route read
    // back above matches); the forward pass after the last harvest sees every
    // pair done and does nothing.
    bool replayed = false;
    std::vector<uint64_t> loop_key;
    const bool graph_ok = graph_env && tc && !sharded && !h_stats && !ctx->profile_all && samples > 0 &&
                          npairs <= loop_graph_max_pairs(ctx);
    if (graph_ok) {
        loop_key = make_key(acc16, memo);
        uint32_t* d_iter = nullptr;
        TRY(dev_arr(ctx, "m.iter", 1, &d_iter));
        if (ctx->ws_gen != loop_key.back()) loop_key = make_key(acc16, memo);  // (first use of m.iter)
        if (spec && spec->key == loop_key) {  // the speculative replay was the right one
            replayed = true;
            ctx->total_launches += spec->launches;
        }
        fnl_context::LoopGraph* lg = nullptr;
        for (auto& g : ctx->graphs)
            if (g.key == loop_key) lg = &g;
        if (!replayed && !lg && ctx->last_key == loop_key && ctx->failed_key != loop_key) {
            // capture the iteration into the WHILE node's body graph
            fnl_context::LoopGraph ng;
            ng.key = loop_key;
            cudaGraphConditionalHandle handle;
            cudaGraphNodeParams cp{};
            cudaGraphNode_t wnode;
            FNL_CUDA_TRY(cudaGraphCreate(&ng.graph, 0));
            FNL_CUDA_TRY(cudaGraphConditionalHandleCreate(&handle, ng.graph, 1, cudaGraphCondAssignDefault));
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = handle;
            cp.conditional.type = cudaGraphCondTypeWhile;
            cp.conditional.size = 1;
            if (!ctx->cap_stream) FNL_CUDA_TRY(cudaStreamCreateWithFlags(&ctx->cap_stream, cudaStreamNonBlocking));
            const cudaStream_t user = s;
            const bool timing = ctx->timing;
            const uint64_t gen0 = ctx->ws_gen, l0 = ctx->total_launches;
            ctx->stream = s = ctx->cap_stream;
            ctx->timing = false;  // no event marks inside the graph
            m.iter = d_iter;
            int rc = FNL_OK;
            cudaGraph_t captured = nullptr;
            // main graph: prefix -> WHILE node
            cudaError_t ce = cudaStreamBeginCaptureToGraph(s, ng.graph, nullptr, nullptr, 0,
                                                           cudaStreamCaptureModeThreadLocal);
            if (ce == cudaSuccess) {
                rc = prefix();
                if (rc == FNL_OK) rc = cudaMemsetAsync(d_iter, 0, 4, s) == cudaSuccess ? FNL_OK : FNL_ERUNTIME;
                cudaStreamCaptureStatus cs_status;
                const cudaGraphNode_t* deps = nullptr;
                size_t ndeps = 0;
                if (rc == FNL_OK) {
                    ce = cudaStreamGetCaptureInfo(s, &cs_status, nullptr, nullptr, &deps, &ndeps);
                    if (ce == cudaSuccess) ce = cudaGraphAddNode(&wnode, ng.graph, deps, ndeps, &cp);
                    if (ce == cudaSuccess)
                        ce = cudaStreamUpdateCaptureDependencies(s, &wnode, 1, cudaStreamSetCaptureDependencies);
                }
                const cudaError_t ee = cudaStreamEndCapture(s, &captured);
                if (ce == cudaSuccess) ce = ee;
            }
            // WHILE body: one iteration
            if (ce == cudaSuccess && rc == FNL_OK)
                ce = cudaStreamBeginCaptureToGraph(s, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                                   cudaStreamCaptureModeThreadLocal);
            if (ce == cudaSuccess && rc == FNL_OK) {
                rc = reverse_pass();
                if (rc == FNL_OK) rc = fnl::launch_harvest(m, 0, s) == cudaSuccess ? FNL_OK : FNL_ERUNTIME;
                if (rc == FNL_OK) rc = fnl::launch_loop_cond(m, handle, s) == cudaSuccess ? FNL_OK : FNL_ERUNTIME;
                if (rc == FNL_OK) rc = nn_pass(P1, p1, m.active_u, P2, p2, m.active_v);
                ce = cudaStreamEndCapture(s, &captured);
            }
            ctx->stream = s = user;
            ctx->timing = timing;
            // launches per replay: the prefix plus one iteration (+ harvest, condition)
            ng.launches = ctx->total_launches - l0 + 2;
            ctx->total_launches = l0;
            if (ce == cudaSuccess && rc == FNL_OK && ctx->ws_gen == gen0)
                ce = cudaGraphInstantiate(&ng.exec, ng.graph, 0);
            if (getenv("FNL_LOOP_GRAPH_DEBUG"))
                fprintf(stderr, "fnl loop graph: capture ce=%d (%s) rc=%d gen %d exec %d\n", (int)ce,
                        cudaGetErrorString(ce), rc, (int)(ctx->ws_gen == gen0), ng.exec != nullptr);
            if (ce != cudaSuccess || rc != FNL_OK || ctx->ws_gen != gen0 || !ng.exec) {
                // not capturable here: keep the host-driven loop
                cudaGetLastError();
                if (ng.exec) cudaGraphExecDestroy(ng.exec);
                cudaGraphDestroy(ng.graph);
                m.iter = nullptr;
                ctx->failed_key = loop_key;
            } else {
                if (ctx->graphs.size() >= 4) {
                    cudaGraphExecDestroy(ctx->graphs.front().exec);
                    cudaGraphDestroy(ctx->graphs.front().graph);
                    ctx->graphs.erase(ctx->graphs.begin());
                }
                ctx->graphs.push_back(ng);
                lg = &ctx->graphs.back();
            }
        }
        if (getenv("FNL_LOOP_GRAPH_DEBUG"))  // tests: which calls replay
            fprintf(stderr, "fnl loop graph: replay %d graphs %zu\n", lg != nullptr, ctx->graphs.size());
        if (lg && !replayed) {
            FNL_CUDA_TRY(cudaGraphLaunch(lg->exec, s));
            ctx->total_launches += lg->launches;  // (one iteration's worth)
            replayed = true;
        }
    }
    if (!replayed) TRY(prefix());
    for (uint32_t t = 1; t <= T && samples > 0 && !replayed; ++t) {
        timer.begin(kPhaseReverse);
        TRY(reverse_pass());
        timer.end();
        timer.begin(kPhaseHarvest);
        {
            fnl::ProfScope prof(ctx, FNL_KCLASS_HARVEST);
            FNL_CUDA_TRY(fnl::launch_harvest(m, t, s));
        }
        timer.end();
        ctx->total_launches += 1;
        if (tc) {
            // Lagged convergence check: iteration t is enqueued before the
            // host looks at the done count of iteration t-1, so the GPU never
            // idles on the round trip.  Passes enqueued after the last pair
            // finished skip every pair on the device (done flags) and change
            // nothing; every rank of a sharded run sees the same counts, so
            // the collectives stay matched.
            FNL_CUDA_TRY(cudaMemcpyAsync(lag_done + (t & 1), m.n_done, 4, cudaMemcpyDeviceToHost, s));
            FNL_CUDA_TRY(cudaEventRecord(lag_ev[t & 1], s));
            if (t >= 2) {
                FNL_CUDA_TRY(cudaEventSynchronize(lag_ev[(t - 1) & 1]));
                if (lag_done[(t - 1) & 1] >= npairs) break;
            }
        } else {
            unsigned int ndone = 0;
            FNL_CUDA_TRY(cudaMemcpyAsync(&ndone, m.n_done, 4, cudaMemcpyDeviceToHost, s));
            FNL_CUDA_TRY(cudaStreamSynchronize(s));
            if (ndone >= npairs) break;
        }
        timer.begin(kPhaseForward);
        TRY(nn_pass(P1, p1, m.active_u, P2, p2, m.active_v));
        timer.end();
    }
    if (graph_ok && !replayed) ctx->last_key = make_key(acc16, memo);

    if (peer) {
        unsigned int err = 0;
        FNL_CUDA_TRY(cudaMemcpyAsync(&err, barrier_err, 4, cudaMemcpyDeviceToHost, s));
        FNL_CUDA_TRY(cudaStreamSynchronize(s));
        if (err) return fail(FNL_ERUNTIME, "sharded reciprocal_match: peer-memory barrier timed out (a rank stopped)");
    }

    // ---- stats back to host and the reference's accounting
    if (h_stats) {
        std::vector<uint32_t> st((size_t)npairs * fnl::kStatWords);
        std::vector<unsigned long long> cnt((size_t)max_calls * npairs * 2);
        std::vector<unsigned long long> ms1(npairs), ms2(npairs);
        std::vector<uint32_t> npr(npairs);
        FNL_CUDA_TRY(cudaMemcpyAsync(st.data(), m.stats, st.size() * 4, cudaMemcpyDeviceToHost, s));
        FNL_CUDA_TRY(cudaMemcpyAsync(cnt.data(), counters, cnt.size() * 8, cudaMemcpyDeviceToHost, s));
        if (!tc) {
            FNL_CUDA_TRY(cudaMemcpyAsync(ms1.data(), P1.map_sat, npairs * 8, cudaMemcpyDeviceToHost, s));
            FNL_CUDA_TRY(cudaMemcpyAsync(ms2.data(), P2.map_sat, npairs * 8, cudaMemcpyDeviceToHost, s));
        }
        FNL_CUDA_TRY(cudaMemcpyAsync(npr.data(), m.n_pairs, npairs * 4, cudaMemcpyDeviceToHost, s));
        std::vector<unsigned long long> tsat_h(2 * (size_t)npairs), ties_h(2 * (size_t)npairs);
        FNL_CUDA_TRY(cudaMemcpyAsync(tsat_h.data(), tsat, tsat_h.size() * 8, cudaMemcpyDeviceToHost, s));
        FNL_CUDA_TRY(cudaMemcpyAsync(ties_h.data(), near_ties, ties_h.size() * 8, cudaMemcpyDeviceToHost, s));
        FNL_CUDA_TRY(cudaStreamSynchronize(s));
        double phase_us[4] = {0, 0, 0, 0};
        timer.collect(phase_us);
        const uint64_t bs = cfg->block_size;
        for (uint32_t p = 0; p < npairs; ++p) {
            const uint32_t* ps = st.data() + (size_t)p * fnl::kStatWords;
            fnl_run_stats& o = h_stats[p];
            memset(&o, 0, sizeof(o));
            o.samples = samples;
            o.subsample_us = phase_us[kPhaseSubsample];
            o.forward_nn_us = phase_us[kPhaseForward];
            o.reverse_nn_us = phase_us[kPhaseReverse];
            o.harvest_us = phase_us[kPhaseHarvest];
            o.iterations = ps[fnl::kStatIters];
            o.converged = ps[fnl::kStatConverged];
            o.duplicates_dropped = ps[fnl::kStatDups];
            o.matches = npr[p];
            o.history_len = std::min<uint32_t>(ps[fnl::kStatHistLen], FNL_MAX_ITERS);
            for (uint32_t i = 0; i < o.history_len; ++i) o.active_history[i] = ps[fnl::kStatHist + i];
            // rebuild the call sequence: fwd(S), then rev(active_{t-1}) and, except
            // after the last iteration, fwd(active_t)
            struct Call { uint64_t nq, nt; bool fwd; };
            std::vector<Call> calls;
            if (samples > 0) calls.push_back({samples, p2, true});
            uint32_t prev = samples;
            for (uint32_t t = 1; t <= o.iterations; ++t) {
                calls.push_back({prev, p1, false});
                const uint32_t cur = o.active_history[t - 1];
                if (t < o.iterations) calls.push_back({cur, p2, true});
                prev = cur;
            }
            for (size_t c = 0; c < calls.size(); ++c) {
                const Call& k = calls[c];
                o.query_rows += k.nq;
                if (backend == FNL_BACKEND_BRUTEFORCE) continue;
                const uint64_t nqb = ceil_div(k.nq, bs), ntb = ceil_div(k.nt, bs);
                const unsigned long long qs = c < max_calls ? cnt[(c * npairs + p) * 2 + 0] : 0;
                const unsigned long long ds = c < max_calls ? cnt[(c * npairs + p) * 2 + 1] : 0;
                const unsigned long long tsat = k.fwd ? ms2[p] : ms1[p];
                o.a_block_fetches += nqb;
                if (backend == FNL_BACKEND_DOUBLE) {
                    o.b_block_fetches += nqb * ntb;
                    if (hyb) o.half_saturation_events += nqb * tsat + ntb * qs + ds;
                } else {
                    o.b_block_fetches += nqb;
                    if (hyb) o.half_saturation_events += tsat + qs + ds;
                }
            }
            if (tensor) o.half_saturation_events = tsat_h[p] + tsat_h[npairs + p];
            if (tc) {
                o.near_tie_rows = ties_h[p];
                o.rescan_rows = ties_h[npairs + p];
                o.tensor_route = 1;
            }
            o.computed_query_rows = o.query_rows;
            if (memo) {
                uint64_t rev_logical = 0;
                for (const Call& k : calls)
                    if (!k.fwd) rev_logical += k.nq;
                o.computed_query_rows = o.query_rows - rev_logical + ps[fnl::kStatRevComputed];
            }
        }
    }
    timing_harvest(ctx);
    return FNL_OK;
}

}  // namespace

extern "C" int fnl_reciprocal_match(fnl_context* ctx, const float* h_d1, uint32_t h1, uint32_t w1,
                                    const float* h_d2, uint32_t h2, uint32_t w2, uint32_t dim,
                                    const fnl_match_config* cfg, int backend, uint32_t* h_pairs,
                                    uint32_t* n_pairs, fnl_run_stats* stats) {
    TRY(check_device(ctx));
    TRY(check_cfg(cfg));
    const uint64_t n1 = (uint64_t)h1 * w1 * dim, n2 = (uint64_t)h2 * w2 * dim;
    float *d1, *d2;
    TRY(dev_arr(ctx, "rm.d1", n1, &d1));
    TRY(dev_arr(ctx, "rm.d2", n2, &d2));
    FNL_CUDA_TRY(cudaMemcpyAsync(d1, h_d1, n1 * 4, cudaMemcpyHostToDevice, ctx->stream));
    FNL_CUDA_TRY(cudaMemcpyAsync(d2, h_d2, n2 * 4, cudaMemcpyHostToDevice, ctx->stream));
    const uint32_t stride = derived_stride(h1, w1, cfg->k, cfg->grid_stride);
    const uint32_t samples = ((h1 + stride - 1) / stride) * ((w1 + stride - 1) / stride);
    uint32_t *dp, *dn;
    TRY(dev_arr(ctx, "rm.pairs", (size_t)3 * std::max<uint32_t>(samples, 1), &dp));
    TRY(dev_arr(ctx, "rm.np", 1, &dn));
    fnl_run_stats local;
    TRY(run_match(ctx, 1, d1, h1, w1, d2, h2, w2, dim, cfg, backend, dp, dn,
                  stats ? stats : &local, true));
    uint32_t n = 0;
    FNL_CUDA_TRY(cudaMemcpyAsync(&n, dn, 4, cudaMemcpyDeviceToHost, ctx->stream));
    FNL_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (n && h_pairs)
        FNL_CUDA_TRY(cudaMemcpyAsync(h_pairs, dp, (size_t)n * 12, cudaMemcpyDeviceToHost, ctx->stream));
    FNL_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (n_pairs) *n_pairs = n;
    return FNL_OK;
}

extern "C" int fnl_reciprocal_match_sharded(fnl_context* ctx, fnl_comm* comm, const float* h_d1, uint32_t h1,
                                            uint32_t w1, const float* h_d2, uint32_t h2, uint32_t w2, uint32_t dim,
                                            const fnl_match_config* cfg, int backend, uint32_t* h_pairs,
                                            uint32_t* n_pairs, fnl_run_stats* stats) {
    TRY(check_device(ctx));
    TRY(check_cfg(cfg));
    if (!comm) return fail(FNL_EINVAL, "fnl_reciprocal_match_sharded: null communicator");
    int nranks = 0, rank = 0;
    fnl::comm_size(comm, &nranks, &rank);
    const uint64_t n1 = (uint64_t)h1 * w1 * dim, n2 = (uint64_t)h2 * w2 * dim;
    float *d1, *d2;
    TRY(dev_arr(ctx, "rms.d1", n1, &d1));
    TRY(dev_arr(ctx, "rms.d2", n2, &d2));
    FNL_CUDA_TRY(cudaMemcpyAsync(d1, h_d1, n1 * 4, cudaMemcpyHostToDevice, ctx->stream));
    FNL_CUDA_TRY(cudaMemcpyAsync(d2, h_d2, n2 * 4, cudaMemcpyHostToDevice, ctx->stream));
    const uint32_t stride = derived_stride(h1, w1, cfg->k, cfg->grid_stride);
    const uint32_t samples = ((h1 + stride - 1) / stride) * ((w1 + stride - 1) / stride);
    const uint32_t cap = std::max<uint32_t>(samples, 1);
    uint32_t *dp, *dn;
    long long* keys;
    TRY(dev_arr(ctx, "rms.pairs", (size_t)3 * cap, &dp));
    TRY(dev_arr(ctx, "rms.np", 1, &dn));
    TRY(dev_arr(ctx, "rms.keys", cap, &keys));
    fnl_shard_spec spec{};
    spec.rank = (uint32_t)rank;
    spec.count = (uint32_t)nranks;
    spec.d_keys = reinterpret_cast<int64_t*>(keys);
    spec.keys_capacity = cap;
    spec.comm = comm;
    fnl_run_stats local;
    TRY(run_match(ctx, 1, d1, h1, w1, d2, h2, w2, dim, cfg, backend, dp, dn, stats ? stats : &local, true, &spec));
    uint32_t n = 0;
    FNL_CUDA_TRY(cudaMemcpyAsync(&n, dn, 4, cudaMemcpyDeviceToHost, ctx->stream));
    FNL_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (n && h_pairs)
        FNL_CUDA_TRY(cudaMemcpyAsync(h_pairs, dp, (size_t)n * 12, cudaMemcpyDeviceToHost, ctx->stream));
    FNL_CUDA_TRY(cudaStreamSynchronize(ctx->stream));
    if (n_pairs) *n_pairs = n;
    return FNL_OK;
}

extern "C" int fnl_reciprocal_match_batch_device(fnl_context* ctx, uint32_t npairs,
                                                 const float* d_d1, const float* d_d2, uint32_t h,
                                                 uint32_t w, uint32_t dim,
                                                 const fnl_match_config* cfg, int backend,
                                                 uint32_t* d_pairs, uint32_t* d_n_pairs,
                                                 fnl_run_stats* h_stats) {
    TRY(check_device(ctx));
    if (npairs == 0) return FNL_OK;
    return run_match(ctx, npairs, d_d1, h, w, d_d2, h, w, dim, cfg, backend, d_pairs, d_n_pairs,
                     h_stats, false);
}

extern "C" int fnl_reciprocal_match_sharded_device(fnl_context* ctx, uint32_t npairs, const float* d_d1,
                                                   const float* d_d2, uint32_t h, uint32_t w, uint32_t dim,
                                                   const fnl_match_config* cfg, int backend,
                                                   const fnl_shard_spec* shard, uint32_t* d_pairs,
                                                   uint32_t* d_n_pairs, fnl_run_stats* h_stats) {
    TRY(check_device(ctx));
    if (!shard) return fail(FNL_EINVAL, "fnl_reciprocal_match_sharded_device: null shard spec");
    if (npairs == 0) return FNL_OK;
    return run_match(ctx, npairs, d_d1, h, w, d_d2, h, w, dim, cfg, backend, d_pairs, d_n_pairs, h_stats, false,
                     shard);
}

extern "C" int fnl_reciprocal_match_batch(fnl_context* ctx, uint32_t npairs, const float* h_d1,
                                          const float* h_d2, uint32_t h, uint32_t w, uint32_t dim,
                                          const fnl_match_config* cfg, int backend,
                                          uint32_t* h_pairs, uint32_t* n_pairs,
                                          fnl_run_stats* stats) {
    TRY(check_device(ctx));
    TRY(check_cfg(cfg));
    if (npairs == 0) return FNL_OK;
    const uint64_t per_map = (uint64_t)h * w * dim;
    const uint32_t stride = derived_stride(h, w, cfg->k, cfg->grid_stride);
    const uint32_t samples = ((h + stride - 1) / stride) * ((w + stride - 1) / stride);
    const uint32_t cap = std::max<uint32_t>(samples, 1);
    // Sub-batches double-buffered: the copy engine uploads sub-batch k+1 while
    // sub-batch k is matched.  Sizes ramp 8, 16, 32, 32, ... so the one upload
    // that nothing overlaps (the first) is short, while later sub-batches are
    // large enough to amortise the per-call work (measured: 16-pair chunks
    // 1124 pairs/s, 32-pair 1171, ramp: see bench e2e).
    static const uint32_t sub_env = getenv("FNL_BATCH_SUB") ? (uint32_t)atoi(getenv("FNL_BATCH_SUB")) : 0;
    const uint32_t max_sub = std::min<uint32_t>(npairs, sub_env ? sub_env : 32);
    std::vector<std::pair<uint32_t, uint32_t>> sched;  // (first pair, count)
    for (uint32_t first = 0, want = sub_env ? max_sub : 8; first < npairs;) {
        const uint32_t n = std::min(std::min(want, max_sub), npairs - first);
        sched.push_back({first, n});
        first += n;
        want = std::min(2 * want, max_sub);  // capped: a doubling uint32 would wrap to 0 after 29 sub-batches
    }
    const uint32_t sub = max_sub;
    float* dbuf[2][2];
    TRY(dev_arr(ctx, "mb.d1a", sub * per_map, &dbuf[0][0]));
    TRY(dev_arr(ctx, "mb.d2a", sub * per_map, &dbuf[0][1]));
    TRY(dev_arr(ctx, "mb.d1b", sub * per_map, &dbuf[1][0]));
    TRY(dev_arr(ctx, "mb.d2b", sub * per_map, &dbuf[1][1]));
    uint32_t *dp, *dn;
    TRY(dev_arr(ctx, "mb.pairs", (size_t)sub * 3 * cap, &dp));
    TRY(dev_arr(ctx, "mb.np", sub, &dn));
    cudaEvent_t ready[2], consumed[2];
    for (int i = 0; i < 2; ++i) {
        cudaEventCreateWithFlags(&ready[i], cudaEventDisableTiming);
        cudaEventCreateWithFlags(&consumed[i], cudaEventDisableTiming);
        cudaEventRecord(consumed[i], ctx->stream);
    }
    auto upload = [&](size_t idx, int slot) -> int {
        const uint32_t first = sched[idx].first, n = sched[idx].second;
        FNL_CUDA_TRY(cudaStreamWaitEvent(ctx->copy_stream, consumed[slot], 0));
        // 32 MB pieces: H2D copies share one copy engine in FIFO order, so a
        // single 600 MB copy would hold the matcher's small per-pass H2D
        // transfers (work lists) hostage for ~11 ms (measured with CUPTI)
        constexpr size_t kPiece = (size_t)32 << 20;
        for (int m = 0; m < 2; ++m) {
            const char* src = reinterpret_cast<const char*>((m ? h_d2 : h_d1) + first * per_map);
            char* dst = reinterpret_cast<char*>(dbuf[slot][m]);
            const size_t bytes = (size_t)n * per_map * 4;
            for (size_t off = 0; off < bytes; off += kPiece)
                FNL_CUDA_TRY(cudaMemcpyAsync(dst + off, src + off, std::min(kPiece, bytes - off),
                                             cudaMemcpyHostToDevice, ctx->copy_stream));
        }
        FNL_CUDA_TRY(cudaEventRecord(ready[slot], ctx->copy_stream));
        return FNL_OK;
    };
    // A large pinned H2D cudaMemcpyAsync still blocks the calling host thread
    // for much of the copy (measured), and run_match drives its loop from the
    // host, so the uploads run on their own host thread, at most one
    // sub-batch ahead of the matcher (two device buffers).
    std::mutex mu;
    std::condition_variable cv;
    size_t uploaded = 0, consumed_n = 0;
    bool abort = false;
    int up_status = FNL_OK;
    std::string up_error;
    const int device = ctx->device;
    std::thread uploader([&] {
        cudaSetDevice(device);
        for (size_t k = 0; k < sched.size(); ++k) {
            {
                std::unique_lock<std::mutex> lk(mu);
                cv.wait(lk, [&] { return abort || k < consumed_n + 2; });
                if (abort) return;
            }
            const int rc = upload(k, (int)(k & 1));
            std::lock_guard<std::mutex> lk(mu);
            if (rc != FNL_OK) {
                up_status = rc;
                up_error = fnl_last_error();
                abort = true;
                cv.notify_all();
                return;
            }
            uploaded = k + 1;
            cv.notify_all();
        }
    });
    // results come back through pinned staging (a pageable D2H would block)
    uint32_t* pin_out = nullptr;
    int st = fnl::ws_pinned(ctx, "mb.out.pin", ((size_t)sub * 3 * cap + sub) * 4, (void**)&pin_out);
    for (size_t k = 0; st == FNL_OK && k < sched.size(); ++k) {
        const int slot = k & 1;
        const uint32_t first = sched[k].first, n = sched[k].second;
        {
            std::unique_lock<std::mutex> lk(mu);
            cv.wait(lk, [&] { return abort || uploaded > k; });
            if (abort) {
                st = fail(up_status ? up_status : FNL_ERUNTIME, "batch upload: " + up_error);
                break;
            }
        }
        cudaStreamWaitEvent(ctx->stream, ready[slot], 0);
        st = run_match(ctx, n, dbuf[slot][0], h, w, dbuf[slot][1], h, w, dim, cfg, backend, dp,
                       dn, stats ? stats + first : nullptr, true);
        if (st) break;
        cudaEventRecord(consumed[slot], ctx->stream);
        uint32_t* pin_cnt = pin_out + (size_t)sub * 3 * cap;
        cudaMemcpyAsync(pin_cnt, dn, n * 4, cudaMemcpyDeviceToHost, ctx->stream);
        if (h_pairs) cudaMemcpyAsync(pin_out, dp, (size_t)n * 3 * cap * 4, cudaMemcpyDeviceToHost, ctx->stream);
        cudaError_t e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) {
            st = fnl::fail_cuda(e, "batch readback", __FILE__, __LINE__);
            break;
        }
        {
            std::lock_guard<std::mutex> lk(mu);
            consumed_n = k + 1;
            cv.notify_all();
        }
        if (h_pairs) memcpy(h_pairs + (size_t)first * 3 * cap, pin_out, (size_t)n * 3 * cap * 4);
        if (n_pairs) memcpy(n_pairs + first, pin_cnt, n * 4);
    }
    {
        std::lock_guard<std::mutex> lk(mu);
        abort = true;
        cv.notify_all();
    }
    uploader.join();
    cudaStreamSynchronize(ctx->copy_stream);
    for (int i = 0; i < 2; ++i) {
        cudaEventDestroy(ready[i]);
        cudaEventDestroy(consumed[i]);
    }
    return st;
}

extern "C" int fnl_confidence_compact_device(fnl_context* ctx, uint32_t npairs, const float* d_d1,
                                             const float* d_d2, uint32_t h, uint32_t w, uint32_t dim, int metric,
                                             float max_distance, uint32_t* d_pairs, uint32_t* d_n_pairs,
                                             uint32_t cap, uint32_t* d_dropped) {
    TRY(check_device(ctx));
    if (!valid_metric(metric)) return fail(FNL_EINVAL, "confidence_compact: bad metric");
    if (npairs == 0) return FNL_OK;
    if (!d_d1 || !d_d2 || !d_pairs || !d_n_pairs || dim == 0 || cap == 0)
        return fail(FNL_EINVAL, "confidence_compact: null buffer or empty shape");
    fnl::ConfArgs a{};
    a.d1 = d_d1;
    a.d2 = d_d2;
    a.map1_stride = a.map2_stride = (uint64_t)h * w * dim;
    a.dim = dim;
    a.l2 = metric == FNL_METRIC_L2;
    a.max_dist = max_distance;
    a.pairs = d_pairs;
    a.n_pairs = d_n_pairs;
    a.cap = cap;
    a.dropped = d_dropped;
    fnl::ProfScope prof(ctx, FNL_KCLASS_HARVEST);
    FNL_CUDA_TRY(fnl::launch_confidence_compact(a, npairs, ctx->stream));
    ctx->total_launches += 1;
    return FNL_OK;
}

// ============================================================== diagnostics
extern "C" int fnl_tensor_selftest(fnl_context* ctx, const float* h_q, const float* h_t, uint32_t dim,
                                   int metric, int mode, float* h_scores) {
    TRY(check_device(ctx));
    float *dq, *dt, *dout;
    TRY(dev_arr(ctx, "st.q", (size_t)256 * dim, &dq));
    TRY(dev_arr(ctx, "st.t", (size_t)128 * dim, &dt));
    TRY(dev_arr(ctx, "st.out", (size_t)256 * 128, &dout));
    FNL_CUDA_TRY(cudaMemcpyAsync(dq, h_q, (size_t)256 * dim * 4, cudaMemcpyHostToDevice, ctx->stream));
    FNL_CUDA_TRY(cudaMemcpyAsync(dt, h_t, (size_t)128 * dim * 4, cudaMemcpyHostToDevice, ctx->stream));
    TRY(fnl::tensor_selftest_scores(ctx, dq, dt, dim, metric == FNL_METRIC_L2, mode, dout));
    FNL_CUDA_TRY(cudaMemcpy(h_scores, dout, (size_t)256 * 128 * 4, cudaMemcpyDeviceToHost));
    return FNL_OK;
}

// ============================================================== mutual NN
namespace {

// Dense mutual NN (src/reciprocal.cpp:82-95): NN of every D1 pixel in D2 and
// of every D2 pixel in D1, then the pairs that agree.  Tensor route: both maps
// packed once, both directions back to back on the device (tensor_mutual_dense),
// resolved in full precision (mutual_nn_exact) or on the binary16-rounded rows
// (mutual_nn_tensor); else the CUDA-core exact scan K4.
int mutual_nn_run(fnl_context* ctx, const char* who, const float* h_d1, uint32_t h1, uint32_t w1,
                  const float* h_d2, uint32_t h2, uint32_t w2, uint32_t dim, int metric, bool rounded,
                  uint32_t* h_pairs, uint32_t* n_pairs) {
    TRY(check_device(ctx));
    if (!valid_metric(metric)) return fail(FNL_EINVAL, std::string(who) + ": bad metric");
    const uint32_t p1 = h1 * w1, p2 = h2 * w2;
    if (p1 == 0 || p2 == 0 || dim == 0) return fail(FNL_EINVAL, std::string(who) + ": empty map");
    const bool l2 = metric == FNL_METRIC_L2;
    float *d1, *d2;
    uint32_t *fwd, *bwd, *pairs, *cnt;
    TRY(dev_arr(ctx, "mu.d1", (size_t)p1 * dim, &d1));
    TRY(dev_arr(ctx, "mu.d2", (size_t)p2 * dim, &d2));
    TRY(dev_arr(ctx, "mu.fwd", p1, &fwd));
    TRY(dev_arr(ctx, "mu.bwd", p2, &bwd));
    TRY(dev_arr(ctx, "mu.pairs", (size_t)2 * p1 + 2, &pairs));
    TRY(dev_arr(ctx, "mu.cnt", 1, &cnt));
    cudaStream_t s = ctx->stream;
    FNL_CUDA_TRY(cudaMemcpyAsync(d1, h_d1, (size_t)p1 * dim * 4, cudaMemcpyHostToDevice, s));
    FNL_CUDA_TRY(cudaMemcpyAsync(d2, h_d2, (size_t)p2 * dim * 4, cudaMemcpyHostToDevice, s));
    bool routed = false, checked = false;
    if (rounded || !force_cuda_core()) {
        // (the pack also finds non-finite inputs: validated like the
        // reference FeatureMap, D1 first)
        unsigned long long hb[2] = {~0ull, ~0ull};
        TRY(fnl::tensor_mutual_dense(ctx, d1, p1, d2, p2, dim, l2, rounded ? fnl::kResolveRounded : fnl::kResolveFull,
                                     fwd, bwd, &routed, hb));
        if (hb[0] != ~0ull) return fail(FNL_EINVAL, nonfinite_msg(hb[0]));
        if (hb[1] != ~0ull) return fail(FNL_EINVAL, nonfinite_msg(hb[1]));
        checked = dim + (l2 ? 2u : 0u) <= fnl::kPackK;
    }
    if (!routed) {
        unsigned long long *k1, *k2, *bad;
        TRY(dev_arr(ctx, "mu.k1", p1, &k1));
        TRY(dev_arr(ctx, "mu.k2", p2, &k2));
        TRY(dev_arr(ctx, "mu.bad", 1, &bad));
        FNL_CUDA_TRY(cudaMemsetAsync(k1, 0xFF, (size_t)p1 * 8, s));
        FNL_CUDA_TRY(cudaMemsetAsync(k2, 0xFF, (size_t)p2 * 8, s));
        FNL_CUDA_TRY(cudaMemsetAsync(bad, 0xFF, 8, s));
        Prepared P1, P2;
        TRY(prepare_maps(ctx, "mu.p1", d1, 1, p1, dim, rounded, !checked, &P1, bad));
        if (!checked) {
            unsigned long long hb = ~0ull;
            FNL_CUDA_TRY(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, s));
            FNL_CUDA_TRY(cudaStreamSynchronize(s));
            if (hb != ~0ull) return fail(FNL_EINVAL, nonfinite_msg(hb));
        }
        TRY(prepare_maps(ctx, "mu.p2", d2, 1, p2, dim, rounded, !checked, &P2, bad));
        if (!checked) {
            unsigned long long hb = ~0ull;
            FNL_CUDA_TRY(cudaMemcpyAsync(&hb, bad, 8, cudaMemcpyDeviceToHost, s));
            FNL_CUDA_TRY(cudaStreamSynchronize(s));
            if (hb != ~0ull) return fail(FNL_EINVAL, nonfinite_msg(hb));
        }
        auto pass = [&](const float* q, uint32_t nq, const float* t, uint32_t nt, unsigned long long* keys,
                        uint32_t* out) -> int {
            fnl::ScanArgs sa{};
            sa.qmap = q;
            sa.qcount_const = nq;
            sa.tmap = t;
            sa.nt = nt;
            sa.dim = dim;
            sa.keys = keys;
            sa.keys_pair_stride = nq;
            fnl::FinalizeArgs fa{};
            fa.keys = keys;
            fa.keys_pair_stride = nq;
            fa.qcount_const = nq;
            fa.nearest = out;
            fa.nearest_pair_stride = nq;
            fa.dot = !l2;
            return exact_nn(ctx, sa, nq, 1, l2, false, fa);
        };
        TRY(pass(P1.data, p1, P2.data, p2, k1, fwd));
        TRY(pass(P2.data, p2, P1.data, p1, k2, bwd));
    }
    FNL_CUDA_TRY(fnl::launch_mutual_filter(fwd, bwd, p1, pairs, cnt, s));
    uint32_t n = 0;
    FNL_CUDA_TRY(cudaMemcpyAsync(&n, cnt, 4, cudaMemcpyDeviceToHost, s));
    FNL_CUDA_TRY(cudaStreamSynchronize(s));
    if (n && h_pairs) FNL_CUDA_TRY(cudaMemcpyAsync(h_pairs, pairs, (size_t)n * 8, cudaMemcpyDeviceToHost, s));
    FNL_CUDA_TRY(cudaStreamSynchronize(s));
    timing_harvest(ctx);
    if (n_pairs) *n_pairs = n;
    return FNL_OK;
}

}  // namespace

extern "C" int fnl_mutual_nn(fnl_context* ctx, const float* h_d1, uint32_t h1, uint32_t w1,
                             const float* h_d2, uint32_t h2, uint32_t w2, uint32_t dim, int metric,
                             uint32_t* h_pairs, uint32_t* n_pairs) {
    return mutual_nn_run(ctx, "mutual_nn_exact", h_d1, h1, w1, h_d2, h2, w2, dim, metric, false, h_pairs, n_pairs);
}

// Dense mutual NN on the binary16-rounded maps (the tensor backend's contract).
extern "C" int fnl_mutual_nn_tensor(fnl_context* ctx, const float* h_d1, uint32_t h1, uint32_t w1,
                                    const float* h_d2, uint32_t h2, uint32_t w2, uint32_t dim, int metric,
                                    uint32_t* h_pairs, uint32_t* n_pairs) {
    return mutual_nn_run(ctx, "mutual_nn_tensor", h_d1, h1, w1, h_d2, h2, w2, dim, metric, true, h_pairs, n_pairs);
}

// ---------------------------------------------------------------- peer memory
namespace {
__global__ void fill_i64_kernel(long long* p, uint64_t n, long long v) {
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        p[i] = v;
}
}  // namespace

extern "C" int fnl_p2p_alloc(fnl_context* ctx, uint64_t bytes, int fill_key_none, void** d_ptr) {
    TRY(check_device(ctx));
    if (!d_ptr || bytes == 0) return fail(FNL_EINVAL, "fnl_p2p_alloc: null output or zero size");
    if (fill_key_none && bytes % 8) return fail(FNL_EINVAL, "fnl_p2p_alloc: key buffers are int64");
    void* p = nullptr;
    FNL_CUDA_TRY(cudaMalloc(&p, bytes));
    if (fill_key_none) {
        const uint64_t n = bytes / 8;
        fill_i64_kernel<<<(unsigned)std::min<uint64_t>(1024, (n + 255) / 256), 256>>>(
            static_cast<long long*>(p), n, 0x7FFFFFFFFFFFFFFFll);
        FNL_CUDA_TRY(cudaGetLastError());
    } else {
        FNL_CUDA_TRY(cudaMemset(p, 0, bytes));
    }
    FNL_CUDA_TRY(cudaDeviceSynchronize());
    *d_ptr = p;
    return FNL_OK;
}

extern "C" int fnl_p2p_free(void* d_ptr) {
    if (d_ptr) FNL_CUDA_TRY(cudaFree(d_ptr));
    return FNL_OK;
}

extern "C" int fnl_ipc_handle(const void* d_ptr, unsigned char handle[64]) {
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "CUDA IPC handles are 64 bytes");
    if (!d_ptr || !handle) return fail(FNL_EINVAL, "fnl_ipc_handle: null pointer");
    cudaIpcMemHandle_t h;
    FNL_CUDA_TRY(cudaIpcGetMemHandle(&h, const_cast<void*>(d_ptr)));
    memcpy(handle, &h, 64);
    return FNL_OK;
}

extern "C" int fnl_ipc_open(fnl_context* ctx, const unsigned char handle[64], void** d_ptr) {
    TRY(check_device(ctx));
    if (!handle || !d_ptr) return fail(FNL_EINVAL, "fnl_ipc_open: null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    FNL_CUDA_TRY(cudaIpcOpenMemHandle(d_ptr, h, cudaIpcMemLazyEnablePeerAccess));
    return FNL_OK;
}

extern "C" int fnl_ipc_close(void* d_ptr) {
    if (d_ptr) FNL_CUDA_TRY(cudaIpcCloseMemHandle(d_ptr));
    return FNL_OK;
}
