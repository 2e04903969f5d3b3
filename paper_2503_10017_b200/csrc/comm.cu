// comm.cu -- native NCCL for the C5 key reduction (include/fastnn_b200.h,
// fnl_comm_*).  The reference has no distributed code; this is what lets a C
// or C++ caller shard one oversized pair's target columns over the GPUs of a
// node without a Python all-reduce: run_match calls
// ncclAllReduce(int64, ncclMin) on the context stream once per NN pass.
//
// libnccl.so.2 is opened at first use (dlopen), so the library has no
// link-time NCCL dependency: inside a process that already loaded torch's
// NCCL the same copy is reused (same soname), elsewhere the system one.
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <mutex>
#include <string>

#include "fastnn_b200.h"
#include "fnl_common.cuh"
#include "fnl_internal.h"

using fnl::fail;

namespace {

struct NcclApi {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                               cudaStream_t) = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
    ncclResult_t (*get_version)(int*) = nullptr;
    std::string error;
    bool ok = false;
};

NcclApi& api() {
    static NcclApi a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            a.error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(sym("ncclAllReduce"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
        a.get_version = reinterpret_cast<decltype(a.get_version)>(sym("ncclGetVersion"));
        a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_reduce && a.error_string;
        if (!a.ok) a.error = "libnccl.so.2 lacks the expected symbols";
    });
    return a;
}

int nccl_fail(ncclResult_t r, const char* what) {
    return fail(FNL_ERUNTIME, std::string("NCCL ") + what + ": " + api().error_string(r));
}

}  // namespace

struct fnl_comm {
    ncclComm_t comm = nullptr;
    int nranks = 0;
    int rank = 0;
    int device = 0;
};

extern "C" int fnl_nccl_unique_id(unsigned char id[128]) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    if (!id) return fail(FNL_EINVAL, "fnl_nccl_unique_id: null output");
    NcclApi& a = api();
    if (!a.ok) return fail(FNL_ERUNTIME, a.error);
    ncclUniqueId u;
    const ncclResult_t r = a.get_unique_id(&u);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    memcpy(id, &u, 128);
    return FNL_OK;
}

extern "C" int fnl_comm_create(fnl_context* ctx, const unsigned char id[128], int nranks, int rank,
                               fnl_comm** out) {
    if (!ctx || !id || !out) return fail(FNL_EINVAL, "fnl_comm_create: null argument");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(FNL_EINVAL, "fnl_comm_create: rank must be < nranks");
    *out = nullptr;
    NcclApi& a = api();
    if (!a.ok) return fail(FNL_ERUNTIME, a.error);
    int dev = 0;
    FNL_CUDA_TRY(cudaGetDevice(&dev));
    ncclUniqueId u;
    memcpy(&u, id, 128);
    ncclComm_t c = nullptr;
    const ncclResult_t r = a.comm_init_rank(&c, nranks, u, rank);  // collective over the ranks
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommInitRank");
    auto* fc = new fnl_comm();
    fc->comm = c;
    fc->nranks = nranks;
    fc->rank = rank;
    fc->device = dev;
    *out = fc;
    return FNL_OK;
}

extern "C" int fnl_comm_destroy(fnl_comm* comm) {
    if (!comm) return FNL_OK;
    NcclApi& a = api();
    const ncclResult_t r = a.ok ? a.comm_destroy(comm->comm) : ncclSuccess;
    delete comm;
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommDestroy");
    return FNL_OK;
}

extern "C" int fnl_comm_info(const fnl_comm* comm, int* nranks, int* rank, int* nccl_version) {
    if (!comm) return fail(FNL_EINVAL, "fnl_comm_info: null communicator");
    if (nranks) *nranks = comm->nranks;
    if (rank) *rank = comm->rank;
    if (nccl_version) {
        *nccl_version = 0;
        if (api().get_version) api().get_version(nccl_version);
    }
    return FNL_OK;
}

namespace fnl {
// in-place MIN all-reduce of int64 keys on `stream` (run_match's C5 step)
int comm_allreduce_min_i64(fnl_comm* comm, long long* d_keys, uint64_t count, cudaStream_t stream) {
    NcclApi& a = api();
    if (!a.ok) return fail(FNL_ERUNTIME, a.error);
    const ncclResult_t r = a.all_reduce(d_keys, d_keys, count, ncclInt64, ncclMin, comm->comm, stream);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
    return FNL_OK;
}
int comm_size(const fnl_comm* comm, int* nranks, int* rank) {
    *nranks = comm->nranks;
    *rank = comm->rank;
    return FNL_OK;
}
}  // namespace fnl
