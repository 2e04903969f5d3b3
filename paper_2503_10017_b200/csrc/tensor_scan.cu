// tensor_scan.cu -- placeholder until the tcgen05 kernel lands.
#include "fastnn_b200.h"
#include "fnl_internal.h"
#include "tensor_scan.h"

namespace fnl {
int tensor_nn_dense(fnl_context*, const float*, uint32_t, const float*, uint32_t, uint32_t, bool,
                    uint32_t*, float*) {
    return fail(FNL_ERUNTIME, "tensor backend not built yet");
}
int tensor_nn_gathered(fnl_context*, uint32_t, const float*, uint64_t, const uint32_t*, uint32_t,
                       const uint32_t*, const uint8_t*, const float*, uint64_t, uint32_t, uint32_t,
                       bool, uint32_t*, uint32_t) {
    return fail(FNL_ERUNTIME, "tensor backend not built yet");
}
uint64_t tensor_near_tie_rows(fnl_context*, uint32_t) { return 0; }
}  // namespace fnl
