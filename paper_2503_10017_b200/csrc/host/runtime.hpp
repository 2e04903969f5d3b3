// runtime.hpp -- glue between the drop-in C++ API and the C-ABI.
//
// Each calling thread owns one fnl_context (GPU + stream + workspace), so
// concurrent callers never share device state.  C-ABI status
// codes become the reference's exception classes.
#pragma once

#include <stdexcept>
#include <string>

#include "fastnn/reciprocal.hpp"
#include "fastnn_b200.h"

namespace fastnn::b200 {

// Context of the calling thread on the selected device (FASTNN_DEVICE env or
// set_device(), default 0).  Throws std::runtime_error when no GPU is usable:
// there is no CPU fallback.
fnl_context* context();
void set_device(int device);
int current_device();

// reciprocal_match over raw row-major buffers (no FeatureMap copy); the
// FeatureMap overload and the Python binding both land here.
MatchOutcome reciprocal_match_raw(const float* d1, std::uint32_t h1, std::uint32_t w1, const float* d2,
                                  std::uint32_t h2, std::uint32_t w2, std::uint32_t dim1,
                                  std::uint32_t dim2, const MatchConfig& cfg, NnBackend backend);

inline void check(int status) {
    if (status == FNL_OK) return;
    const std::string msg = fnl_last_error();
    if (status == FNL_EINVAL) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}

}  // namespace fastnn::b200
