// tensor_scan.h -- K3: tcgen05 HybridCast score + certified argmax (tensor_scan.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

struct fnl_context;

namespace fnl {

// Dense: every row of d_q (nq x dim fp32) against d_t (nt x dim fp32).
int tensor_nn_dense(fnl_context* ctx, const float* d_q, uint32_t nq, const float* d_t, uint32_t nt,
                    uint32_t dim, bool l2, uint32_t* d_nearest, float* d_min_dist);

// Gathered, batched over pairs, driven by the matcher state: queries of pair p
// are rows ids[p*cap + i] (i < n_active[p]) of qmap + p*q_stride; pairs with
// done[p] are skipped.  Winners land in out[p*out_stride + i].
int tensor_nn_gathered(fnl_context* ctx, uint32_t npairs, const float* qmap, uint64_t q_stride,
                       const uint32_t* ids, uint32_t cap, const uint32_t* n_active,
                       const uint8_t* done, const float* tmap, uint64_t t_stride, uint32_t nt,
                       uint32_t dim, bool l2, uint32_t* out, uint32_t out_stride);

// Rows of pair p re-decided by the exact chain since the matcher started.
uint64_t tensor_near_tie_rows(fnl_context* ctx, uint32_t pair);

}  // namespace fnl
