// fnl_common.cuh -- shared device helpers of the FastNN-Lite sm_100a kernels.
//
// Numeric contract (reference /root/reference/proj):
//  * per-pair distance = fmaf chain over channels in order, dot negated
//    (src/kernels.cpp:31-43); kernels are built with --fmad=false and use
//    __fmaf_rn explicitly so nvcc fuses nothing else;
//  * binary16 rounding = RNE, |x| >= 65520 clamps to +-65504 and is counted
//    (src/half.cpp:15-47); cvt.rn.f16.f32 would overflow to inf instead;
//  * argmin = strict <, lowest index on exact ties, order independent
//    (src/kernels.cpp:287-300, :202-229).  We realise it as a min over packed
//    64-bit keys (orderable(dist) << 32 | index), which is associative and
//    commutative, so any CTA split or atomic order gives the same answer.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace fnl {

constexpr float kHalfMax = 65504.0f;
constexpr float kHalfOverflow = 65520.0f;

// binary16 round trip with the reference's saturation rule.
__device__ __forceinline__ float half_round_sat(float x, uint32_t& sat) {
    // branch-free (selects), so it stays if-converted inside unrolled scans
    const bool over = fabsf(x) >= kHalfOverflow;  // false for NaN
    sat += over ? 1u : 0u;
    const float r = __half2float(__float2half_rn(x));
    return over ? copysignf(kHalfMax, x) : r;
}
__device__ __forceinline__ float half_round_nosat(float x) {
    return __half2float(__float2half_rn(x));
}

// Monotone map float -> u32 (total order matching <, with -0 == +0 and NaN
// treated as +inf so it can never displace a real candidate).
__device__ __forceinline__ uint32_t orderable(float d) {
    uint32_t b = __float_as_uint(d);
    if ((b & 0x7FFFFFFFu) > 0x7F800000u) b = 0x7F800000u;  // NaN -> +inf
    if (b == 0x80000000u) b = 0u;                           // -0 -> +0
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__device__ __host__ __forceinline__ float from_orderable(uint32_t o) {
    uint32_t b = (o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o;
#ifdef __CUDA_ARCH__
    return __uint_as_float(b);
#else
    float f;
    __builtin_memcpy(&f, &b, 4);
    return f;
#endif
}
__device__ __forceinline__ uint64_t pack_key(float d, uint32_t idx) {
    return (static_cast<uint64_t>(orderable(d)) << 32) | idx;
}

// Reference per-pair chain over `dim` channels (src/kernels.cpp:31-43).
template <bool kL2>
__device__ __forceinline__ float chain(const float* __restrict__ a, const float* __restrict__ b,
                                       uint32_t dim) {
    float acc = 0.0f;
    for (uint32_t c = 0; c < dim; ++c) {
        if constexpr (kL2) {
            const float d = __fsub_rn(a[c], b[c]);
            acc = __fmaf_rn(d, d, acc);
        } else {
            acc = __fmaf_rn(a[c], b[c], acc);
        }
    }
    return kL2 ? acc : -acc;
}

__device__ __forceinline__ uint32_t warp_sum(uint32_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

}  // namespace fnl

#define FNL_CUDA_TRY(expr)                                                        \
    do {                                                                          \
        cudaError_t _e = (expr);                                                  \
        if (_e != cudaSuccess) return ::fnl::fail_cuda(_e, #expr, __FILE__, __LINE__); \
    } while (0)
