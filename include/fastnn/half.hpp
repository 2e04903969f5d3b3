// fastnn/half.hpp -- binary16 conversion contract (drop-in for ref half.hpp).
//
// Round to nearest even; |x| >= 65520 and infinities clamp to +-65504 and set
// *saturated (never fatal); NaN becomes the canonical quiet NaN; -0 survives.
#pragma once

#include <cstdint>

namespace fastnn {

std::uint16_t float_to_half_bits(float x, bool* saturated = nullptr);
float half_bits_to_float(std::uint16_t h);
float to_half_round(float x);
float to_half_round(float x, bool& saturated);

inline constexpr float kHalfMax = 65504.0f;

}  // namespace fastnn
