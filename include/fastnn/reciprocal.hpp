// fastnn/reciprocal.hpp -- L3 iterative reciprocal matcher (drop-in for ref
// reciprocal.hpp).  The whole loop (NN queries, cycle check, harvest,
// compaction, termination) runs on the GPU; see DESIGN.md.
#pragma once

#include <cstdint>
#include <vector>

#include "fastnn/core.hpp"
#include "fastnn/instrument.hpp"
#include "fastnn/nn.hpp"

namespace fastnn {

// Centred row-major grid, one sample per stride x stride cell (stride 0: derived
// from k as round(sqrt(H*W/k))); std::invalid_argument when both are zero.
std::vector<PixelId> grid_subsample(const FeatureMap& map, std::uint32_t k, std::uint32_t stride);

// Exhaustive mutual nearest neighbours, lowest-index ties.
MatchSet mutual_nn_exact(const FeatureMap& D1, const FeatureMap& D2, DistanceMetric metric);

struct MatcherState {
    std::uint32_t iteration = 0;
    std::vector<std::uint32_t> active_u;
    std::vector<std::uint32_t> active_v;
    MatchSet collected;
    std::uint32_t converged_count = 0;
};

struct MatchOutcome {
    MatchSet matches;
    RunReport report;
};

MatchOutcome reciprocal_match(const FeatureMap& D1, const FeatureMap& D2, const MatchConfig& cfg,
                              NnBackend backend, unsigned threads = 1);

}  // namespace fastnn
