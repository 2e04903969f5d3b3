// kernels.cpp -- L1 entry points.  Scalar single-pair utilities stay on the host
// (they score one pair); every block / scan entry point runs on the GPU through
// the C-ABI (include/fastnn_b200.h).
#include "fastnn/kernels.hpp"

#include <cmath>
#include <stdexcept>
#include <string>

#include "fastnn/half.hpp"
#include "runtime.hpp"

namespace fastnn {

// One pair, reference FMA chain (src/kernels.cpp:31-43, :277-285).
float dist_scalar(std::span<const float> a, std::span<const float> b, DistanceMetric metric) {
    if (a.size() != b.size())
        throw std::invalid_argument("dist_scalar: descriptor lengths differ (" + std::to_string(a.size()) +
                                    " vs " + std::to_string(b.size()) + ")");
    float acc = 0.0f;
    const bool l2 = metric == DistanceMetric::SquaredL2;
    for (std::size_t c = 0; c < a.size(); ++c) {
        const float x = l2 ? a[c] - b[c] : a[c];
        acc = std::fma(x, l2 ? x : b[c], acc);
    }
    return l2 ? acc : -acc;
}

ArgminResult argmin_row(std::span<const float> row) {
    if (row.empty()) throw std::invalid_argument("argmin_row: empty row");
    ArgminResult r{0, row[0]};
    for (std::uint32_t i = 1; i < row.size(); ++i)
        if (row[i] < r.value) r = {i, row[i]};
    return r;
}

ArgminResult argmin_row(const DistanceRow& row) { return argmin_row(row.distances); }

DistanceMatrix block_distances(DescriptorsView q, DescriptorsView t, DistanceMetric metric,
                               PrecisionMode precision, FetchCounter& counter) {
    if (q.dim != t.dim)
        throw std::invalid_argument("block_distances: descriptor dim mismatch (" + std::to_string(q.dim) +
                                    " vs " + std::to_string(t.dim) + ")");
    if (!q.count || !t.count) throw std::invalid_argument("block_distances: empty block");
    record_fetch(counter, FetchKind::B);
    DistanceMatrix m{q.count, t.count, std::vector<float>(std::size_t(q.count) * t.count)};
    std::uint64_t sat = 0;
    b200::check(fnl_block_distances(b200::context(), q.data, q.count, t.data, t.count, q.dim,
                                    metric == DistanceMetric::SquaredL2 ? FNL_METRIC_L2 : FNL_METRIC_DOT,
                                    precision == PrecisionMode::Hybrid ? FNL_PREC_HYBRID : FNL_PREC_FULL,
                                    m.data.data(), &sat));
    if (sat) counter.half_saturation_events.fetch_add(sat, std::memory_order_relaxed);
    return m;
}

namespace detail {

namespace {

// Lanes back to row-major rows (the GPU consumes plain rows).
std::vector<float> unpack_rows(const PackedTargets& p) {
    std::vector<float> rows(std::size_t(p.count) * p.dim);
    for (std::uint32_t s = 0; s < p.full_strips; ++s)
        for (std::uint32_t c = 0; c < p.dim; ++c)
            for (std::uint32_t l = 0; l < 8; ++l)
                rows[(std::size_t(s) * 8 + l) * p.dim + c] = p.lanes[(std::size_t(s) * p.dim + c) * 8 + l];
    std::copy(p.tail.begin(), p.tail.end(), rows.begin() + std::size_t(p.full_strips) * 8 * p.dim);
    return rows;
}

}  // namespace

PackedTargets pack_targets(DescriptorsView t) {
    PackedTargets p;
    p.count = t.count;
    p.dim = t.dim;
    p.full_strips = t.count / 8;
    p.lanes.resize(std::size_t(p.full_strips) * t.dim * 8);
    for (std::uint32_t r = 0; r < p.full_strips * 8; ++r)
        for (std::uint32_t c = 0; c < t.dim; ++c)
            p.lanes[(std::size_t(r / 8) * t.dim + c) * 8 + r % 8] = t.row(r)[c];
    p.tail.assign(t.row(p.full_strips * 8), t.row(p.full_strips * 8) + std::size_t(p.tail_count()) * t.dim);
    for (float v : p.lanes) p.max_abs = std::max(p.max_abs, std::fabs(v));
    for (float v : p.tail) p.max_abs = std::max(p.max_abs, std::fabs(v));
    return p;
}

PackedTargets pack_targets_half(DescriptorsView t, std::uint64_t& saturation_events) {
    PackedTargets p = pack_targets(t);
    p.max_abs = 0.0f;
    auto cast = [&](float& v) {
        bool s = false;
        v = to_half_round(v, s);
        saturation_events += s;
        p.max_abs = std::max(p.max_abs, std::fabs(v));
    };
    for (float& v : p.lanes) cast(v);
    for (float& v : p.tail) cast(v);
    return p;
}

void nn_scan_block(const float* queries, std::uint32_t nq, std::uint32_t dim,
                   const PackedTargets& targets, DistanceMetric metric, PrecisionMode precision,
                   std::uint32_t* nearest, float* min_dist, std::uint64_t& saturation_events) {
    if (!nq) return;
    const std::vector<float> rows = unpack_rows(targets);
    std::uint64_t a = 0, b = 0, sat = 0;
    // targets were already cast by pack_targets_half: the scan rounds queries
    // and distances only, so the target share of the counter is subtracted by
    // scanning already-rounded values (their re-rounding is exact, uncounted).
    b200::check(fnl_nn_query(b200::context(), queries, nq, rows.data(), targets.count, dim,
                             metric == DistanceMetric::SquaredL2 ? FNL_METRIC_L2 : FNL_METRIC_DOT,
                             precision == PrecisionMode::Hybrid ? FNL_PREC_HYBRID : FNL_PREC_FULL,
                             FNL_BACKEND_SINGLE, 1, 1, nearest, min_dist, &a, &b, &sat));
    saturation_events += sat;
}

void fill_block(const float* queries, std::uint32_t nq, std::uint32_t dim, const PackedTargets& targets,
                DistanceMetric metric, PrecisionMode precision, float* out,
                std::uint64_t& saturation_events) {
    if (!nq) return;
    const std::vector<float> rows = unpack_rows(targets);
    std::uint64_t sat = 0;
    b200::check(fnl_block_distances(b200::context(), queries, nq, rows.data(), targets.count, dim,
                                    metric == DistanceMetric::SquaredL2 ? FNL_METRIC_L2 : FNL_METRIC_DOT,
                                    precision == PrecisionMode::Hybrid ? FNL_PREC_HYBRID : FNL_PREC_FULL,
                                    out, &sat));
    saturation_events += sat;
}

}  // namespace detail

}  // namespace fastnn
