// reciprocal.cpp -- L3 entry points (reference src/reciprocal.cpp surface).
// grid_subsample is index arithmetic returned to the caller; the matcher and
// the exhaustive mutual search run on the GPU (match_loop.cu / exact_scan.cu /
// tensor_scan.cu) through the C-ABI.
#include "fastnn/reciprocal.hpp"

#include <cmath>
#include <cstring>

#include "fastnn/sharded.hpp"
#include <stdexcept>

#include "runtime.hpp"

namespace fastnn {

namespace {

std::vector<std::uint32_t> axis(std::uint32_t extent, std::uint32_t stride) {
    const std::uint32_t n = (extent + stride - 1) / stride;
    if (n == 1) return {extent / 2};
    std::vector<std::uint32_t> pos(n);
    for (std::uint32_t i = 0; i < n; ++i) pos[i] = std::min(stride / 2 + i * stride, extent - 1);
    return pos;
}

int metric_code(DistanceMetric m) { return m == DistanceMetric::SquaredL2 ? FNL_METRIC_L2 : FNL_METRIC_DOT; }

int backend_code(NnBackend b) {
    switch (b) {
        case NnBackend::Bruteforce: return FNL_BACKEND_BRUTEFORCE;
        case NnBackend::DoubleLoop: return FNL_BACKEND_DOUBLE;
        case NnBackend::SingleLoop: return FNL_BACKEND_SINGLE;
        case NnBackend::HybridCast: return FNL_BACKEND_HYBRIDCAST;
        case NnBackend::Tensor: return FNL_BACKEND_TENSOR;
    }
    throw std::invalid_argument("reciprocal_match: unknown backend");
}

}  // namespace

std::vector<PixelId> grid_subsample(const FeatureMap& map, std::uint32_t k, std::uint32_t stride) {
    if (!stride) {
        if (!k) throw std::invalid_argument("grid_subsample: one of k or stride must be >= 1");
        const double cells = double(map.pixel_count()) / double(k);
        stride = std::max<std::uint32_t>(1, static_cast<std::uint32_t>(std::lround(std::sqrt(cells))));
    }
    std::vector<PixelId> ids;
    const auto rows = axis(map.height, stride), cols = axis(map.width, stride);
    ids.reserve(rows.size() * cols.size());
    for (std::uint32_t h : rows)
        for (std::uint32_t w : cols) ids.push_back(pixel_id_from_coord({w, h}, map.width));
    return ids;
}

MatchSet mutual_nn_exact(const FeatureMap& D1, const FeatureMap& D2, DistanceMetric metric) {
    if (D1.dim != D2.dim)
        throw std::invalid_argument("mutual_nn_exact: descriptor dim mismatch (" + std::to_string(D1.dim) +
                                    " vs " + std::to_string(D2.dim) + ")");
    std::vector<std::uint32_t> flat(2 * std::size_t(D1.pixel_count()) + 2);
    std::uint32_t n = 0;
    b200::check(fnl_mutual_nn(b200::context(), D1.data.data(), D1.height, D1.width, D2.data.data(),
                              D2.height, D2.width, D1.dim, metric_code(metric), flat.data(), &n));
    MatchSet out;
    out.pairs.reserve(n);
    for (std::uint32_t k = 0; k < n; ++k) out.pairs.push_back({flat[2 * k], flat[2 * k + 1], 0});
    return out;
}

MatchOutcome reciprocal_match(const FeatureMap& D1, const FeatureMap& D2, const MatchConfig& cfg,
                              NnBackend backend, unsigned /*threads*/) {
    return b200::reciprocal_match_raw(D1.data.data(), D1.height, D1.width, D2.data.data(), D2.height,
                                      D2.width, D1.dim, D2.dim, cfg, backend);
}

namespace {

// MatchOutcome from the C-ABI outputs: the MatchSet in harvest order and the
// RunReport, field for field as src/reciprocal.cpp:105-111, :195-205 fill it
MatchOutcome make_outcome(const std::vector<std::uint32_t>& flat, std::uint32_t n, const fnl_run_stats& st,
                          std::uint32_t h1, std::uint32_t w1, std::uint32_t h2, std::uint32_t w2,
                          std::uint32_t dim, const MatchConfig& cfg, NnBackend backend) {
    MatchOutcome out;
    out.matches.pairs.reserve(n);
    for (std::uint32_t k = 0; k < n; ++k)
        out.matches.pairs.push_back({flat[3 * k], flat[3 * k + 1], flat[3 * k + 2]});
    RunReport& r = out.report;
    const bool hybrid = backend == NnBackend::HybridCast || backend == NnBackend::Tensor ||
                        (backend != NnBackend::Bruteforce && cfg.precision == PrecisionMode::Hybrid);
    r.backend = to_string(backend);
    r.metric = to_string(cfg.metric);
    r.precision = hybrid ? "hybrid" : "full";
    r.height1 = h1;
    r.width1 = w1;
    r.height2 = h2;
    r.width2 = w2;
    r.dim = dim;
    r.k = cfg.k;
    r.grid_stride = cfg.grid_stride;
    r.max_iters = cfg.max_iters;
    r.convergence_fraction = cfg.convergence_fraction;
    r.block_size = cfg.block_size;
    r.subsample_us = st.subsample_us;
    r.forward_nn_us = st.forward_nn_us;
    r.reverse_nn_us = st.reverse_nn_us;
    r.harvest_us = st.harvest_us;
    r.samples = st.samples;
    r.iterations = st.iterations;
    r.converged = st.converged;
    r.converged_fraction = st.samples ? double(st.converged) / st.samples : 0.0;
    r.a_block_fetches = st.a_block_fetches;
    r.b_block_fetches = st.b_block_fetches;
    r.half_saturation_events = st.half_saturation_events;
    r.half_saturated = st.half_saturation_events > 0;
    r.matches_emitted = n;
    r.duplicates_dropped = st.duplicates_dropped;
    r.active_history.assign(st.active_history, st.active_history + st.history_len);
    return out;
}

fnl_match_config c_config(const MatchConfig& cfg) {
    return fnl_match_config{cfg.k, cfg.grid_stride, cfg.max_iters, cfg.convergence_fraction,
                            metric_code(cfg.metric),
                            cfg.precision == PrecisionMode::Hybrid ? FNL_PREC_HYBRID : FNL_PREC_FULL,
                            cfg.block_size};
}

}  // namespace

MatchOutcome b200::reciprocal_match_raw(const float* d1, std::uint32_t h1, std::uint32_t w1,
                                        const float* d2, std::uint32_t h2, std::uint32_t w2,
                                        std::uint32_t dim1, std::uint32_t dim2, const MatchConfig& cfg,
                                        NnBackend backend) {
    cfg.validate();
    if (dim1 != dim2)
        throw std::invalid_argument("reciprocal_match: descriptor dim mismatch (" + std::to_string(dim1) +
                                    " vs " + std::to_string(dim2) + ")");
    const std::uint32_t dim = dim1;
    const FeatureMap D1shape(h1, w1, 1);
    const fnl_match_config c = c_config(cfg);
    const std::size_t samples = grid_subsample(D1shape, cfg.k, cfg.grid_stride).size();
    std::vector<std::uint32_t> flat(3 * std::max<std::size_t>(samples, 1));
    std::uint32_t n = 0;
    fnl_run_stats st{};
    b200::check(fnl_reciprocal_match(b200::context(), d1, h1, w1, d2, h2, w2, dim, &c, backend_code(backend),
                                     flat.data(), &n, &st));
    return make_outcome(flat, n, st, h1, w1, h2, w2, dim, cfg, backend);
}

// ---------------------------------------------------------------- C5 extension
NcclCommunicator::Id NcclCommunicator::unique_id() {
    Id id{};
    b200::check(fnl_nccl_unique_id(id.data()));
    return id;
}

NcclCommunicator::NcclCommunicator(const Id& id, int nranks, int rank) : nranks_(nranks), rank_(rank) {
    b200::check(fnl_comm_create(b200::context(), id.data(), nranks, rank, &comm_));
}

NcclCommunicator::~NcclCommunicator() { fnl_comm_destroy(comm_); }

MatchOutcome reciprocal_match_sharded(const FeatureMap& D1, const FeatureMap& D2, const MatchConfig& cfg,
                                      NnBackend backend, const NcclCommunicator& comm) {
    cfg.validate();
    if (D1.dim != D2.dim)
        throw std::invalid_argument("reciprocal_match: descriptor dim mismatch (" + std::to_string(D1.dim) +
                                    " vs " + std::to_string(D2.dim) + ")");
    const fnl_match_config c = c_config(cfg);
    const std::size_t samples = grid_subsample(D1, cfg.k, cfg.grid_stride).size();
    std::vector<std::uint32_t> flat(3 * std::max<std::size_t>(samples, 1));
    std::uint32_t n = 0;
    fnl_run_stats st{};
    b200::check(fnl_reciprocal_match_sharded(b200::context(), comm.handle(), D1.data.data(), D1.height, D1.width,
                                             D2.data.data(), D2.height, D2.width, D1.dim, &c,
                                             backend_code(backend), flat.data(), &n, &st));
    return make_outcome(flat, n, st, D1.height, D1.width, D2.height, D2.width, D1.dim, cfg, backend);
}

}  // namespace fastnn
