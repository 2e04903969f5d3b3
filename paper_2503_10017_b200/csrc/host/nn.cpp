// nn.cpp -- L2 search entry points (reference src/nn.cpp surface).  Argument
// checks and messages follow the reference (src/nn.cpp:10-22); the search
// itself is one GPU scan whatever the backend, and the backend only selects
// the logical counter law reported on the FetchCounter.
#include "fastnn/nn.hpp"

#include <stdexcept>

#include "runtime.hpp"

namespace fastnn {

namespace {

void check_dims(std::uint32_t da, std::uint32_t db, const char* who) {
    if (da != db)
        throw std::invalid_argument(std::string(who) + ": descriptor dim mismatch (" + std::to_string(da) +
                                    " vs " + std::to_string(db) + ")");
}

void check_partition(const BlockPartition& part, std::uint32_t count, const char* who) {
    if (part.total_pixels != count)
        throw std::invalid_argument(std::string(who) + ": partition covers " +
                                    std::to_string(part.total_pixels) + " pixels but the map has " +
                                    std::to_string(count));
    if (part.ranges.empty()) throw std::invalid_argument(std::string(who) + ": empty partition");
}

int metric_code(DistanceMetric m) { return m == DistanceMetric::SquaredL2 ? FNL_METRIC_L2 : FNL_METRIC_DOT; }
int precision_code(PrecisionMode p) { return p == PrecisionMode::Hybrid ? FNL_PREC_HYBRID : FNL_PREC_FULL; }

NnResult run(DescriptorsView q, DescriptorsView t, DistanceMetric metric, PrecisionMode precision,
             int backend, std::uint32_t qb, std::uint32_t tb, FetchCounter* counter) {
    NnResult r;
    r.nearest.resize(q.count);
    r.min_dist.resize(q.count);
    std::uint64_t a = 0, b = 0, sat = 0;
    b200::check(fnl_nn_query(b200::context(), q.data, q.count, t.data, t.count, q.dim,
                             metric_code(metric), precision_code(precision), backend, qb, tb,
                             r.nearest.data(), r.min_dist.data(), &a, &b, &sat));
    if (counter) {
        counter->a_block_fetches.fetch_add(a, std::memory_order_relaxed);
        counter->b_block_fetches.fetch_add(b, std::memory_order_relaxed);
        if (sat) counter->half_saturation_events.fetch_add(sat, std::memory_order_relaxed);
    }
    return r;
}

}  // namespace

std::string to_string(NnBackend b) {
    switch (b) {
        case NnBackend::Bruteforce: return "bruteforce";
        case NnBackend::DoubleLoop: return "double";
        case NnBackend::SingleLoop: return "single";
        case NnBackend::HybridCast: return "hybrid";
        case NnBackend::Tensor: return "tensor";
    }
    return "?";
}

NnBackend backend_from_string(const std::string& s) {
    if (s == "bruteforce") return NnBackend::Bruteforce;
    if (s == "double") return NnBackend::DoubleLoop;
    if (s == "single") return NnBackend::SingleLoop;
    if (s == "hybrid") return NnBackend::HybridCast;
    if (s == "tensor") return NnBackend::Tensor;
    throw std::invalid_argument("unknown backend '" + s +
                                "' (expected bruteforce, double, single, hybrid or tensor)");
}

NnResult nn_query_bruteforce(DescriptorsView q, DescriptorsView t, DistanceMetric metric) {
    check_dims(q.dim, t.dim, "nn_bruteforce");
    if (!t.count) throw std::invalid_argument("nn_bruteforce: no target pixels");
    return run(q, t, metric, PrecisionMode::Full, FNL_BACKEND_BRUTEFORCE, 0, 0, nullptr);
}

NnResult nn_query_double_loop(DescriptorsView q, DescriptorsView t, const BlockPartition& pq,
                              const BlockPartition& pt, DistanceMetric metric, PrecisionMode precision,
                              FetchCounter& counter, unsigned /*threads*/) {
    check_dims(q.dim, t.dim, "nn_double_loop");
    check_partition(pq, q.count, "nn_double_loop(A)");
    check_partition(pt, t.count, "nn_double_loop(B)");
    return run(q, t, metric, precision, FNL_BACKEND_DOUBLE, pq.num_blocks(), pt.num_blocks(), &counter);
}

NnResult nn_query_single_loop(DescriptorsView q, DescriptorsView t, const BlockPartition& pq,
                              DistanceMetric metric, PrecisionMode precision, FetchCounter& counter,
                              unsigned /*threads*/) {
    check_dims(q.dim, t.dim, "nn_single_loop");
    check_partition(pq, q.count, "nn_single_loop(A)");
    if (!t.count) throw std::invalid_argument("nn_single_loop: no target pixels");
    return run(q, t, metric, precision, FNL_BACKEND_SINGLE, pq.num_blocks(), 0, &counter);
}

NnResult nn_query_tensor(DescriptorsView q, DescriptorsView t, DistanceMetric metric) {
    check_dims(q.dim, t.dim, "nn_tensor");
    if (!t.count) throw std::invalid_argument("nn_tensor: no target pixels");
    return run(q, t, metric, PrecisionMode::Hybrid, FNL_BACKEND_TENSOR, 0, 0, nullptr);
}

NnResult nn_bruteforce(const FeatureMap& A, const FeatureMap& B, DistanceMetric metric) {
    return nn_query_bruteforce(DescriptorsView::of(A), DescriptorsView::of(B), metric);
}

NnResult nn_double_loop(const FeatureMap& A, const FeatureMap& B, const BlockPartition& pa,
                        const BlockPartition& pb, DistanceMetric metric, PrecisionMode precision,
                        FetchCounter& counter, unsigned threads) {
    return nn_query_double_loop(DescriptorsView::of(A), DescriptorsView::of(B), pa, pb, metric,
                                precision, counter, threads);
}

NnResult nn_single_loop(const FeatureMap& A, const FeatureMap& B, const BlockPartition& pa,
                        DistanceMetric metric, PrecisionMode precision, FetchCounter& counter,
                        unsigned threads) {
    return nn_query_single_loop(DescriptorsView::of(A), DescriptorsView::of(B), pa, metric, precision,
                                counter, threads);
}

NnResult nn_hybridcast(const FeatureMap& A, const FeatureMap& B, const BlockPartition& pa,
                       DistanceMetric metric, FetchCounter& counter, unsigned threads) {
    return nn_single_loop(A, B, pa, metric, PrecisionMode::Hybrid, counter, threads);
}

}  // namespace fastnn
