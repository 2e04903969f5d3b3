// instrument.cpp -- RunReport renderings (reference contract docs/formats.md:72-91,
// golden zero report tests/acceptance.cpp:354-386).  One ordered field visitor
// drives JSON, CSV and parsing so the three can never drift apart.
#include "fastnn/instrument.hpp"

#include <algorithm>
#include <sstream>
#include <stdexcept>

#include <json.hpp>

namespace fastnn {

const char* const kRunReportCsvHeader =
    "backend,metric,precision,height1,width1,height2,width2,dim,k,grid_stride,max_iters,"
    "convergence_fraction,block_size,seed,subsample_us,forward_nn_us,reverse_nn_us,harvest_us,"
    "a_block_fetches,b_block_fetches,iterations,samples,converged,converged_fraction,"
    "half_saturated,half_saturation_events,hybrid_full_argmin_agreement,matches_emitted,"
    "duplicates_dropped";

namespace {

// Calls v(name, member) for every scalar field in contract order.
template <typename R, typename V>
void visit_fields(R& r, V&& v) {
    v("backend", r.backend);
    v("metric", r.metric);
    v("precision", r.precision);
    v("height1", r.height1);
    v("width1", r.width1);
    v("height2", r.height2);
    v("width2", r.width2);
    v("dim", r.dim);
    v("k", r.k);
    v("grid_stride", r.grid_stride);
    v("max_iters", r.max_iters);
    v("convergence_fraction", r.convergence_fraction);
    v("block_size", r.block_size);
    v("seed", r.seed);
    v("subsample_us", r.subsample_us);
    v("forward_nn_us", r.forward_nn_us);
    v("reverse_nn_us", r.reverse_nn_us);
    v("harvest_us", r.harvest_us);
    v("a_block_fetches", r.a_block_fetches);
    v("b_block_fetches", r.b_block_fetches);
    v("iterations", r.iterations);
    v("samples", r.samples);
    v("converged", r.converged);
    v("converged_fraction", r.converged_fraction);
    v("half_saturated", r.half_saturated);
    v("half_saturation_events", r.half_saturation_events);
    v("hybrid_full_argmin_agreement", r.hybrid_full_argmin_agreement);
    v("matches_emitted", r.matches_emitted);
    v("duplicates_dropped", r.duplicates_dropped);
}

constexpr const char* kAgreement = "hybrid_full_argmin_agreement";

}  // namespace

std::string render_report(const RunReport& r, ReportFormat format) {
    if (format == ReportFormat::Json) {
        nlohmann::ordered_json j;
        visit_fields(r, [&](const char* name, const auto& value) {
            if constexpr (std::is_same_v<std::decay_t<decltype(value)>, double>) {
                if (std::string(name) == kAgreement && value < 0.0) {
                    j[name] = nullptr;
                    return;
                }
            }
            j[name] = value;
        });
        j["active_history"] = r.active_history;
        return j.dump(2) + "\n";
    }
    std::ostringstream head, row;
    bool first = true;
    visit_fields(r, [&](const char* name, const auto& value) {
        if (!first) row << ',';
        first = false;
        using T = std::decay_t<decltype(value)>;
        if constexpr (std::is_same_v<T, bool>) {
            row << (value ? 1 : 0);
        } else if constexpr (std::is_same_v<T, double>) {
            if (!(std::string(name) == kAgreement && value < 0.0)) row << value;
        } else {
            row << value;
        }
    });
    return std::string(kRunReportCsvHeader) + "\n" + row.str() + "\n";
}

RunReport parse_report_json(const std::string& text) {
    const auto j = nlohmann::json::parse(text);
    RunReport r;
    visit_fields(r, [&](const char* name, auto& value) {
        using T = std::decay_t<decltype(value)>;
        const auto& node = j.at(name);
        if constexpr (std::is_same_v<T, double>) {
            value = node.is_null() ? -1.0 : node.get<double>();
        } else {
            value = node.get<T>();
        }
    });
    r.active_history = j.at("active_history").get<std::vector<std::uint32_t>>();
    return r;
}

double argmin_agreement(std::span<const std::uint32_t> a, std::span<const std::uint32_t> b) {
    if (a.size() != b.size())
        throw std::invalid_argument("argmin_agreement: arrays must have equal length");
    if (a.empty()) return 1.0;
    std::size_t same = 0;
    for (std::size_t i = 0; i < a.size(); ++i) same += a[i] == b[i];
    return static_cast<double>(same) / static_cast<double>(a.size());
}

double median(std::vector<double> v) {
    if (v.empty()) throw std::invalid_argument("median: empty sample");
    const std::size_t n = v.size(), mid = n / 2;
    std::nth_element(v.begin(), v.begin() + mid, v.end());
    if (n % 2) return v[mid];
    const double hi = v[mid];
    const double lo = *std::max_element(v.begin(), v.begin() + mid);
    return 0.5 * (lo + hi);
}

}  // namespace fastnn
