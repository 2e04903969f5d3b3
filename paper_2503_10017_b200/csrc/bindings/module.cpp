// module.cpp -- the `_fastnn` Python surface (drop-in for the reference
// bindings/module.cpp:64-260): the same 14 functions, argument names, defaults,
// dtypes, return shapes and dict keys, plus batch / device-resident entry points
// and instrumentation.  GPU work runs with the GIL released.
#include <array>
#include <pybind11/numpy.h>
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include <cstring>

#include "fastnn/half.hpp"
#include "fastnn/instrument.hpp"
#include "fastnn/io.hpp"
#include "fastnn/kernels.hpp"
#include "fastnn/nn.hpp"
#include "fastnn/reciprocal.hpp"
#include "runtime.hpp"

namespace py = pybind11;
using F32 = py::array_t<float, py::array::c_style | py::array::forcecast>;
using U32Array = py::array_t<std::uint32_t>;

namespace {

fastnn::FeatureMap to_map(const F32& a) {
    if (a.ndim() != 3) throw std::invalid_argument("feature map must have shape (H, W, d)");
    return fastnn::FeatureMap::from_data(static_cast<std::uint32_t>(a.shape(0)),
                                         static_cast<std::uint32_t>(a.shape(1)),
                                         static_cast<std::uint32_t>(a.shape(2)),
                                         std::vector<float>(a.data(), a.data() + a.size()));
}

py::array from_map(const fastnn::FeatureMap& m) {
    py::array_t<float> a({py::ssize_t(m.height), py::ssize_t(m.width), py::ssize_t(m.dim)});
    std::memcpy(a.mutable_data(), m.data.data(), m.data.size() * sizeof(float));
    return a;
}

template <typename T>
py::array_t<T> vec_array(const std::vector<T>& v) {
    py::array_t<T> a(py::ssize_t(v.size()));
    if (!v.empty()) std::memcpy(a.mutable_data(), v.data(), v.size() * sizeof(T));
    return a;
}

py::dict nn_dict(const fastnn::NnResult& r, const fastnn::FetchCounter& c) {
    py::dict d;
    d["nearest"] = vec_array(r.nearest);
    d["min_dist"] = vec_array(r.min_dist);
    d["a_block_fetches"] = c.a_fetches();
    d["b_block_fetches"] = c.b_fetches();
    d["half_saturation_events"] = c.saturations();
    return d;
}

fastnn::MatchConfig make_cfg(std::uint32_t k, std::uint32_t stride, std::uint32_t max_iters,
                             double convergence, const std::string& metric,
                             const std::string& precision, std::uint32_t block_size) {
    fastnn::MatchConfig cfg;
    cfg.k = k;
    cfg.grid_stride = k > 0 ? 0 : stride;  // bindings/module.cpp:236
    cfg.max_iters = max_iters;
    cfg.convergence_fraction = convergence;
    cfg.metric = fastnn::metric_from_string(metric);
    cfg.precision = fastnn::precision_from_string(precision);
    cfg.block_size = block_size;
    return cfg;
}

fnl_match_config c_cfg(const fastnn::MatchConfig& c) {
    return {c.k, c.grid_stride, c.max_iters, c.convergence_fraction,
            c.metric == fastnn::DistanceMetric::SquaredL2 ? FNL_METRIC_L2 : FNL_METRIC_DOT,
            c.precision == fastnn::PrecisionMode::Hybrid ? FNL_PREC_HYBRID : FNL_PREC_FULL,
            c.block_size};
}

int c_backend(fastnn::NnBackend b) {
    switch (b) {
        case fastnn::NnBackend::Bruteforce: return FNL_BACKEND_BRUTEFORCE;
        case fastnn::NnBackend::DoubleLoop: return FNL_BACKEND_DOUBLE;
        case fastnn::NnBackend::SingleLoop: return FNL_BACKEND_SINGLE;
        case fastnn::NnBackend::HybridCast: return FNL_BACKEND_HYBRIDCAST;
        case fastnn::NnBackend::Tensor: return FNL_BACKEND_TENSOR;
    }
    return FNL_BACKEND_SINGLE;
}

py::dict stats_dict(const fnl_run_stats& s) {
    py::dict d;
    d["samples"] = s.samples;
    d["iterations"] = s.iterations;
    d["converged"] = s.converged;
    d["duplicates_dropped"] = s.duplicates_dropped;
    d["matches"] = s.matches;
    d["active_history"] = std::vector<std::uint32_t>(s.active_history, s.active_history + s.history_len);
    d["a_block_fetches"] = s.a_block_fetches;
    d["b_block_fetches"] = s.b_block_fetches;
    d["half_saturation_events"] = s.half_saturation_events;
    d["near_tie_rows"] = s.near_tie_rows;
    d["rescan_rows"] = s.rescan_rows;
    d["tensor_route"] = s.tensor_route;
    d["computed_query_rows"] = s.computed_query_rows;
    d["query_rows"] = s.query_rows;
    d["forward_nn_us"] = s.forward_nn_us;
    d["reverse_nn_us"] = s.reverse_nn_us;
    d["harvest_us"] = s.harvest_us;
    return d;
}

void check_shape3(const F32& a, const char* who) {
    if (a.ndim() != 3) throw std::invalid_argument(std::string(who) + ": feature map must have shape (H, W, d)");
    if (a.shape(0) == 0 || a.shape(1) == 0 || a.shape(2) == 0)
        throw std::invalid_argument("FeatureMap: height, width and dim must all be >= 1");
}

}  // namespace

// `stream` arguments: None = the library's own stream; otherwise a CUDA
// stream handle as torch reports it (torch.cuda.Stream.cuda_stream), where 0
// is the legacy default stream (cudaStreamLegacy == (cudaStream_t)0x1), not
// "no stream" -- so work is ordered with torch's current stream.
static void* stream_handle(const py::object& s) {
    if (s.is_none()) return nullptr;
    const auto h = s.cast<std::uintptr_t>();
    return h == 0 ? reinterpret_cast<void*>(std::uintptr_t(1)) : reinterpret_cast<void*>(h);
}

PYBIND11_MODULE(_fastnn, m) {
    m.doc() = "B200-native fast reciprocal nearest-neighbour matching (FastNN-Lite / HybridCast)";

    m.def("gen_random",
          [](std::uint32_t h, std::uint32_t w, std::uint32_t d, std::uint64_t seed, bool normalize) {
              return from_map(fastnn::gen_random(h, w, d, seed, normalize));
          },
          py::arg("height"), py::arg("width"), py::arg("dim"), py::arg("seed"), py::arg("normalize") = true);

    m.def("gen_matched_pair",
          [](std::uint32_t h, std::uint32_t w, std::uint32_t d, std::uint64_t seed, double sigma,
             const std::string& permute) {
              const auto p = fastnn::gen_matched_pair(h, w, d, seed, sigma, fastnn::permute_from_string(permute));
              py::dict out;
              out["d1"] = from_map(p.d1);
              out["d2"] = from_map(p.d2);
              out["truth"] = vec_array(p.truth.map);
              out["noise_sigma"] = p.truth.noise_sigma;
              out["permute"] = permute;
              return out;
          },
          py::arg("height"), py::arg("width"), py::arg("dim"), py::arg("seed"),
          py::arg("noise_sigma") = 0.0, py::arg("permute") = "random");

    m.def("write_fmap", [](const F32& a, const std::string& path) { fastnn::save_fmap(to_map(a), path); },
          py::arg("map"), py::arg("path"));
    m.def("read_fmap", [](const std::string& path) { return from_map(fastnn::load_fmap(path)); },
          py::arg("path"));

    m.def("dist_scalar",
          [](const std::vector<float>& a, const std::vector<float>& b, const std::string& metric) {
              return fastnn::dist_scalar(a, b, fastnn::metric_from_string(metric));
          },
          py::arg("a"), py::arg("b"), py::arg("metric") = "l2");

    m.def("to_half_round", [](float x) { return fastnn::to_half_round(x); }, py::arg("x"),
          "nearest binary16 value, round to nearest even, widened back to float32");

    m.def("block_distances",
          [](const F32& q, const F32& t, const std::string& metric, const std::string& precision) {
              if (q.ndim() != 2 || t.ndim() != 2)
                  throw std::invalid_argument("block_distances expects 2-D (n, d) arrays");
              const fastnn::DescriptorsView qv{q.data(), std::uint32_t(q.shape(0)), std::uint32_t(q.shape(1))};
              const fastnn::DescriptorsView tv{t.data(), std::uint32_t(t.shape(0)), std::uint32_t(t.shape(1))};
              const auto mt = fastnn::metric_from_string(metric);
              const auto pr = fastnn::precision_from_string(precision);
              fastnn::FetchCounter c;
              fastnn::DistanceMatrix dm;
              {
                  py::gil_scoped_release nogil;
                  dm = fastnn::block_distances(qv, tv, mt, pr, c);
              }
              py::array_t<float> out({py::ssize_t(dm.rows), py::ssize_t(dm.cols)});
              std::memcpy(out.mutable_data(), dm.data.data(), dm.data.size() * sizeof(float));
              return out;
          },
          py::arg("queries"), py::arg("targets"), py::arg("metric") = "l2", py::arg("precision") = "full");

    m.def("nn_bruteforce",
          [](const F32& A, const F32& B, const std::string& metric) {
              const auto a = to_map(A), b = to_map(B);
              const auto mt = fastnn::metric_from_string(metric);
              fastnn::FetchCounter c;
              fastnn::NnResult r;
              {
                  py::gil_scoped_release nogil;
                  r = fastnn::nn_bruteforce(a, b, mt);
              }
              return nn_dict(r, c);
          },
          py::arg("A"), py::arg("B"), py::arg("metric") = "l2");

    m.def("nn_double_loop",
          [](const F32& A, const F32& B, std::uint32_t bs, const std::string& metric,
             const std::string& precision, unsigned threads) {
              const auto a = to_map(A), b = to_map(B);
              const auto pa = fastnn::make_partition(a.pixel_count(), bs);
              const auto pb = fastnn::make_partition(b.pixel_count(), bs);
              const auto mt = fastnn::metric_from_string(metric);
              const auto pr = fastnn::precision_from_string(precision);
              fastnn::FetchCounter c;
              fastnn::NnResult r;
              {
                  py::gil_scoped_release nogil;
                  r = fastnn::nn_double_loop(a, b, pa, pb, mt, pr, c, threads);
              }
              return nn_dict(r, c);
          },
          py::arg("A"), py::arg("B"), py::arg("block_size") = 4096, py::arg("metric") = "l2",
          py::arg("precision") = "full", py::arg("threads") = 1);

    m.def("nn_single_loop",
          [](const F32& A, const F32& B, std::uint32_t bs, const std::string& metric,
             const std::string& precision, unsigned threads) {
              const auto a = to_map(A), b = to_map(B);
              const auto pa = fastnn::make_partition(a.pixel_count(), bs);
              const auto mt = fastnn::metric_from_string(metric);
              const auto pr = fastnn::precision_from_string(precision);
              fastnn::FetchCounter c;
              fastnn::NnResult r;
              {
                  py::gil_scoped_release nogil;
                  r = fastnn::nn_single_loop(a, b, pa, mt, pr, c, threads);
              }
              return nn_dict(r, c);
          },
          py::arg("A"), py::arg("B"), py::arg("block_size") = 4096, py::arg("metric") = "l2",
          py::arg("precision") = "full", py::arg("threads") = 1);

    m.def("nn_hybridcast",
          [](const F32& A, const F32& B, std::uint32_t bs, const std::string& metric, unsigned threads) {
              const auto a = to_map(A), b = to_map(B);
              const auto pa = fastnn::make_partition(a.pixel_count(), bs);
              const auto mt = fastnn::metric_from_string(metric);
              fastnn::FetchCounter c;
              fastnn::NnResult r;
              {
                  py::gil_scoped_release nogil;
                  r = fastnn::nn_hybridcast(a, b, pa, mt, c, threads);
              }
              return nn_dict(r, c);
          },
          py::arg("A"), py::arg("B"), py::arg("block_size") = 4096, py::arg("metric") = "l2",
          py::arg("threads") = 1);

    m.def("grid_subsample",
          [](std::uint32_t h, std::uint32_t w, std::uint32_t k, std::uint32_t stride) {
              const fastnn::FeatureMap shape(h, w, 1);
              std::vector<std::uint32_t> ids;
              for (const auto p : fastnn::grid_subsample(shape, k, stride)) ids.push_back(p.index);
              return vec_array(ids);
          },
          py::arg("height"), py::arg("width"), py::arg("k") = 0, py::arg("stride") = 8);

    // The maps go straight from the numpy buffers to the device (no FeatureMap
    // copy); finiteness is validated on the GPU with the reference's message.
    m.def("mutual_nn_exact",
          [](const F32& D1, const F32& D2, const std::string& metric) {
              check_shape3(D1, "mutual_nn_exact");
              check_shape3(D2, "mutual_nn_exact");
              if (D1.shape(2) != D2.shape(2)) {
                  (void)to_map(D1);  // the reference validates both maps before the dims
                  (void)to_map(D2);
                  throw std::invalid_argument("mutual_nn_exact: descriptor dim mismatch (" +
                                              std::to_string(D1.shape(2)) + " vs " + std::to_string(D2.shape(2)) +
                                              ")");
              }
              const auto mt = fastnn::metric_from_string(metric);
              const std::uint32_t h1 = std::uint32_t(D1.shape(0)), w1 = std::uint32_t(D1.shape(1));
              std::vector<std::uint32_t> pairs(2 * std::size_t(h1) * w1 + 2);
              std::uint32_t n = 0;
              {
                  py::gil_scoped_release nogil;
                  fastnn::b200::check(fnl_mutual_nn(
                      fastnn::b200::context(), D1.data(), h1, w1, D2.data(), std::uint32_t(D2.shape(0)),
                      std::uint32_t(D2.shape(1)), std::uint32_t(D1.shape(2)),
                      mt == fastnn::DistanceMetric::SquaredL2 ? FNL_METRIC_L2 : FNL_METRIC_DOT, pairs.data(), &n));
              }
              U32Array out({py::ssize_t(n), py::ssize_t(2)});
              std::memcpy(out.mutable_data(), pairs.data(), std::size_t(n) * 8);
              return out;
          },
          py::arg("D1"), py::arg("D2"), py::arg("metric") = "l2");

    m.def("mutual_nn_tensor",
          [](const F32& D1, const F32& D2, const std::string& metric) {
              if (D1.ndim() != 3 || D2.ndim() != 3 || D1.shape(2) != D2.shape(2))
                  throw std::invalid_argument("mutual_nn_tensor: expects (H, W, d) maps with equal d");
              const auto mt = fastnn::metric_from_string(metric);
              const std::uint32_t h1 = std::uint32_t(D1.shape(0)), w1 = std::uint32_t(D1.shape(1));
              std::vector<std::uint32_t> pairs(2 * std::size_t(h1) * w1 + 2);
              std::uint32_t n = 0;
              {
                  py::gil_scoped_release nogil;
                  fastnn::b200::check(fnl_mutual_nn_tensor(
                      fastnn::b200::context(), D1.data(), h1, w1, D2.data(), std::uint32_t(D2.shape(0)),
                      std::uint32_t(D2.shape(1)), std::uint32_t(D1.shape(2)),
                      mt == fastnn::DistanceMetric::SquaredL2 ? FNL_METRIC_L2 : FNL_METRIC_DOT, pairs.data(), &n));
              }
              U32Array out({py::ssize_t(n), py::ssize_t(2)});
              std::memcpy(out.mutable_data(), pairs.data(), std::size_t(n) * 8);
              return out;
          },
          py::arg("D1"), py::arg("D2"), py::arg("metric") = "l2",
          "dense mutual NN on the tensor cores; equals mutual_nn_exact on binary16-rounded maps");

    // The maps go straight from the numpy buffers to the device (no FeatureMap
    // copy); finiteness is validated on the GPU with the reference's message.
    m.def("reciprocal_match",
          [](const F32& D1, const F32& D2, const std::string& backend, std::uint32_t k,
             std::uint32_t stride, std::uint32_t max_iters, double convergence,
             const std::string& metric, const std::string& precision, std::uint32_t block_size,
             unsigned threads) {
              check_shape3(D1, "reciprocal_match");
              check_shape3(D2, "reciprocal_match");
              const auto cfg = make_cfg(k, stride, max_iters, convergence, metric, precision, block_size);
              const auto be = fastnn::backend_from_string(backend);
              (void)threads;
              fastnn::MatchOutcome out;
              {
                  py::gil_scoped_release nogil;
                  out = fastnn::b200::reciprocal_match_raw(
                      D1.data(), std::uint32_t(D1.shape(0)), std::uint32_t(D1.shape(1)), D2.data(),
                      std::uint32_t(D2.shape(0)), std::uint32_t(D2.shape(1)), std::uint32_t(D1.shape(2)),
                      std::uint32_t(D2.shape(2)), cfg, be);
              }
              U32Array pairs({py::ssize_t(out.matches.pairs.size()), py::ssize_t(3)});
              auto v = pairs.mutable_unchecked<2>();
              for (py::ssize_t r = 0; r < py::ssize_t(out.matches.pairs.size()); ++r) {
                  v(r, 0) = out.matches.pairs[r].i;
                  v(r, 1) = out.matches.pairs[r].j;
                  v(r, 2) = out.matches.pairs[r].iteration;
              }
              return py::make_tuple(pairs, fastnn::render_report(out.report, fastnn::ReportFormat::Json));
          },
          py::arg("D1"), py::arg("D2"), py::arg("backend") = "single", py::arg("k") = 0,
          py::arg("stride") = 8, py::arg("max_iters") = 10, py::arg("convergence") = 0.99,
          py::arg("metric") = "l2", py::arg("precision") = "full", py::arg("block_size") = 4096,
          py::arg("threads") = 1);

    // ------------------------------------------------------------ extensions
    m.def("nn_tensor",
          [](const F32& A, const F32& B, const std::string& metric) {
              const auto a = to_map(A), b = to_map(B);
              const auto mt = fastnn::metric_from_string(metric);
              fastnn::FetchCounter c;
              fastnn::NnResult r;
              {
                  py::gil_scoped_release nogil;
                  r = fastnn::nn_query_tensor(fastnn::DescriptorsView::of(a), fastnn::DescriptorsView::of(b), mt);
              }
              return nn_dict(r, c);
          },
          py::arg("A"), py::arg("B"), py::arg("metric") = "dot",
          "tcgen05 HybridCast NN of every pixel of A in B (binary16 in, fp32 accumulate/compare, "
          "near ties re-decided exactly)");

    // Batched host-buffer matcher: npairs stacked (n, H, W, d) maps, H2D copies
    // pipelined with compute.  Returns (pairs[n, samples, 3], counts[n], stats).
    m.def("reciprocal_match_batch",
          [](const F32& D1, const F32& D2, const std::string& backend, std::uint32_t k,
             std::uint32_t stride, std::uint32_t max_iters, double convergence,
             const std::string& metric, const std::string& precision, std::uint32_t block_size) {
              if (D1.ndim() != 4 || D2.ndim() != 4)
                  throw std::invalid_argument("reciprocal_match_batch expects (n, H, W, d) arrays");
              for (int i = 0; i < 4; ++i)
                  if (D1.shape(i) != D2.shape(i))
                      throw std::invalid_argument("reciprocal_match_batch: D1 and D2 shapes differ");
              const auto cfg = make_cfg(k, stride, max_iters, convergence, metric, precision, block_size);
              cfg.validate();
              const auto cc = c_cfg(cfg);
              const int be = c_backend(fastnn::backend_from_string(backend));
              const std::uint32_t n = std::uint32_t(D1.shape(0)), h = std::uint32_t(D1.shape(1)),
                                  w = std::uint32_t(D1.shape(2)), d = std::uint32_t(D1.shape(3));
              const fastnn::FeatureMap shape(h, w, 1);
              const std::size_t cap = std::max<std::size_t>(1, fastnn::grid_subsample(shape, cfg.k, cfg.grid_stride).size());
              U32Array pairs({py::ssize_t(n), py::ssize_t(cap), py::ssize_t(3)});
              U32Array counts{py::ssize_t(n)};
              std::vector<fnl_run_stats> st(n);
              {
                  py::gil_scoped_release nogil;
                  fastnn::b200::check(fnl_reciprocal_match_batch(fastnn::b200::context(), n, D1.data(), D2.data(),
                                                                 h, w, d, &cc, be, pairs.mutable_data(),
                                                                 counts.mutable_data(), st.data()));
              }
              py::list stats;
              for (const auto& s : st) stats.append(stats_dict(s));
              return py::make_tuple(pairs, counts, stats);
          },
          py::arg("D1"), py::arg("D2"), py::arg("backend") = "tensor", py::arg("k") = 0,
          py::arg("stride") = 8, py::arg("max_iters") = 10, py::arg("convergence") = 0.99,
          py::arg("metric") = "dot", py::arg("precision") = "full", py::arg("block_size") = 4096);

    // Device-resident matcher (maps and outputs are device pointers, e.g.
    // torch.Tensor.data_ptr()); returns per-pair stats.
    m.def("reciprocal_match_device",
          [](std::uintptr_t d1, std::uintptr_t d2, std::uint32_t n, std::uint32_t h, std::uint32_t w,
             std::uint32_t d, std::uintptr_t out_pairs, std::uintptr_t out_counts,
             const std::string& backend, std::uint32_t k, std::uint32_t stride, std::uint32_t max_iters,
             double convergence, const std::string& metric, const std::string& precision,
             std::uint32_t block_size, py::object stream, py::object max_distance, bool with_stats) {
              const bool conf = !max_distance.is_none();
              const float max_dist = conf ? max_distance.cast<float>() : 0.0f;
              void* const sh = stream_handle(stream);  // with the GIL held
              const auto cfg = make_cfg(k, stride, max_iters, convergence, metric, precision, block_size);
              cfg.validate();
              const auto cc = c_cfg(cfg);
              const int be = c_backend(fastnn::backend_from_string(backend));
              std::vector<fnl_run_stats> st(n);
              {
                  py::gil_scoped_release nogil;
                  fnl_context* ctx = fastnn::b200::context();
                  fastnn::b200::check(fnl_context_set_stream(ctx, sh));
                  int rc = fnl_reciprocal_match_batch_device(
                      ctx, n, reinterpret_cast<const float*>(d1), reinterpret_cast<const float*>(d2), h, w, d,
                      &cc, be, reinterpret_cast<std::uint32_t*>(out_pairs),
                      reinterpret_cast<std::uint32_t*>(out_counts), with_stats ? st.data() : nullptr);
                  if (rc == FNL_OK && conf) {
                      // confidence-thresholded compaction of the finished MatchSets (extension)
                      const fastnn::FeatureMap shape(h, w, 1);
                      const std::uint32_t cap = std::max<std::uint32_t>(
                          1, std::uint32_t(fastnn::grid_subsample(shape, cfg.k, cfg.grid_stride).size()));
                      rc = fnl_confidence_compact_device(
                          ctx, n, reinterpret_cast<const float*>(d1), reinterpret_cast<const float*>(d2), h, w, d,
                          cc.metric, max_dist, reinterpret_cast<std::uint32_t*>(out_pairs),
                          reinterpret_cast<std::uint32_t*>(out_counts), cap, nullptr);
                  }
                  fnl_context_set_stream(ctx, nullptr);
                  fastnn::b200::check(rc);
              }
              py::list stats;
              if (with_stats)
                  for (const auto& s : st) stats.append(stats_dict(s));
              return stats;
          },
          py::arg("d1"), py::arg("d2"), py::arg("npairs"), py::arg("height"), py::arg("width"),
          py::arg("dim"), py::arg("out_pairs"), py::arg("out_counts"), py::arg("backend") = "tensor",
          py::arg("k") = 0, py::arg("stride") = 8, py::arg("max_iters") = 10,
          py::arg("convergence") = 0.99, py::arg("metric") = "dot", py::arg("precision") = "full",
          py::arg("block_size") = 4096, py::arg("stream") = py::none(), py::arg("max_distance") = py::none(),
          py::arg("with_stats") = true);

    // Target-sharded matcher (config C5).  `reduce(count)` must MIN-all-reduce
    // the first `count` int64 entries of the caller's key buffer (`keys`, a
    // device pointer with `keys_capacity` entries) across the shards, on the
    // current stream -- e.g. torch.distributed.all_reduce(keys[:count], MIN).
    m.def("reciprocal_match_sharded_device",
          [](std::uintptr_t d1, std::uintptr_t d2, std::uint32_t n, std::uint32_t h, std::uint32_t w,
             std::uint32_t d, std::uintptr_t out_pairs, std::uintptr_t out_counts, std::uintptr_t keys,
             std::uint64_t keys_capacity, std::uint32_t rank, std::uint32_t count, py::object reduce,
             const std::string& backend, std::uint32_t k, std::uint32_t stride, std::uint32_t max_iters,
             double convergence, const std::string& metric, std::uint32_t block_size, py::object stream,
             std::uintptr_t comm) {
              void* const sh = stream_handle(stream);  // with the GIL held
              const auto cfg = make_cfg(k, stride, max_iters, convergence, metric, "full", block_size);
              cfg.validate();
              const auto cc = c_cfg(cfg);
              const int be = c_backend(fastnn::backend_from_string(backend));
              std::vector<fnl_run_stats> st(n);
              if (reduce.is_none() && !comm)
                  throw std::invalid_argument("reciprocal_match_sharded_device: a reduce callback or comm is required");
              struct Ctx {
                  py::object fn;
                  std::string err;
              } cb{reduce, {}};
              fnl_shard_spec spec{};
              spec.rank = rank;
              spec.count = count;
              spec.d_keys = reinterpret_cast<std::int64_t*>(keys);
              spec.keys_capacity = keys_capacity;
              spec.user = &cb;
              spec.comm = reinterpret_cast<fnl_comm*>(comm);  // native NCCL: the library reduces itself
              if (!spec.comm) spec.reduce = [](void* user, std::int64_t*, std::uint64_t cnt, void*) -> int {
                  auto* c = static_cast<Ctx*>(user);
                  py::gil_scoped_acquire gil;
                  try {
                      c->fn(cnt);
                      return 0;
                  } catch (const std::exception& e) {
                      c->err = e.what();
                      return 1;
                  }
              };
              int rc;
              {
                  py::gil_scoped_release nogil;
                  fnl_context* ctx = fastnn::b200::context();
                  fastnn::b200::check(fnl_context_set_stream(ctx, sh));
                  rc = fnl_reciprocal_match_sharded_device(
                      ctx, n, reinterpret_cast<const float*>(d1), reinterpret_cast<const float*>(d2), h, w, d,
                      &cc, be, &spec, reinterpret_cast<std::uint32_t*>(out_pairs),
                      reinterpret_cast<std::uint32_t*>(out_counts), st.data());
                  fnl_context_set_stream(ctx, nullptr);
              }
              if (rc != FNL_OK && !cb.err.empty()) throw std::runtime_error("shard reduce callback: " + cb.err);
              fastnn::b200::check(rc);
              py::list stats;
              for (const auto& s : st) stats.append(stats_dict(s));
              return stats;
          },
          py::arg("d1"), py::arg("d2"), py::arg("npairs"), py::arg("height"), py::arg("width"),
          py::arg("dim"), py::arg("out_pairs"), py::arg("out_counts"), py::arg("keys"),
          py::arg("keys_capacity"), py::arg("shard_rank"), py::arg("shard_count"), py::arg("reduce"),
          py::arg("backend") = "tensor", py::arg("k") = 0, py::arg("stride") = 8, py::arg("max_iters") = 10,
          py::arg("convergence") = 0.99, py::arg("metric") = "dot", py::arg("block_size") = 4096,
          py::arg("stream") = py::none(), py::arg("comm") = 0);

    // Native NCCL communicator for the C5 key reduction (fnl_comm_*): rank 0
    // makes the id, every rank creates its communicator (collective).
    m.def("nccl_unique_id", [] {
        unsigned char id[128];
        fastnn::b200::check(fnl_nccl_unique_id(id));
        return py::bytes(reinterpret_cast<const char*>(id), 128);
    });
    m.def("comm_create",
          [](py::bytes id, int nranks, int rank) {
              const std::string s = id;
              if (s.size() != 128) throw std::invalid_argument("comm_create: the NCCL id is 128 bytes");
              fnl_comm* c = nullptr;
              {
                  py::gil_scoped_release nogil;
                  fastnn::b200::check(fnl_comm_create(fastnn::b200::context(),
                                                      reinterpret_cast<const unsigned char*>(s.data()), nranks,
                                                      rank, &c));
              }
              return reinterpret_cast<std::uintptr_t>(c);
          },
          py::arg("id"), py::arg("nranks"), py::arg("rank"));
    m.def("comm_destroy", [](std::uintptr_t c) { fastnn::b200::check(fnl_comm_destroy(reinterpret_cast<fnl_comm*>(c))); });
    m.def("comm_info", [](std::uintptr_t c) {
        int n = 0, r = 0, v = 0;
        fastnn::b200::check(fnl_comm_info(reinterpret_cast<const fnl_comm*>(c), &n, &r, &v));
        return py::make_tuple(n, r, v);
    });

    // Same, with the peer-memory transport (keys pushed into every rank's
    // buffer by the merge epilogues, peer-memory barrier instead of NCCL).
    // Returns (stats, barrier_seq).
    m.def("reciprocal_match_p2p_device",
          [](std::uintptr_t d1, std::uintptr_t d2, std::uint32_t n, std::uint32_t h, std::uint32_t w,
             std::uint32_t d, std::uintptr_t out_pairs, std::uintptr_t out_counts, std::uint64_t keys_capacity,
             std::uint32_t rank, const std::vector<std::uintptr_t>& peer_keys,
             const std::vector<std::uintptr_t>& peer_flags, std::uint64_t barrier_seq, const std::string& backend,
             std::uint32_t k, std::uint32_t stride, std::uint32_t max_iters, double convergence,
             const std::string& metric, std::uint32_t block_size, py::object stream) {
              void* const sh = stream_handle(stream);  // with the GIL held
              if (peer_keys.size() != peer_flags.size() || rank >= peer_keys.size())
                  throw std::invalid_argument("reciprocal_match_p2p_device: one key buffer and flag per rank");
              const auto cfg = make_cfg(k, stride, max_iters, convergence, metric, "full", block_size);
              cfg.validate();
              const auto cc = c_cfg(cfg);
              const int be = c_backend(fastnn::backend_from_string(backend));
              std::vector<fnl_run_stats> st(n);
              std::vector<std::int64_t*> pk;
              std::vector<std::uint32_t*> pf;
              for (auto v : peer_keys) pk.push_back(reinterpret_cast<std::int64_t*>(v));
              for (auto v : peer_flags) pf.push_back(reinterpret_cast<std::uint32_t*>(v));
              fnl_shard_spec spec{};
              spec.rank = rank;
              spec.count = std::uint32_t(pk.size());
              spec.d_keys = pk[rank];
              spec.keys_capacity = keys_capacity;
              spec.peer_keys = pk.data();
              spec.peer_flags = pf.data();
              spec.barrier_seq = &barrier_seq;
              int rc;
              {
                  py::gil_scoped_release nogil;
                  fnl_context* ctx = fastnn::b200::context();
                  fastnn::b200::check(fnl_context_set_stream(ctx, sh));
                  rc = fnl_reciprocal_match_sharded_device(
                      ctx, n, reinterpret_cast<const float*>(d1), reinterpret_cast<const float*>(d2), h, w, d,
                      &cc, be, &spec, reinterpret_cast<std::uint32_t*>(out_pairs),
                      reinterpret_cast<std::uint32_t*>(out_counts), st.data());
                  fnl_context_set_stream(ctx, nullptr);
              }
              fastnn::b200::check(rc);
              py::list stats;
              for (const auto& s : st) stats.append(stats_dict(s));
              return py::make_tuple(stats, barrier_seq);
          },
          py::arg("d1"), py::arg("d2"), py::arg("npairs"), py::arg("height"), py::arg("width"),
          py::arg("dim"), py::arg("out_pairs"), py::arg("out_counts"), py::arg("keys_capacity"),
          py::arg("shard_rank"), py::arg("peer_keys"), py::arg("peer_flags"), py::arg("barrier_seq"),
          py::arg("backend") = "tensor", py::arg("k") = 0, py::arg("stride") = 8, py::arg("max_iters") = 10,
          py::arg("convergence") = 0.99, py::arg("metric") = "dot", py::arg("block_size") = 4096,
          py::arg("stream") = py::none());
    m.def("p2p_alloc",
          [](std::uint64_t bytes, bool fill_key_none) {
              void* p = nullptr;
              fastnn::b200::check(fnl_p2p_alloc(fastnn::b200::context(), bytes, fill_key_none ? 1 : 0, &p));
              return reinterpret_cast<std::uintptr_t>(p);
          },
          py::arg("bytes"), py::arg("fill_key_none") = false);
    m.def("p2p_free", [](std::uintptr_t p) { fastnn::b200::check(fnl_p2p_free(reinterpret_cast<void*>(p))); });
    m.def("ipc_handle", [](std::uintptr_t p) {
        unsigned char h[64];
        fastnn::b200::check(fnl_ipc_handle(reinterpret_cast<const void*>(p), h));
        return py::bytes(reinterpret_cast<const char*>(h), 64);
    });
    m.def("ipc_open", [](py::bytes handle) {
        const std::string s = handle;
        if (s.size() != 64) throw std::invalid_argument("ipc_open: handles are 64 bytes");
        void* p = nullptr;
        fastnn::b200::check(fnl_ipc_open(fastnn::b200::context(),
                                         reinterpret_cast<const unsigned char*>(s.data()), &p));
        return reinterpret_cast<std::uintptr_t>(p);
    });
    m.def("ipc_close", [](std::uintptr_t p) { fastnn::b200::check(fnl_ipc_close(reinterpret_cast<void*>(p))); });

    m.def("kernel_timing",
          [](bool reset) {
              double ms = 0;
              std::uint64_t launches = 0, total = 0;
              fastnn::b200::check(fnl_kernel_timing(fastnn::b200::context(), reset, &ms, &launches, &total));
              py::dict d;
              d["score_ms"] = ms;
              d["score_launches"] = launches;
              d["total_launches"] = total;
              return d;
          },
          py::arg("reset") = false,
          "device time and launch count of the dominant scoring kernel since the last reset");

    m.def("loop_graph_max_pairs",
          [](int max_pairs) {
              int prev = 0;
              fastnn::b200::check(fnl_loop_graph_max_pairs(fastnn::b200::context(), max_pairs, &prev));
              return prev;
          },
          py::arg("max_pairs") = -1,
          "Largest batch whose reciprocal loop replays as a CUDA graph on this thread's context (0: off; "
          "negative: query only); returns the previous value.");
    m.def("kernel_profile",
          [](int enable, bool reset) {
              double ms[FNL_KCLASS_COUNT] = {};
              std::uint64_t n[FNL_KCLASS_COUNT] = {};
              fastnn::b200::check(fnl_kernel_profile(fastnn::b200::context(), enable, reset ? 1 : 0, ms, n));
              static const char* names[FNL_KCLASS_COUNT] = {"score", "pack", "gather", "merge",
                                                            "rescan", "harvest", "attention", "other"};
              py::dict d;
              for (int c = 0; c < FNL_KCLASS_COUNT; ++c) {
                  py::dict e;
                  e["ms"] = ms[c];
                  e["launches"] = n[c];
                  d[names[c]] = e;
              }
              return d;
          },
          py::arg("enable") = -1, py::arg("reset") = false,
          "per-kernel-class device time (CUDA events) since the last reset; enable=1/0 turns the "
          "breakdown of the non-score classes on/off");

    m.def("_flashmatch_fwd",
          [](std::uintptr_t q, std::uintptr_t k, std::uintptr_t v, std::uintptr_t o, std::uint32_t batch,
             std::uint32_t heads, std::uint32_t nq, std::uint32_t nkv, std::uint32_t head_dim, float scale,
             std::array<std::uint64_t, 3> qs, std::array<std::uint64_t, 3> ks, std::array<std::uint64_t, 3> vs,
             std::array<std::uint64_t, 3> os, py::object stream) {
              fnl_context* ctx = fastnn::b200::context();
              void* const sh = stream_handle(stream);
              fastnn::b200::check(fnl_context_set_stream(ctx, sh));
              fnl_attention_desc d{};
              d.q = reinterpret_cast<const void*>(q);
              d.k = reinterpret_cast<const void*>(k);
              d.v = reinterpret_cast<const void*>(v);
              d.o = reinterpret_cast<void*>(o);
              d.batch = batch;
              d.heads = heads;
              d.nq = nq;
              d.nkv = nkv;
              d.head_dim = head_dim;
              d.scale = scale;
              for (int i = 0; i < 3; ++i) {
                  d.q_stride[i] = qs[i];
                  d.k_stride[i] = ks[i];
                  d.v_stride[i] = vs[i];
                  d.o_stride[i] = os[i];
              }
              const int st = fnl_flashmatch_fwd(ctx, &d);
              fnl_context_set_stream(ctx, nullptr);
              fastnn::b200::check(st);
          },
          py::arg("q"), py::arg("k"), py::arg("v"), py::arg("o"), py::arg("batch"), py::arg("heads"),
          py::arg("nq"), py::arg("nkv"), py::arg("head_dim"), py::arg("scale"), py::arg("q_strides"),
          py::arg("k_strides"), py::arg("v_strides"), py::arg("o_strides"), py::arg("stream") = py::none(),
          "K7 FlashMatch attention on raw device pointers (binary16, head_dim 64); see flashmatch.py");

    m.def("_flashmatch_trace", []() {
        std::vector<unsigned long long> v(64);
        fnl_context* ctx = fastnn::b200::context();
        fastnn::b200::check(fnl_context_synchronize(ctx));
        fastnn::b200::check(fnl_flashmatch_trace(ctx, v.data()));
        return v;
    });

    m.def("_tensor_selftest",
          [](const F32& q, const F32& t, const std::string& metric, int mode) {
              if (q.ndim() != 2 || t.ndim() != 2 || q.shape(0) != 256 || t.shape(0) != 128 || q.shape(1) != t.shape(1))
                  throw std::invalid_argument("_tensor_selftest expects q (256, d), t (128, d)");
              py::array_t<float> out({py::ssize_t(256), py::ssize_t(128)});
              fastnn::b200::check(fnl_tensor_selftest(fastnn::b200::context(), q.data(), t.data(),
                                                      std::uint32_t(q.shape(1)),
                                                      metric == "l2" ? FNL_METRIC_L2 : FNL_METRIC_DOT, mode,
                                                      out.mutable_data()));
              return out;
          },
          py::arg("queries"), py::arg("targets"), py::arg("metric") = "dot", py::arg("mode") = 1);

    // host-side report rendering, exposed for the golden-format tests
    m.def("_render_report",
          [](py::dict d, const std::string& format) {
              fastnn::RunReport r;
              auto get = [&](const char* k, auto& v) {
                  if (d.contains(k)) v = d[k].cast<std::decay_t<decltype(v)>>();
              };
              get("backend", r.backend); get("metric", r.metric); get("precision", r.precision);
              get("height1", r.height1); get("width1", r.width1); get("height2", r.height2); get("width2", r.width2);
              get("dim", r.dim); get("k", r.k); get("grid_stride", r.grid_stride); get("max_iters", r.max_iters);
              get("convergence_fraction", r.convergence_fraction); get("block_size", r.block_size); get("seed", r.seed);
              get("subsample_us", r.subsample_us); get("forward_nn_us", r.forward_nn_us);
              get("reverse_nn_us", r.reverse_nn_us); get("harvest_us", r.harvest_us);
              get("a_block_fetches", r.a_block_fetches); get("b_block_fetches", r.b_block_fetches);
              get("iterations", r.iterations); get("samples", r.samples); get("converged", r.converged);
              get("converged_fraction", r.converged_fraction); get("half_saturated", r.half_saturated);
              get("half_saturation_events", r.half_saturation_events);
              if (d.contains("hybrid_full_argmin_agreement") && !d["hybrid_full_argmin_agreement"].is_none())
                  r.hybrid_full_argmin_agreement = d["hybrid_full_argmin_agreement"].cast<double>();
              get("matches_emitted", r.matches_emitted); get("duplicates_dropped", r.duplicates_dropped);
              get("active_history", r.active_history);
              return fastnn::render_report(r, format == "csv" ? fastnn::ReportFormat::Csv : fastnn::ReportFormat::Json);
          },
          py::arg("report"), py::arg("format") = "json");
    m.def("_parse_report", [](const std::string& text) {
        return fastnn::render_report(fastnn::parse_report_json(text), fastnn::ReportFormat::Json);
    });

    m.def("device_count", [] {
        int n = 0;
        fnl_device_count(&n);
        return n;
    });
    m.def("set_device", [](int dev) { fastnn::b200::set_device(dev); }, py::arg("device"));
    m.def("abi_version", [] { return fnl_abi_version(); });
}
