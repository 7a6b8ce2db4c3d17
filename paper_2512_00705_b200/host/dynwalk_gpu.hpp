// dynwalk_gpu.hpp -- header-only C++ shim: the reference's host API for the
// walk path, executed by the B200 engine through the C ABI (dynwalk_b200.h).
//
// Drop-in for the reference (compile inside its tree, link libdynwalk_b200.so):
//
//   dynwalk::run_queries(g, model, params, queries, opts)          runtime.hpp:85-86
//     -> dynwalk::gpu::run_queries(g, model, params, queries, opts)  (same signature)
//   dynwalk::profile_edge_cost_ratio(g, model, cfg)                cost_model.hpp:39-40
//     -> dynwalk::gpu::profile_edge_cost_ratio(g, model, cfg)
//   dynwalk::selection_ratio_sweep(base, model, params, alphas, q, opts)  runtime.hpp:99-103
//     -> dynwalk::gpu::selection_ratio_sweep(...)                        (same signature)
//   dynwalk::write_paths(file, dynwalk::run_queries(...).paths)         runtime.cpp:280-291
//     -> dynwalk::gpu::run_queries_write_paths(g, model, params, q, opts, file)
//
// Semantics kept: query order, path[0] = start, length
// <= min(L, max_steps) + 1, empty path + query_errors++ for an out-of-range
// start, RunStats counters exactly as runtime.cpp:141-149, output independent
// of the device count.  Errors surface as dynwalk::Error with the reference's
// wording.  Options the GPU runtime does not implement (ForceIts, ForceAls,
// check_bounds, bound_scale != 1, collect_cv) throw dynwalk::Error naming the
// option; the CPU run_queries still serves them.  DslWalk models are compiled
// into the walk kernel (dsl_codegen.hpp, dw_model_compile); their device
// calibration is not supported, so pass CostModelParams explicitly.
// Walker randomness is the Philox (seed, walker, step) stream, so paths equal
// the reference samplers driven by that stream (tests/golden/ref_walks.json),
// not the mt19937 stream of the CPU run_queries.
#pragma once

#include <algorithm>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <span>
#include <string>
#include <tuple>
#include <type_traits>
#include <variant>
#include <vector>

#include "dsl_codegen.hpp"
#include "dynwalk/cost_model.hpp"
#include "dynwalk/graph.hpp"
#include "dynwalk/rng.hpp"
#include "dynwalk/runtime.hpp"
#include "dynwalk_b200.h"

namespace dynwalk::gpu {

inline void check(int rc) {
    if (rc != DW_OK) throw Error(dw_last_error());
}

// Device replicas of one immutable Graph (graph.hpp:47).
class DeviceGraph {
public:
    // one replica per device in `devices` (dw_graph_create)
    explicit DeviceGraph(const Graph& g, std::vector<int> devices = {0}) {
        const std::uint32_t nv = g.num_vertices();
        std::vector<double> nmax(nv), nsum(nv);
        for (std::uint32_t v = 0; v < nv; ++v) {
            nmax[v] = g.node_prop_max(v);
            nsum[v] = g.node_prop_sum(v);
        }
        dw_graph_desc d{};
        d.num_vertices = nv;
        d.num_edges = g.num_edges();
        d.row_offsets = g.row_offsets().data();
        d.col_indices = g.col_indices().data();
        d.edge_props = g.edge_props().data();
        d.edge_labels = g.has_labels() ? g.edge_labels().data() : nullptr;
        d.node_prop_max = nmax.data();
        d.node_prop_sum = nsum.data();
        check(dw_graph_create(&d, devices.data(), static_cast<int>(devices.size()), &h_));
    }
    ~DeviceGraph() { dw_graph_destroy(h_); }
    DeviceGraph(const DeviceGraph&) = delete;
    DeviceGraph& operator=(const DeviceGraph&) = delete;
    dw_graph_t handle() const { return h_; }

private:
    dw_graph_t h_ = nullptr;
};

namespace detail {

// A DslWalk compiled into the walk kernel (dsl_codegen.hpp + dw_model_compile),
// cached by program source so each program compiles once per process.
inline dw_custom_model_t compiled_dsl(const DslWalk& w) {
    static std::mutex mu;
    static std::map<std::string, dw_custom_model_t> cache;
    const dsl::Program& prog = w.program();
    const DslCode code = dsl_codegen(prog, w.analysis(), w.max_steps());
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find(code.source);
    if (it != cache.end()) return it->second;
    dw_custom_model_t h = nullptr;
    check(dw_model_compile(code.source.c_str(), w.max_steps(),
                           code.label_aggregates ? DW_CUSTOM_LABEL_AGGREGATES : 0u, &h));
    cache.emplace(code.source, h);
    return h;
}

// AnyModel (models.hpp:200) -> dw_model_desc; the device functor is picked by
// kind inside the library (compile-time specialised kernels); a DslWalk is
// compiled to its own kernel.
struct ModelDesc {
    dw_model_desc d{};
    std::vector<std::uint16_t> schema;
};

inline ModelDesc to_desc(const AnyModel& model) {
    ModelDesc m;
    std::visit(
        [&](const auto& v) {
            using T = std::decay_t<decltype(v)>;
            if constexpr (!std::is_same_v<T, DslWalk>) m.d.weighted = v.weighted ? 1 : 0;
            if constexpr (std::is_same_v<T, StaticWalk>) {
                m.d.kind = DW_MODEL_STATIC;
            } else if constexpr (std::is_same_v<T, Node2Vec>) {
                m.d.kind = DW_MODEL_NODE2VEC;
                m.d.a = v.a;
                m.d.b = v.b;
            } else if constexpr (std::is_same_v<T, MetaPath>) {
                m.d.kind = DW_MODEL_METAPATH;
                m.schema.assign(v.schema.begin(), v.schema.end());
            } else if constexpr (std::is_same_v<T, SecondOrderPr>) {
                m.d.kind = DW_MODEL_PR2;
                m.d.gamma = v.gamma;
            } else if constexpr (std::is_same_v<T, DslWalk>) {
                m.d.kind = DW_MODEL_CUSTOM;
                m.d.custom = compiled_dsl(v);
            }
        },
        model);
    m.d.schema = m.schema.empty() ? nullptr : m.schema.data();
    m.d.schema_len = static_cast<std::uint32_t>(m.schema.size());
    return m;
}

inline int to_mode(SamplerMode mode) {
    switch (mode) {
    case SamplerMode::Adaptive: return DW_MODE_ADAPTIVE;
    case SamplerMode::ForceErvs: return DW_MODE_FORCE_ERVS;
    case SamplerMode::ForceErjs: return DW_MODE_FORCE_ERJS;
    case SamplerMode::ErvsNoJump: return DW_MODE_ERVS_NOJUMP;
    case SamplerMode::ForceIts: return DW_MODE_FORCE_ITS;
    case SamplerMode::ForceAls: return DW_MODE_FORCE_ALS;
    }
    return -1;
}

// FNV-1a over a strided sample (<= ~4K positions) of every CSR array.  Graphs
// built in a loop (selection_ratio_sweep, repeated synthesize_weights) free and
// reallocate their vectors, and a new graph can land on the old addresses; the
// sample tells such graphs apart at O(4K) cost per call.
inline std::uint64_t sample_fingerprint(const Graph& g) {
    std::uint64_t h = 1469598103934665603ull;
    auto mix = [&h](std::uint64_t v) {
        h ^= v;
        h *= 1099511628211ull;
    };
    auto sample = [&mix](auto span) {
        const std::size_t n = span.size();
        const std::size_t step = std::max<std::size_t>(1, n / 4096);
        mix(n);
        for (std::size_t i = 0; i < n; i += step) {
            std::uint64_t v = 0;
            std::memcpy(&v, &span[i], sizeof(span[i]));
            mix(v);
        }
        if (n) {
            std::uint64_t v = 0;
            std::memcpy(&v, &span[n - 1], sizeof(span[n - 1]));
            mix(v);
        }
    };
    sample(g.row_offsets());
    sample(g.col_indices());
    sample(g.edge_props());
    if (g.has_labels()) sample(g.edge_labels());
    return h;
}

// Cached replicas keyed by graph identity: addresses plus the sampled content
// fingerprint (arrays are never mutated in place: set_edge_props replaces the
// vector).  An edit that touches none of the sampled positions is not seen;
// callers that rewrite graphs in place should pass a DeviceGraph explicitly.
using CacheKey = std::tuple<const Graph*, const void*, const void*, const void*, std::uint64_t,
                            std::uint64_t>;
struct ReplicaCache {
    std::mutex mu;
    std::map<CacheKey, std::shared_ptr<DeviceGraph>> map;
    std::vector<int> devices;  // empty: every visible device
};
inline ReplicaCache& replica_cache() {
    static ReplicaCache c;
    return c;
}

// The devices a Graph is replicated on when the reference signatures are
// called with a `const Graph&`: every visible GPU (walkers are split over
// them; output does not depend on the count), or the list set_devices() gave.
inline std::vector<int> default_devices() {
    ReplicaCache& c = replica_cache();
    if (!c.devices.empty()) return c.devices;
    int n = 0;
    dw_device_count(&n);
    std::vector<int> all;
    for (int d = 0; d < n; ++d) all.push_back(d);
    if (all.empty()) all.push_back(0);  // dw_graph_create reports the missing device
    return all;
}

inline std::shared_ptr<DeviceGraph> cached(const Graph& g) {
    ReplicaCache& c = replica_cache();
    const CacheKey k{&g, g.col_indices().data(), g.edge_props().data(),
                     g.has_labels() ? static_cast<const void*>(g.edge_labels().data()) : nullptr,
                     g.num_edges(), sample_fingerprint(g)};
    std::lock_guard<std::mutex> lk(c.mu);
    auto it = c.map.find(k);
    if (it != c.map.end()) return it->second;
    if (c.map.size() >= 4) c.map.clear();
    auto dg = std::make_shared<DeviceGraph>(g, default_devices());
    c.map.emplace(k, dg);
    return dg;
}

}  // namespace detail

// Restricts the replicas behind the `const Graph&` overloads to `devices`
// (empty: every visible GPU); drops replicas cached for another list.
inline void set_devices(std::vector<int> devices) {
    detail::ReplicaCache& c = detail::replica_cache();
    std::lock_guard<std::mutex> lk(c.mu);
    c.devices = std::move(devices);
    c.map.clear();
}

namespace detail {

}  // namespace detail

namespace detail {

inline dw_run_opts to_opts(const CostModelParams& params, const RunOptions& opts) {
    if (opts.workers < 1) throw Error("worker count must be >= 1");  // runtime.cpp:194
    if (opts.check_bounds) throw Error("RunOptions.check_bounds is not supported by the GPU runtime");
    if (opts.bound_scale != 1.0)
        throw Error("RunOptions.bound_scale is not supported by the GPU runtime");
    if (opts.collect_cv) throw Error("RunOptions.collect_cv is not supported by the GPU runtime");
    dw_run_opts o{};
    o.mode = to_mode(opts.mode);
    o.walk_length = opts.walk_length;
    o.seed = opts.seed;
    o.erjs_cap_per_degree = opts.erjs_cap_per_degree;
    o.edge_cost_ratio = params.edge_cost_ratio;
    o.qid_base = 0;
    return o;
}

inline RunStats to_stats(const dw_run_stats& st) {
    RunStats s;
    s.queries = st.queries;
    s.query_errors = st.query_errors;
    s.dead_ends = st.dead_ends;
    s.steps = st.steps;
    s.select_ervs = st.select_ervs;
    s.select_erjs = st.select_erjs;
    s.trials = st.trials;
    s.weight_reads = st.weight_reads;
    s.rng_draws = st.rng_draws;
    s.erjs_fallbacks = st.erjs_fallbacks;
    for (std::size_t b = 0; b < s.selection_by_degree.size(); ++b) {
        s.selection_by_degree[b][0] = st.selection_by_degree[b][0];
        s.selection_by_degree[b][1] = st.selection_by_degree[b][1];
    }
    s.wall_ms = st.total_ms;
    return s;
}

}  // namespace detail

inline RunResult run_queries(const DeviceGraph& dg, const AnyModel& model,
                             const CostModelParams& params, std::span<const VertexId> queries,
                             const RunOptions& opts) {
    const dw_run_opts o = detail::to_opts(params, opts);
    const detail::ModelDesc m = detail::to_desc(model);
    const std::size_t nq = queries.size();
    const std::size_t stride = static_cast<std::size_t>(opts.walk_length) + 1;
    // compact transfer: offsets + the ids that exist (dw_run_compact)
    std::vector<VertexId> flat(std::max<std::size_t>(nq * stride, 1));
    std::vector<std::uint64_t> offsets(nq + 1);
    dw_run_stats st{};
    check(dw_run_compact(dg.handle(), &m.d, queries.data(), nq, &o, offsets.data(), flat.data(),
                         flat.size(), &st));

    RunResult rr;
    rr.paths.resize(nq);
    std::vector<std::uint32_t> lengths(nq);
    for (std::size_t i = 0; i < nq; ++i) {
        rr.paths[i].assign(flat.begin() + offsets[i], flat.begin() + offsets[i + 1]);
        lengths[i] = static_cast<std::uint32_t>(offsets[i + 1] - offsets[i]);
    }
    rr.stats = detail::to_stats(st);
    rr.stats.path_lengths = std::move(lengths);
    return rr;
}

// write_paths(path, run_queries(g, model, params, queries, opts).paths)
// (runtime.cpp:280-291) in one pass: the text is formatted on the device and
// written batch by batch while later batches walk, so host memory stays
// bounded for any number of queries (BASELINE config 5).  The file is
// byte-identical; the returned RunStats has no path_lengths.
inline RunStats run_queries_write_paths(const DeviceGraph& dg, const AnyModel& model,
                                        const CostModelParams& params,
                                        std::span<const VertexId> queries, const RunOptions& opts,
                                        const std::string& path) {
    const dw_run_opts o = detail::to_opts(params, opts);
    const detail::ModelDesc m = detail::to_desc(model);
    dw_run_stats st{};
    check(dw_run_write_paths(dg.handle(), &m.d, queries.data(), queries.size(), &o, path.c_str(),
                             &st));
    return detail::to_stats(st);
}

inline RunStats run_queries_write_paths(const Graph& g, const AnyModel& model,
                                        const CostModelParams& params,
                                        std::span<const VertexId> queries, const RunOptions& opts,
                                        const std::string& path) {
    return run_queries_write_paths(*detail::cached(g), model, params, queries, opts, path);
}

// Same signature as dynwalk::run_queries (runtime.hpp:85-86).
inline RunResult run_queries(const Graph& g, const AnyModel& model, const CostModelParams& params,
                             std::span<const VertexId> queries, const RunOptions& opts) {
    return run_queries(*detail::cached(g), model, params, queries, opts);
}

// Same signature as dynwalk::selection_ratio_sweep (runtime.hpp:96-103): per
// alpha, the base graph's properties are regenerated as Pareto(alpha) with one
// draw seed for every row (runtime.cpp:249-278), the queries walk adaptively
// on the GPU, and the row reports the eRJS / eRVS selection split.
inline std::vector<SweepRow> selection_ratio_sweep(const Graph& base, const AnyModel& model,
                                                   const CostModelParams& params,
                                                   std::span<const double> alphas,
                                                   std::span<const VertexId> queries,
                                                   const RunOptions& opts) {
    RunOptions adaptive = opts;
    adaptive.mode = SamplerMode::Adaptive;
    WeightGenSpec spec;
    spec.kind = WeightGenSpec::Kind::Pareto;
    spec.seed = derive_seed(opts.seed, 0x7377656570ULL);  // shared by every row
    std::vector<SweepRow> rows;
    rows.reserve(alphas.size());
    for (const double alpha : alphas) {
        spec.alpha = alpha;
        const Graph g = synthesize_weights(base, spec);
        const DeviceGraph dg(g);  // one upload per row, never a stale cache entry
        const RunStats s = run_queries(dg, model, params, queries, adaptive).stats;
        const std::uint64_t total = s.select_erjs + s.select_ervs;
        SweepRow row{};
        row.alpha = alpha;
        row.erjs_steps = s.select_erjs;
        row.ervs_steps = s.select_ervs;
        if (total) {
            row.pct_erjs = 100.0 * static_cast<double>(s.select_erjs) / static_cast<double>(total);
            row.pct_ervs = 100.0 - row.pct_erjs;
        }
        rows.push_back(row);
    }
    return rows;
}

// Same signature as dynwalk::profile_edge_cost_ratio (cost_model.hpp:39-40);
// the random / sequential micro-passes run on device 0 with every
// ProfileConfig field forwarded.
inline CostModelParams profile_edge_cost_ratio(const Graph& g, const AnyModel& model,
                                               const ProfileConfig& cfg) {
    if (!(cfg.node_fraction > 0.0) || cfg.node_fraction > 1.0)
        throw Error("profile node_fraction must be in (0, 1]");
    if (cfg.neighbors_per_node == 0 || cfg.repetitions == 0)
        throw Error("profile neighbors_per_node and repetitions must be >= 1");
    const detail::ModelDesc m = detail::to_desc(model);
    const dw_profile_config pc{cfg.node_fraction, cfg.min_nodes, cfg.neighbors_per_node,
                               cfg.repetitions, cfg.seed};
    CostModelParams p;
    check(dw_calibrate_ex(detail::cached(g)->handle(), &m.d, &pc, &p.edge_cost_ratio));
    p.profiled = true;
    return p;
}

// The micro-pass ratio refined by timing the walk kernel itself at a few
// thresholds around it (dw_tune_ratio): the threshold decide_sampler should
// use on this device.  Not in the reference; same inputs as
// profile_edge_cost_ratio.
inline CostModelParams tune_edge_cost_ratio(const Graph& g, const AnyModel& model,
                                            const ProfileConfig& cfg,
                                            std::uint32_t walk_length = 80) {
    const detail::ModelDesc m = detail::to_desc(model);
    const dw_profile_config pc{cfg.node_fraction, cfg.min_nodes, cfg.neighbors_per_node,
                               cfg.repetitions, cfg.seed};
    CostModelParams p;
    check(dw_tune_ratio(detail::cached(g)->handle(), &m.d, &pc, walk_length, &p.edge_cost_ratio));
    p.profiled = true;
    return p;
}

}  // namespace dynwalk::gpu
