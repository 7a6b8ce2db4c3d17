// ref_harness.cpp -- extern "C" harness over the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile together with the
// reference's own translation units (read in place from /root/reference/proj,
// never copied) into oracle/_ref/libdynwalk_ref.so.  Used by tests/ to pin the
// C oracle and the GPU path against the reference itself, and by bench.py's
// --impl reference leg (the reference CPU run_queries, timed on host cores).
//
// Two walk drivers:
//  * ref_run            -> dynwalk::run_queries (src/runtime.cpp:192-247),
//                          stock mt19937 streams per query;
//  * ref_run_philox     -> the reference walk loop (src/runtime.cpp:59-153)
//                          restated over the reference's own public templates
//                          decide_sampler / sample_erjs / sample_ervs /
//                          sample_ervs_nojump, with a Philox counter Rng keyed
//                          by (seed, walker, step) -- the stream the GPU uses.
//                          (walk_query itself sits in an anonymous namespace
//                          and hard-codes CountingRng, runtime.cpp:37,65.)
#include <atomic>
#include <chrono>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "dynwalk/cost_model.hpp"
#include "dynwalk/gen.hpp"
#include "dynwalk/graph.hpp"
#include "dynwalk/models.hpp"
#include "dynwalk/rng.hpp"
#include "dynwalk/runtime.hpp"
#include "dynwalk/dsl/parser.hpp"
#include "dynwalk/dsl/analyzer.hpp"
#include "dsl_codegen.hpp"
#include "dynwalk/samplers.hpp"

#include "oracle.h"

namespace dw = dynwalk;

namespace {

thread_local std::string tl_error;
// DSL program for ModelDesc kind 4 (ref_set_dsl_source); parsed with the
// reference's own parser, so the reference's DslWalk is what runs
std::string tl_dsl_source;  // set before a run (tests are single-threaded)

struct ModelDesc {
    int kind;
    int weighted;
    double a, b, gamma;
    const std::uint16_t* schema;
    std::uint32_t schema_len;
};

dw::AnyModel make_model(const ModelDesc& d, const dw::Graph* g = nullptr) {
    if (d.kind == 4) {
        if (!g) throw dw::Error("DSL model needs the graph");
        return dw::DslWalk(dw::dsl::parse(tl_dsl_source, "<test>"), *g);
    }
    switch (d.kind) {
    case 0: return dw::StaticWalk{d.weighted != 0};
    case 1: return dw::Node2Vec{d.a, d.b, d.weighted != 0};
    case 2: {
        std::vector<dw::Label> schema(d.schema, d.schema + d.schema_len);
        return dw::MetaPath{schema, d.weighted != 0};
    }
    case 3: return dw::SecondOrderPr{d.gamma, d.weighted != 0};
    }
    throw dw::Error("unknown model kind");
}

// Philox Rng satisfying the reference Rng concept (rng.hpp:31-57 bit maps).
class PhiloxRng {
public:
    PhiloxRng(std::uint64_t seed, std::uint64_t qid) : seed_(seed), qid_(qid) {}
    void start_step(std::uint32_t step) {
        step_ = step;
        idx_ = 0;
    }
    std::uint64_t next_u64() {
        ++draws_;
        return orc_walker_draw(seed_, qid_, step_, idx_++);
    }
    double uniform01() { return static_cast<double>(next_u64() >> 11) * 0x1.0p-53; }
    double open01() { return (static_cast<double>(next_u64() >> 11) + 0.5) * 0x1.0p-53; }
    std::uint64_t bounded(std::uint64_t n) {
        return static_cast<std::uint64_t>((static_cast<unsigned __int128>(next_u64()) * n) >> 64);
    }
    std::uint64_t draw_count() const { return draws_; }

private:
    std::uint64_t seed_, qid_;
    std::uint32_t step_ = 0;
    std::uint64_t idx_ = 0;
    std::uint64_t draws_ = 0;
};

void bucket(orc_stats& s, std::uint32_t degree, bool erjs) {  // runtime.cpp:42-46
    std::uint32_t b = 0;
    while (b < 31 && (1u << (b + 1)) <= degree) ++b;
    ++s.sel_by_deg[b][erjs ? 1 : 0];
}

template <typename Model>
void walk_philox(const dw::Graph& g, const Model& model, const dw::CostModelParams& params,
                 int mode, std::uint32_t walk_length, std::uint64_t seed, std::uint64_t cap,
                 dw::VertexId start, std::uint64_t qid, std::vector<dw::VertexId>& path,
                 orc_stats& ls) {
    dw::WalkerState st;
    st.reset(qid, start);
    PhiloxRng rng(seed, qid);
    const std::uint32_t target = std::min(walk_length, model.max_steps());
    const bool boundable = model.estimation_flag() != dw::EstimationFlag::None;
    while (st.step < target) {
        const std::uint32_t d = g.degree(st.cur);
        if (d == 0) break;
        rng.start_step(st.step);
        dw::SampleOutcome out;
        if (mode == ORC_ADAPTIVE) {
            const dw::SamplerDecision dec = dw::decide_sampler(g, st, model, params);
            const bool erjs = dec.choice == dw::SamplerChoice::Erjs;
            bucket(ls, d, erjs);
            if (erjs) {
                ++ls.select_erjs;
                out = dw::sample_erjs(g, st, model, rng, dw::BoundEstimate{dec.est_max}, cap);
            } else {
                ++ls.select_ervs;
                out = dw::sample_ervs(g, st, model, rng);
            }
        } else if (mode == ORC_FORCE_ERVS) {
            ++ls.select_ervs;
            bucket(ls, d, false);
            out = dw::sample_ervs(g, st, model, rng);
        } else if (mode == ORC_ERVS_NOJUMP) {
            ++ls.select_ervs;
            bucket(ls, d, false);
            out = dw::sample_ervs_nojump(g, st, model, rng);
        } else if (mode == ORC_FORCE_ERJS) {
            if (!boundable) {
                ++ls.select_ervs;
                bucket(ls, d, false);
                out = dw::sample_ervs(g, st, model, rng);
            } else {
                ++ls.select_erjs;
                bucket(ls, d, true);
                out = dw::sample_erjs(g, st, model, rng,
                                      dw::BoundEstimate{model.estimate_bound(g, st)}, cap);
            }
        } else {
            throw dw::Error("unsupported sampler mode");
        }
        ++ls.steps;
        ls.trials += out.trials;
        ls.weight_reads += out.weight_reads;
        ls.rng_draws += out.rng_draws;
        if (out.fell_back) ++ls.erjs_fallbacks;
        if (out.dead_end()) {
            ++ls.dead_ends;
            break;
        }
        st.advance(g, out.next);
    }
    path = std::move(st.path);
}

void add_stats(orc_stats& into, const orc_stats& f) {
    into.queries += f.queries;
    into.query_errors += f.query_errors;
    into.dead_ends += f.dead_ends;
    into.steps += f.steps;
    into.select_ervs += f.select_ervs;
    into.select_erjs += f.select_erjs;
    into.trials += f.trials;
    into.weight_reads += f.weight_reads;
    into.rng_draws += f.rng_draws;
    into.erjs_fallbacks += f.erjs_fallbacks;
    for (int b = 0; b < 33; ++b)
        for (int k = 0; k < 2; ++k) into.sel_by_deg[b][k] += f.sel_by_deg[b][k];
}

void emit_paths(const std::vector<std::vector<dw::VertexId>>& paths, std::uint32_t stride,
                std::uint32_t* out, std::uint32_t* lengths) {
    for (std::size_t i = 0; i < paths.size(); ++i) {
        if (lengths) lengths[i] = static_cast<std::uint32_t>(paths[i].size());
        if (!out) continue;
        std::uint32_t* row = out + i * stride;
        for (std::uint32_t k = 0; k < stride; ++k)
            row[k] = k < paths[i].size() ? paths[i][k] : dw::kInvalidVertex;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return tl_error.c_str(); }

void* ref_graph_from_csr(std::uint32_t nv, std::uint64_t ne, const std::uint64_t* row,
                         const std::uint32_t* col, const float* prop,
                         const std::uint16_t* label) {
    try {
        std::vector<dw::EdgeRecord> edges(ne);
        for (std::uint32_t v = 0; v < nv; ++v)
            for (std::uint64_t e = row[v]; e < row[v + 1]; ++e)
                edges[e] = dw::EdgeRecord{v, col[e], prop[e], label ? label[e] : dw::Label{0}};
        return new dw::Graph(dw::Graph::build(std::move(edges), label != nullptr, false, nv));
    } catch (const std::exception& ex) {
        tl_error = ex.what();
        return nullptr;
    }
}

// kind 0 = uniform, 1 = ba (gen.cpp:96-103)
void* ref_graph_gen(int kind, std::uint32_t n, std::uint32_t deg, std::uint64_t seed,
                    int mirror) {
    try {
        dw::TopologySpec spec;
        spec.kind = kind == 1 ? dw::TopologySpec::Kind::PreferentialAttachment
                              : dw::TopologySpec::Kind::UniformRandom;
        spec.n = n;
        spec.deg = deg;
        spec.seed = seed;
        spec.mirror = mirror != 0;
        return new dw::Graph(dw::generate_topology(spec));
    } catch (const std::exception& ex) {
        tl_error = ex.what();
        return nullptr;
    }
}

// kind 0 uniform, 1 labels, 2 pareto, 3 degree (graph.cpp:302-352)
int ref_synth(void* gp, int kind, double low, double high, double alpha, std::uint64_t seed) {
    try {
        dw::WeightGenSpec spec;
        spec.kind = kind == 0   ? dw::WeightGenSpec::Kind::UniformReal
                    : kind == 1 ? dw::WeightGenSpec::Kind::UniformIntLabel
                    : kind == 2 ? dw::WeightGenSpec::Kind::Pareto
                                : dw::WeightGenSpec::Kind::DegreeBased;
        spec.low = low;
        spec.high = high;
        spec.alpha = alpha;
        spec.seed = seed;
        auto* g = static_cast<dw::Graph*>(gp);
        *g = dw::synthesize_weights(*g, spec);
        return 0;
    } catch (const std::exception& ex) {
        tl_error = ex.what();
        return -1;
    }
}

void ref_set_dsl_source(const char* src) { tl_dsl_source = src ? src : ""; }

// The product's DSL -> CUDA codegen (host/dsl_codegen.hpp) applied to the
// reference's parse and analysis of `src`; test infrastructure for the GPU
// DSL parity tests.  Returns the source length (or -1), writes at most cap
// bytes.
long ref_dsl_codegen(const char* src, char* out, std::uint64_t cap, std::uint32_t* max_steps,
                     std::uint32_t* flags) {
    try {
        const dw::dsl::Program prog = dw::dsl::parse(src, "<test>");
        const dw::dsl::AnalysisResult res = dw::dsl::analyze(prog);
        std::uint32_t ms = 0xFFFFFFFFu;
        for (const auto& [name, value] : prog.scalar_params)
            if (name == "walk_length") ms = static_cast<std::uint32_t>(value);
        const auto code = dw::gpu::detail::dsl_codegen(prog, res, ms);
        if (max_steps) *max_steps = ms;
        if (flags) *flags = code.label_aggregates ? 1u : 0u;
        if (out && cap) {
            const std::size_t n = std::min<std::size_t>(code.source.size(), cap - 1);
            std::memcpy(out, code.source.data(), n);
            out[n] = '\0';
        }
        return static_cast<long>(code.source.size());
    } catch (const std::exception& ex) {
        tl_error = ex.what();
        return -1;
    }
}

// DWG1 binary CSR cache (graph.cpp:217-300), for the device loader's tests
int ref_save_binary(const void* gp, const char* path) {
    try {
        dw::save_binary(*static_cast<const dw::Graph*>(gp), path);
        return 0;
    } catch (const std::exception& ex) {
        tl_error = ex.what();
        return -1;
    }
}

void* ref_load_binary(const char* path) {
    try {
        return new dw::Graph(dw::load_binary(path));
    } catch (const std::exception& ex) {
        tl_error = ex.what();
        return nullptr;
    }
}

void ref_graph_free(void* g) { delete static_cast<dw::Graph*>(g); }

void ref_graph_dims(const void* gp, std::uint32_t* nv, std::uint64_t* ne, int* has_labels) {
    const auto* g = static_cast<const dw::Graph*>(gp);
    *nv = g->num_vertices();
    *ne = g->num_edges();
    *has_labels = g->has_labels() ? 1 : 0;
}

void ref_graph_copy(const void* gp, std::uint64_t* row, std::uint32_t* col, float* prop,
                    std::uint16_t* label, double* nmax, double* nsum) {
    const auto* g = static_cast<const dw::Graph*>(gp);
    const auto r = g->row_offsets();
    const auto c = g->col_indices();
    const auto p = g->edge_props();
    if (row) std::memcpy(row, r.data(), r.size_bytes());
    if (col) std::memcpy(col, c.data(), c.size_bytes());
    if (prop) std::memcpy(prop, p.data(), p.size_bytes());
    if (label && g->has_labels()) {
        const auto l = g->edge_labels();
        std::memcpy(label, l.data(), l.size_bytes());
    }
    for (std::uint32_t v = 0; v < g->num_vertices(); ++v) {
        if (nmax) nmax[v] = g->node_prop_max(v);
        if (nsum) nsum[v] = g->node_prop_sum(v);
    }
}

// dynwalk::run_queries, stock reference path (mt19937 per query).
int ref_run(const void* gp, const ModelDesc* md, int mode, std::uint32_t walk_length,
            std::uint32_t workers, std::uint64_t seed, std::uint64_t cap, double ratio,
            const std::uint32_t* queries, std::uint64_t nq, std::uint32_t* paths,
            std::uint32_t* lengths, orc_stats* stats, double* wall_ms) {
    try {
        const auto* g = static_cast<const dw::Graph*>(gp);
        dw::RunOptions opts;
        opts.mode = mode == ORC_ADAPTIVE     ? dw::SamplerMode::Adaptive
                    : mode == ORC_FORCE_ERVS ? dw::SamplerMode::ForceErvs
                    : mode == ORC_FORCE_ERJS ? dw::SamplerMode::ForceErjs
                                             : dw::SamplerMode::ErvsNoJump;
        opts.walk_length = walk_length;
        opts.workers = workers;
        opts.seed = seed;
        opts.erjs_cap_per_degree = cap;
        dw::CostModelParams params;
        params.edge_cost_ratio = ratio;
        const dw::AnyModel model = make_model(*md, g);
        const dw::RunResult rr =
            dw::run_queries(*g, model, params, std::span<const dw::VertexId>(queries, nq), opts);
        emit_paths(rr.paths, walk_length + 1, paths, lengths);
        if (stats) {
            std::memset(stats, 0, sizeof(*stats));
            const dw::RunStats& s = rr.stats;
            stats->queries = s.queries;
            stats->query_errors = s.query_errors;
            stats->dead_ends = s.dead_ends;
            stats->steps = s.steps;
            stats->select_ervs = s.select_ervs;
            stats->select_erjs = s.select_erjs;
            stats->trials = s.trials;
            stats->weight_reads = s.weight_reads;
            stats->rng_draws = s.rng_draws;
            stats->erjs_fallbacks = s.erjs_fallbacks;
            for (int b = 0; b < 33; ++b)
                for (int k = 0; k < 2; ++k) stats->sel_by_deg[b][k] = s.selection_by_degree[b][k];
        }
        if (wall_ms) *wall_ms = rr.stats.wall_ms;
        return 0;
    } catch (const std::exception& ex) {
        tl_error = ex.what();
        return -1;
    }
}

// Reference walk loop over the reference sampler templates, Philox streams.
int ref_run_philox(const void* gp, const ModelDesc* md, int mode, std::uint32_t walk_length,
                   std::uint32_t workers, std::uint64_t seed, std::uint64_t cap, double ratio,
                   const std::uint32_t* queries, std::uint64_t nq, std::uint32_t* paths,
                   std::uint32_t* lengths, orc_stats* stats, double* wall_ms) {
    try {
        const auto* g = static_cast<const dw::Graph*>(gp);
        dw::CostModelParams params;
        params.edge_cost_ratio = ratio;
        const dw::AnyModel model = make_model(*md, g);
        std::vector<std::vector<dw::VertexId>> out(nq);
        orc_stats total;
        std::memset(&total, 0, sizeof total);
        std::atomic<std::uint64_t> next{0};
        std::mutex mu;
        std::exception_ptr first;
        const auto t0 = std::chrono::steady_clock::now();
        auto worker = [&]() {
            orc_stats ls;
            std::memset(&ls, 0, sizeof ls);
            try {
                for (;;) {
                    const std::uint64_t i = next.fetch_add(1, std::memory_order_relaxed);
                    if (i >= nq) break;
                    ++ls.queries;
                    if (queries[i] >= g->num_vertices()) {
                        ++ls.query_errors;
                        continue;
                    }
                    std::visit(
                        [&](const auto& m) {
                            walk_philox(*g, m, params, mode, walk_length, seed, cap, queries[i],
                                        i, out[i], ls);
                        },
                        model);
                }
            } catch (...) {
                std::lock_guard<std::mutex> lk(mu);
                if (!first) first = std::current_exception();
            }
            std::lock_guard<std::mutex> lk(mu);
            add_stats(total, ls);
        };
        std::vector<std::thread> pool;
        for (std::uint32_t w = 1; w < workers; ++w) pool.emplace_back(worker);
        worker();
        for (auto& t : pool) t.join();
        if (first) std::rethrow_exception(first);
        const auto t1 = std::chrono::steady_clock::now();
        emit_paths(out, walk_length + 1, paths, lengths);
        if (stats) *stats = total;
        if (wall_ms) *wall_ms = std::chrono::duration<double, std::milli>(t1 - t0).count();
        return 0;
    } catch (const std::exception& ex) {
        tl_error = ex.what();
        return -1;
    }
}

// profile_edge_cost_ratio (cost_model.cpp:37-126) with the CLI's defaults.
double ref_profile_ratio(const void* gp, const ModelDesc* md, std::uint64_t seed) {
    try {
        dw::ProfileConfig cfg;
        cfg.seed = seed;
        const auto* g = static_cast<const dw::Graph*>(gp);
        return dw::profile_edge_cost_ratio(*g, make_model(*md, g), cfg)
            .edge_cost_ratio;
    } catch (const std::exception& ex) {
        tl_error = ex.what();
        return -1.0;
    }
}

}  // extern "C"
