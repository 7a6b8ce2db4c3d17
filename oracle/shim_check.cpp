// shim_check.cpp -- TEST INFRASTRUCTURE: drives the product C++ shim
// (paper_2512_00705_b200/host/dynwalk_gpu.hpp) from inside the reference's own
// types.  Graphs come from the reference generators (gen.cpp, graph.cpp), the
// walk goes through dynwalk::gpu::run_queries with the reference signature,
// and the result (paths, lengths, RunStats) is written for tests/ to compare
// against tests/golden/ref_walks.json.
//
// usage: shim_check key=value ...   (see tests/test_gpu_shim.py)
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>

#include "dynwalk/dsl/parser.hpp"
#include "dynwalk/gen.hpp"
#include "dynwalk/rng.hpp"
#include "dynwalk_gpu.hpp"

namespace dw = dynwalk;

int main(int argc, char** argv) {
    std::map<std::string, std::string> kv;
    for (int i = 1; i < argc; ++i) {
        const char* eq = std::strchr(argv[i], '=');
        if (!eq) continue;
        kv[std::string(argv[i], static_cast<std::size_t>(eq - argv[i]))] = eq + 1;
    }
    auto get = [&](const char* k, const char* def) {
        auto it = kv.find(k);
        return it == kv.end() ? std::string(def) : it->second;
    };
    try {
        dw::TopologySpec topo;
        topo.kind = get("graph", "ba") == "ba" ? dw::TopologySpec::Kind::PreferentialAttachment
                                               : dw::TopologySpec::Kind::UniformRandom;
        topo.n = std::stoul(get("n", "300"));
        topo.deg = std::stoul(get("deg", "5"));
        topo.seed = std::stoull(get("gseed", "11"));
        topo.mirror = true;
        dw::Graph g = dw::generate_topology(topo);
        dw::WeightGenSpec w;
        w.kind = get("weights", "uniform") == "pareto" ? dw::WeightGenSpec::Kind::Pareto
                                                       : dw::WeightGenSpec::Kind::UniformReal;
        w.low = std::stod(get("low", "1"));
        w.high = std::stod(get("high", "5"));
        w.alpha = std::stod(get("alpha", "1"));
        w.seed = topo.seed + 100;
        g = dw::synthesize_weights(g, w);
        if (get("labels", "") != "") {
            const std::string l = get("labels", "");
            dw::WeightGenSpec ls;
            ls.kind = dw::WeightGenSpec::Kind::UniformIntLabel;
            ls.low = std::stod(l.substr(0, l.find(',')));
            ls.high = std::stod(l.substr(l.find(',') + 1));
            ls.seed = topo.seed + 200;
            g = dw::synthesize_weights(g, ls);
        }
        dw::ModelParams mp;
        mp.a = std::stod(get("a", "2"));
        mp.b = std::stod(get("b", "0.5"));
        mp.gamma = std::stod(get("gamma", "0.2"));
        mp.schema.clear();
        std::istringstream ss(get("schema", "0,1,2,3,4"));
        for (std::string t; std::getline(ss, t, ',');) mp.schema.push_back(std::stoul(t));
        std::string name = get("model", "node2vec");
        if (get("weighted", "1") == "0") name += "-unw";
        // dsl=<file>: a DslWalk parsed by the reference, compiled for the GPU by the shim
        const dw::AnyModel model = get("dsl", "") != ""
                                       ? dw::AnyModel(dw::DslWalk(dw::dsl::parse_file(get("dsl", "")), g))
                                       : dw::make_builtin_model(name, mp);

        dw::RunOptions opts;
        opts.mode = dw::parse_sampler_mode(get("mode", "adaptive"));
        opts.walk_length = std::stoul(get("L", "20"));
        opts.seed = std::stoull(get("seed", "7"));
        opts.workers = 1;
        dw::CostModelParams params;
        params.edge_cost_ratio = std::stod(get("ratio", "1.2"));
        const std::vector<dw::VertexId> queries = dw::all_vertices(g);

        // sweep=a1,a2,...: dynwalk::gpu::selection_ratio_sweep, one JSON row per alpha
        if (get("sweep", "") != "") {
            std::vector<double> alphas;
            std::istringstream as(get("sweep", ""));
            for (std::string t; std::getline(as, t, ',');) alphas.push_back(std::stod(t));
            const auto rows = dw::gpu::selection_ratio_sweep(g, model, params, alphas, queries, opts);
            std::cout << "[";
            for (std::size_t i = 0; i < rows.size(); ++i)
                std::cout << (i ? "," : "") << "{\"alpha\":" << rows[i].alpha
                          << ",\"erjs_steps\":" << rows[i].erjs_steps
                          << ",\"ervs_steps\":" << rows[i].ervs_steps
                          << ",\"pct_erjs\":" << rows[i].pct_erjs << "}";
            std::cout << "]" << std::endl;
            return 0;
        }

        // write=<file>: the one-pass GPU walk + write_paths; also writes
        // <file>.ref from the run_queries paths through the reference's write_paths
        if (get("write", "") != "") {
            const std::string file = get("write", "");
            const dw::RunStats ws =
                dw::gpu::run_queries_write_paths(g, model, params, queries, opts, file);
            const dw::RunResult rr2 = dw::gpu::run_queries(g, model, params, queries, opts);
            dw::write_paths(file + ".ref", rr2.paths);
            std::cout << "{\"steps\":" << ws.steps << ",\"steps_rq\":" << rr2.stats.steps << "}"
                      << std::endl;
            return 0;
        }

        const dw::RunResult rr = dw::gpu::run_queries(g, model, params, queries, opts);

        const std::string out = get("out", "shim_out");
        std::ofstream pf(out + ".paths", std::ios::binary);
        const std::uint32_t stride = opts.walk_length + 1;
        for (const auto& p : rr.paths)
            for (std::uint32_t k = 0; k < stride; ++k) {
                const std::uint32_t v = k < p.size() ? p[k] : dw::kInvalidVertex;
                pf.write(reinterpret_cast<const char*>(&v), 4);
            }
        std::ofstream lf(out + ".lengths", std::ios::binary);
        for (const auto& p : rr.paths) {
            const std::uint32_t n = static_cast<std::uint32_t>(p.size());
            lf.write(reinterpret_cast<const char*>(&n), 4);
        }
        const dw::RunStats& s = rr.stats;
        std::cout << "{\"queries\":" << s.queries << ",\"query_errors\":" << s.query_errors
                  << ",\"dead_ends\":" << s.dead_ends << ",\"steps\":" << s.steps
                  << ",\"select_ervs\":" << s.select_ervs << ",\"select_erjs\":" << s.select_erjs
                  << ",\"trials\":" << s.trials << ",\"weight_reads\":" << s.weight_reads
                  << ",\"rng_draws\":" << s.rng_draws << ",\"erjs_fallbacks\":" << s.erjs_fallbacks
                  << ",\"selection_by_degree\":[";
        for (std::size_t b = 0; b < s.selection_by_degree.size(); ++b)
            std::cout << (b ? "," : "") << "[" << s.selection_by_degree[b][0] << ","
                      << s.selection_by_degree[b][1] << "]";
        std::cout << "]}" << std::endl;
        // profile through the shim as well (cost_model.hpp:39-40 signature)
        if (get("profile", "0") == "1") {
            dw::ProfileConfig cfg;
            cfg.seed = 1;
            const dw::CostModelParams p = dw::gpu::profile_edge_cost_ratio(g, model, cfg);
            std::cerr << "profiled_ratio=" << p.edge_cost_ratio << std::endl;
        }
        return 0;
    } catch (const dw::Error& e) {
        std::cerr << "dynwalk::Error: " << e.what() << std::endl;
        return 2;
    }
}
