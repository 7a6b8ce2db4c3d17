/*
 * dynwalk_b200.h -- C ABI of the B200-native dynamic random-walk engine.
 *
 * This is the drop-in boundary for the reference's hot path (BASELINE.json
 * north_star).  Plain pointers and sizes only, no C++ or torch
 * types.  Each entry point names the reference interface it replaces
 * (paths relative to /root/reference/proj).  The C++ shim with the reference's
 * exact signatures (dynwalk::gpu::run_queries, ...) is header-only on top of
 * this ABI: paper_2512_00705_b200/host/dynwalk_gpu.hpp; INTEGRATION.md shows
 * the binding.
 *
 * Conventions
 *  - Every function returns 0 on success or a negative DW_E* code; the
 *    message (reference wording where one exists) is in dw_last_error(),
 *    thread-local.  No exception crosses the ABI.
 *  - The caller owns all host arrays; dw_graph_create copies them.  The
 *    handle owns one device replica of the graph per device (read-only after
 *    create; graph.hpp:47 "Immutable after construction").
 *  - dw_run blocks; it drives every device of the handle from the calling
 *    thread with one stream per device.  Reentrant on distinct handles.
 */
#ifndef DYNWALK_B200_H
#define DYNWALK_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DW_ABI_VERSION 2
#define DW_INVALID_VERTEX 0xFFFFFFFFu /* kInvalidVertex, types.hpp:13 */

enum {
    DW_OK = 0,
    DW_EINVAL = -1,   /* bad argument / contract violation (dynwalk::Error) */
    DW_ECUDA = -2,    /* CUDA runtime failure (no device, OOM, launch) */
    DW_EMODEL = -3,   /* model contract violation inside the walk */
    DW_EUNSUPPORTED = -4
};

/* Graph CSR as dynwalk::Graph holds it (graph.hpp:55-126, 257-263). */
typedef struct dw_graph_desc {
    uint32_t num_vertices;
    uint64_t num_edges;
    const uint64_t* row_offsets;   /* [nv+1] */
    const uint32_t* col_indices;   /* [ne], each slice sorted by target */
    const float* edge_props;       /* [ne], > 0 and finite */
    const uint16_t* edge_labels;   /* [ne] or NULL (graph.hpp:226-228: label 0) */
    const double* node_prop_max;   /* [nv] or NULL: recomputed (graph.cpp:83-98) */
    const double* node_prop_sum;   /* [nv] or NULL: recomputed, left-to-right */
} dw_graph_desc;

/* Synthetic R-MAT workload built on the device. */
typedef struct dw_rmat_desc {
    uint32_t scale;         /* V = 2^scale */
    uint32_t edge_factor;   /* edge_factor/2 * V undirected samples, mirrored */
    uint64_t seed;          /* topology: derive_seed(seed, "rmat") */
    int weights;            /* 0 uniform[low,high), 2 pareto(alpha), -1 none (1.0) */
    double low, high, alpha;
    uint64_t weight_seed;
    int labels;             /* 1: labels uniform in [label_low, label_high] */
    uint32_t label_low, label_high;
    uint64_t label_seed;
} dw_rmat_desc;

typedef struct dw_graph_s* dw_graph_t;

/* Builtin models (models.hpp:33-164); a user model compiles in as a device
 * functor (paper_2512_00705_b200/csrc/dw_models.cuh). */
enum {
    DW_MODEL_STATIC = 0,
    DW_MODEL_NODE2VEC = 1,
    DW_MODEL_METAPATH = 2,
    DW_MODEL_PR2 = 3,
    DW_MODEL_CUSTOM = 4 /* a DslWalk compiled with dw_model_compile */
};

/* A DslWalk model (models.hpp:170-198) compiled into the walk kernel. */
typedef struct dw_custom_model_s* dw_custom_model_t;

typedef struct dw_model_desc {
    int kind;
    int weighted;
    double a, b;              /* node2vec return / in-out parameters */
    double gamma;             /* second-order pagerank mixing */
    const uint16_t* schema;   /* metapath label schema */
    uint32_t schema_len;      /* <= DW_MAX_SCHEMA */
    dw_custom_model_t custom; /* DW_MODEL_CUSTOM only */
} dw_model_desc;
#define DW_MAX_SCHEMA 128

/* SamplerMode (runtime.hpp:15).  ITS/ALS are CPU comparison baselines and
 * are rejected with DW_EUNSUPPORTED. */
enum {
    DW_MODE_ADAPTIVE = 0,
    DW_MODE_FORCE_ERVS = 1,
    DW_MODE_FORCE_ERJS = 2,
    DW_MODE_ERVS_NOJUMP = 3,
    DW_MODE_FORCE_ITS = 4,
    DW_MODE_FORCE_ALS = 5
};

/* RunOptions (runtime.hpp:17-32) + CostModelParams (cost_model.hpp:19-22). */
typedef struct dw_run_opts {
    int mode;
    uint32_t walk_length;          /* default 80 */
    uint64_t seed;
    uint64_t erjs_cap_per_degree;  /* default 64 */
    double edge_cost_ratio;        /* decide_sampler threshold, > 0 */
    uint64_t qid_base;             /* global id of queries[0] (RNG key; sharding) */
    /* [nq] global walker ids (RNG keys) of the queries, or NULL: qid_base + i.
     * Lets one shard of a partitioned run walk any subset of the global ids
     * (hash-partitioned walkers) with the streams, and so the
     * paths, of the unpartitioned run.  Host memory for dw_run /
     * dw_run_compact / dw_run_write_paths, device memory for dw_run_device. */
    const uint64_t* qids;
    /* Tier-2 eRJS hand-off (FlexiWalker's bounded per-lane rejection,
     * PAPER.md:760-765; not in the reference): when > 0, an eRJS step that
     * has run max(32, ceil(erjs_handoff * d / edge_cost_ratio)) trials
     * without acceptance -- trials worth erjs_handoff reservoir passes over
     * the row under the cost model (cost_model.hpp:46-56) -- falls back to
     * the reservoir pass exactly as the reference's cap overrun does
     * (samplers.hpp:174-177).  The sampled distribution is unchanged (a
     * mixture of two exact samplers); paths equal the oracle run with the
     * same rule, not the reference's.  0 (default) = the reference's rule,
     * bit-exact. */
    double erjs_handoff;
} dw_run_opts;

/* RunStats (runtime.hpp:53-73) minus host-only fields. */
typedef struct dw_run_stats {
    uint64_t queries, query_errors, dead_ends, steps;
    uint64_t select_ervs, select_erjs, select_its, select_als;
    uint64_t trials, weight_reads, rng_draws, erjs_fallbacks;
    uint64_t selection_by_degree[33][2]; /* [floor(log2 d)][0 ervs, 1 erjs] */
    double kernel_ms;                    /* device time of the walk, max over devices */
    double total_ms;                     /* incl. H2D/D2H inside dw_run */
    uint64_t kernel_launches;            /* walk-path kernels launched */
    uint64_t algorithmic_bytes;          /* SURVEY §8(d) minimal-sector bytes of the walk */
} dw_run_stats;

int dw_abi_version(void);
const char* dw_last_error(void);
int dw_device_count(int* n);

/* Replaces Graph construction + the implicit sharing of `const Graph&`
 * across workers (runtime.cpp:192-247): one device replica per device. */
int dw_graph_create(const dw_graph_desc* desc, const int* devices, int ndev, dw_graph_t* out);
int dw_graph_generate_rmat(const dw_rmat_desc* desc, const int* devices, int ndev,
                           dw_graph_t* out);
/* Loads a DWG1 binary CSR cache (dynwalk::save_binary, graph.cpp:243-256)
 * straight onto the devices: the file streams through pinned staging buffers
 * into device arrays, and Graph::build's invariants (graph.cpp:15-81: slices
 * stable-sorted by target, referenced ids extend the vertex count) are
 * re-established on the device instead of the host round-trip that
 * load_binary makes (graph.cpp:258-291).  Error messages follow load_binary. */
int dw_graph_load_dwg1(const char* path, const int* devices, int ndev, dw_graph_t* out);
int dw_graph_destroy(dw_graph_t g);
int dw_graph_info(dw_graph_t g, uint32_t* num_vertices, uint64_t* num_edges, int* has_labels,
                  uint32_t* max_degree);
/* Copies replica 0 back to host arrays (any may be NULL). */
int dw_graph_download(dw_graph_t g, uint64_t* row_offsets, uint32_t* col_indices,
                      float* edge_props, uint16_t* edge_labels, double* node_prop_max,
                      double* node_prop_sum);

/* ProfileConfig (cost_model.hpp:9-15). */
typedef struct dw_profile_config {
    double node_fraction;         /* share of nodes probed per round, (0, 1]; default 0.01 */
    uint32_t min_nodes;           /* probe at least this many (graph permitting); default 64 */
    uint32_t neighbors_per_node;  /* >= 1; default 32 */
    uint32_t repetitions;         /* >= 1; default 5 (the median is returned) */
    uint64_t seed;
} dw_profile_config;

/* Replaces profile_edge_cost_ratio (cost_model.hpp:39-40, cost_model.cpp:37-126):
 * random-neighbour vs sequential weight evaluation timed on device 0, the
 * median per-edge time ratio over cfg->repetitions.  Errors follow the
 * reference (node_fraction outside (0, 1], zero neighbours or repetitions,
 * no node with out-edges). */
int dw_calibrate_ex(dw_graph_t g, const dw_model_desc* model, const dw_profile_config* cfg,
                    double* ratio);
/* The B200 refinement of dw_calibrate_ex: the micro-passes price an eRJS
 * trial and an eRVS visit in isolation, but the walk kernel overlaps both with
 * other lanes' phases, so the best threshold is found by walking.  Starting
 * from the micro-pass ratio r0, times the walk kernel itself (adaptive,
 * `walk_length` steps, 0 = 80) on a sample of uniformly drawn start vertices
 * at r0 x {1/2, 1/sqrt2, 1, sqrt2, 2} (median of min(repetitions, 3)
 * launches each) and returns the vertex of the least-squares parabola through
 * walker-steps/s over log2(ratio), kept inside that range (the best sampled
 * ratio if the fit is not concave).  Decisions stay the reference's
 * decide_sampler; only the threshold it is given changes. */
int dw_tune_ratio(dw_graph_t g, const dw_model_desc* model, const dw_profile_config* cfg,
                  uint32_t walk_length, double* ratio);
/* dw_calibrate_ex with the ProfileConfig defaults and `seed`. */
int dw_calibrate(dw_graph_t g, const dw_model_desc* model, uint64_t seed, double* ratio);

/* Compiles a DslWalk weight function into the walk kernel.
 * `source` is the CUDA model functor that paper_2512_00705_b200/host/
 * dsl_codegen.hpp generates from the reference's parsed program and analysis
 * (dsl::Program, dsl::AnalysisResult); NVRTC compiles it against the kernel
 * template this library was built from, for every sampler mode.  max_steps is
 * DslWalk::max_steps(); flags bit 0: the estimators read per-node label
 * MAX/SUM (built on the device at first use).  No interpretation happens on
 * the device.  Errors: DW_EUNSUPPORTED without NVRTC, DW_EMODEL with the
 * compiler log. */
#define DW_CUSTOM_LABEL_AGGREGATES 1u
int dw_model_compile(const char* source, uint32_t max_steps, uint32_t flags,
                     dw_custom_model_t* out);
int dw_model_free(dw_custom_model_t model);

/* Replaces run_queries (runtime.hpp:85-86, runtime.cpp:192-247).
 * queries: host [nq].  paths: host [nq][walk_length+1], DW_INVALID_VERTEX
 * padded, or NULL (discard).  lengths: host [nq] (0 = query error) or NULL.
 * Walkers are cut into batches that go round-robin over the handle's devices;
 * every device walks while the host drains finished batches in query order,
 * and the output does not depend on the device count (the RNG is keyed by the
 * global walker id). */
int dw_run(dw_graph_t g, const dw_model_desc* model, const uint32_t* queries, uint64_t nq,
           const dw_run_opts* opts, uint32_t* paths, uint32_t* lengths, dw_run_stats* stats);

/* run_queries with compact output, the layout of RunResult.paths
 * (vector<vector<VertexId>>, runtime.hpp:75-78) flattened: path i is
 * flat[offsets[i] .. offsets[i+1]), empty on a query error.  offsets: host
 * [nq + 1]; flat: host, flat_capacity ids (nq * (walk_length + 1) always
 * suffices).  Only the ids that exist cross PCIe, not the padding. */
int dw_run_compact(dw_graph_t g, const dw_model_desc* model, const uint32_t* queries,
                   uint64_t nq, const dw_run_opts* opts, uint64_t* offsets, uint32_t* flat,
                   uint64_t flat_capacity, dw_run_stats* stats);

/* run_queries + write_paths (runtime.cpp:280-291) as one streamed sink: the
 * paths are formatted as text on the device ("id id ... id\n" per query in
 * query order, "\n" for an empty path) and written batch by batch while the
 * next batches walk; device and host memory stay bounded for any nq.  The
 * file is byte-identical to write_paths on the same paths. */
int dw_run_write_paths(dw_graph_t g, const dw_model_desc* model, const uint32_t* queries,
                       uint64_t nq, const dw_run_opts* opts, const char* path,
                       dw_run_stats* stats);

/* Device-resident variant on replica `replica`: d_queries / d_paths /
 * d_lengths are device pointers on that device (d_paths, d_lengths may be
 * NULL), `stream` a cudaStream_t (NULL = the replica's stream).  Enqueues and
 * returns; stats are valid after dw_run_device_sync.  When every path length
 * is known before the walk (node2vec with a, b > 0, adaptive or force-erjs,
 * no edge into a vertex without neighbours, >= 2^20 queries) the walkers that
 * cannot move are written first and the walk runs over the others; the call
 * then waits for that ~1 ms pre-pass (the walk's grid is sized by its count)
 * before it enqueues the walk, and dw_run_device_sync verifies the lengths
 * (re-running every walker if one walk ended early). */
int dw_run_device(dw_graph_t g, int replica, const dw_model_desc* model,
                  const uint32_t* d_queries, uint64_t nq, const dw_run_opts* opts,
                  uint32_t* d_paths, uint32_t* d_lengths, void* stream);
int dw_run_device_sync(dw_graph_t g, int replica, dw_run_stats* stats);

/* Self-test of the device math the reservoir samplers use (samplers.hpp:
 * 82-97 std::log / std::exp): y[i] = log(x[i]) (fn 0) or exp(x[i]) (fn 1)
 * computed by CUDA libdevice on device 0, host arrays in and out.  Lets the
 * test suite measure where libdevice and the host libm disagree. */
int dw_selftest_math(int fn, const double* x, double* y, uint64_t n);

/* Pinned host buffers for dw_run (cudaMallocHost). */
int dw_host_alloc(size_t bytes, void** out);
int dw_host_free(void* p);

#ifdef __cplusplus
}
#endif
#endif
