/*
 * oracle.h -- CPU restatement of the reference dynamic random-walk path.
 *
 * TEST INFRASTRUCTURE ONLY.  This library is the checker for the B200 product
 * path (paper_2512_00705_b200/csrc).  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product
 * never links, loads or calls anything in oracle/.
 *
 * Every function cites the reference file:line it restates; paths are
 * relative to /root/reference/proj.  Parity is pinned two ways (see
 * DESIGN.md "Oracle"):
 *   1. tests/golden/stats_walk.txt (the reference CLI golden) is reproduced
 *      counter-for-counter in mt19937 mode;
 *   2. paths + counters equal the reference's own run_queries
 *      (oracle/_ref/libdynwalk_ref.so, built from the reference sources) on
 *      randomized graphs, all modes, all builtin models.
 */
#ifndef DYNWALK_ORACLE_H
#define DYNWALK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ORC_INVALID 0xFFFFFFFFu

/* CSR graph, same arrays as dynwalk::Graph (include/dynwalk/graph.hpp:55-126). */
typedef struct orc_graph {
    uint32_t nv;
    uint64_t ne;
    uint64_t* row;   /* nv+1 */
    uint32_t* col;   /* ne, each slice sorted by target */
    float* prop;     /* ne */
    uint16_t* label; /* ne or NULL */
    double* nmax;    /* nv: max prop per slice, ascending edge order */
    double* nsum;    /* nv: left-to-right double sum */
} orc_graph;

enum { ORC_STATIC = 0, ORC_NODE2VEC = 1, ORC_METAPATH = 2, ORC_PR2 = 3 };
enum { ORC_ADAPTIVE = 0, ORC_FORCE_ERVS = 1, ORC_FORCE_ERJS = 2, ORC_ERVS_NOJUMP = 3 };
enum { ORC_RNG_MT19937 = 0, ORC_RNG_PHILOX = 1 };

typedef struct orc_model {
    int kind;
    int weighted;
    double a, b, gamma;
    const uint16_t* schema;
    uint32_t schema_len;
} orc_model;

typedef struct orc_opts {
    int mode;
    uint32_t walk_length;
    uint64_t seed;
    uint64_t cap_per_degree;
    double edge_cost_ratio;
    int rng; /* ORC_RNG_* */
    uint64_t qid_base; /* global id of queries[0] (walker-stream key) */
    const uint64_t* qids; /* [nq] global walker ids, or NULL: qid_base + i */
    double erjs_handoff;  /* tier-2 hand-off (include/dynwalk_b200.h), 0 = off */
} orc_opts;

void orc_libm(int fn, const double* x, double* y, uint64_t n);

/* Mirrors RunStats (include/dynwalk/runtime.hpp:53-73), GPU-relevant fields. */
typedef struct orc_stats {
    uint64_t queries, query_errors, dead_ends, steps;
    uint64_t select_ervs, select_erjs;
    uint64_t trials, weight_reads, rng_draws, erjs_fallbacks;
    uint64_t sel_by_deg[33][2];
} orc_stats;

/* ---- RNG ---- */
uint64_t orc_derive_seed(uint64_t seed, uint64_t stream);
void orc_mt19937_64(uint64_t seed, uint64_t n, uint64_t* out);
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
/* draw `idx` of the (seed, qid, step) walker stream */
uint64_t orc_walker_draw(uint64_t seed, uint64_t qid, uint32_t step, uint64_t idx);

/* ---- graph ---- */
orc_graph* orc_graph_build(const uint32_t* src, const uint32_t* dst, const float* prop,
                           const uint16_t* label, uint64_t n, int has_labels, int mirror,
                           uint64_t nv_hint);
orc_graph* orc_graph_from_csr(uint32_t nv, uint64_t ne, const uint64_t* row,
                              const uint32_t* col, const float* prop, const uint16_t* label);
void orc_graph_free(orc_graph* g);
void orc_recompute_aggregates(orc_graph* g);
int orc_has_edge(const orc_graph* g, uint32_t v, uint32_t u);

orc_graph* orc_gen_uniform(uint32_t n, uint32_t deg, uint64_t seed, int mirror);
orc_graph* orc_gen_ba(uint32_t n, uint32_t deg, uint64_t seed, int mirror);
/* reference synthesize_weights (mt19937): kind 0 uniform, 1 labels, 2 pareto, 3 degree */
int orc_synth_weights(orc_graph* g, int kind, double low, double high, double alpha,
                      uint64_t seed);

/* New synthetic workload (no reference counterpart):
 * R-MAT edge sampling, mirrored CSR, Philox weights/labels keyed by edge index. */
void orc_rmat_samples(uint32_t scale, uint64_t nsamples, uint64_t seed, uint32_t* src,
                      uint32_t* dst);
orc_graph* orc_gen_rmat(uint32_t scale, uint32_t edge_factor, uint64_t seed);
int orc_synth_philox(orc_graph* g, int kind, double low, double high, double alpha,
                     uint64_t seed);
/* multi-threaded orc_gen_rmat + orc_synth_philox(uniform) for large scales */
orc_graph* orc_gen_rmat_par(uint32_t scale, uint32_t edge_factor, uint64_t seed, double low,
                            double high, uint64_t wseed, int nthreads);

/* ---- walks ---- */
int orc_run(const orc_graph* g, const orc_model* m, const orc_opts* o, const uint32_t* queries,
            uint64_t nq, uint32_t* paths, uint32_t* lengths, orc_stats* stats, int nthreads);
/* exact transition probabilities (samplers.hpp:272-288); returns 0 dead end, -1 error, d */
int64_t orc_transition_probs(const orc_graph* g, const orc_model* m, uint32_t cur,
                             uint32_t prev, uint32_t step, double* probs);
/* decide_sampler (cost_model.hpp:46-56): 1 = eRJS, 0 = eRVS */
int orc_decide(const orc_graph* g, const orc_model* m, uint32_t cur, uint32_t prev,
               uint32_t step, double ratio, double* est_max, double* est_sum);
double orc_weight(const orc_graph* g, const orc_model* m, uint32_t cur, uint32_t prev,
                  uint32_t step, uint64_t e);
const char* orc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
