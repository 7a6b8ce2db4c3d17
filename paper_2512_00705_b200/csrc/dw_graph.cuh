// dw_graph.cuh -- device graph construction and calibration (host-callable).
#pragma once
#include "dw_models.cuh"

namespace dwb {

struct DeviceGraphBuffers {
    NodeRec* nodes = nullptr;
    EdgeRec* edges = nullptr;
    uint16_t* labels = nullptr;
    uint32_t* hslots = nullptr;  // membership hash sets (dw_member.cuh)
    FatRec* fat = nullptr;       // fat edge records (optional accelerator)
    FatRec32* fat32 = nullptr;   // compact fat records (when the 64 B ones exceed the cap)
    uint32_t* twin = nullptr;    // slim layout: per edge (v -> u), v's range in N(u)
                                 // (lo | cnt << 24; cnt 255 = unknown), or null
    double2* lagg = nullptr;     // per-node label MAX/SUM, built on first DSL use
    uint32_t* lab2 = nullptr;    // labels packed 2 bits each when all are < 4, or null
    unsigned long long nbuckets = 0;
    uint32_t nv = 0;
    unsigned long long ne = 0;
    uint32_t max_degree = 0;
};

// Packs CSR arrays already on the device into NodeRec/EdgeRec.  nmax/nsum may
// be null: they are then recomputed per node in ascending edge order
// (graph.cpp:83-98), bit-identical to the host.
cudaError_t pack_graph(const unsigned long long* d_row, const uint32_t* d_col, const float* d_prop,
                       const double* d_nmax, const double* d_nsum, DeviceGraphBuffers& out,
                       cudaStream_t s);

// Optional accelerators built once the packed graph is final and the build's
// temporaries are freed: the fat edge records (skipped when they would crowd
// HBM).  Every graph constructor calls it last.
cudaError_t finish_graph(DeviceGraphBuffers& g, cudaStream_t s);

// R-MAT topology + mirrored CSR + Philox weights/labels on the device.
// Definition identical to oracle.c orc_gen_rmat / orc_synth_philox.
struct RmatSpec {
    uint32_t scale, edge_factor;
    unsigned long long seed;       // derive_seed(seed, "rmat") / "perm" applied inside
    int weights;                   // 0 uniform, 2 pareto, -1 none
    double low, high, alpha;
    unsigned long long weight_seed;
    int labels;
    uint32_t label_low, label_high;
    unsigned long long label_seed;
};
cudaError_t build_rmat(const RmatSpec& spec, DeviceGraphBuffers& out, cudaStream_t s);

// Unpacks the device graph into separate device arrays (for downloads).
cudaError_t unpack_graph(const DeviceGraphBuffers& g, unsigned long long* d_row, uint32_t* d_col,
                         float* d_prop, double* d_nmax, double* d_nsum, cudaStream_t s);

// ProfileConfig (cost_model.hpp:9-15), validated by the caller.
struct ProfileSpec {
    double node_fraction;         // share of nodes probed per round
    uint32_t min_nodes;           // probe at least this many (graph permitting)
    uint32_t neighbors_per_node;  // weights evaluated per probed node
    uint32_t repetitions;         // median over this many timed repetitions
    unsigned long long seed;
};

// K4: the two profiling micro-passes of profile_edge_cost_ratio
// (cost_model.cpp:37-126) on the device; returns the median ratio.
cudaError_t calibrate_ratio(const DeviceGraphBuffers& g, int model_kind, bool weighted,
                            const ModelParams& mp, const ProfileSpec& cfg, cudaStream_t s,
                            double* ratio);

unsigned long long host_derive_seed(unsigned long long seed, unsigned long long stream);

// Per-node {MAX, SUM} over the row's labels in ascending edge order, the
// DslWalk preprocess step (models.cpp:19-35); zero rows without labels.
cudaError_t build_label_aggregates(DeviceGraphBuffers& g, cudaStream_t s);

// ---- text sink (dw_run_write_paths): write_paths' format, runtime.cpp:280-291
// bytes[i] = text size of path i ("id id ... id\n", "\n" when empty)
cudaError_t path_text_bytes(const uint32_t* paths, const uint32_t* lengths, unsigned long long n,
                            unsigned long long stride, uint32_t* bytes, cudaStream_t s);
// text[toffs[i] - toffs[0] ..) = path i as text
cudaError_t path_text_write(const uint32_t* paths, const uint32_t* lengths, unsigned long long n,
                            unsigned long long stride, const unsigned long long* toffs, char* text,
                            cudaStream_t s);

// ---- DWG1 loads (dw_graph_load_dwg1) ----------------------------------------
// Re-establishes Graph::build's invariants (graph.cpp:15-81) on a CSR that was
// streamed to the device as stored in the file: vertices referenced beyond the
// offsets array extend the vertex count (*d_row is reallocated), unsorted
// slices are stable-sorted by target (props and labels follow), and every prop
// must be strictly positive and finite (graph.hpp:51).  *status: 0 ok,
// 1 bad prop, 2 vertex id overflow, 3 unsorted slices above 2^31 edges.
cudaError_t prepare_loaded_csr(unsigned long long** d_row, uint32_t* nv, unsigned long long ne,
                               uint32_t* d_col, float* d_prop, uint16_t* d_label, int* status,
                               cudaStream_t s);

// ---- path compaction (dw_run_compact) ----------------------------------------
// offs[0..n] = base + exclusive prefix sum of lengths[0..n) (offs[n] = base +
// total); base is read from *d_base (device scalar) and *d_base is advanced by
// the batch total, so consecutive batches on one stream produce global
// offsets.  tmp/tmp_bytes: CUB scratch, query with tmp = nullptr.
cudaError_t path_offsets(const uint32_t* lengths, unsigned long long n, unsigned long long* offs,
                         unsigned long long* d_base, void* tmp, size_t& tmp_bytes,
                         cudaStream_t s);
// flat[offs[i] - offs[0] ..) = paths[i * stride .. + lengths[i]], one warp per
// walker (flat holds one batch, offs its global offsets)
cudaError_t compact_paths(const uint32_t* paths, const uint32_t* lengths, unsigned long long n,
                          unsigned long long stride, const unsigned long long* offs,
                          uint32_t* flat, cudaStream_t s);

// ---- direct compact runs (dw_capi.cu run_direct) ------------------------------
// lengths[i] = the path length query i has unless its walk stops early (0 for
// a start >= nv, 1 for a start without neighbours or target 0, else target+1)
cudaError_t predict_lengths(const uint32_t* queries, unsigned long long n, const NodeRec* nodes,
                            uint32_t nv, uint32_t target, uint32_t* lengths, cudaStream_t s);
// out[c] = offs[min(c << shift, n)] for c = 0..nchunks
cudaError_t chunk_bounds(const unsigned long long* offs, unsigned long long n, uint32_t shift,
                         unsigned long long nchunks, unsigned long long* out, cudaStream_t s);
// Walkers whose path is final before the walk: writes length-1 paths at
// offs, adds their queries and query errors to counters, and turns
// lengths[i] into the "walks" flag (length > 1).
cudaError_t trivial_walkers(const uint32_t* queries, unsigned long long n, uint32_t* lengths,
                            const unsigned long long* offs, uint32_t* flat,
                            unsigned long long* counters, cudaStream_t s);
// cq / cqid / coffs[pos[i]] = queries[i], its walker id (qids[i] or
// qid_base + i) and offs[i] (offs null: i * stride) for every i with flag[i]
cudaError_t walker_list(const uint32_t* queries, const unsigned long long* qids,
                        unsigned long long qid_base, unsigned long long n, const uint32_t* flag,
                        const unsigned long long* pos, const unsigned long long* offs,
                        unsigned long long stride, uint32_t* cq, unsigned long long* cqid,
                        unsigned long long* coffs, cudaStream_t s);
// dw_run_device's listed walks: lengths[i] = len[i] (predicted), paths[i *
// stride] = queries[i] for length-1 walkers, queries / query errors counted,
// len[i] <- (len[i] > 1)
cudaError_t trivial_rows(const uint32_t* queries, unsigned long long n, uint32_t* len,
                         uint32_t* paths, unsigned long long stride, uint32_t* lengths,
                         unsigned long long* counters, cudaStream_t s);
// chunk copy ranges of a direct run (see dw_graph.cu direct_bounds_kernel)
cudaError_t direct_bounds(const unsigned long long* coffs, const unsigned long long* d_nt,
                          const unsigned long long* total, uint32_t shift, unsigned long long kmax,
                          unsigned long long* out, cudaStream_t s);
// *flag |= 1 if some edge's target has no neighbours (a walk can end early)
cudaError_t sink_targets(const NodeRec* nodes, const EdgeRec* edges, unsigned long long ne,
                         int* flag, cudaStream_t s);

}  // namespace dwb
