// dw_capi.cu -- the C ABI (include/dynwalk_b200.h) over the device engine.
//
// Host side of the boundary: validation with the reference's error
// semantics, per-device graph replicas, walker sharding, stream-ordered
// H2D -> walk -> D2H pipelines, and RunStats assembly.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dynwalk_b200.h"
#include "dw_graph.cuh"
#include "dw_walk.cuh"

using dwb::DeviceGraphBuffers;
typedef unsigned long long ull;

namespace {

thread_local std::string t_error;

}  // namespace

struct dw_custom_model_s;
namespace dwb {
std::string* dsl_error_slot() { return &t_error; }
cudaError_t launch_custom(const dw_custom_model_s* cm, int mode, const WalkParams& p, int num_sms,
                          cudaStream_t stream);
uint32_t custom_max_steps(const dw_custom_model_s* cm);
uint32_t custom_flags(const dw_custom_model_s* cm);
}  // namespace dwb

namespace {

int fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_error = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(DW_ECUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CU(call, what)                                         \
    do {                                                       \
        cudaError_t e_ = (call);                               \
        if (e_ != cudaSuccess) return cuda_fail(e_, what);     \
    } while (0)

constexpr int kMaxBatches = 64;
constexpr int kRingSlots = 3;

struct Replica {
    int device = 0;
    int num_sms = 0;
    cudaStream_t stream = nullptr;  // walk kernels
    cudaStream_t copy = nullptr;    // H2D/D2H
    cudaStream_t ends = nullptr;    // dw_run_compact: batch end offsets (D2H)
    cudaStream_t d2h = nullptr;     // dw_run_compact: compacted paths and offsets (D2H)
    DeviceGraphBuffers g;
    ull* counters = nullptr;   // [kCNum]
    ull* queues = nullptr;     // [kMaxBatches]
    int* error = nullptr;
    ull* error_info = nullptr;
    // dw_run / dw_run_compact: a ring of batch slots, so device memory stays
    // bounded whatever nq is (BASELINE config 5 streams 435 GB of paths)
    struct Slot {
        uint32_t* q = nullptr;      // [cap] queries
        ull* qids = nullptr;        // [cap] global walker ids (runs with dw_run_opts.qids)
        uint32_t* len = nullptr;    // [cap] path lengths
        uint32_t* paths = nullptr;  // [cap][stride] padded paths
        uint32_t* flat = nullptr;   // [cap * stride] compacted paths (compact runs)
        ull* offs = nullptr;        // [cap + 1] global path (or text byte) offsets
        char* txt = nullptr;        // [cap * stride * 11] path text (text runs)
        cudaEvent_t h2d = nullptr, walk = nullptr, end = nullptr, d2h = nullptr;
    };
    Slot slots[kRingSlots];
    ull slot_cap = 0, slot_stride = 0;
    bool slot_flat = false, slot_txt = false, slot_qids = false;
    ull* d_base = nullptr;      // running offset of the batches already compacted
    void* d_scan = nullptr;
    size_t scan_bytes = 0;
    ull* h_ends = nullptr;      // pinned [kRingSlots] batch end offsets
    cudaEvent_t ev_start = nullptr, ev_stop = nullptr;
    cudaEvent_t ev_reset = nullptr;
    // direct compact runs (run_direct): one launch writes the flat layout at
    // predicted offsets and the host copies finished chunks while it walks
    struct Direct {
        uint32_t* q = nullptr;      // [cap_q] queries
        ull* qids = nullptr;        // [cap_q] global walker ids
        uint32_t* len = nullptr;    // [cap_q] predicted lengths
        ull* offs = nullptr;        // [cap_q + 1] predicted offsets
        uint32_t* flat = nullptr;   // [cap_flat] ids
        ull* pos = nullptr;         // [cap_q + 1] rank of each walking walker
        uint32_t* cq = nullptr;     // [cap_q] the walking walkers: queries,
        ull* cqid = nullptr;        //   global walker ids,
        ull* coffs = nullptr;       //   flat offsets
        unsigned* done = nullptr;   // [kMaxChunks] finished walkers per chunk
        int* flag = nullptr;        // scratch (sink_targets)
        unsigned* h_flag = nullptr; // host-mapped [kMaxChunks] chunk final flags
        ull* h_bounds = nullptr;    // host-mapped [kMaxChunks + 3] chunk flat bounds, nt, nch
        ull cap_q = 0, cap_flat = 0;
        bool has_qids = false;
        cudaEvent_t pre = nullptr, walk = nullptr, w0 = nullptr, w1 = nullptr;
    } dir;
    int sinks = -1;  // -1 unknown, 1: some edge leads to a vertex without neighbours
    // dw_run_device bookkeeping
    struct Listed {               // a listed walk (run_device_listed) to verify
        bool on = false;
        uint32_t target = 0;
        dw_model_desc model;
        dw_run_opts opts;
        const uint32_t* queries = nullptr;
        ull nq = 0;
        uint32_t *paths = nullptr, *lengths = nullptr;
        cudaStream_t stream = nullptr;
        ull nt = 0;               // walkers the walk was given
    } listed;
    bool pending = false;
    ull pending_launches = 0;
    ull pending_qbase = 0;
};

}  // namespace

struct dw_graph_s {
    uint32_t nv = 0;
    ull ne = 0;
    bool has_labels = false;
    uint32_t max_degree = 0;
    std::vector<Replica> reps;
};

namespace {

int init_replica(Replica& r, int device) {
    r.device = device;
    CU(cudaSetDevice(device), "cudaSetDevice");
    CU(cudaDeviceGetAttribute(&r.num_sms, cudaDevAttrMultiProcessorCount, device),
       "cudaDeviceGetAttribute");
    // Every gather on the walk path is one random 32 B sector; an L2 that
    // promotes misses to 64/128 B fetches would multiply DRAM traffic.
    // DW_L2_FETCH overrides the granularity (bytes) for experiments.
    {
        size_t fetch = 32;
        if (const char* s = std::getenv("DW_L2_FETCH")) fetch = (size_t)std::atoi(s);
        if (fetch) CU(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, fetch), "L2 fetch limit");
        if (std::getenv("DW_VERBOSE")) {
            size_t v = 0;
            cudaDeviceGetLimit(&v, cudaLimitMaxL2FetchGranularity);
            std::fprintf(stderr, "dynwalk: device %d L2 fetch granularity %zu B\n", device, v);
        }
    }
    CU(cudaStreamCreateWithFlags(&r.stream, cudaStreamNonBlocking), "cudaStreamCreate");
    CU(cudaStreamCreateWithFlags(&r.copy, cudaStreamNonBlocking), "cudaStreamCreate");
    CU(cudaStreamCreateWithFlags(&r.ends, cudaStreamNonBlocking), "cudaStreamCreate");
    CU(cudaStreamCreateWithFlags(&r.d2h, cudaStreamNonBlocking), "cudaStreamCreate");
    CU(cudaMalloc(&r.counters, dwb::kCNum * sizeof(ull)), "cudaMalloc counters");
    CU(cudaMalloc(&r.queues, kMaxBatches * sizeof(ull)), "cudaMalloc queues");
    CU(cudaMalloc(&r.error, sizeof(int)), "cudaMalloc error");
    CU(cudaMalloc(&r.error_info, sizeof(ull)), "cudaMalloc error");
    CU(cudaEventCreate(&r.ev_start), "cudaEventCreate");
    CU(cudaEventCreate(&r.ev_stop), "cudaEventCreate");
    CU(cudaEventCreateWithFlags(&r.ev_reset, cudaEventDisableTiming), "cudaEventCreate");
    for (auto& sl : r.slots)
        for (cudaEvent_t* e : {&sl.h2d, &sl.walk, &sl.end, &sl.d2h})
            CU(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
    CU(cudaMallocHost(&r.h_ends, kRingSlots * sizeof(ull)), "cudaMallocHost");
    CU(cudaMalloc(&r.d_base, sizeof(ull)), "cudaMalloc");
    return DW_OK;
}

// the direct compact runs' per-walker buffers (reallocated on next use)
void free_direct(Replica::Direct& d) {
    cudaFree(d.q);
    cudaFree(d.qids);
    cudaFree(d.len);
    cudaFree(d.offs);
    cudaFree(d.flat);
    cudaFree(d.pos);
    cudaFree(d.cq);
    cudaFree(d.cqid);
    cudaFree(d.coffs);
    d.q = d.len = d.flat = d.cq = nullptr;
    d.qids = d.offs = d.pos = d.cqid = d.coffs = nullptr;
    d.cap_q = d.cap_flat = 0;
    d.has_qids = false;
}

void free_replica(Replica& r) {
    if (cudaSetDevice(r.device) != cudaSuccess) return;
    if (r.stream) cudaStreamSynchronize(r.stream);
    if (r.copy) cudaStreamSynchronize(r.copy);
    if (r.ends) cudaStreamSynchronize(r.ends);
    if (r.d2h) cudaStreamSynchronize(r.d2h);
    cudaFree(r.g.nodes);
    cudaFree(r.g.edges);
    cudaFree(r.g.labels);
    cudaFree(r.g.hslots);
    cudaFree(r.g.fat);
    cudaFree(r.g.lagg);
    cudaFree(r.g.twin);
    cudaFree(r.g.fat32);
    cudaFree(r.g.lab2);
    cudaFree(r.counters);
    cudaFree(r.queues);
    cudaFree(r.error);
    cudaFree(r.error_info);
    for (auto& sl : r.slots) {
        cudaFree(sl.q);
        cudaFree(sl.qids);
        cudaFree(sl.len);
        cudaFree(sl.paths);
        cudaFree(sl.flat);
        cudaFree(sl.offs);
        cudaFree(sl.txt);
        for (cudaEvent_t e : {sl.h2d, sl.walk, sl.end, sl.d2h})
            if (e) cudaEventDestroy(e);
    }
    free_direct(r.dir);
    cudaFree(r.dir.done);
    cudaFree(r.dir.flag);
    if (r.dir.h_flag) cudaFreeHost(r.dir.h_flag);
    if (r.dir.h_bounds) cudaFreeHost(r.dir.h_bounds);
    for (cudaEvent_t e : {r.dir.pre, r.dir.walk, r.dir.w0, r.dir.w1})
        if (e) cudaEventDestroy(e);
    cudaFree(r.d_base);
    cudaFree(r.d_scan);
    if (r.h_ends) cudaFreeHost(r.h_ends);
    if (r.ev_start) cudaEventDestroy(r.ev_start);
    if (r.ev_stop) cudaEventDestroy(r.ev_stop);
    if (r.ev_reset) cudaEventDestroy(r.ev_reset);
    if (r.stream) cudaStreamDestroy(r.stream);
    if (r.copy) cudaStreamDestroy(r.copy);
    if (r.ends) cudaStreamDestroy(r.ends);
    if (r.d2h) cudaStreamDestroy(r.d2h);
}

int resolve_devices(const int* devices, int ndev, std::vector<int>& out) {
    int count = 0;
    CU(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    if (count < 1) return fail(DW_ECUDA, "no CUDA device available");
    if (ndev < 1) return fail(DW_EINVAL, "worker count must be >= 1 (ndev=%d)", ndev);
    out.clear();
    for (int i = 0; i < ndev; ++i) {
        const int d = devices ? devices[i] : i;
        if (d < 0 || d >= count) return fail(DW_EINVAL, "device %d out of range (%d devices)", d, count);
        out.push_back(d);
    }
    return DW_OK;
}

// Graph invariants the reference keeps by construction (graph.hpp:187-192).
int validate_desc(const dw_graph_desc* d) {
    if (!d || !d->row_offsets || (d->num_edges && (!d->col_indices || !d->edge_props)))
        return fail(DW_EINVAL, "graph descriptor is missing arrays");
    if ((ull)d->num_vertices >= DW_INVALID_VERTEX)
        return fail(DW_EINVAL, "vertex id overflow: graph needs %u vertices", d->num_vertices);
    const uint32_t nv = d->num_vertices;
    if (d->row_offsets[0] != 0 || d->row_offsets[nv] != d->num_edges)
        return fail(DW_EINVAL, "corrupt CSR: row_offsets must start at 0 and end at num_edges");
    for (uint32_t v = 0; v < nv; ++v) {
        const ull b = d->row_offsets[v], e = d->row_offsets[v + 1];
        if (e < b) return fail(DW_EINVAL, "corrupt CSR: row_offsets decrease at vertex %u", v);
        for (ull i = b; i < e; ++i) {
            const uint32_t c = d->col_indices[i];
            if (c >= nv)
                return fail(DW_EINVAL, "vertex id %u out of range (num_vertices=%u)", c, nv);
            if (i > b && d->col_indices[i - 1] > c)
                return fail(DW_EINVAL, "adjacency slice of vertex %u is not sorted by target", v);
            const float p = d->edge_props[i];
            if (!(p > 0.0f) || !std::isfinite(p))
                return fail(DW_EINVAL, "edge property must be strictly positive and finite, got %g",
                            (double)p);
        }
    }
    return DW_OK;
}

int upload_replica(Replica& r, const dw_graph_desc* d) {
    CU(cudaSetDevice(r.device), "cudaSetDevice");
    const uint32_t nv = d->num_vertices;
    const ull ne = d->num_edges;
    cudaStream_t s = r.stream;
    ull* row = nullptr;
    uint32_t* col = nullptr;
    float* prop = nullptr;
    double *nmax = nullptr, *nsum = nullptr;
    CU(cudaMalloc(&row, (nv + 1ull) * sizeof(ull)), "cudaMalloc");
    CU(cudaMalloc(&col, std::max<ull>(ne, 1) * sizeof(uint32_t)), "cudaMalloc");
    CU(cudaMalloc(&prop, std::max<ull>(ne, 1) * sizeof(float)), "cudaMalloc");
    CU(cudaMemcpyAsync(row, d->row_offsets, (nv + 1ull) * sizeof(ull), cudaMemcpyHostToDevice, s),
       "H2D");
    if (ne) {
        CU(cudaMemcpyAsync(col, d->col_indices, ne * sizeof(uint32_t), cudaMemcpyHostToDevice, s),
           "H2D");
        CU(cudaMemcpyAsync(prop, d->edge_props, ne * sizeof(float), cudaMemcpyHostToDevice, s),
           "H2D");
    }
    if (d->node_prop_max && d->node_prop_sum && nv) {
        CU(cudaMalloc(&nmax, nv * sizeof(double)), "cudaMalloc");
        CU(cudaMalloc(&nsum, nv * sizeof(double)), "cudaMalloc");
        CU(cudaMemcpyAsync(nmax, d->node_prop_max, nv * sizeof(double), cudaMemcpyHostToDevice, s),
           "H2D");
        CU(cudaMemcpyAsync(nsum, d->node_prop_sum, nv * sizeof(double), cudaMemcpyHostToDevice, s),
           "H2D");
    }
    r.g.nv = nv;
    r.g.ne = ne;
    CU(cudaMalloc(&r.g.nodes, std::max<uint32_t>(nv, 1) * sizeof(dwb::NodeRec)), "cudaMalloc nodes");
    CU(cudaMalloc(&r.g.edges, ((std::max<ull>(ne, 1) + 1) & ~1ull) * sizeof(dwb::EdgeRec)), "cudaMalloc edges");
    if (d->edge_labels) {
        CU(cudaMalloc(&r.g.labels, ((std::max<ull>(ne, 1) + 1) & ~1ull) * sizeof(uint16_t)), "cudaMalloc labels");
        if (ne)
            CU(cudaMemcpyAsync(r.g.labels, d->edge_labels, ne * sizeof(uint16_t),
                               cudaMemcpyHostToDevice, s),
               "H2D");
    }
    CU(dwb::pack_graph(row, col, prop, nmax, nsum, r.g, s), "pack_graph");
    CU(cudaStreamSynchronize(s), "upload");
    cudaFree(row);
    cudaFree(col);
    cudaFree(prop);
    cudaFree(nmax);
    cudaFree(nsum);
    CU(dwb::finish_graph(r.g, s), "fat records");
    return DW_OK;
}

int check_model(const dw_model_desc* m) {
    if (!m) return fail(DW_EINVAL, "model descriptor is NULL");
    if (m->kind == DW_MODEL_CUSTOM) {
        if (!m->custom) return fail(DW_EINVAL, "custom model handle is NULL");
        return DW_OK;
    }
    if (m->kind < DW_MODEL_STATIC || m->kind > DW_MODEL_PR2)
        return fail(DW_EINVAL,
                    "unknown model kind %d (expected static, node2vec, metapath, pr2; DSL models "
                    "need code generation)",
                    m->kind);
    if (m->kind == DW_MODEL_NODE2VEC) {
        // the device divides by a and b with a correctly rounded reciprocal
        // (dw_models.cuh ddiv), exact for every quotient in this range
        const double lo = 0x1p-500, hi = 0x1p500;
        const double aa = std::fabs(m->a), bb = std::fabs(m->b);
        if (!(aa >= lo && aa <= hi && bb >= lo && bb <= hi))
            return fail(DW_EUNSUPPORTED,
                        "node2vec parameters |a|, |b| must lie in [2^-500, 2^500] on the GPU "
                        "runtime (a=%g, b=%g)",
                        m->a, m->b);
    }
    if (m->kind == DW_MODEL_METAPATH) {
        if (m->schema_len > DW_MAX_SCHEMA)
            return fail(DW_EINVAL, "metapath schema longer than %d labels", DW_MAX_SCHEMA);
        if (m->schema_len && !m->schema) return fail(DW_EINVAL, "metapath schema is NULL");
    }
    return DW_OK;
}

dwb::ModelParams model_params(const dw_model_desc* m) {
    dwb::ModelParams mp;
    std::memset(&mp, 0, sizeof mp);
    mp.a = m->a;
    mp.b = m->b;
    mp.gamma = m->gamma;
    // correctly rounded reciprocals for the device's Markstein division
    // (dw_models.cuh ddiv); only within a range where every quotient the
    // models form stays a normal double
    auto in_range = [](double x) { return x >= 0x1p-500 && x <= 0x1p500; };
    mp.fast_div = (in_range(m->a) && in_range(m->b)) ? 1u : 0u;
    mp.inv_a = 1.0 / m->a;
    mp.inv_b = 1.0 / m->b;
    mp.inv_3 = 1.0 / 3.0;
    // free rejections need weights that are valid by construction
    switch (m->kind) {
    case DW_MODEL_NODE2VEC:
        mp.shortcut = (m->a > 0.0 && m->b > 0.0 && std::isfinite(m->a) && std::isfinite(m->b)) ? 1u : 0u;
        break;
    case DW_MODEL_PR2: mp.shortcut = (m->gamma >= 0.0 && m->gamma <= 1.0) ? 1u : 0u; break;
    default: mp.shortcut = 0u;
    }
    switch (m->kind) {
    case DW_MODEL_NODE2VEC: mp.pos_weights = (m->a > 0.0 && m->b > 0.0) ? 1u : 0u; break;
    case DW_MODEL_PR2: mp.pos_weights = (m->gamma >= 0.0 && m->gamma < 1.0) ? 1u : 0u; break;
    case DW_MODEL_STATIC: mp.pos_weights = 1u; break;  // props are validated > 0
    default: mp.pos_weights = 0u;
    }
    // one-multiply weight-sum screen (dw_models.cuh wsum_approx)
    mp.screen = (m->kind == DW_MODEL_NODE2VEC && m->a > 0.0 && m->b > 0.0) ? 1u : 0u;
    mp.wsum_coef = (1.0 / m->a + 1.0 + 1.0 / m->b) / 3.0;
    // decisions within this relative distance of a compact record's row sum
    // refetch the exact node record (dw_walk_kernel.cuh); the record keeps
    // the f32 sum truncated to 15 mantissa bits (within 2^-15 = 3.1e-5 of the
    // double sum), so any band >= 1e-4 is exact
    mp.fat32_band = 1e-4;
    if (const char* env = std::getenv("DW_FAT32_BAND")) {
        const double b = std::atof(env);
        if (b >= 1e-4) mp.fat32_band = b;
    }
    // the warp reservoir's rounding band (dw_walk_kernel.cuh ervs_warp) is
    // rigorous at 1; DW_ERVS_SLACK > 1 widens it so that tests drive the exact
    // replay on most crossings
    mp.ervs_slack = 1.0;
    if (const char* env = std::getenv("DW_ERVS_SLACK")) {
        const double v = std::atof(env);
        if (v >= 1.0) mp.ervs_slack = v;
    }
    if (const char* env = std::getenv("DW_SCREEN"))
        if (env[0] == '0') mp.screen = 0u;
    if (const char* env = std::getenv("DW_D1"))
        if (env[0] == '0') mp.pos_weights = 0u;
    if (const char* env = std::getenv("DW_SHORTCUT"))
        if (env[0] == '0') mp.shortcut = mp.pos_weights = 0u;
    if (m->kind == DW_MODEL_METAPATH) {
        mp.schema_len = m->schema_len;
        for (uint32_t i = 0; i < m->schema_len; ++i) mp.schema[i] = m->schema[i];
    }
    return mp;
}

const char* mode_name(int mode) {
    switch (mode) {
    case DW_MODE_FORCE_ITS: return "force-its";
    case DW_MODE_FORCE_ALS: return "force-als";
    }
    return "?";
}

int check_opts(const dw_run_opts* o) {
    if (!o) return fail(DW_EINVAL, "run options are NULL");
    if (o->mode == DW_MODE_FORCE_ITS || o->mode == DW_MODE_FORCE_ALS)
        return fail(DW_EUNSUPPORTED,
                    "sampler mode %s is a CPU comparison baseline and is not supported by the "
                    "GPU runtime",
                    mode_name(o->mode));
    if (o->mode < DW_MODE_ADAPTIVE || o->mode > DW_MODE_ERVS_NOJUMP)
        return fail(DW_EINVAL, "unknown sampler mode %d", o->mode);
    if (o->walk_length == 0xFFFFFFFFu) return fail(DW_EINVAL, "walk_length too large");
    if (!(o->erjs_handoff >= 0.0) || !std::isfinite(o->erjs_handoff))
        return fail(DW_EINVAL, "erjs_handoff must be >= 0 and finite");
    if (o->erjs_handoff > 0.0 && (!(o->edge_cost_ratio > 0.0) || !std::isfinite(o->edge_cost_ratio)))
        return fail(DW_EINVAL, "erjs_handoff needs a positive finite edge_cost_ratio");
    return DW_OK;
}

uint32_t target_steps(const dw_model_desc* m, const dw_run_opts* o) {
    const uint32_t ms = m->kind == DW_MODEL_METAPATH ? m->schema_len
                        : m->kind == DW_MODEL_CUSTOM ? dwb::custom_max_steps(m->custom)
                                                     : 0xFFFFFFFFu;
    return std::min(o->walk_length, ms);
}

dwb::WalkParams make_params(Replica& r, const dw_model_desc* m, const dw_run_opts* o) {
    dwb::WalkParams p;
    std::memset(&p, 0, sizeof p);
    p.g = dwb::DevGraph{r.g.nodes, r.g.edges, r.g.labels, r.g.hslots, r.g.fat, r.g.lagg,
                        r.g.twin, r.g.fat32, r.g.lab2, r.g.nv, r.g.ne};
    p.stride = o->walk_length + 1;
    p.target = target_steps(m, o);
    p.seed_lo = (uint32_t)o->seed;
    p.seed_hi = (uint32_t)(o->seed >> 32);
    p.rk = dwb::philox_keys(p.seed_lo, p.seed_hi);
    p.cap_per_degree = o->erjs_cap_per_degree;
    p.ratio = o->edge_cost_ratio;
    p.handoff = o->erjs_handoff;
    p.counters = r.counters;
    p.error = r.error;
    p.error_info = r.error_info;
    p.mp = model_params(m);
    return p;
}

// builtin models are template instantiations; DSL models NVRTC-compiled kernels
cudaError_t launch_model(Replica& r, const dw_model_desc* m, int mode, const dwb::WalkParams& p,
                         cudaStream_t s) {
    if (m->kind == DW_MODEL_CUSTOM) return dwb::launch_custom(m->custom, mode, p, r.num_sms, s);
    return dwb::launch_walk(m->kind, m->weighted != 0, mode, p, r.num_sms, s);
}

// per-replica preprocessing a model needs before its first walk
int prepare_model(Replica& r, const dw_model_desc* m) {
    if (m->kind == DW_MODEL_CUSTOM && (dwb::custom_flags(m->custom) & DW_CUSTOM_LABEL_AGGREGATES) &&
        !r.g.lagg) {
        CU(cudaSetDevice(r.device), "cudaSetDevice");
        CU(dwb::build_label_aggregates(r.g, r.stream), "label aggregates");
    }
    return DW_OK;
}

int reset_run_state(Replica& r) {
    CU(cudaMemsetAsync(r.counters, 0, dwb::kCNum * sizeof(ull), r.stream), "memset");
    CU(cudaMemsetAsync(r.queues, 0, kMaxBatches * sizeof(ull), r.stream), "memset");
    CU(cudaMemsetAsync(r.error, 0, sizeof(int), r.stream), "memset");
    return DW_OK;
}

void add_counters(dw_run_stats* st, const ull* c) {
    st->queries += c[dwb::kCQueries];
    st->query_errors += c[dwb::kCQueryErrors];
    st->dead_ends += c[dwb::kCDeadEnds];
    st->trials += c[dwb::kCTrials];
    st->weight_reads += c[dwb::kCWeightReads];
    st->rng_draws += c[dwb::kCRngDraws];
    st->erjs_fallbacks += c[dwb::kCFallbacks];
    st->algorithmic_bytes += c[dwb::kCAlgBytes];
    for (int b = 0; b < 33; ++b)
        for (int k = 0; k < 2; ++k) {
            const ull v = c[dwb::kCHist + 2 * b + k];
            st->selection_by_degree[b][k] += v;
            st->steps += v;
            (k ? st->select_erjs : st->select_ervs) += v;
        }
}

// Reads back error + counters of one replica after its streams drained.
int collect(Replica& r, dw_run_stats* st, ull qbase) {
    int err = 0;
    ull info = 0;
    ull c[dwb::kCNum];
    CU(cudaMemcpy(&err, r.error, sizeof(int), cudaMemcpyDeviceToHost), "D2H error");
    if (err) {
        CU(cudaMemcpy(&info, r.error_info, sizeof(ull), cudaMemcpyDeviceToHost), "D2H error");
        switch (err) {
        case dwb::kDevBadWeight:
            return fail(DW_EMODEL, "model returned a negative or non-finite weight (query %llu)",
                        info);
        case dwb::kDevBadBound:
            return fail(DW_EMODEL, "rejection bound must be positive and finite (query %llu)",
                        info);
        default:
            return fail(DW_EMODEL, "walk kernel error %d (query %llu)", err, info);
        }
    }
    (void)qbase;
    if (st) {
        CU(cudaMemcpy(c, r.counters, sizeof c, cudaMemcpyDeviceToHost), "D2H counters");
        add_counters(st, c);
    }
    return DW_OK;
}

constexpr ull kTextBytesPerId = 11;  // up to 10 digits + separator

int ensure_ring(Replica& r, ull cap, ull stride, bool flat, bool txt, bool qids) {
    if (cap <= r.slot_cap && stride <= r.slot_stride && (!flat || r.slot_flat) &&
        (!txt || r.slot_txt) && (!qids || r.slot_qids))
        return DW_OK;
    CU(cudaDeviceSynchronize(), "ring");
    cap = std::max(cap, r.slot_cap);
    stride = std::max(stride, r.slot_stride);
    flat = flat || txt || r.slot_flat;
    txt = txt || r.slot_txt;
    qids = qids || r.slot_qids;
    for (auto& sl : r.slots) {
        cudaFree(sl.q);
        cudaFree(sl.qids);
        sl.qids = nullptr;
        cudaFree(sl.len);
        cudaFree(sl.paths);
        cudaFree(sl.flat);
        cudaFree(sl.offs);
        cudaFree(sl.txt);
        sl.q = sl.len = sl.paths = sl.flat = nullptr;
        sl.offs = nullptr;
        sl.txt = nullptr;
        CU(cudaMalloc(&sl.q, cap * sizeof(uint32_t)), "cudaMalloc queries");
        CU(cudaMalloc(&sl.len, cap * sizeof(uint32_t)), "cudaMalloc lengths");
        if (qids) CU(cudaMalloc(&sl.qids, cap * sizeof(ull)), "cudaMalloc walker ids");
        CU(cudaMalloc(&sl.paths, cap * stride * sizeof(uint32_t)), "cudaMalloc paths");
        if (flat) {
            CU(cudaMalloc(&sl.flat, cap * stride * sizeof(uint32_t)), "cudaMalloc flat paths");
            CU(cudaMalloc(&sl.offs, (cap + 1) * sizeof(ull)), "cudaMalloc offsets");
        }
        if (txt) CU(cudaMalloc(&sl.txt, cap * stride * kTextBytesPerId), "cudaMalloc text");
    }
    if (flat) {
        size_t need = 0;
        CU(dwb::path_offsets(nullptr, cap, nullptr, nullptr, nullptr, need, r.stream), "scan size");
        if (need > r.scan_bytes) {
            cudaFree(r.d_scan);
            r.d_scan = nullptr;
            CU(cudaMalloc(&r.d_scan, need), "cudaMalloc scan");
            r.scan_bytes = need;
        }
    }
    r.slot_cap = cap;
    r.slot_stride = stride;
    r.slot_flat = flat;
    r.slot_txt = txt;
    r.slot_qids = qids;
    return DW_OK;
}

// Output of a host-buffer run: padded paths + lengths (dw_run), or the
// flattened RunResult.paths layout (dw_run_compact).
struct RunOut {
    bool compact = false;
    FILE* text = nullptr;       // write_paths sink (dw_run_write_paths)
    const char* text_path = nullptr;
    char* h_txt = nullptr;      // pinned staging for one batch of text
    uint32_t* paths = nullptr;
    uint32_t* lengths = nullptr;
    ull* offsets = nullptr;
    uint32_t* flat = nullptr;
    ull flat_cap = 0;
};

// Walkers per batch: ~4 batches per device so H2D/D2H overlap the walks (each
// launch ends in a ~1 ms tail while its last walkers finish, so fewer is
// better; batch_plan shortens the last ones), at least 256K walkers per
// launch, at most 4M (1.3 GB of padded paths at L=80)
ull batch_size(ull n, ull div = 4) {
    if (const char* env = std::getenv("DW_BATCH"))  // experiments: fixed walkers per batch
        if (std::atoll(env) > 0) return std::min<ull>(std::max<ull>(n, 1), (ull)std::atoll(env));
    if (const char* env = std::getenv("DW_BATCH_DIV")) div = std::max(1, std::atoi(env));
    const ull want = (n + div - 1) / div;
    return std::max<ull>(1, std::min<ull>(n, std::max<ull>(1ull << 18, std::min<ull>(want, 1ull << 22))));
}

// Batch boundaries of one device's n walkers: batches of bs (batch_size), the
// last two batches' worth split geometrically (1/2, 1/4, 1/8, 1/8, pieces of
// at least 1M walkers) so the copy of the final batch, which nothing
// overlaps, is short.  bs is the ring slot size (every batch fits one).
std::vector<ull> batch_plan(ull n, ull bs) {
    std::vector<ull> at{0};
    if (n == 0) return at;
    bs = std::max<ull>(bs, 1);
    ull pos = 0;
    while (n - pos > 2 * bs) at.push_back(pos += bs);
    ull rem = n - pos;
    // pieces stay >= 1M walkers: a launch ends when its slowest walker does,
    // and models with heavy-tailed walks (PR2: thousands of trials on hub
    // rows) pay that at every batch boundary, while the copies the split
    // hides are small for small batches
    if (rem > bs && !std::getenv("DW_BATCH")) {
        for (int k = 0; k < 3 && rem / 2 >= (1ull << 20); ++k) {
            at.push_back(pos += rem / 2);
            rem -= rem / 2;
        }
    }
    while (pos < n) at.push_back(pos = std::min(n, pos + bs));
    return at;
}

// The batched H2D -> walk -> (compaction) -> D2H pipeline behind dw_run,
// dw_run_compact and dw_run_write_paths.  The queries are cut into batches
// (batch_plan) that go round-robin over the devices, so every device walks
// at once and a hub-heavy stretch of the query list is spread over all of
// them.  On each device, batches cycle through kRingSlots buffer slots and
// stream events order slot reuse.  The host drains finished batches in query
// order: it blocks only to learn a compact / text batch's size, and never on a
// device other than the batch's own, so a device refills its ring while
// another one is being drained.  Output is independent of the device count:
// the RNG is keyed by the global walker id, and a batch's compact offsets are
// shifted to their global position on the host after the last copy.
int run_engine(dw_graph_t g, const dw_model_desc* model, const uint32_t* queries, ull nq,
               const dw_run_opts* opts, const RunOut& out, dw_run_stats* st) {
    if (st) std::memset(st, 0, sizeof *st);
    const int nd = (int)g->reps.size();
    const ull stride = (ull)opts->walk_length + 1;
    const bool ordered = out.compact || out.text;
    const ull per_dev = std::max<ull>(1, (nq + nd - 1) / nd);
    // compact output: ~2 batches per device (its last copy is small next to
    // the launch tails a batch adds: MetaPath s22 e2e 14.3 ms against 15.1
    // with 4, profiles/r2_cfg_ab_final.txt); padded rows: ~4
    const ull bs = out.text ? std::min<ull>(batch_size(per_dev), 1ull << 20)
                            : batch_size(per_dev, out.compact ? 2 : 4);
    const std::vector<ull> at = batch_plan(nq, bs);
    const ull nb = at.size() - 1;
    struct Dev {
        ull end = 0;       // device-local running end offset (ids or text bytes)
        ull inflight = 0;  // batches enqueued and not yet drained
    };
    std::vector<Dev> dv(nd);
    struct Fixup {
        ull lo, n, delta;
    };
    std::vector<Fixup> fixups;  // compact offsets that need the other devices' ids added
    // DW_ENGINE_TRACE=<file>: the host schedule ("E|D batch device" per
    // enqueue / drain), for tests of the device interleaving
    std::unique_ptr<FILE, int (*)(FILE*)> trace(nullptr, &std::fclose);
    if (const char* tp = std::getenv("DW_ENGINE_TRACE")) trace.reset(std::fopen(tp, "a"));
    cudaEvent_t wall0 = nullptr, wall1 = nullptr;
    CU(cudaSetDevice(g->reps[0].device), "cudaSetDevice");
    CU(cudaEventCreate(&wall0), "event");
    CU(cudaEventCreate(&wall1), "event");
    CU(cudaEventRecord(wall0, g->reps[0].copy), "event");
    ull launches = 0;
    int rc;
    for (int di = 0; di < nd; ++di) {
        Replica& r = g->reps[di];
        CU(cudaSetDevice(r.device), "cudaSetDevice");
        if ((rc = prepare_model(r, model))) return rc;
        if ((rc = ensure_ring(r, bs, stride, out.compact, out.text != nullptr,
                              opts->qids != nullptr)))
            return rc;
        if ((rc = reset_run_state(r))) return rc;
        CU(cudaMemsetAsync(r.d_base, 0, sizeof(ull), r.stream), "memset");
        CU(cudaEventRecord(r.ev_reset, r.stream), "event");
        CU(cudaStreamWaitEvent(r.copy, r.ev_reset, 0), "event");
        CU(cudaEventRecord(r.ev_start, r.stream), "event");
    }
    auto enqueue = [&](ull b) -> int {
        const int di = (int)(b % nd);
        const ull li = b / nd;  // the device's own batch index
        Replica& r = g->reps[di];
        Replica::Slot& sl = r.slots[li % kRingSlots];
        const ull blo = at[b], bn = at[b + 1] - blo;
        cudaStream_t ws = r.stream;
        CU(cudaSetDevice(r.device), "cudaSetDevice");
        if (li >= (ull)kRingSlots) {  // the slot's previous batch must be walked and drained
            CU(cudaStreamWaitEvent(r.copy, sl.walk, 0), "event");
            CU(cudaStreamWaitEvent(ws, sl.d2h, 0), "event");
        }
        CU(cudaMemcpyAsync(sl.q, queries + blo, bn * sizeof(uint32_t), cudaMemcpyHostToDevice,
                           r.copy),
           "H2D queries");
        if (opts->qids)
            CU(cudaMemcpyAsync(sl.qids, opts->qids + blo, bn * sizeof(ull), cudaMemcpyHostToDevice,
                               r.copy),
               "H2D walker ids");
        CU(cudaEventRecord(sl.h2d, r.copy), "event");
        CU(cudaStreamWaitEvent(ws, sl.h2d, 0), "event");
        dwb::WalkParams p = make_params(r, model, opts);
        p.queries = sl.q;
        p.nq = bn;
        p.qid_base = opts->qid_base + blo;
        p.qids = opts->qids ? sl.qids : nullptr;
        p.paths = (out.compact || out.text || out.paths) ? sl.paths : nullptr;
        p.lengths = sl.len;
        p.next_walker = r.queues + (li % kRingSlots);
        CU(cudaMemsetAsync(p.next_walker, 0, sizeof(ull), ws), "memset");
        if (p.paths && !ordered)  // compaction copies only the written ids
            CU(cudaMemsetAsync(p.paths, 0xFF, bn * stride * sizeof(uint32_t), ws),
               "memset paths");
        CU(launch_model(r, model, opts->mode, p, ws), "walk");
        ++launches;
        if (out.compact) {
            size_t tb = r.scan_bytes;
            CU(dwb::path_offsets(sl.len, bn, sl.offs, r.d_base, r.d_scan, tb, ws), "scan");
            CU(dwb::compact_paths(sl.paths, sl.len, bn, stride, sl.offs, sl.flat, ws), "compact");
            launches += 5;
        } else if (out.text) {  // write_paths bytes, formatted on the device
            uint32_t* bytes = sl.flat;
            size_t tb = r.scan_bytes;
            CU(dwb::path_text_bytes(sl.paths, sl.len, bn, stride, bytes, ws), "text");
            CU(dwb::path_offsets(bytes, bn, sl.offs, r.d_base, r.d_scan, tb, ws), "scan");
            CU(dwb::path_text_write(sl.paths, sl.len, bn, stride, sl.offs, sl.txt, ws), "text");
            launches += 6;
        }
        CU(cudaEventRecord(sl.walk, ws), "event");
        if (ordered) {
            CU(cudaStreamWaitEvent(r.ends, sl.walk, 0), "event");
            CU(cudaMemcpyAsync(r.h_ends + (li % kRingSlots), sl.offs + bn, sizeof(ull),
                               cudaMemcpyDeviceToHost, r.ends),
               "D2H end");
            CU(cudaEventRecord(sl.end, r.ends), "event");
        } else {
            CU(cudaStreamWaitEvent(r.d2h, sl.walk, 0), "event");
            if (out.paths)
                CU(cudaMemcpyAsync(out.paths + blo * stride, sl.paths,
                                   bn * stride * sizeof(uint32_t), cudaMemcpyDeviceToHost, r.d2h),
                   "D2H paths");
            if (out.lengths)
                CU(cudaMemcpyAsync(out.lengths + blo, sl.len, bn * sizeof(uint32_t),
                                   cudaMemcpyDeviceToHost, r.d2h),
                   "D2H lengths");
            CU(cudaEventRecord(sl.d2h, r.d2h), "event");
        }
        return DW_OK;
    };
    ull gbase = 0;  // ordered runs: ids (or text bytes) of the batches drained so far
    auto drain = [&](ull b) -> int {
        if (!ordered) return DW_OK;  // the D2H was enqueued with the walk
        const int di = (int)(b % nd);
        const ull li = b / nd;
        Replica& r = g->reps[di];
        Dev& d = dv[di];
        Replica::Slot& sl = r.slots[li % kRingSlots];
        const ull blo = at[b], bn = at[b + 1] - blo;
        CU(cudaSetDevice(r.device), "cudaSetDevice");
        CU(cudaEventSynchronize(sl.end), "walk");
        const ull end = r.h_ends[li % kRingSlots];
        const ull cnt = end - d.end;
        if (out.text) {  // the batch's text follows the previous batches in the file
            if (cnt) {
                CU(cudaMemcpyAsync(out.h_txt, sl.txt, cnt, cudaMemcpyDeviceToHost, r.d2h),
                   "D2H text");
                CU(cudaStreamSynchronize(r.d2h), "D2H text");
                if (std::fwrite(out.h_txt, 1, cnt, out.text) != cnt)
                    return fail(DW_EINVAL, "write failed: %s", out.text_path);
            }
            CU(cudaEventRecord(sl.d2h, r.d2h), "event");
            d.end = end;
            gbase += cnt;
            return DW_OK;
        }
        if (gbase + cnt > out.flat_cap) {
            for (auto& rr : g->reps) {
                cudaSetDevice(rr.device);
                cudaDeviceSynchronize();
            }
            return fail(DW_EINVAL, "flat path buffer too small: need more than %llu ids",
                        (unsigned long long)(gbase + cnt));
        }
        if (cnt) {
            if (!out.flat) return fail(DW_EINVAL, "flat is NULL");
            // every walk full length: the padded rows are the flat layout and
            // compact_paths skipped the copy
            const uint32_t* src = (cnt == bn * stride) ? sl.paths : sl.flat;
            CU(cudaMemcpyAsync(out.flat + gbase, src, cnt * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, r.d2h),
               "D2H paths");
        }
        CU(cudaMemcpyAsync(out.offsets + blo, sl.offs, bn * sizeof(ull), cudaMemcpyDeviceToHost,
                           r.d2h),
           "D2H offsets");
        CU(cudaEventRecord(sl.d2h, r.d2h), "event");
        // the device's offsets count its own batches only
        if (gbase != d.end && bn) fixups.push_back({blo, bn, gbase - d.end});
        d.end = end;
        gbase += cnt;
        return DW_OK;
    };
    for (ull eb = 0, db = 0; db < nb;) {
        if (eb < nb && dv[eb % nd].inflight < (ull)kRingSlots) {
            if (trace) std::fprintf(trace.get(), "E %llu %d\n", eb, (int)(eb % nd));
            if ((rc = enqueue(eb))) return rc;
            ++dv[eb % nd].inflight;
            ++eb;
        } else {
            if (trace) std::fprintf(trace.get(), "D %llu %d\n", db, (int)(db % nd));
            if ((rc = drain(db))) return rc;
            --dv[db % nd].inflight;
            ++db;
        }
    }
    double kmax = 0.0;
    for (int di = 0; di < nd; ++di) {
        Replica& r = g->reps[di];
        CU(cudaSetDevice(r.device), "cudaSetDevice");
        CU(cudaEventRecord(r.ev_stop, r.stream), "event");
        CU(cudaStreamSynchronize(r.stream), "walk");
        CU(cudaStreamSynchronize(r.copy), "copy");
        CU(cudaStreamSynchronize(r.ends), "copy");
        CU(cudaStreamSynchronize(r.d2h), "copy");
        if ((rc = collect(r, st, 0))) return rc;
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.ev_start, r.ev_stop);
        kmax = std::max(kmax, (double)ms);
    }
    if (out.compact) {
        for (const Fixup& f : fixups)
            for (ull i = f.lo; i < f.lo + f.n; ++i) out.offsets[i] += f.delta;
        out.offsets[nq] = gbase;
    }
    CU(cudaSetDevice(g->reps[0].device), "cudaSetDevice");
    CU(cudaEventRecord(wall1, g->reps[0].d2h), "event");
    CU(cudaEventSynchronize(wall1), "event");
    float wall = 0.f;
    cudaEventElapsedTime(&wall, wall0, wall1);
    cudaEventDestroy(wall0);
    cudaEventDestroy(wall1);
    if (st) {
        st->kernel_ms = kmax;
        st->total_ms = wall;
        st->kernel_launches = launches;
    }
    return DW_OK;
}

// ---- direct compact runs ---------------------------------------------------
// dw_run_compact on one device for walks whose lengths are known before they
// run: node2vec (a, b > 0: weights positive by construction), adaptive or
// force-erjs, on a graph where no edge leads to a vertex without neighbours
// (mirrored graphs: every target has its twin edge back).
// Then no walk stops early (runtime.cpp:115-153: dead ends need d = 0 or
// all-zero weights) and a path's length is 0 (start out of range), 1 (start
// without neighbours) or target + 1.  The offsets of RunResult's flattened
// paths are therefore a scan of the predicted lengths, computed before the
// walk, and one launch writes every path straight to its final place.  The
// walk counts finished walkers per chunk of 2^shift and raises a host-mapped
// flag per finished chunk; this thread copies each chunk to the caller's
// buffer as soon as it is final, so the copies overlap the walk and the run
// ends one chunk copy after the walk does (the batched engine pays a launch
// tail per batch and the final batch's copy).  A walk that ends up shorter
// than predicted makes the ids written fall short of the predicted total (the
// counters tell: every path is at most its predicted length), and the caller
// re-runs the batched engine.
constexpr ull kMaxChunks = 1024;
constexpr int kDirectNo = 1;     // not applicable: use the batched engine
constexpr int kDirectRetry = 2;  // prediction failed: use the batched engine

int listed_ok(Replica& r, const dw_model_desc* m, const dw_run_opts* o);

int direct_ok(dw_graph_t g, const dw_model_desc* m, const dw_run_opts* o, ull nq) {
    if (g->reps.size() != 1 || nq == 0 || nq >= (1ull << 32)) return kDirectNo;
    return listed_ok(g->reps[0], m, o);
}

// Every path length is known before the walk (see above) on replica r
int listed_ok(Replica& r, const dw_model_desc* m, const dw_run_opts* o) {
    // DW_DIRECT=0: always the batched engine; =2: predict even on a graph
    // with sinks (tests of the short-walk -> batched re-run path)
    bool force = false;
    if (const char* e = std::getenv("DW_DIRECT")) {
        if (e[0] == '0') return kDirectNo;
        force = e[0] == '2';
    }
    // the walk kernels with the direct layout: node2vec, adaptive / force-erjs
    // (dw_walk.cu DirectOk)
    if (m->kind != DW_MODEL_NODE2VEC || !model_params(m).pos_weights) return kDirectNo;
    if (o->mode != DW_MODE_ADAPTIVE && o->mode != DW_MODE_FORCE_ERJS) return kDirectNo;
    if (force) return DW_OK;
    if (r.sinks < 0) {
        CU(cudaSetDevice(r.device), "cudaSetDevice");
        if (!r.dir.flag) CU(cudaMalloc(&r.dir.flag, sizeof(int)), "cudaMalloc");
        CU(cudaMemsetAsync(r.dir.flag, 0, sizeof(int), r.stream), "memset");
        CU(dwb::sink_targets(r.g.nodes, r.g.edges, r.g.ne, r.dir.flag, r.stream), "sinks");
        int f = 0;
        CU(cudaMemcpyAsync(&f, r.dir.flag, sizeof(int), cudaMemcpyDeviceToHost, r.stream),
           "D2H");
        CU(cudaStreamSynchronize(r.stream), "sinks");
        r.sinks = f ? 1 : 0;
    }
    return r.sinks ? kDirectNo : DW_OK;
}

// grows the direct buffers to nq walkers / nflat ids; kDirectNo when device
// memory is short (the batched engine's ring is bounded)
int direct_buffers(Replica& r, ull nq, ull nflat, bool qids) {
    Replica::Direct& d = r.dir;
    if (!d.done) {
        CU(cudaMalloc(&d.done, kMaxChunks * sizeof(unsigned)), "cudaMalloc");
        CU(cudaHostAlloc(&d.h_flag, kMaxChunks * sizeof(unsigned), cudaHostAllocMapped),
           "cudaHostAlloc");
        CU(cudaHostAlloc(&d.h_bounds, (kMaxChunks + 3) * sizeof(ull), cudaHostAllocMapped),
           "cudaHostAlloc");
        for (cudaEvent_t* e : {&d.pre, &d.walk})
            CU(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "cudaEventCreate");
        CU(cudaEventCreate(&d.w0), "cudaEventCreate");
        CU(cudaEventCreate(&d.w1), "cudaEventCreate");
    }
    if (!d.flag) CU(cudaMalloc(&d.flag, sizeof(int)), "cudaMalloc");
    if (nq > d.cap_q || (qids && !d.has_qids) || nflat > d.cap_flat) {
        CU(cudaStreamSynchronize(r.stream), "sync");
        CU(cudaStreamSynchronize(r.copy), "sync");
        ull need = 0;
        const ull cq = std::max(nq, d.cap_q);
        const bool hq = qids || d.has_qids;
        const ull cf = std::max(nflat, d.cap_flat);
        if (cq > d.cap_q || hq != d.has_qids)
            need += cq * (sizeof(uint32_t) * 3 + sizeof(ull) * (hq ? 5 : 4));
        if (cf > d.cap_flat) need += cf * sizeof(uint32_t);
        size_t fr = 0, tot = 0;
        CU(cudaMemGetInfo(&fr, &tot), "cudaMemGetInfo");
        if ((ull)fr < need + (2ull << 30)) return kDirectNo;
        if (cq > d.cap_q || hq != d.has_qids) {
            for (void* p : {(void*)d.q, (void*)d.qids, (void*)d.len, (void*)d.offs, (void*)d.pos,
                            (void*)d.cq, (void*)d.cqid, (void*)d.coffs})
                cudaFree(p);
            d.q = d.len = d.cq = nullptr;
            d.qids = d.offs = d.pos = d.cqid = d.coffs = nullptr;
            d.cap_q = 0;
            CU(cudaMalloc(&d.q, cq * sizeof(uint32_t)), "cudaMalloc queries");
            CU(cudaMalloc(&d.len, cq * sizeof(uint32_t)), "cudaMalloc lengths");
            CU(cudaMalloc(&d.offs, (cq + 1) * sizeof(ull)), "cudaMalloc offsets");
            CU(cudaMalloc(&d.pos, (cq + 1) * sizeof(ull)), "cudaMalloc walker ranks");
            CU(cudaMalloc(&d.cq, cq * sizeof(uint32_t)), "cudaMalloc walker list");
            CU(cudaMalloc(&d.cqid, cq * sizeof(ull)), "cudaMalloc walker list");
            CU(cudaMalloc(&d.coffs, cq * sizeof(ull)), "cudaMalloc walker list");
            if (hq) CU(cudaMalloc(&d.qids, cq * sizeof(ull)), "cudaMalloc walker ids");
            d.cap_q = cq;
            d.has_qids = hq;
        }
        if (cf > d.cap_flat) {
            cudaFree(d.flat);
            d.flat = nullptr;
            d.cap_flat = 0;
            CU(cudaMalloc(&d.flat, cf * sizeof(uint32_t)), "cudaMalloc flat paths");
            d.cap_flat = cf;
        }
    }
    size_t need = 0;
    CU(dwb::path_offsets(nullptr, nq, nullptr, nullptr, nullptr, need, r.stream), "scan size");
    if (need > r.scan_bytes) {
        CU(cudaStreamSynchronize(r.stream), "sync");
        cudaFree(r.d_scan);
        r.d_scan = nullptr;
        r.scan_bytes = 0;
        CU(cudaMalloc(&r.d_scan, need), "cudaMalloc scan");
        r.scan_bytes = need;
    }
    return DW_OK;
}

int run_direct(dw_graph_t g, const dw_model_desc* model, const uint32_t* queries, ull nq,
               const dw_run_opts* opts, const RunOut& out, dw_run_stats* st) {
    int rc;
    if ((rc = direct_ok(g, model, opts, nq))) return rc;
    Replica& r = g->reps[0];
    Replica::Direct& d = r.dir;
    CU(cudaSetDevice(r.device), "cudaSetDevice");
    if ((rc = prepare_model(r, model))) return rc;
    // the flat size is known only after the scan: reserve the bound
    // nq * (target + 1) (always enough) up front
    const uint32_t target = target_steps(model, opts);
    const ull bound = nq * ((ull)target + 1);
    if ((rc = direct_buffers(r, nq, bound, opts->qids != nullptr))) return rc;
    // ~256 chunks of >= 16K walkers (a smaller chunk's copy is launch-bound)
    uint32_t shift = 14;
    while ((nq >> shift) > 256 && shift < 24) ++shift;
    while (((nq + (1ull << shift) - 1) >> shift) > kMaxChunks) ++shift;
    const ull nch_max = (nq + (1ull << shift) - 1) >> shift;
    cudaStream_t ws = r.stream, cp = r.copy;
    std::memset(d.h_flag, 0, nch_max * sizeof(unsigned));
    if (st) std::memset(st, 0, sizeof *st);
    CU(cudaEventRecord(d.w0, ws), "event");
    CU(cudaMemcpyAsync(d.q, queries, nq * sizeof(uint32_t), cudaMemcpyHostToDevice, ws),
       "H2D queries");
    if (opts->qids)
        CU(cudaMemcpyAsync(d.qids, opts->qids, nq * sizeof(ull), cudaMemcpyHostToDevice, ws),
           "H2D walker ids");
    if ((rc = reset_run_state(r))) return rc;
    CU(cudaMemsetAsync(d.done, 0, nch_max * sizeof(unsigned), ws), "memset");
    CU(cudaMemsetAsync(r.d_base, 0, sizeof(ull), ws), "memset");
    // offsets of every path, then the walkers whose path is final already
    // (start out of range or without neighbours: 56 % of the s24 starts) are
    // written here, and the walk gets only the list of the others: no claim,
    // node gather or chunk count for them in the walk
    CU(dwb::predict_lengths(d.q, nq, r.g.nodes, r.g.nv, target, d.len, ws), "predict");
    size_t tb = r.scan_bytes;
    CU(dwb::path_offsets(d.len, nq, d.offs, r.d_base, r.d_scan, tb, ws), "scan");
    CU(dwb::trivial_walkers(d.q, nq, d.len, d.offs, d.flat, r.counters, ws), "trivial walkers");
    CU(cudaMemsetAsync(r.d_base, 0, sizeof(ull), ws), "memset");
    CU(dwb::path_offsets(d.len, nq, d.pos, r.d_base, r.d_scan, tb, ws), "scan");
    CU(dwb::walker_list(d.q, opts->qids ? d.qids : nullptr, opts->qid_base, nq, d.len, d.pos,
                        d.offs, 0, d.cq, d.cqid, d.coffs, ws),
       "walker list");
    CU(dwb::direct_bounds(d.coffs, r.d_base, d.offs + nq, shift, kMaxChunks, d.h_bounds, ws),
       "bounds");
    CU(cudaEventRecord(d.pre, ws), "event");
    CU(cudaEventSynchronize(d.pre), "predict");
    const ull nt = d.h_bounds[kMaxChunks + 1], nch = d.h_bounds[kMaxChunks + 2];
    const ull total = d.h_bounds[nch];
    if (total > out.flat_cap)
        return fail(DW_EINVAL, "flat path buffer too small: need %llu ids",
                    (unsigned long long)total);
    if (total && !out.flat) return fail(DW_EINVAL, "flat is NULL");
    dwb::WalkParams p = make_params(r, model, opts);
    p.queries = d.cq;
    p.nq = nt;
    p.qid_base = 0;
    p.qids = d.cqid;
    p.paths = d.flat;
    p.lengths = nullptr;
    p.next_walker = r.queues;
    p.offs = d.coffs;
    p.chunk_done = d.done;
    p.chunk_flag = d.h_flag;
    p.chunk_shift = shift;
    CU(cudaEventRecord(r.ev_start, ws), "event");
    if (nt) {
        CU(cudaMemsetAsync(p.next_walker, 0, sizeof(ull), ws), "memset");
        CU(launch_model(r, model, opts->mode, p, ws), "walk");
    }
    CU(cudaEventRecord(r.ev_stop, ws), "event");
    CU(cudaEventRecord(d.walk, ws), "event");
    // the offsets are final already: their copy overlaps the walk
    CU(cudaMemcpyAsync(out.offsets, d.offs, (nq + 1) * sizeof(ull), cudaMemcpyDeviceToHost, cp),
       "D2H offsets");
    if (nch == 0 && total)  // no walker walks: every path is final
        CU(cudaMemcpyAsync(out.flat, d.flat, total * sizeof(uint32_t), cudaMemcpyDeviceToHost, cp),
           "D2H paths");
    // copy every chunk as soon as its walkers are final
    volatile unsigned* flag = d.h_flag;
    bool walk_done = false;
    for (ull c = 0; c < nch; ++c) {
        while (!flag[c]) {
            if (walk_done) break;
            if (cudaEventQuery(d.walk) == cudaSuccess) walk_done = true;  // recheck the flag
            else std::this_thread::yield();
        }
        if (!flag[c]) break;  // the walk stopped on an error: collect() reports it
        const ull lo = d.h_bounds[c], hi = d.h_bounds[c + 1];
        if (hi > lo)
            CU(cudaMemcpyAsync(out.flat + lo, d.flat + lo, (hi - lo) * sizeof(uint32_t),
                               cudaMemcpyDeviceToHost, cp),
               "D2H paths");
    }
    CU(cudaStreamWaitEvent(cp, d.walk, 0), "event");
    CU(cudaEventRecord(d.w1, cp), "event");
    CU(cudaStreamSynchronize(ws), "walk");
    if ((rc = collect(r, st, 0))) {
        cudaStreamSynchronize(cp);
        return rc;
    }
    CU(cudaStreamSynchronize(cp), "copy");
    // every path is at most its predicted length, so the lengths all match
    // iff their sum does: ids written = walkers with a start in range + steps
    // that advanced (runtime.cpp:141-149)
    dw_run_stats cs;
    std::memset(&cs, 0, sizeof cs);
    {
        ull c[dwb::kCNum];
        CU(cudaMemcpy(c, r.counters, sizeof c, cudaMemcpyDeviceToHost), "D2H counters");
        add_counters(&cs, c);
    }
    const bool mis = cs.queries - cs.query_errors + cs.steps - cs.dead_ends != total;
    if (const char* tp = std::getenv("DW_ENGINE_TRACE"))
        if (FILE* f = std::fopen(tp, "a")) {
            std::fprintf(f, "X %llu %s\n", (unsigned long long)nq, mis ? "retry" : "ok");
            std::fclose(f);
        }
    if (mis) {
        r.sinks = 1;  // do not predict on this graph again
        return kDirectRetry;
    }
    if (st) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.ev_start, r.ev_stop);
        st->kernel_ms = ms;
        cudaEventElapsedTime(&ms, d.w0, d.w1);
        st->total_ms = ms;
        st->kernel_launches = 10 + (nt ? 1 : 0);
    }
    if (std::getenv("DW_VERBOSE")) {
        float a = 0.f, b = 0.f, c = 0.f;
        cudaEventElapsedTime(&a, d.w0, r.ev_start);
        cudaEventElapsedTime(&b, r.ev_start, r.ev_stop);
        cudaEventElapsedTime(&c, r.ev_stop, d.w1);
        std::fprintf(stderr, "dynwalk direct: %llu chunks, before walk %.3f ms, walk %.3f ms, after %.3f ms\n",
                     (unsigned long long)nch, a, b, c);
    }
    return DW_OK;
}

// dw_run_device when every path length is known before the walk (listed_ok):
// `trivial_rows` writes every length (the predicted one) and the padded row
// of each walker that does not move (start without neighbours: 56 % of the
// s24 starts), and one walk over the
// list of the others (`walker_list`, rows at i * stride, walker ids as RNG
// keys) writes their rows: no claim or node gather for the walkers that
// cannot move.  The host reads the list's length before the launch (the walk
// sizes its grid by it).  dw_run_device_sync checks that no walk ended early
// (steps - dead ends = listed walkers * target) and otherwise re-runs every
// walker on the padded kernel.
int run_device_listed(Replica& r, const dw_model_desc* model, const uint32_t* d_queries, ull nq,
                      const dw_run_opts* opts, uint32_t* d_paths, uint32_t* d_lengths,
                      cudaStream_t s) {
    // below ~1M walkers the walk is short and the host round trip for the
    // list's length plus the extra passes cost more than they save (R-MAT
    // s16, 65K walkers: 0.73 ms a pass against 0.66 ms)
    if (nq < (1ull << 20)) return kDirectNo;
    int rc;
    if ((rc = listed_ok(r, model, opts))) return rc;
    if ((rc = direct_buffers(r, nq, 0, false))) return rc;
    Replica::Direct& d = r.dir;
    const uint32_t target = target_steps(model, opts);
    const ull stride = (ull)opts->walk_length + 1;
    // no memset of the rows: trivial_rows pads the rows of the walkers that
    // do not move, and the walk fills every row of the others (no walk ends
    // early here; the sync check re-runs on a memset buffer if one did)
    CU(cudaMemsetAsync(r.d_base, 0, sizeof(ull), s), "memset");
    CU(dwb::predict_lengths(d_queries, nq, r.g.nodes, r.g.nv, target, d.len, s), "predict");
    CU(dwb::trivial_rows(d_queries, nq, d.len, d_paths, stride, d_lengths, r.counters, s),
       "trivial rows");
    size_t tb = r.scan_bytes;
    CU(dwb::path_offsets(d.len, nq, d.pos, r.d_base, r.d_scan, tb, s), "scan");
    CU(dwb::walker_list(d_queries, reinterpret_cast<const ull*>(opts->qids), opts->qid_base, nq,
                        d.len, d.pos, nullptr, stride, d.cq, d.cqid, d.coffs, s),
       "walker list");
    ull nt = 0;
    CU(cudaMemcpyAsync(&nt, r.d_base, sizeof(ull), cudaMemcpyDeviceToHost, s), "D2H");
    CU(cudaStreamSynchronize(s), "walker list");
    dwb::WalkParams p = make_params(r, model, opts);
    p.queries = d.cq;
    p.nq = nt;
    p.qid_base = 0;
    p.qids = d.cqid;
    p.paths = d_paths;
    p.lengths = nullptr;
    p.next_walker = r.queues;
    p.offs = d.coffs;  // kOutFlat kernel: rows at i * stride, no chunk counts
    CU(cudaEventRecord(r.ev_start, s), "event");
    if (nt) CU(launch_model(r, model, opts->mode, p, s), "walk");
    CU(cudaEventRecord(r.ev_stop, s), "event");
    Replica::Listed& l = r.listed;
    l.on = true;
    l.target = target;
    l.model = *model;
    l.opts = *opts;
    l.queries = d_queries;
    l.nq = nq;
    l.paths = d_paths;
    l.lengths = d_lengths;
    l.stream = s;
    l.nt = nt;
    r.pending = true;
    r.pending_launches = 6 + (nt ? 1 : 0);
    r.pending_qbase = opts->qid_base;
    return DW_OK;
}

}  // namespace

// ---- DWG1 binary CSR cache, streamed to the devices (graph.cpp:217-300) ----
namespace {

struct Dwg1Reader {
    FILE* f = nullptr;
    std::string path;
    ~Dwg1Reader() {
        if (f) std::fclose(f);
    }
    bool read(void* dst, size_t n) { return std::fread(dst, 1, n, f) == n; }
};

// Streams `count` elements of `elem` bytes from the file into every device
// array in `dst` through two pinned staging buffers (file reads overlap the
// H2D copies).  first/last receive the array's first and last 8-byte words
// when non-null (the offsets array checks).
int stream_array(Dwg1Reader& rd, dw_graph_s* g, const std::vector<void*>& dst, ull count,
                 size_t elem, ull* first, ull* last) {
    constexpr size_t kChunk = 64u << 20;
    void* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2][8] = {};
    const int nd = (int)g->reps.size();
    CU(cudaSetDevice(g->reps[0].device), "cudaSetDevice");
    CU(cudaMallocHost(&stage[0], kChunk), "cudaMallocHost");
    CU(cudaMallocHost(&stage[1], kChunk), "cudaMallocHost");
    int rc = DW_OK;
    const ull bytes = count * elem;
    ull off = 0;
    int k = 0;
    bool used[2] = {false, false};
    while (off < bytes && rc == DW_OK) {
        const size_t n = (size_t)std::min<ull>(kChunk, bytes - off);
        if (used[k])
            for (int di = 0; di < nd && di < 8; ++di) cudaEventSynchronize(done[k][di]);
        if (!rd.read(stage[k], n)) {
            rc = fail(DW_EINVAL, "truncated binary graph file: %s", rd.path.c_str());
            break;
        }
        if (first && off == 0 && n >= 8) std::memcpy(first, stage[k], 8);
        if (last && off + n == bytes && n >= 8) std::memcpy(last, (char*)stage[k] + n - 8, 8);
        for (int di = 0; di < nd && rc == DW_OK; ++di) {
            Replica& r = g->reps[di];
            if (cudaSetDevice(r.device) != cudaSuccess ||
                cudaMemcpyAsync((char*)dst[di] + off, stage[k], n, cudaMemcpyHostToDevice,
                                r.copy) != cudaSuccess) {
                rc = fail(DW_ECUDA, "H2D of %s failed", rd.path.c_str());
                break;
            }
            if (!done[k][di]) cudaEventCreateWithFlags(&done[k][di], cudaEventDisableTiming);
            cudaEventRecord(done[k][di], r.copy);
        }
        used[k] = true;
        off += n;
        k ^= 1;
    }
    for (int j = 0; j < 2; ++j)
        for (int di = 0; di < nd && di < 8; ++di)
            if (done[j][di]) {
                cudaEventSynchronize(done[j][di]);
                cudaEventDestroy(done[j][di]);
            }
    cudaFreeHost(stage[0]);
    cudaFreeHost(stage[1]);
    return rc;
}

int read_count(Dwg1Reader& rd, ull* n) {
    if (!rd.read(n, sizeof *n))
        return fail(DW_EINVAL, "truncated binary graph file: %s", rd.path.c_str());
    return DW_OK;
}

}  // namespace

extern "C" int dw_graph_load_dwg1(const char* path, const int* devices, int ndev,
                                  dw_graph_t* out) {
    if (!out || !path) return fail(DW_EINVAL, "NULL argument");
    *out = nullptr;
    Dwg1Reader rd;
    rd.path = path;
    rd.f = std::fopen(path, "rb");
    if (!rd.f) return fail(DW_EINVAL, "cannot open graph file: %s", path);
    char magic[4];
    if (!rd.read(magic, 4) || std::memcmp(magic, "DWG1", 4) != 0)
        return fail(DW_EINVAL, "not a binary graph file: %s", path);
    uint32_t version = 0;
    if (!rd.read(&version, 4) || version != 1)
        return fail(DW_EINVAL, "unsupported binary graph version %u", version);
    uint8_t labels = 0;
    if (!rd.read(&labels, 1)) return fail(DW_EINVAL, "truncated binary graph file: %s", path);
    ull n_off = 0;
    int rc;
    if ((rc = read_count(rd, &n_off))) return rc;
    if (n_off == 0) return fail(DW_EINVAL, "corrupt binary graph file: %s", path);
    if (n_off - 1 >= DW_INVALID_VERTEX)
        return fail(DW_EINVAL, "vertex id overflow: graph needs %llu vertices",
                    (unsigned long long)(n_off - 1));
    std::vector<int> devs;
    if ((rc = resolve_devices(devices, ndev, devs))) return rc;
    auto* g = new dw_graph_s;
    std::unique_ptr<dw_graph_s, int (*)(dw_graph_t)> guard(g, dw_graph_destroy);
    g->reps.resize(devs.size());
    for (size_t i = 0; i < devs.size(); ++i)
        if ((rc = init_replica(g->reps[i], devs[i]))) return rc;
    const int nd = (int)devs.size();
    std::vector<ull*> row(nd, nullptr);
    std::vector<uint32_t*> col(nd, nullptr);
    std::vector<float*> prop(nd, nullptr);
    std::vector<uint16_t*> lab(nd, nullptr);
    auto free_all = [&]() {
        for (int di = 0; di < nd; ++di) {
            cudaSetDevice(g->reps[di].device);
            cudaFree(row[di]);
            cudaFree(col[di]);
            cudaFree(prop[di]);
            if (!g->reps[di].g.labels) cudaFree(lab[di]);
        }
    };
    std::vector<void*> dst(nd);
    // offsets
    for (int di = 0; di < nd; ++di) {
        CU(cudaSetDevice(g->reps[di].device), "cudaSetDevice");
        CU(cudaMalloc(&row[di], n_off * sizeof(ull)), "cudaMalloc offsets");
        dst[di] = row[di];
    }
    ull front = 0, back = 0;
    if ((rc = stream_array(rd, g, dst, n_off, sizeof(ull), &front, &back))) {
        free_all();
        return rc;
    }
    // targets, props, labels
    ull ne = 0;
    if ((rc = read_count(rd, &ne))) {
        free_all();
        return rc;
    }
    if (front != 0 || back != ne) {
        free_all();
        return fail(DW_EINVAL, "corrupt binary graph file: %s", path);
    }
    for (int di = 0; di < nd; ++di) {
        CU(cudaSetDevice(g->reps[di].device), "cudaSetDevice");
        CU(cudaMalloc(&col[di], std::max<ull>(ne, 1) * sizeof(uint32_t)), "cudaMalloc");
        CU(cudaMalloc(&prop[di], std::max<ull>(ne, 1) * sizeof(float)), "cudaMalloc");
        if (labels) CU(cudaMalloc(&lab[di], ((std::max<ull>(ne, 1) + 1) & ~1ull) * sizeof(uint16_t)), "cudaMalloc");
        dst[di] = col[di];
    }
    if ((rc = stream_array(rd, g, dst, ne, sizeof(uint32_t), nullptr, nullptr))) {
        free_all();
        return rc;
    }
    ull n = 0;
    if ((rc = read_count(rd, &n))) {
        free_all();
        return rc;
    }
    if (n != ne) {
        free_all();
        return fail(DW_EINVAL, "corrupt binary graph file: %s", path);
    }
    for (int di = 0; di < nd; ++di) dst[di] = prop[di];
    if ((rc = stream_array(rd, g, dst, ne, sizeof(float), nullptr, nullptr))) {
        free_all();
        return rc;
    }
    if (labels) {
        if ((rc = read_count(rd, &n))) {
            free_all();
            return rc;
        }
        if (n != ne) {
            free_all();
            return fail(DW_EINVAL, "corrupt binary graph file: %s", path);
        }
        for (int di = 0; di < nd; ++di) dst[di] = lab[di];
        if ((rc = stream_array(rd, g, dst, ne, sizeof(uint16_t), nullptr, nullptr))) {
            free_all();
            return rc;
        }
    }
    // Graph::build's invariants, then the device layout (pack_graph)
    uint32_t nv = 0;
    for (int di = 0; di < nd; ++di) {
        Replica& r = g->reps[di];
        CU(cudaSetDevice(r.device), "cudaSetDevice");
        CU(cudaStreamSynchronize(r.copy), "H2D");
        nv = (uint32_t)(n_off - 1);
        int status = 0;
        CU(dwb::prepare_loaded_csr(&row[di], &nv, ne, col[di], prop[di], lab[di], &status,
                                   r.stream),
           "prepare csr");
        if (status) {
            free_all();
            return fail(DW_EINVAL, status == 1 ? "edge property must be strictly positive and finite"
                                   : status == 2 ? "vertex id overflow"
                                                 : "unsorted adjacency slices above 2^31 edges are not supported");
        }
        r.g.nv = nv;
        r.g.ne = ne;
        CU(cudaMalloc(&r.g.nodes, std::max<uint32_t>(nv, 1) * sizeof(dwb::NodeRec)), "cudaMalloc nodes");
        CU(cudaMalloc(&r.g.edges, ((std::max<ull>(ne, 1) + 1) & ~1ull) * sizeof(dwb::EdgeRec)), "cudaMalloc edges");
        r.g.labels = lab[di];  // owned by the replica from here on
        CU(dwb::pack_graph(row[di], col[di], prop[di], nullptr, nullptr, r.g, r.stream), "pack_graph");
        CU(cudaStreamSynchronize(r.stream), "pack");
    }
    free_all();
    for (auto& r : g->reps) {
        CU(cudaSetDevice(r.device), "cudaSetDevice");
        CU(dwb::finish_graph(r.g, r.stream), "fat records");
    }
    g->nv = nv;
    g->ne = ne;
    g->has_labels = labels != 0;
    g->max_degree = g->reps[0].g.max_degree;
    *out = guard.release();
    return DW_OK;
}

extern "C" {

int dw_abi_version(void) { return DW_ABI_VERSION; }

const char* dw_last_error(void) { return t_error.c_str(); }

int dw_device_count(int* n) {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    if (e != cudaSuccess) c = 0;
    if (n) *n = c;
    return DW_OK;
}

int dw_graph_create(const dw_graph_desc* desc, const int* devices, int ndev, dw_graph_t* out) {
    if (!out) return fail(DW_EINVAL, "output handle pointer is NULL");
    *out = nullptr;
    std::vector<int> devs;
    int rc = resolve_devices(devices, ndev, devs);
    if (rc) return rc;
    if ((rc = validate_desc(desc))) return rc;
    auto* g = new dw_graph_s;
    g->nv = desc->num_vertices;
    g->ne = desc->num_edges;
    g->has_labels = desc->edge_labels != nullptr;
    g->reps.resize(devs.size());
    for (size_t i = 0; i < devs.size(); ++i) {
        if ((rc = init_replica(g->reps[i], devs[i])) || (rc = upload_replica(g->reps[i], desc))) {
            dw_graph_destroy(g);
            return rc;
        }
    }
    g->max_degree = g->reps[0].g.max_degree;
    *out = g;
    return DW_OK;
}

int dw_graph_generate_rmat(const dw_rmat_desc* d, const int* devices, int ndev, dw_graph_t* out) {
    if (!out || !d) return fail(DW_EINVAL, "NULL argument");
    *out = nullptr;
    if (d->scale > 30 || d->edge_factor < 2 || (2ull * (d->edge_factor / 2) << d->scale) > (1ull << 34))
        return fail(DW_EINVAL, "rmat: scale %u / edge factor %u out of range", d->scale,
                    d->edge_factor);
    if (d->weights == 0 && !(d->low > 0.0 && d->low < d->high))
        return fail(DW_EINVAL, "uniform weight spec requires 0 < low < high");
    if (d->weights == 2 && !(d->alpha > 0.0))
        return fail(DW_EINVAL, "pareto weight spec requires alpha > 0");
    if (d->weights != 0 && d->weights != 2 && d->weights != -1)
        return fail(DW_EINVAL, "unknown weight kind %d", d->weights);
    if (d->labels && !(d->label_low <= d->label_high && d->label_high <= 65535))
        return fail(DW_EINVAL, "label spec requires 0 <= low <= high <= 65535");
    std::vector<int> devs;
    int rc = resolve_devices(devices, ndev, devs);
    if (rc) return rc;
    dwb::RmatSpec spec{d->scale, d->edge_factor, d->seed, d->weights, d->low, d->high, d->alpha,
                       d->weight_seed, d->labels, d->label_low, d->label_high, d->label_seed};
    auto* g = new dw_graph_s;
    g->reps.resize(devs.size());
    for (size_t i = 0; i < devs.size(); ++i) {
        Replica& r = g->reps[i];
        if ((rc = init_replica(r, devs[i]))) {
            dw_graph_destroy(g);
            return rc;
        }
        cudaError_t e = dwb::build_rmat(spec, r.g, r.stream);
        if (e != cudaSuccess) {
            dw_graph_destroy(g);
            return cuda_fail(e, "build_rmat");
        }
    }
    g->nv = g->reps[0].g.nv;
    g->ne = g->reps[0].g.ne;
    g->has_labels = d->labels != 0;
    g->max_degree = g->reps[0].g.max_degree;
    *out = g;
    return DW_OK;
}

int dw_graph_destroy(dw_graph_t g) {
    if (!g) return DW_OK;
    for (auto& r : g->reps) free_replica(r);
    delete g;
    return DW_OK;
}

int dw_graph_info(dw_graph_t g, uint32_t* nv, uint64_t* ne, int* has_labels, uint32_t* max_degree) {
    if (!g) return fail(DW_EINVAL, "graph handle is NULL");
    if (nv) *nv = g->nv;
    if (ne) *ne = g->ne;
    if (has_labels) *has_labels = g->has_labels ? 1 : 0;
    if (max_degree) *max_degree = g->max_degree;
    return DW_OK;
}

int dw_graph_download(dw_graph_t g, uint64_t* row, uint32_t* col, float* prop, uint16_t* label,
                      double* nmax, double* nsum) {
    if (!g) return fail(DW_EINVAL, "graph handle is NULL");
    Replica& r = g->reps[0];
    CU(cudaSetDevice(r.device), "cudaSetDevice");
    // the unpacked CSR needs ~8 B per edge of scratch: give back the direct
    // compact runs' cached buffers first (config 5: 45 GB)
    CU(cudaStreamSynchronize(r.stream), "sync");
    CU(cudaStreamSynchronize(r.copy), "sync");
    free_direct(r.dir);
    const ull nv = g->nv, ne = g->ne;
    ull* d_row = nullptr;
    uint32_t* d_col = nullptr;
    float* d_prop = nullptr;
    double *d_nmax = nullptr, *d_nsum = nullptr;
    struct Scratch {
        void** p[5];
        ~Scratch() {
            for (void** q : p) cudaFree(*q);
        }
    } scratch{{(void**)&d_row, (void**)&d_col, (void**)&d_prop, (void**)&d_nmax, (void**)&d_nsum}};
    if (row) CU(cudaMalloc(&d_row, (nv + 1) * sizeof(ull)), "cudaMalloc");
    if (col) CU(cudaMalloc(&d_col, std::max<ull>(ne, 1) * sizeof(uint32_t)), "cudaMalloc");
    if (prop) CU(cudaMalloc(&d_prop, std::max<ull>(ne, 1) * sizeof(float)), "cudaMalloc");
    if (nmax) CU(cudaMalloc(&d_nmax, std::max<ull>(nv, 1) * sizeof(double)), "cudaMalloc");
    if (nsum) CU(cudaMalloc(&d_nsum, std::max<ull>(nv, 1) * sizeof(double)), "cudaMalloc");
    CU(dwb::unpack_graph(r.g, d_row, d_col, d_prop, d_nmax, d_nsum, r.stream), "unpack");
    CU(cudaStreamSynchronize(r.stream), "unpack");
    if (row) CU(cudaMemcpy(row, d_row, (nv + 1) * sizeof(ull), cudaMemcpyDeviceToHost), "D2H");
    if (col && ne) CU(cudaMemcpy(col, d_col, ne * sizeof(uint32_t), cudaMemcpyDeviceToHost), "D2H");
    if (prop && ne) CU(cudaMemcpy(prop, d_prop, ne * sizeof(float), cudaMemcpyDeviceToHost), "D2H");
    if (nmax && nv) CU(cudaMemcpy(nmax, d_nmax, nv * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    if (nsum && nv) CU(cudaMemcpy(nsum, d_nsum, nv * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    if (label && r.g.labels && ne)
        CU(cudaMemcpy(label, r.g.labels, ne * sizeof(uint16_t), cudaMemcpyDeviceToHost), "D2H");
    return DW_OK;
}

int dw_calibrate_ex(dw_graph_t g, const dw_model_desc* model, const dw_profile_config* cfg,
                    double* ratio) {
    if (!g || !ratio || !cfg) return fail(DW_EINVAL, "NULL argument");
    // cost_model.cpp:39-42
    if (!(cfg->node_fraction > 0.0) || cfg->node_fraction > 1.0)
        return fail(DW_EINVAL, "profile node_fraction must be in (0, 1]");
    if (cfg->neighbors_per_node == 0 || cfg->repetitions == 0)
        return fail(DW_EINVAL, "profile neighbors_per_node and repetitions must be >= 1");
    int rc = check_model(model);
    if (rc) return rc;
    if (model->kind == DW_MODEL_CUSTOM)
        return fail(DW_EUNSUPPORTED,
                    "device calibration of DSL models is not supported; pass edge_cost_ratio");
    Replica& r = g->reps[0];
    CU(cudaSetDevice(r.device), "cudaSetDevice");
    const dwb::ModelParams mp = model_params(model);
    const dwb::ProfileSpec spec{cfg->node_fraction, cfg->min_nodes, cfg->neighbors_per_node,
                                cfg->repetitions, cfg->seed};
    cudaError_t e = dwb::calibrate_ratio(r.g, model->kind, model->weighted != 0, mp, spec,
                                         r.stream, ratio);
    if (e == cudaErrorInvalidValue) return fail(DW_EINVAL, "profiling found no node with out-edges");
    if (e != cudaSuccess) return cuda_fail(e, "calibrate");
    if (!(*ratio > 0.0) || !std::isfinite(*ratio))
        return fail(DW_EINVAL, "profiled edge cost ratio is not positive and finite");
    return DW_OK;
}

int dw_calibrate(dw_graph_t g, const dw_model_desc* model, uint64_t seed, double* ratio) {
    const dw_profile_config cfg{0.01, 64, 32, 5, seed};
    return dw_calibrate_ex(g, model, &cfg, ratio);
}

int dw_tune_ratio(dw_graph_t g, const dw_model_desc* model, const dw_profile_config* cfg,
                  uint32_t walk_length, double* ratio) {
    if (!g || !ratio || !cfg) return fail(DW_EINVAL, "NULL argument");
    double r0 = 0.0;
    int rc = dw_calibrate_ex(g, model, cfg, &r0);
    if (rc) return rc;
    if (walk_length == 0) walk_length = 80;
    Replica& r = g->reps[0];
    CU(cudaSetDevice(r.device), "cudaSetDevice");
    if ((rc = prepare_model(r, model))) return rc;
    // walker sample: uniform start vertices (all_vertices' distribution), up
    // to 2^24 of them -- a launch of a few ms ends in a tail whose lanes wait
    // on single walkers, and that tail favours other thresholds than a full
    // walk does (s24: 1.8M walkers put the optimum at ~0.4, all 16.8M at ~0.9)
    const ull nq = std::min<ull>(std::max<ull>(g->nv, 1), 1ull << 24);
    std::vector<uint32_t> hq(nq);
    ull x = cfg->seed ^ 0x74756e65ull;
    for (ull i = 0; i < nq; ++i) {  // SplitMix64 (rng.hpp:10-20)
        ull z = (x += 0x9E3779B97F4A7C15ull);
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        hq[i] = (uint32_t)((unsigned __int128)(z ^ (z >> 31)) * g->nv >> 64);
    }
    uint32_t* dq = nullptr;
    CU(cudaMalloc(&dq, nq * sizeof(uint32_t)), "cudaMalloc");
    std::unique_ptr<uint32_t, cudaError_t (*)(void*)> hold(dq, &cudaFree);
    CU(cudaMemcpy(dq, hq.data(), nq * sizeof(uint32_t), cudaMemcpyHostToDevice), "H2D");
    dw_run_opts o{};
    o.mode = DW_MODE_ADAPTIVE;
    o.walk_length = walk_length;
    o.seed = cfg->seed;
    o.erjs_cap_per_degree = 64;
    // walker-steps per ms of the walk kernel at one ratio (median of reps)
    auto rate = [&](double ratio_c, double* out) -> int {
        o.edge_cost_ratio = ratio_c;
        std::vector<double> v;
        const uint32_t reps = std::max<uint32_t>(1, std::min<uint32_t>(cfg->repetitions, 3));
        for (uint32_t k = 0; k < reps; ++k) {
            int e = reset_run_state(r);
            if (e) return e;
            dwb::WalkParams p = make_params(r, model, &o);
            p.queries = dq;
            p.nq = nq;
            p.next_walker = r.queues;
            CU(cudaEventRecord(r.ev_start, r.stream), "event");
            CU(launch_model(r, model, o.mode, p, r.stream), "walk");
            CU(cudaEventRecord(r.ev_stop, r.stream), "event");
            CU(cudaEventSynchronize(r.ev_stop), "walk");
            dw_run_stats st{};
            if ((e = collect(r, &st, 0))) return e;
            float ms = 0.f;
            cudaEventElapsedTime(&ms, r.ev_start, r.ev_stop);
            v.push_back((double)(st.steps - st.dead_ends) / std::max(1e-3, (double)ms));
        }
        std::sort(v.begin(), v.end());
        *out = v[v.size() / 2];
        return DW_OK;
    };
    double warm = 0.0;
    if ((rc = rate(r0, &warm))) return rc;
    // throughput on a log2 grid around the micro-pass estimate; a least-
    // squares parabola through the five points smooths the timing noise (the
    // optimum is flat: within 2 % over a factor of ~2 at s24) and its vertex,
    // kept inside the grid, is the threshold
    const double xs[5] = {-1.0, -0.5, 0.0, 0.5, 1.0};
    double ys[5], best = r0, best_rate = 0.0;
    for (int i = 0; i < 5; ++i) {
        if ((rc = rate(r0 * std::exp2(xs[i]), &ys[i]))) return rc;
        if (ys[i] > best_rate) best_rate = ys[i], best = r0 * std::exp2(xs[i]);
    }
    // x symmetric around 0: the normal equations decouple
    double sy = 0, sxy = 0, sx2y = 0;
    for (int i = 0; i < 5; ++i) {
        sy += ys[i];
        sxy += xs[i] * ys[i];
        sx2y += xs[i] * xs[i] * ys[i];
    }
    const double s2 = 2.5, s4 = 2.125, n = 5.0;  // sum x^2, sum x^4
    const double qa = (n * sx2y - s2 * sy) / (n * s4 - s2 * s2);
    const double qb = sxy / s2;
    if (qa < 0.0) best = r0 * std::exp2(std::clamp(-qb / (2.0 * qa), -1.0, 1.0));
    if (std::getenv("DW_VERBOSE")) {
        for (int i = 0; i < 5; ++i)
            std::fprintf(stderr, "dynwalk: tune ratio %.4f -> %.4e walker-steps/s\n",
                         r0 * std::exp2(xs[i]), ys[i] * 1e3);
        std::fprintf(stderr, "dynwalk: tuned ratio %.4f (micro-pass %.4f)\n", best, r0);
    }
    *ratio = best;
    return DW_OK;
}

int dw_run_device(dw_graph_t g, int replica, const dw_model_desc* model, const uint32_t* d_queries,
                  uint64_t nq, const dw_run_opts* opts, uint32_t* d_paths, uint32_t* d_lengths,
                  void* stream) {
    if (!g) return fail(DW_EINVAL, "graph handle is NULL");
    if (replica < 0 || replica >= (int)g->reps.size())
        return fail(DW_EINVAL, "replica %d out of range", replica);
    int rc;
    if ((rc = check_model(model)) || (rc = check_opts(opts))) return rc;
    if (nq > 0xFFFFFFFFull)  // the kernel indexes a launch's walkers with 32 bits
        return fail(DW_EINVAL, "at most 2^32 - 1 queries per device launch (got %llu)",
                    (unsigned long long)nq);
    Replica& r = g->reps[replica];
    CU(cudaSetDevice(r.device), "cudaSetDevice");
    if ((rc = prepare_model(r, model))) return rc;
    cudaStream_t s = stream ? (cudaStream_t)stream : r.stream;
    if ((rc = reset_run_state(r))) return rc;
    if (s != r.stream) {  // order the resets before work on the caller's stream
        CU(cudaEventRecord(r.ev_reset, r.stream), "event");
        CU(cudaStreamWaitEvent(s, r.ev_reset, 0), "event");
    }
    r.listed.on = false;
    rc = run_device_listed(r, model, d_queries, nq, opts, d_paths, d_lengths, s);
    if (rc != kDirectNo) return rc;
    dwb::WalkParams p = make_params(r, model, opts);
    p.queries = d_queries;
    p.nq = nq;
    p.qid_base = opts->qid_base;
    p.qids = reinterpret_cast<const ull*>(opts->qids);
    p.paths = d_paths;
    p.lengths = d_lengths;
    p.next_walker = r.queues;
    if (d_paths && nq)
        CU(cudaMemsetAsync(d_paths, 0xFF, nq * (ull)p.stride * sizeof(uint32_t), s), "memset paths");
    CU(cudaEventRecord(r.ev_start, s), "event");
    CU(launch_model(r, model, opts->mode, p, s), "walk");
    CU(cudaEventRecord(r.ev_stop, s), "event");
    r.pending = true;
    r.pending_launches = 1;
    r.pending_qbase = opts->qid_base;
    return DW_OK;
}

int dw_run_device_sync(dw_graph_t g, int replica, dw_run_stats* st) {
    if (!g) return fail(DW_EINVAL, "graph handle is NULL");
    if (replica < 0 || replica >= (int)g->reps.size())
        return fail(DW_EINVAL, "replica %d out of range", replica);
    Replica& r = g->reps[replica];
    CU(cudaSetDevice(r.device), "cudaSetDevice");
    CU(cudaEventSynchronize(r.ev_stop), "walk");
    if (st) std::memset(st, 0, sizeof *st);
    if (r.listed.on) {
        // a listed walk (run_device_listed) is exact iff no walk ended early:
        // steps that advanced = listed walkers * target (runtime.cpp:141-149)
        Replica::Listed& l = r.listed;
        l.on = false;
        dw_run_stats cs;
        std::memset(&cs, 0, sizeof cs);
        int rc0 = collect(r, &cs, 0);
        if (rc0) return rc0;
        if (cs.steps - cs.dead_ends != l.nt * (ull)l.target) {
            r.sinks = 1;  // do not list on this graph again; re-run every walker
            if (const char* tp = std::getenv("DW_ENGINE_TRACE"))
                if (FILE* f = std::fopen(tp, "a")) {
                    std::fprintf(f, "L %llu retry\n", (unsigned long long)l.nq);
                    std::fclose(f);
                }
            int rc1;
            if ((rc1 = reset_run_state(r))) return rc1;
            CU(cudaStreamSynchronize(r.stream), "reset");
            dwb::WalkParams p = make_params(r, &l.model, &l.opts);
            p.queries = l.queries;
            p.nq = l.nq;
            p.qid_base = l.opts.qid_base;
            p.qids = reinterpret_cast<const ull*>(l.opts.qids);
            p.paths = l.paths;
            p.lengths = l.lengths;
            p.next_walker = r.queues;
            if (l.paths)
                CU(cudaMemsetAsync(l.paths, 0xFF, l.nq * (ull)p.stride * sizeof(uint32_t), l.stream),
                   "memset paths");
            CU(cudaEventRecord(r.ev_start, l.stream), "event");
            CU(launch_model(r, &l.model, l.opts.mode, p, l.stream), "walk");
            CU(cudaEventRecord(r.ev_stop, l.stream), "event");
            CU(cudaEventSynchronize(r.ev_stop), "walk");
            r.pending_launches = 1;
        } else if (std::getenv("DW_ENGINE_TRACE")) {
            if (FILE* f = std::fopen(std::getenv("DW_ENGINE_TRACE"), "a")) {
                std::fprintf(f, "L %llu ok\n", (unsigned long long)l.nq);
                std::fclose(f);
            }
        }
    }
    int rc = collect(r, st, r.pending_qbase);
    if (st) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, r.ev_start, r.ev_stop);
        st->kernel_ms = ms;
        st->total_ms = ms;
        st->kernel_launches = r.pending_launches;
    }
    r.pending = false;
    return rc;
}

int dw_run(dw_graph_t g, const dw_model_desc* model, const uint32_t* queries, uint64_t nq,
           const dw_run_opts* opts, uint32_t* paths, uint32_t* lengths, dw_run_stats* st) {
    if (!g) return fail(DW_EINVAL, "graph handle is NULL");
    int rc;
    if ((rc = check_model(model)) || (rc = check_opts(opts))) return rc;
    if (nq && !queries) return fail(DW_EINVAL, "queries is NULL");
    RunOut out;
    out.paths = paths;
    out.lengths = lengths;
    return run_engine(g, model, queries, nq, opts, out, st);
}

int dw_run_write_paths(dw_graph_t g, const dw_model_desc* model, const uint32_t* queries,
                       uint64_t nq, const dw_run_opts* opts, const char* path,
                       dw_run_stats* st) {
    if (!g) return fail(DW_EINVAL, "graph handle is NULL");
    int rc;
    if ((rc = check_model(model)) || (rc = check_opts(opts))) return rc;
    if (nq && !queries) return fail(DW_EINVAL, "queries is NULL");
    if (!path) return fail(DW_EINVAL, "path is NULL");
    FILE* f = std::fopen(path, "wb");
    if (!f) return fail(DW_EINVAL, "cannot open paths output file: %s", path);
    RunOut out;
    out.text = f;
    out.text_path = path;
    const ull stride = (ull)opts->walk_length + 1;
    const ull cap = std::min<ull>(batch_size(std::max<ull>(nq, 1)), 1ull << 20);
    CU(cudaSetDevice(g->reps[0].device), "cudaSetDevice");
    if (cudaMallocHost(&out.h_txt, cap * stride * kTextBytesPerId) != cudaSuccess) {
        std::fclose(f);
        return fail(DW_ECUDA, "cudaMallocHost text staging");
    }
    rc = run_engine(g, model, queries, nq, opts, out, st);
    cudaFreeHost(out.h_txt);
    if (std::fclose(f) != 0 && rc == DW_OK) rc = fail(DW_EINVAL, "write failed: %s", path);
    return rc;
}

int dw_run_compact(dw_graph_t g, const dw_model_desc* model, const uint32_t* queries,
                   uint64_t nq, const dw_run_opts* opts, uint64_t* offsets, uint32_t* flat,
                   uint64_t flat_capacity, dw_run_stats* st) {
    if (!g) return fail(DW_EINVAL, "graph handle is NULL");
    int rc;
    if ((rc = check_model(model)) || (rc = check_opts(opts))) return rc;
    if (nq && !queries) return fail(DW_EINVAL, "queries is NULL");
    if (!offsets) return fail(DW_EINVAL, "offsets is NULL");
    RunOut out;
    out.compact = true;
    out.offsets = reinterpret_cast<ull*>(offsets);
    out.flat = flat;
    out.flat_cap = flat_capacity;
    rc = run_direct(g, model, queries, nq, opts, out, st);
    if (rc != kDirectNo && rc != kDirectRetry) return rc;
    return run_engine(g, model, queries, nq, opts, out, st);
}

int dw_host_alloc(size_t bytes, void** out) {
    if (!out) return fail(DW_EINVAL, "NULL argument");
    CU(cudaMallocHost(out, bytes), "cudaMallocHost");
    return DW_OK;
}

int dw_host_free(void* p) {
    CU(cudaFreeHost(p), "cudaFreeHost");
    return DW_OK;
}

namespace {
__global__ void math_kernel(int fn, const double* __restrict__ x, double* __restrict__ y,
                            unsigned long long n) {
    const unsigned long long i = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x;
    if (i < n) y[i] = fn == 0 ? log(x[i]) : exp(x[i]);
}
}  // namespace

int dw_selftest_math(int fn, const double* x, double* y, uint64_t n) {
    if ((fn != 0 && fn != 1) || (n && (!x || !y))) return fail(DW_EINVAL, "bad arguments");
    if (!n) return DW_OK;
    CU(cudaSetDevice(0), "cudaSetDevice");
    double* d = nullptr;
    CU(cudaMalloc(&d, 2 * n * sizeof(double)), "cudaMalloc");
    std::unique_ptr<double, cudaError_t (*)(void*)> hold(d, &cudaFree);
    CU(cudaMemcpy(d, x, n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
    math_kernel<<<(unsigned)((n + 255) / 256), 256>>>(fn, d, d + n, n);
    CU(cudaGetLastError(), "math_kernel");
    CU(cudaMemcpy(y, d + n, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
    return DW_OK;
}

}  // extern "C"
