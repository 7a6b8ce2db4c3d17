// dw_graph.cu -- device graph construction and K4 calibration.
//
// build_rmat: R-MAT sampling, mirroring, CSR by one 64-bit radix sort of
// (src, dst) keys, Philox weights keyed by edge index, left-to-right
// aggregates.  The CSR equals Graph::build(mirror=true) on the same samples
// (graph.cpp:15-81): the reference stable-sorts each slice by target and
// equal targets are indistinguishable before weights are synthesized per
// edge, so a full key sort yields the identical arrays.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "dw_graph.cuh"
#include "dw_walk_kernel.cuh"  // ervs_visit: K4 prices the walk's own reservoir step

namespace dwb {

typedef unsigned long long ull;

#define DW_TRY(x)                              \
    do {                                       \
        cudaError_t e_ = (x);                  \
        if (e_ != cudaSuccess) return e_;      \
    } while (0)

static inline unsigned grid_for(ull n, int threads) {
    ull b = (n + threads - 1) / threads;
    if (b > 65535ull * 64) b = 65535ull * 64;
    return (unsigned)(b ? b : 1);
}

// ---- SplitMix64 / derive_seed (rng.hpp:10-25) -------------------------------
ull host_derive_seed(ull seed, ull stream) {
    ull st = seed ^ (stream * 0x9e3779b97f4a7c15ULL + 0x2545f4914f6cdd1dULL);
    auto next = [&]() {
        ull z = (st += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    };
    next();
    return next();
}

// ---- packing ---------------------------------------------------------------
__global__ void pack_edges_kernel(const uint32_t* __restrict__ col, const float* __restrict__ prop,
                                  EdgeRec* __restrict__ out, ull ne) {
    for (ull e = blockIdx.x * (ull)blockDim.x + threadIdx.x; e < ne;
         e += (ull)gridDim.x * blockDim.x)
        out[e] = EdgeRec{col[e], prop[e]};
}

// one thread per node; sequential ascending-order max/sum (graph.cpp:87-97)
__global__ void pack_nodes_kernel(const ull* __restrict__ row, const float* __restrict__ prop,
                                  const double* __restrict__ nmax, const double* __restrict__ nsum,
                                  NodeRec* __restrict__ out, uint32_t nv,
                                  unsigned* __restrict__ max_degree) {
    for (ull v = blockIdx.x * (ull)blockDim.x + threadIdx.x; v < nv;
         v += (ull)gridDim.x * blockDim.x) {
        const ull b = row[v], e = row[v + 1];
        double mx = 0.0, sum = 0.0;
        if (nmax && nsum) {
            mx = nmax[v];
            sum = nsum[v];
        } else {
            for (ull i = b; i < e; ++i) {
                const double p = prop[i];
                if (p > mx) mx = p;
                sum += p;
            }
        }
        NodeRec r;
        r.begin = b;
        r.degree = (uint32_t)(e - b);
        r.hoff = 0;
        r.hmax = mx;
        r.hsum = sum;
        out[v] = r;
        atomicMax(max_degree, r.degree);
    }
}

// ---- membership hash sets (dw_member.cuh) ----------------------------------
__global__ void bucket_count_kernel(const NodeRec* __restrict__ nodes, uint32_t nv,
                                    uint32_t* __restrict__ counts) {
    for (ull v = blockIdx.x * (ull)blockDim.x + threadIdx.x; v < nv;
         v += (ull)gridDim.x * blockDim.x)
        counts[v] = hash_buckets(nodes[v].degree);
}

__global__ void set_hoff_kernel(NodeRec* __restrict__ nodes, uint32_t nv,
                                const uint32_t* __restrict__ offs) {
    for (ull v = blockIdx.x * (ull)blockDim.x + threadIdx.x; v < nv;
         v += (ull)gridDim.x * blockDim.x)
        nodes[v].hoff = offs[v];
}

// one warp per row: lanes insert the row's targets (coalesced reads)
__global__ void hash_insert_kernel(const NodeRec* __restrict__ nodes, uint32_t nv,
                                   const EdgeRec* __restrict__ edges, uint32_t* __restrict__ hslots) {
    const ull warp = (blockIdx.x * (ull)blockDim.x + threadIdx.x) >> 5;
    const ull nwarps = ((ull)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    for (ull v = warp; v < nv; v += nwarps) {
        const NodeRec nr = nodes[v];
        if (nr.degree == 0) continue;
        const uint32_t lg = hash_log2_buckets(nr.degree);
        const uint32_t mask = (1u << lg) - 1u;
        for (ull i = lane; i < nr.degree; i += 32) {
            const uint32_t u = edges[nr.begin + i].col;
            uint32_t b = hash_bucket(u, lg);
            for (bool done = false; !done;) {
                uint32_t* slot = hslots + 8ull * (nr.hoff + b);
                for (int k = 0; k < 8; ++k) {
                    const uint32_t old = atomicCAS(slot + k, kHashEmpty, u);
                    if (old == kHashEmpty || old == u) {
                        done = true;
                        break;
                    }
                }
                b = (b + 1) & mask;
            }
        }
    }
}

// ---- fat edge records (dw_common.cuh FatRec) --------------------------------
// first index i in [0, d) with col[b + i] >= key (the row is sorted by target)
__device__ __forceinline__ uint32_t row_lower_bound(const EdgeRec* __restrict__ edges, ull b,
                                                    uint32_t d, uint32_t key) {
    uint32_t lo = 0, hi = d;
    while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (load_col(edges + b + mid) < key)
            lo = mid + 1;
        else
            hi = mid;
    }
    return lo;
}

// one warp per row v: record e = (v -> u) gets u's node data and the range of
// v in N(u) (its return edges when a walker stands on u having come from v)
// per node: bit l (l < kMaskLabels) iff the row has an edge labelled l, bit
// kMaskLabels iff it has a label >= kMaskLabels (MetaPath dead-row detection)
__global__ void label_mask_kernel(const NodeRec* __restrict__ nodes, uint32_t nv,
                                  const uint16_t* __restrict__ labels, uint8_t* __restrict__ mask) {
    const ull warp = (blockIdx.x * (ull)blockDim.x + threadIdx.x) >> 5;
    const ull nwarps = ((ull)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    for (ull v = warp; v < nv; v += nwarps) {
        const NodeRec nr = nodes[v];
        uint32_t m = 0;
        for (ull i = lane; i < nr.degree; i += 32) {
            const uint32_t l = labels[nr.begin + i];
            m |= l < kMaskLabels ? (1u << l) : (1u << kMaskLabels);
        }
        m = __reduce_or_sync(0xFFFFFFFFu, m);
        if (lane == 0) mask[v] = (uint8_t)m;
    }
}

// Triangle bound of the step v -> u (record of edge v -> u): the largest prop
// h(u -> w) over w in N(v), w != v -- the edges whose node2vec/PR2 weight is
// the "in N(prev)" case at cur = u, prev = v (models.hpp:62-69, 128-138).
// Encoded in 8 bits against hmax(u): 0 = no such edge; q >= 1: every such
// prop is <= hmax(u) * (q + 1) / 256 (exact in double); 255 = unknown (the
// intersection was not computed: more than `work` probes; DW_TRI_WORK, default
// kTriWork, 0 = never).  The walk turns
// it into a tighter non-return maximum (dw_models.cuh nonreturn_max), so more
// eRJS trials are rejected without a gather and fewer need a membership
// probe; outcomes are unchanged because it is an upper bound.
constexpr uint32_t kTriWork = 1024;
__device__ uint32_t tri_q(const EdgeRec* __restrict__ edges, const uint32_t* __restrict__ hslots,
                          uint32_t v, const NodeRec& nvr, uint32_t u, const NodeRec& nur,
                          uint32_t work) {
    const uint32_t du = nur.degree, dv = nvr.degree;
    const ull work_a = du;                                          // probe N(v) per edge of u
    const ull work_b = (ull)dv * (ull)(33 - __clz(du | 1u));        // search u's row per w
    if ((work_a < work_b ? work_a : work_b) > work) return 255u;
    DevGraph g{};
    g.hslots = hslots;
    float m = -1.0f;
    if (work_a <= work_b) {
        for (uint32_t i = 0; i < du; ++i) {
            const EdgeRec er = edges[nur.begin + i];
            if (er.col != v && member(g, dv, nvr.hoff, er.col) && er.h > m) m = er.h;
        }
    } else {
        for (uint32_t j = 0; j < dv; ++j) {
            const uint32_t w = edges[nvr.begin + j].col;
            if (w == v) continue;
            uint32_t lo = row_lower_bound(edges, nur.begin, du, w);
            for (; lo < du && edges[nur.begin + lo].col == w; ++lo)
                if (edges[nur.begin + lo].h > m) m = edges[nur.begin + lo].h;
        }
    }
    if (m < 0.0f) return 0u;
    // q = floor(256 m / hmax), nudged up so rounding cannot make it too small
    const double r = 256.0 * (double)m / nur.hmax * (1.0 + 0x1.0p-40);
    const uint32_t q = r >= 255.0 ? 255u : (uint32_t)r;
    return q < 1u ? 1u : q;
}

// tri_q of every edge, once for both record layouts (one warp per row)
__global__ void tri_build_kernel(const NodeRec* __restrict__ nodes, uint32_t nv,
                                 const EdgeRec* __restrict__ edges,
                                 const uint32_t* __restrict__ hslots, uint32_t work,
                                 uint8_t* __restrict__ tq) {
    const ull warp = (blockIdx.x * (ull)blockDim.x + threadIdx.x) >> 5;
    const ull nwarps = ((ull)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    for (ull v = warp; v < nv; v += nwarps) {
        const NodeRec nr = nodes[v];
        for (ull i = lane; i < nr.degree; i += 32) {
            const ull e = nr.begin + i;
            const uint32_t u = load_col(edges + e);
            tq[e] = (uint8_t)tri_q(edges, hslots, (uint32_t)v, nr, u, nodes[u], work);
        }
    }
}

__global__ void fat_build_kernel(const NodeRec* __restrict__ nodes, uint32_t nv,
                                 const EdgeRec* __restrict__ edges,
                                 const uint16_t* __restrict__ labels,
                                 const uint8_t* __restrict__ lmask, const uint8_t* __restrict__ tq,
                                 FatRec* __restrict__ fat) {
    const ull warp = (blockIdx.x * (ull)blockDim.x + threadIdx.x) >> 5;
    const ull nwarps = ((ull)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    for (ull v = warp; v < nv; v += nwarps) {
        const NodeRec nr = nodes[v];
        for (ull i = lane; i < nr.degree; i += 32) {
            const ull e = nr.begin + i;
            const EdgeRec er = edges[e];
            const NodeRec nu = nodes[er.col];
            const uint32_t lo = row_lower_bound(edges, nu.begin, nu.degree, (uint32_t)v);
            const uint32_t hi = v == 0xFFFFFFFFull
                                    ? nu.degree
                                    : row_lower_bound(edges, nu.begin, nu.degree, (uint32_t)v + 1);
            FatRec f;
            f.col = er.col;
            f.h = er.h;
            f.tbegin_label = (nu.begin & kBeginMask) |
                             ((ull)(labels ? labels[e] : (uint16_t)0) << 40) |
                             ((ull)(lmask ? lmask[er.col] : 1u) << 56);
            f.tdeg = nu.degree;
            f.thoff = nu.hoff;
            f.twin_lo = lo;
            // multiplicity (24 bits; 0xFFFFFF = too many to describe) | triangle bound << 24
            f.twin_cnt = (hi - lo >= 0xFFFFFFu ? 0xFFFFFFu : hi - lo) |
                         ((uint32_t)tq[e] << 24);
            f.thmax = nu.hmax;
            f.thsum = nu.hsum;
            f.aux[0] = f.aux[1] = f.aux[2] = f.aux[3] = 0;
            fat[e] = f;
        }
    }
}

// Slim layout: the fat record's return-edge range alone, 4 B per edge, so the
// slim walk keeps its free rejections (the walker fetches twin[e] of the edge
// it took together with the next node record).  lo | cnt << 24; cnt 255 marks
// a range it cannot describe (degree >= 2^24 or >= 255 parallel edges).
__global__ void twin_build_kernel(const NodeRec* __restrict__ nodes, uint32_t nv,
                                  const EdgeRec* __restrict__ edges, uint32_t* __restrict__ twin) {
    const ull warp = (blockIdx.x * (ull)blockDim.x + threadIdx.x) >> 5;
    const ull nwarps = ((ull)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    for (ull v = warp; v < nv; v += nwarps) {
        const NodeRec nr = nodes[v];
        for (ull i = lane; i < nr.degree; i += 32) {
            const ull e = nr.begin + i;
            const NodeRec nu = nodes[load_col(edges + e)];
            const uint32_t lo = row_lower_bound(edges, nu.begin, nu.degree, (uint32_t)v);
            const uint32_t hi = v == 0xFFFFFFFFull
                                    ? nu.degree
                                    : row_lower_bound(edges, nu.begin, nu.degree, (uint32_t)v + 1);
            const uint32_t cnt = hi - lo;
            twin[e] = (nu.degree >= (1u << 24) || cnt >= 255u) ? (255u << 24) : (lo | (cnt << 24));
        }
    }
}

static cudaError_t build_twin(DeviceGraphBuffers& g, cudaStream_t s) {
    g.twin = nullptr;
    if (g.fat || g.ne == 0) return cudaSuccess;
    if (const char* env = getenv("DW_TWIN"))
        if (env[0] == '0') return cudaSuccess;
    size_t free_b = 0, total_b = 0;
    DW_TRY(cudaMemGetInfo(&free_b, &total_b));
    const ull need = g.ne * sizeof(uint32_t);
    if (need + (2ull << 30) > free_b) return cudaSuccess;
    DW_TRY(cudaMallocAsync(&g.twin, need, s));
    twin_build_kernel<<<grid_for((ull)g.nv * 32, 256), 256, 0, s>>>(g.nodes, g.nv, g.edges, g.twin);
    DW_TRY(cudaGetLastError());
    if (getenv("DW_VERBOSE"))
        fprintf(stderr, "dynwalk: slim layout with return-edge ranges (%.1f GB)\n", need / 1e9);
    return cudaStreamSynchronize(s);
}

__global__ void fat32_build_kernel(const NodeRec* __restrict__ nodes, uint32_t nv,
                                   const EdgeRec* __restrict__ edges,
                                   const uint8_t* __restrict__ tq, FatRec32* __restrict__ fat) {
    const ull warp = (blockIdx.x * (ull)blockDim.x + threadIdx.x) >> 5;
    const ull nwarps = ((ull)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    for (ull v = warp; v < nv; v += nwarps) {
        const NodeRec nr = nodes[v];
        for (ull i = lane; i < nr.degree; i += 32) {
            const ull e = nr.begin + i;
            const EdgeRec er = edges[e];
            const NodeRec nu = nodes[er.col];
            const uint32_t lo = row_lower_bound(edges, nu.begin, nu.degree, (uint32_t)v);
            const uint32_t hi = v == 0xFFFFFFFFull
                                    ? nu.degree
                                    : row_lower_bound(edges, nu.begin, nu.degree, (uint32_t)v + 1);
            const uint32_t cnt = hi - lo;
            FatRec32 f;
            f.col = er.col;
            f.h = er.h;
            f.begin_lo = (uint32_t)nu.begin;
            f.begin_hi_deg = (uint32_t)((nu.begin >> 32) & 0xFFu) | (nu.degree << 8);
            f.thoff = nu.hoff;
            f.twin = cnt >= 255u ? (255u << 24) : (lo | (cnt << 24));
            f.thmax = (float)nu.hmax;  // exact: a maximum of f32 props
            // a row sum above FLT_MAX has no f32 neighbour: NaN fails both of
            // the decision's band tests, so the exact node record decides
            // the row sum in the top 24 bits (f32 truncated to 15 mantissa
            // bits: decisions within fat32_band = 1e-4 of it refetch the
            // node record), the triangle bound in the low 8
            const float fs = (float)nu.hsum;
            const uint32_t sb = isfinite(fs) ? __float_as_uint(fs) : 0x7fc00000u;
            f.thsum = __uint_as_float((sb & ~0xFFu) |
                                      (uint32_t)tq[e]);
            fat[e] = f;
        }
    }
}

// Above ~100 GB of fat records the walk slows down instead of speeding up:
// measured on one B200, node2vec (0.5, 2), walker-steps/s fat vs slim:
// s25 (34 GB of records) 6.04e9 vs 4.19e9, s26 (69 GB) 5.87e9 vs 4.20e9,
// s27 (137 GB) 3.27e9 vs 4.42e9 (random gathers spread over 175 GB of HBM).
// DW_FAT=0 disables the layout, DW_FAT=1 builds it whenever it fits.
constexpr unsigned long long kFatMaxBytes = 96ull * 1000 * 1000 * 1000;

// s24: 1024 probes per edge build in 10 s and walk at 8.65e9 walker-steps/s,
// 4096 in 34 s at 8.78e9, 16384 in 59 s at 8.78e9 (profiles/r2_tri_work_s24.txt);
// graphs above 2^30 edges keep 1024 (s27: the build stays under 20 s)
static uint32_t tri_work(ull ne) {
    if (const char* env = getenv("DW_TRI_WORK")) return (uint32_t)std::strtoul(env, nullptr, 10);
    return ne > (1ull << 30) ? kTriWork : 4 * kTriWork;
}

static cudaError_t build_fat(DeviceGraphBuffers& g, cudaStream_t s) {
    g.fat = nullptr;
    g.fat32 = nullptr;
    bool force = false;
    if (const char* env = getenv("DW_FAT")) {
        if (env[0] == '0') return cudaSuccess;
        force = env[0] == '1';
    }
    if (g.ne == 0 || g.ne > kBeginMask) return cudaSuccess;
    // Build temporaries freed with cudaFreeAsync stay in the stream-ordered
    // pool until trimmed; return them first so they count as free.
    auto free_now = [&](size_t* free_b) -> cudaError_t {
        DW_TRY(cudaStreamSynchronize(s));
        int dev = 0;
        cudaMemPool_t pool;
        DW_TRY(cudaGetDevice(&dev));
        DW_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
        DW_TRY(cudaMemPoolTrimTo(pool, 0));
        size_t total_b = 0;
        return cudaMemGetInfo(free_b, &total_b);
    };
    // compact 32 B records for unlabelled graphs whose degrees fit 24 bits:
    // node2vec walks them (+5 % over the 64 B records at s24, and they fit
    // s27), the other models use the 64 B records built next when those fit.
    // Both layouts together stay under kFatMaxBytes and leave 4 GB free.
    // the triangle bounds of every edge (1 B each), shared by both layouts
    uint8_t* tq = nullptr;
    DW_TRY(cudaMallocAsync(&tq, std::max<ull>(g.ne, 1), s));
    tri_build_kernel<<<grid_for((ull)g.nv * 32, 256), 256, 0, s>>>(g.nodes, g.nv, g.edges, g.hslots,
                                                                   tri_work(g.ne), tq);
    DW_TRY(cudaGetLastError());
    struct FreeTq {
        uint8_t* p;
        cudaStream_t s;
        ~FreeTq() { cudaFreeAsync(p, s); }
    } free_tq{tq, s};
    const bool compact_ok = !g.labels && g.max_degree < (1u << 24);
    const char* fenv = getenv("DW_FAT");
    ull used = 0;
    if (compact_ok && !force && g.ne * sizeof(FatRec32) <= kFatMaxBytes) {
        size_t fb = 0;
        DW_TRY(free_now(&fb));
        const ull need32 = g.ne * sizeof(FatRec32);
        if (need32 + (4ull << 30) <= fb) {
            DW_TRY(cudaMallocAsync(&g.fat32, need32, s));
            fat32_build_kernel<<<grid_for((ull)g.nv * 32, 256), 256, 0, s>>>(g.nodes, g.nv, g.edges,
                                                                             tq, g.fat32);
            DW_TRY(cudaGetLastError());
            DW_TRY(cudaStreamSynchronize(s));
            used = need32;
            if (getenv("DW_VERBOSE"))
                fprintf(stderr, "dynwalk: compact 32 B fat records built (%.1f GB)\n", need32 / 1e9);
        }
    }
    if (fenv && fenv[0] == '2') return cudaSuccess;  // compact records only
    if (!force && used + g.ne * sizeof(FatRec) > kFatMaxBytes) {
        if (getenv("DW_VERBOSE"))
            fprintf(stderr, "dynwalk: fat records skipped (%.1f GB + %.1f GB above the %.0f GB cap)\n",
                    g.ne * sizeof(FatRec) / 1e9, used / 1e9, kFatMaxBytes / 1e9);
        return cudaSuccess;
    }
    // the fat layout is an accelerator: skip it when it would crowd HBM
    size_t free_b = 0;
    DW_TRY(free_now(&free_b));
    const ull need = g.ne * sizeof(FatRec);
    const bool fits = need + (4ull << 30) <= free_b;
    if (getenv("DW_VERBOSE"))
        fprintf(stderr, "dynwalk: fat records %s (%.1f GB needed, %.1f GB free)\n",
                fits ? "built" : "skipped", need / 1e9, free_b / 1e9);
    if (!fits) return cudaSuccess;
    DW_TRY(cudaMallocAsync(&g.fat, need, s));
    uint8_t* lmask = nullptr;
    if (g.labels) {
        DW_TRY(cudaMallocAsync(&lmask, std::max<ull>(g.nv, 1), s));
        label_mask_kernel<<<grid_for((ull)g.nv * 32, 256), 256, 0, s>>>(g.nodes, g.nv, g.labels,
                                                                        lmask);
        DW_TRY(cudaGetLastError());
    }
    fat_build_kernel<<<grid_for((ull)g.nv * 32, 256), 256, 0, s>>>(g.nodes, g.nv, g.edges,
                                                                   g.labels, lmask, tq, g.fat);
    DW_TRY(cudaGetLastError());
    if (lmask) DW_TRY(cudaFreeAsync(lmask, s));
    return cudaStreamSynchronize(s);
}

static cudaError_t build_member_index(DeviceGraphBuffers& g, cudaStream_t s) {
    uint32_t* counts = nullptr;
    uint32_t* offs = nullptr;
    const ull n = std::max<ull>(g.nv, 1);
    DW_TRY(cudaMallocAsync(&counts, (n + 1) * sizeof(uint32_t), s));
    DW_TRY(cudaMallocAsync(&offs, (n + 1) * sizeof(uint32_t), s));
    DW_TRY(cudaMemsetAsync(counts, 0, (n + 1) * sizeof(uint32_t), s));
    bucket_count_kernel<<<grid_for(g.nv, 256), 256, 0, s>>>(g.nodes, g.nv, counts);
    // total fits u32 unless sum(next_pow2(2d))/8 >= 2^32 (E >~ 8e9); checked below in u64
    ull* total64 = nullptr;
    DW_TRY(cudaMallocAsync(&total64, sizeof(ull), s));
    size_t tb = 0;
    DW_TRY(cub::DeviceReduce::Sum(nullptr, tb, counts, total64, (int)(g.nv + 1), s));
    void* tmp = nullptr;
    DW_TRY(cudaMallocAsync(&tmp, tb, s));
    DW_TRY(cub::DeviceReduce::Sum(tmp, tb, counts, total64, (int)(g.nv + 1), s));
    DW_TRY(cudaFreeAsync(tmp, s));
    ull total = 0;
    DW_TRY(cudaMemcpyAsync(&total, total64, sizeof(ull), cudaMemcpyDeviceToHost, s));
    DW_TRY(cudaStreamSynchronize(s));
    DW_TRY(cudaFreeAsync(total64, s));
    if (total >= 0xFFFFFFFFull) return cudaErrorInvalidValue;
    tb = 0;
    DW_TRY(cub::DeviceScan::ExclusiveSum(nullptr, tb, counts, offs, (int)(g.nv + 1), s));
    DW_TRY(cudaMallocAsync(&tmp, tb, s));
    DW_TRY(cub::DeviceScan::ExclusiveSum(tmp, tb, counts, offs, (int)(g.nv + 1), s));
    DW_TRY(cudaFreeAsync(tmp, s));
    set_hoff_kernel<<<grid_for(g.nv, 256), 256, 0, s>>>(g.nodes, g.nv, offs);
    g.nbuckets = total;
    DW_TRY(cudaMallocAsync(&g.hslots, std::max<ull>(total, 1) * 32, s));
    DW_TRY(cudaMemsetAsync(g.hslots, 0xFF, std::max<ull>(total, 1) * 32, s));
    hash_insert_kernel<<<grid_for((ull)g.nv * 32, 256), 256, 0, s>>>(g.nodes, g.nv, g.edges,
                                                                      g.hslots);
    DW_TRY(cudaGetLastError());
    DW_TRY(cudaFreeAsync(counts, s));
    DW_TRY(cudaFreeAsync(offs, s));
    return cudaStreamSynchronize(s);
}

cudaError_t pack_graph(const ull* d_row, const uint32_t* d_col, const float* d_prop,
                       const double* d_nmax, const double* d_nsum, DeviceGraphBuffers& g,
                       cudaStream_t s) {
    unsigned* d_maxd = nullptr;
    DW_TRY(cudaMallocAsync(&d_maxd, sizeof(unsigned), s));
    DW_TRY(cudaMemsetAsync(d_maxd, 0, sizeof(unsigned), s));
    if (g.ne) pack_edges_kernel<<<grid_for(g.ne, 256), 256, 0, s>>>(d_col, d_prop, g.edges, g.ne);
    pack_nodes_kernel<<<grid_for(g.nv, 128), 128, 0, s>>>(d_row, d_prop, d_nmax, d_nsum, g.nodes,
                                                          g.nv, d_maxd);
    DW_TRY(cudaGetLastError());
    unsigned h = 0;
    DW_TRY(cudaMemcpyAsync(&h, d_maxd, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    DW_TRY(cudaStreamSynchronize(s));
    g.max_degree = h;
    DW_TRY(cudaFreeAsync(d_maxd, s));
    return build_member_index(g, s);
}

__global__ void label_max_kernel(const uint16_t* __restrict__ label, ull ne,
                                 unsigned* __restrict__ mx) {
    unsigned m = 0;
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < ne; i += (ull)gridDim.x * blockDim.x)
        m = max(m, (unsigned)label[i]);
    m = __reduce_max_sync(0xFFFFFFFFu, m);
    if ((threadIdx.x & 31) == 0 && m) atomicMax(mx, m);
}

__global__ void label_pack_kernel(const uint16_t* __restrict__ label, ull ne,
                                  uint32_t* __restrict__ out, ull nw) {
    for (ull w = blockIdx.x * (ull)blockDim.x + threadIdx.x; w < nw; w += (ull)gridDim.x * blockDim.x) {
        uint32_t v = 0;
        for (uint32_t k = 0; k < 16; ++k) {
            const ull e = w * 16 + k;
            if (e < ne) v |= ((uint32_t)label[e] & 3u) << (2 * k);
        }
        out[w] = v;
    }
}

// Labels packed 2 bits per edge when every label is < 4 (DevGraph::lab2).
// DW_LAB2=0 disables it.
static cudaError_t build_lab2(DeviceGraphBuffers& g, cudaStream_t s) {
    g.lab2 = nullptr;
    if (!g.labels || g.ne == 0) return cudaSuccess;
    if (const char* env = getenv("DW_LAB2"))
        if (env[0] == '0') return cudaSuccess;
    unsigned* d_mx = nullptr;
    DW_TRY(cudaMallocAsync(&d_mx, sizeof(unsigned), s));
    DW_TRY(cudaMemsetAsync(d_mx, 0, sizeof(unsigned), s));
    label_max_kernel<<<grid_for(g.ne, 256) < 4096 ? grid_for(g.ne, 256) : 4096, 256, 0, s>>>(
        g.labels, g.ne, d_mx);
    unsigned mx = 0;
    DW_TRY(cudaMemcpyAsync(&mx, d_mx, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    DW_TRY(cudaStreamSynchronize(s));
    DW_TRY(cudaFreeAsync(d_mx, s));
    if (mx >= 4) return cudaSuccess;
    const ull nw = (g.ne + 15) / 16;
    DW_TRY(cudaMallocAsync(&g.lab2, nw * sizeof(uint32_t), s));
    label_pack_kernel<<<grid_for(nw, 256) < 8192 ? grid_for(nw, 256) : 8192, 256, 0, s>>>(
        g.labels, g.ne, g.lab2, nw);
    DW_TRY(cudaGetLastError());
    return cudaStreamSynchronize(s);
}

cudaError_t finish_graph(DeviceGraphBuffers& g, cudaStream_t s) {
    DW_TRY(build_fat(g, s));
    DW_TRY(build_lab2(g, s));
    return build_twin(g, s);
}

__global__ void unpack_kernel(const NodeRec* __restrict__ nodes, const EdgeRec* __restrict__ edges,
                              uint32_t nv, ull ne, ull* row, uint32_t* col, float* prop,
                              double* nmax, double* nsum) {
    const ull stride = (ull)gridDim.x * blockDim.x;
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < ne; i += stride) {
        if (col) col[i] = edges[i].col;
        if (prop) prop[i] = edges[i].h;
    }
    for (ull v = blockIdx.x * (ull)blockDim.x + threadIdx.x; v < nv; v += stride) {
        if (row) row[v] = nodes[v].begin;
        if (nmax) nmax[v] = nodes[v].hmax;
        if (nsum) nsum[v] = nodes[v].hsum;
    }
    if (row && blockIdx.x == 0 && threadIdx.x == 0) row[nv] = ne;
}

cudaError_t unpack_graph(const DeviceGraphBuffers& g, ull* d_row, uint32_t* d_col, float* d_prop,
                         double* d_nmax, double* d_nsum, cudaStream_t s) {
    unpack_kernel<<<grid_for(std::max<ull>(g.ne, g.nv), 256), 256, 0, s>>>(
        g.nodes, g.edges, g.nv, g.ne, d_row, d_col, d_prop, d_nmax, d_nsum);
    return cudaGetLastError();
}

// ---- R-MAT (definition shared with oracle.c orc_rmat_samples) --------------
#define RMAT_TA 2448131358u   /* floor(0.57 * 2^32) */
#define RMAT_TAB 3264175144u  /* floor(0.76 * 2^32) */
#define RMAT_TABC 4080218931u /* floor(0.95 * 2^32) */

__device__ __forceinline__ uint32_t rmat_perm(uint32_t x, uint32_t scale, ull pk) {
    if (scale == 0) return 0;
    const uint32_t mask = scale >= 32 ? 0xFFFFFFFFu : ((1u << scale) - 1u);
    const uint32_t sh = scale / 2 + 1;
    const uint32_t m1 = ((uint32_t)pk | 1u), a1 = (uint32_t)(pk >> 32);
    const uint32_t m2 = ((uint32_t)(pk >> 17) | 1u), a2 = (uint32_t)(pk >> 7);
    x = (x * m1 + a1) & mask;
    x ^= x >> sh;
    x = (x * m2 + a2) & mask;
    x ^= x >> sh;
    return x & mask;
}

// keys[i] = (src<<32|dst); keys[ns+i] = twin, or the sentinel (nv<<32) for a
// self-loop (Graph::build mirrors only non-self-loops, graph.cpp:17-25)
__global__ void rmat_keys_kernel(uint32_t scale, ull ns, ull ks, ull pk, ull* __restrict__ keys,
                                 ull* __restrict__ self_loops) {
    const uint32_t k0 = (uint32_t)ks, k1 = (uint32_t)(ks >> 32);
    ull loops = 0;
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < ns;
         i += (ull)gridDim.x * blockDim.x) {
        uint32_t u = 0, v = 0;
        U4 rnd{0, 0, 0, 0};
        for (uint32_t lvl = 0; lvl < scale; ++lvl) {
            if ((lvl & 3) == 0)
                rnd = philox4x32_10(U4{lvl >> 2, (uint32_t)i, (uint32_t)(i >> 32), 0x524d4154u},
                                    k0, k1);
            const uint32_t q = lvl & 3;
            const uint32_t r = q == 0 ? rnd.x : q == 1 ? rnd.y : q == 2 ? rnd.z : rnd.w;
            const uint32_t bu = r >= RMAT_TAB;
            const uint32_t bv = (r >= RMAT_TA && r < RMAT_TAB) || r >= RMAT_TABC;
            u = (u << 1) | bu;
            v = (v << 1) | bv;
        }
        u = rmat_perm(u, scale, pk);
        v = rmat_perm(v, scale, pk);
        keys[i] = ((ull)u << 32) | v;
        if (u != v) {
            keys[ns + i] = ((ull)v << 32) | u;
        } else {
            keys[ns + i] = (ull)(1ull << scale) << 32;
            ++loops;
        }
    }
    if (loops) atomicAdd(self_loops, loops);
}

__global__ void keys_to_col_kernel(const ull* __restrict__ keys, uint32_t* __restrict__ col,
                                   ull ne) {
    for (ull e = blockIdx.x * (ull)blockDim.x + threadIdx.x; e < ne;
         e += (ull)gridDim.x * blockDim.x)
        col[e] = (uint32_t)keys[e];
}

// row[v] = first e with key >= v<<32 (keys sorted)
__global__ void row_offsets_kernel(const ull* __restrict__ keys, ull ne, uint32_t nv,
                                   ull* __restrict__ row) {
    for (ull v = blockIdx.x * (ull)blockDim.x + threadIdx.x; v <= nv;
         v += (ull)gridDim.x * blockDim.x) {
        if (v == nv) {
            row[v] = ne;
            continue;
        }
        const ull target = v << 32;
        ull lo = 0, hi = ne;
        while (lo < hi) {
            const ull mid = lo + ((hi - lo) >> 1);
            if (keys[mid] < target)
                lo = mid + 1;
            else
                hi = mid;
        }
        row[v] = lo;
    }
}

__device__ __forceinline__ ull edge_draw(ull seed, ull e, uint32_t tag) {
    const U4 o = philox4x32_10(U4{(uint32_t)e, (uint32_t)(e >> 32), 0u, tag}, (uint32_t)seed,
                               (uint32_t)(seed >> 32));
    return (ull)o.x | ((ull)o.y << 32);
}

// same maps as synthesize_weights (graph.cpp:308-341), Philox keyed by edge
__global__ void synth_props_kernel(float* __restrict__ prop, ull ne, int kind, double low,
                                   double high, double alpha, ull seed) {
    for (ull e = blockIdx.x * (ull)blockDim.x + threadIdx.x; e < ne;
         e += (ull)gridDim.x * blockDim.x) {
        if (kind == 0) {
            const double u = uniform01(edge_draw(seed, e, 0x57474854u));
            prop[e] = (float)(low + u * (high - low));
        } else if (kind == 2) {
            const double u = open01(edge_draw(seed, e, 0x50415245u));
            prop[e] = alpha == 1.0 ? (float)(1.0 / u) : (float)pow(u, -(1.0 / alpha));
        } else {
            prop[e] = 1.0f;
        }
    }
}

__global__ void synth_labels_kernel(uint16_t* __restrict__ label, ull ne, uint32_t lo, ull span,
                                    ull seed) {
    for (ull e = blockIdx.x * (ull)blockDim.x + threadIdx.x; e < ne;
         e += (ull)gridDim.x * blockDim.x)
        label[e] = (uint16_t)(lo + __umul64hi(edge_draw(seed, e, 0x4c41424cu), span));
}

cudaError_t build_rmat(const RmatSpec& spec, DeviceGraphBuffers& g, cudaStream_t s) {
    if (spec.scale > 30 || spec.edge_factor < 2) return cudaErrorInvalidValue;
    const uint32_t nv = 1u << spec.scale;
    const ull ns = (ull)(spec.edge_factor / 2) * nv;
    const ull nkeys = 2 * ns;
    if (nkeys > (1ull << 34)) return cudaErrorInvalidValue;
    const ull ks = host_derive_seed(spec.seed, 0x726d6174ULL);
    const ull pk = host_derive_seed(spec.seed, 0x7065726dULL);

    ull *keys = nullptr, *keys_alt = nullptr, *d_loops = nullptr, *row = nullptr;
    DW_TRY(cudaMallocAsync(&keys, nkeys * sizeof(ull), s));
    DW_TRY(cudaMallocAsync(&keys_alt, nkeys * sizeof(ull), s));
    DW_TRY(cudaMallocAsync(&d_loops, sizeof(ull), s));
    DW_TRY(cudaMemsetAsync(d_loops, 0, sizeof(ull), s));
    rmat_keys_kernel<<<grid_for(ns, 256), 256, 0, s>>>(spec.scale, ns, ks, pk, keys, d_loops);
    DW_TRY(cudaGetLastError());

    cub::DoubleBuffer<ull> db(keys, keys_alt);
    size_t tmp_bytes = 0;
    // 64-bit item count: s27 draws 2^31 directed keys
    DW_TRY(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, db, (long long)nkeys, 0,
                                          32 + spec.scale + 1, s));
    void* tmp = nullptr;
    DW_TRY(cudaMallocAsync(&tmp, tmp_bytes, s));
    DW_TRY(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, db, (long long)nkeys, 0, 32 + spec.scale + 1,
                                          s));
    DW_TRY(cudaFreeAsync(tmp, s));
    ull loops = 0;
    DW_TRY(cudaMemcpyAsync(&loops, d_loops, sizeof(ull), cudaMemcpyDeviceToHost, s));
    DW_TRY(cudaStreamSynchronize(s));
    const ull ne = nkeys - loops;
    const ull* sorted = db.Current();
    ull* spare = db.Alternate();

    g.nv = nv;
    g.ne = ne;
    DW_TRY(cudaMallocAsync(&row, (nv + 1ull) * sizeof(ull), s));
    row_offsets_kernel<<<grid_for(nv + 1ull, 256), 256, 0, s>>>(sorted, ne, nv, row);
    // col and prop live in the spare sort buffer (2*ne*4 bytes <= nkeys*8)
    uint32_t* col = reinterpret_cast<uint32_t*>(spare);
    float* prop = reinterpret_cast<float*>(col + ne);
    keys_to_col_kernel<<<grid_for(ne, 256), 256, 0, s>>>(sorted, col, ne);
    synth_props_kernel<<<grid_for(ne, 256), 256, 0, s>>>(prop, ne, spec.weights, spec.low,
                                                         spec.high, spec.alpha, spec.weight_seed);
    DW_TRY(cudaGetLastError());
    DW_TRY(cudaMallocAsync(&g.edges, ((std::max<ull>(ne, 1) + 1) & ~1ull) * sizeof(EdgeRec), s));
    DW_TRY(cudaMallocAsync(&g.nodes, std::max<uint32_t>(nv, 1) * sizeof(NodeRec), s));
    if (spec.labels) {
        DW_TRY(cudaMallocAsync(&g.labels, ((std::max<ull>(ne, 1) + 1) & ~1ull) * sizeof(uint16_t), s));
        synth_labels_kernel<<<grid_for(ne, 256), 256, 0, s>>>(
            g.labels, ne, spec.label_low, (ull)spec.label_high - spec.label_low + 1,
            spec.label_seed);
        DW_TRY(cudaGetLastError());
    }
    DW_TRY(pack_graph(row, col, prop, nullptr, nullptr, g, s));
    DW_TRY(cudaFreeAsync(keys, s));
    DW_TRY(cudaFreeAsync(keys_alt, s));
    DW_TRY(cudaFreeAsync(d_loops, s));
    DW_TRY(cudaFreeAsync(row, s));
    return finish_graph(g, s);  // after the sort buffers are gone
}

// ---- K4: calibration (cost_model.cpp:37-126) -------------------------------
// Probe state of one sampled node (probe_state, cost_model.cpp:20-33: step 1
// with the first neighbour as prev), built once per calibration so the timed
// passes read it with one coalesced load per warp.
struct ProbeState {
    ull begin;       // row of cur
    uint32_t cur, degree;
    uint32_t prev, prev_degree;
    uint32_t phoff;  // hash set of prev
    uint32_t step;
    double hmax, hsum;
};

template <class M>
__device__ __forceinline__ double eval_weight(const M& m, const Step& S, uint32_t phoff,
                                              const DevGraph& g, ull e) {
    const EdgeRec er = load_edge(g.edges + e);
    const uint16_t lab = (M::kUsesLabels && g.labels) ? g.labels[e] : (uint16_t)0;
    const WeightCase wc = m.weight(S, er.col, er.h, lab);
    if (!M::kSecondOrder || !wc.needs_member) return wc.w;
    return member(g, S.prev_degree, phoff, er.col) ? wc.w_in : wc.w_out;
}

__global__ void probe_states_kernel(DevGraph g, const uint32_t* __restrict__ nodes, uint32_t n,
                                    ProbeState* __restrict__ out) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const uint32_t v = nodes[i];
    const NodeRec nr = load_node(g.nodes + v);
    ProbeState P;
    P.begin = nr.begin;
    P.cur = v;
    P.degree = nr.degree;
    P.hmax = nr.hmax;
    P.hsum = nr.hsum;
    P.prev = kInvalid;
    P.prev_degree = 0;
    P.phoff = 0;
    P.step = 0;
    if (nr.degree) {
        const uint32_t pv = load_col(g.edges + nr.begin);
        const NodeRec pr = load_node(g.nodes + pv);
        if (pr.degree) {
            P.prev = pv;
            P.prev_degree = pr.degree;
            P.phoff = pr.hoff;
            P.step = 1;
        }
    }
    out[i] = P;
}

__global__ void sample_nodes_kernel(DevGraph g, ull seed, ull tries, uint32_t want,
                                    uint32_t* nodes, unsigned* count) {
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < tries;
         i += (ull)gridDim.x * blockDim.x) {
        const U4 b = philox4x32_10(U4{(uint32_t)i, (uint32_t)(i >> 32), 0u, 0x70726f66u},
                                   (uint32_t)seed, (uint32_t)(seed >> 32));
        const uint32_t v = (uint32_t)bounded(lo64(b), g.nv);
        if (g.nodes[v].degree == 0) continue;
        const unsigned slot = atomicAdd(count, 1u);
        if (slot < want) nodes[slot] = v;
    }
}

// One lane per probed node and round, like the walk kernel's per-lane phase
// machine; round r probes the pool's nodes [r*n, (r+1)*n) (mod the pool), so
// consecutive rounds touch different rows of the whole graph, not the same
// cached neighbours: the pool is many times the L2, like the rows a walk
// visits.  Both passes read the same states and visit k = min(d, npn) edges
// per node; they differ in what a visit is (cost_model.cpp:67-98):
//   random     one eRJS trial as the walk kernel runs it: the Philox (x, y)
//              draw, then the weight of a random neighbour only when y is
//              below the row's non-return maximum -- a trial above it is
//              rejected without reading the edge (the free rejection)
//   sequential one eRVS visit as the walk kernel runs it on a short row: the
//              next neighbour's weight (membership included) folded into the
//              A-ExpJ reservoir (ervs_visit: key, jump-threshold and floor
//              draws with their log/exp)
// so the ratio prices the kernel's trial against the kernel's reservoir visit,
// the balance decide_sampler encodes (cost_model.hpp:46-56).  (A warp-wide
// coalesced scan would price a sequential read at a fraction of what the
// walk's reservoir pays per edge, and the decision would then send rows to
// eRVS that the kernel walks faster with rejection.)
// Weights of up to kProbeBatch edges with their loads in flight together (the
// walk kernel keeps a ring of outstanding gathers per lane the same way):
// the edge records first, then the first membership bucket of each.
constexpr int kProbeBatch = 4;
template <class M>
__device__ __forceinline__ void probe_weights(const M& m, const Step& S, uint32_t phoff,
                                              const DevGraph& g, const ull (&e)[kProbeBatch],
                                              const bool (&live)[kProbeBatch],
                                              double (&w)[kProbeBatch]) {
    EdgeRec er[kProbeBatch];
    uint16_t lab[kProbeBatch];
#pragma unroll
    for (int j = 0; j < kProbeBatch; ++j) {
        er[j] = live[j] ? load_edge(g.edges + e[j]) : EdgeRec{0u, 0.f};
        lab[j] = (live[j] && M::kUsesLabels && g.labels) ? g.labels[e[j]] : (uint16_t)0;
    }
    WeightCase wc[kProbeBatch];
    uint4 b0[kProbeBatch], b1[kProbeBatch];
    const uint32_t lg = hash_log2_buckets(S.prev_degree);
#pragma unroll
    for (int j = 0; j < kProbeBatch; ++j) {
        wc[j] = m.weight(S, er[j].col, er[j].h, lab[j]);
        if (live[j] && M::kSecondOrder && wc[j].needs_member && S.prev_degree) {
            const uint4* p = reinterpret_cast<const uint4*>(
                g.hslots + 8ull * (phoff + hash_bucket(er[j].col, lg)));
            b0[j] = __ldg(p);
            b1[j] = __ldg(p + 1);
        }
    }
#pragma unroll
    for (int j = 0; j < kProbeBatch; ++j) {
        w[j] = wc[j].w;
        if (live[j] && M::kSecondOrder && wc[j].needs_member) {
            int r = S.prev_degree ? bucket_lookup(b0[j], b1[j], er[j].col) : 0;
            if (r < 0) r = member(g, S.prev_degree, phoff, er[j].col) ? 1 : 0;
            w[j] = r ? wc[j].w_in : wc[j].w_out;
        }
    }
}

// One lane per probed node and round, like the walk kernel's per-lane phase
// machine; round r probes the pool's nodes [r*n, (r+1)*n) (mod the pool), so
// consecutive rounds touch different rows of the whole graph, not the same
// cached neighbours: the pool is many times the L2, like the rows a walk
// visits.  Both passes read the same states and visit k = min(d, npn) edges
// per node, kProbeBatch at a time; they differ in what a visit is
// (cost_model.cpp:67-98):
//   random     one eRJS trial as the walk kernel runs it: the Philox (x, y)
//              draw, then the weight of a random neighbour only when y is
//              below the row's non-return maximum -- a trial above it is
//              rejected without reading the edge (the free rejection)
//   sequential one eRVS visit as the walk kernel runs it on a short row: the
//              next neighbour's weight (membership included) folded into the
//              A-ExpJ reservoir (ervs_visit: key, jump-threshold and floor
//              draws with their log/exp)
// so the ratio prices the kernel's trial against the kernel's reservoir visit,
// the balance decide_sampler encodes (cost_model.hpp:46-56).  (A warp-wide
// coalesced scan prices a sequential read at a fraction of what the walk's
// reservoir pays per edge, and the decision then sends rows to eRVS that the
// kernel walks faster with rejection.)
template <class M, bool RANDOM>
__global__ void probe_pass_kernel(DevGraph g, __grid_constant__ const ModelParams mp,
                                  const ProbeState* __restrict__ pool, uint32_t pool_n, uint32_t n,
                                  uint32_t npn, int rounds, ull seed, double* sink) {
    M m(mp);
    const uint32_t i0 = blockIdx.x * blockDim.x + threadIdx.x;
    if (i0 >= n) return;
    const PhiloxKeys rk = philox_keys((uint32_t)seed, (uint32_t)(seed >> 32));
    double acc = 0.0;
    for (int r = 0; r < rounds; ++r) {
        const ProbeState P = pool[((ull)r * n + i0) % pool_n];
        Step S;
        S.cur = P.cur;
        S.prev = P.prev;
        S.prev_degree = P.prev_degree;
        S.step = P.step;
        S.degree = P.degree;
        S.hmax = P.hmax;
        S.hsum = P.hsum;
        S.hin = P.hmax;  // no triangle bound in the probe
        S.lmax = S.lsum = 0.0;
        m.prepare(S);
        const uint32_t k = min(S.degree, npn);
        const WalkerKey key{(uint32_t)seed, (uint32_t)(seed >> 32), i0, (uint32_t)r, S.step};
        double bnd = 1.0, mnr = __longlong_as_double(0x7ff0000000000000ll);
        if (RANDOM && M::kBoundable && mp.shortcut) {
            bnd = m.bound(S);
            mnr = m.nonreturn_max(S);
        }
        ErvsState st{-DBL_MAX, 0.0, 0, kInvalid, 0};
        for (uint32_t t0 = 0; t0 < k; t0 += kProbeBatch) {
            ull e[kProbeBatch];
            bool live[kProbeBatch];
            double w[kProbeBatch];
#pragma unroll
            for (int j = 0; j < kProbeBatch; ++j) {
                const uint32_t t = t0 + j;
                live[j] = t < k;
                if (RANDOM) {
                    const U4 b = philox4x32_10_rk(U4{t, S.step, i0, (uint32_t)r}, rk);
                    e[j] = P.begin + bounded(lo64(b), S.degree);
                    live[j] = live[j] && uniform01(hi64(b)) * bnd < mnr;  // else nothing read
                } else {
                    e[j] = P.begin + t;
                }
            }
            probe_weights(m, S, P.phoff, g, e, live, w);
#pragma unroll
            for (int j = 0; j < kProbeBatch; ++j) {
                if (!live[j]) continue;
                if (RANDOM)
                    acc += w[j];
                else
                    st = ervs_visit<false>(st, key, rk, t0 + j, t0 + j, valid_w(w[j]) ? w[j] : 0.0);
            }
        }
        if (!RANDOM) acc += st.best_key + (double)st.best;
    }
    if (acc == -1.0) *sink = acc;  // keeps the loads alive
}

template <class M>
static cudaError_t calibrate_t(const DeviceGraphBuffers& gb, const ModelParams& mp,
                               const ProfileSpec& cfg, cudaStream_t s, double* ratio) {
    DevGraph g{gb.nodes, gb.edges, gb.labels, gb.hslots, gb.fat, gb.lagg, gb.twin, gb.fat32, gb.lab2,
               gb.nv, gb.ne};
    // the probe set of one round (cost_model.cpp:45-54): ceil(fraction * nv),
    // at least min_nodes; the pool holds kPoolRounds such sets (capped at the
    // graph's nodes with out-edges, and at 2^24 states)
    constexpr ull kPoolRounds = 16;
    const uint32_t want = (uint32_t)std::max<ull>(
        (ull)std::ceil(cfg.node_fraction * gb.nv), (ull)cfg.min_nodes);
    const ull pool_want = std::min<ull>(std::max<ull>((ull)want * kPoolRounds, want), 1ull << 24);
    const ull tries = pool_want * 8;
    uint32_t* nodes = nullptr;
    ProbeState* pool = nullptr;
    unsigned* count = nullptr;
    double* sink = nullptr;
    DW_TRY(cudaMallocAsync(&nodes, pool_want * sizeof(uint32_t), s));
    DW_TRY(cudaMallocAsync(&count, sizeof(unsigned), s));
    DW_TRY(cudaMallocAsync(&sink, sizeof(double), s));
    DW_TRY(cudaMemsetAsync(count, 0, sizeof(unsigned), s));
    const ull kseed = host_derive_seed(cfg.seed, 0x70726f66ULL);
    sample_nodes_kernel<<<grid_for(tries, 256), 256, 0, s>>>(g, kseed, tries, (uint32_t)pool_want,
                                                            nodes, count);
    unsigned got = 0;
    DW_TRY(cudaMemcpyAsync(&got, count, sizeof(unsigned), cudaMemcpyDeviceToHost, s));
    DW_TRY(cudaStreamSynchronize(s));
    const uint32_t pool_n = (uint32_t)std::min<ull>(got, pool_want);
    if (pool_n == 0) {
        cudaFreeAsync(nodes, s);
        cudaFreeAsync(count, s);
        cudaFreeAsync(sink, s);
        return cudaErrorInvalidValue;  // "profiling found no node with out-edges"
    }
    const uint32_t n = std::min<uint32_t>(want, pool_n);
    DW_TRY(cudaMallocAsync(&pool, (ull)pool_n * sizeof(ProbeState), s));
    probe_states_kernel<<<(pool_n + 255) / 256, 256, 0, s>>>(g, nodes, pool_n, pool);
    DW_TRY(cudaGetLastError());
    cudaEvent_t e0, e1, e2;
    DW_TRY(cudaEventCreate(&e0));
    DW_TRY(cudaEventCreate(&e1));
    DW_TRY(cudaEventCreate(&e2));
    const unsigned blocks = (unsigned)(((ull)n + 255) / 256);
    const uint32_t npn = cfg.neighbors_per_node;
    auto pass = [&](int rounds, float& t_rand, float& t_seq) -> cudaError_t {
        cudaEventRecord(e0, s);
        probe_pass_kernel<M, true>
            <<<blocks, 256, 0, s>>>(g, mp, pool, pool_n, n, npn, rounds, kseed, sink);
        cudaEventRecord(e1, s);
        probe_pass_kernel<M, false>
            <<<blocks, 256, 0, s>>>(g, mp, pool, pool_n, n, npn, rounds, kseed, sink);
        cudaEventRecord(e2, s);
        DW_TRY(cudaEventSynchronize(e2));
        cudaEventElapsedTime(&t_rand, e0, e1);
        cudaEventElapsedTime(&t_seq, e1, e2);
        return cudaGetLastError();
    };
    float tr = 0, ts = 0;
    DW_TRY(pass(1, tr, ts));  // warm-up
    int rounds = 1;
    // grow until both passes take milliseconds: sub-millisecond passes on a
    // 148-SM part are dominated by launch and tail effects, and the ratio
    // then swings by +-30% between runs
    while (rounds < (1 << 20)) {
        DW_TRY(pass(rounds, tr, ts));
        if (tr > 2.0f && ts > 2.0f) break;
        rounds *= 2;
    }
    std::vector<double> ratios;
    for (uint32_t rep = 0; rep < cfg.repetitions; ++rep) {
        DW_TRY(pass(rounds, tr, ts));
        ratios.push_back((double)tr / (double)ts);
    }
    std::sort(ratios.begin(), ratios.end());
    *ratio = ratios[ratios.size() / 2];
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaEventDestroy(e2);
    cudaFreeAsync(nodes, s);
    cudaFreeAsync(pool, s);
    cudaFreeAsync(count, s);
    cudaFreeAsync(sink, s);
    return cudaStreamSynchronize(s);
}

cudaError_t calibrate_ratio(const DeviceGraphBuffers& g, int kind, bool weighted,
                            const ModelParams& mp, const ProfileSpec& cfg, cudaStream_t s,
                            double* ratio) {
    switch (kind) {
    case 0: return weighted ? calibrate_t<StaticModel<true>>(g, mp, cfg, s, ratio)
                            : calibrate_t<StaticModel<false>>(g, mp, cfg, s, ratio);
    case 1: return weighted ? calibrate_t<Node2VecModel<true>>(g, mp, cfg, s, ratio)
                            : calibrate_t<Node2VecModel<false>>(g, mp, cfg, s, ratio);
    case 2: return weighted ? calibrate_t<MetaPathModel<true>>(g, mp, cfg, s, ratio)
                            : calibrate_t<MetaPathModel<false>>(g, mp, cfg, s, ratio);
    case 3: return weighted ? calibrate_t<Pr2Model<true>>(g, mp, cfg, s, ratio)
                            : calibrate_t<Pr2Model<false>>(g, mp, cfg, s, ratio);
    }
    return cudaErrorInvalidValue;
}

// ---- path compaction (dw_run_compact) ---------------------------------------
// Offsets as three small kernels of 128-thread blocks limited to 32 registers
// (__launch_bounds__(128, 16)): a block of them fits beside three resident
// walk-kernel CTAs (61,440 of 65,536 registers), so a batch's offsets and
// compaction run on a high-priority stream while the next batch walks
// (dw_capi.cu run engine).  Tiles of 1024 walkers: per-tile sums, a one-block
// scan of the tile sums chained through *d_base, per-tile offsets.
constexpr int kScanThreads = 128, kScanItems = 8, kScanTile = kScanThreads * kScanItems;

__device__ __forceinline__ ull block_excl_scan(ull v, ull* s_warp, ull* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    ull x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const ull y = __shfl_up_sync(0xFFFFFFFFu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[w] = x;
    __syncthreads();
    ull wbase = 0, all = 0;
#pragma unroll
    for (int i = 0; i < kScanThreads / 32; ++i) {
        if (i < w) wbase += s_warp[i];
        all += s_warp[i];
    }
    __syncthreads();
    *total = all;
    return wbase + x - v;
}

__global__ void __launch_bounds__(kScanThreads, 16)
    tile_sums_kernel(const uint32_t* __restrict__ len, ull n, ull* __restrict__ sums) {
    __shared__ ull s_warp[kScanThreads / 32];
    const ull t0 = (ull)blockIdx.x * kScanTile;
    ull v = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const ull i = t0 + (ull)k * kScanThreads + threadIdx.x;
        if (i < n) v += len[i];
    }
    ull total;
    block_excl_scan(v, s_warp, &total);
    if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

// sums[t] <- base + exclusive prefix over tiles; offs[n] and *d_base <- the end
__global__ void __launch_bounds__(kScanThreads, 16)
    tile_scan_kernel(ull* __restrict__ sums, ull ntiles, ull n, ull* __restrict__ offs,
                     ull* __restrict__ d_base) {
    __shared__ ull s_warp[kScanThreads / 32];
    ull run = *d_base;
    for (ull c = 0; c < ntiles; c += kScanThreads) {
        const ull i = c + threadIdx.x;
        const ull v = i < ntiles ? sums[i] : 0ull;
        ull total;
        const ull ex = block_excl_scan(v, s_warp, &total);
        if (i < ntiles) sums[i] = run + ex;
        run += total;
    }
    if (threadIdx.x == 0) {
        offs[n] = run;
        *d_base = run;
    }
}

// thread t owns walkers t*8 .. t*8+7 of the tile
__global__ void __launch_bounds__(kScanThreads, 16)
    tile_offsets_kernel(const uint32_t* __restrict__ len, ull n, const ull* __restrict__ sums,
                        ull* __restrict__ offs) {
    __shared__ ull s_warp[kScanThreads / 32];
    const ull i0 = (ull)blockIdx.x * kScanTile + (ull)threadIdx.x * kScanItems;
    uint32_t l[kScanItems];
    ull v = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        l[k] = i0 + k < n ? len[i0 + k] : 0u;
        v += l[k];
    }
    ull total;
    ull o = sums[blockIdx.x] + block_excl_scan(v, s_warp, &total);
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        if (i0 + k < n) offs[i0 + k] = o;
        o += l[k];
    }
}

cudaError_t path_offsets(const uint32_t* lengths, ull n, ull* offs, ull* d_base, void* tmp,
                         size_t& tmp_bytes, cudaStream_t s) {
    const ull ntiles = (n + kScanTile - 1) / kScanTile;
    if (!tmp) {
        tmp_bytes = std::max<ull>(ntiles, 1) * sizeof(ull);
        return cudaSuccess;
    }
    ull* sums = static_cast<ull*>(tmp);
    if (ntiles) {
        tile_sums_kernel<<<(unsigned)ntiles, kScanThreads, 0, s>>>(lengths, n, sums);
        DW_TRY(cudaGetLastError());
    }
    tile_scan_kernel<<<1, kScanThreads, 0, s>>>(sums, ntiles, n, offs, d_base);
    DW_TRY(cudaGetLastError());
    if (ntiles) {
        tile_offsets_kernel<<<(unsigned)ntiles, kScanThreads, 0, s>>>(lengths, n, sums, offs);
        DW_TRY(cudaGetLastError());
    }
    return cudaSuccess;
}

// Padded [n][stride] rows -> flat ids at offs[i] - offs[0].  A block owns
// kCompactRows rows and walks their padded elements with consecutive threads on
// consecutive ids (coalesced both ways); row/column advance incrementally.
// Every row full (no dead end, no early stop) means the padded rows already
// are the flat layout: the kernel returns and the engine copies the padded
// buffer (dw_capi.cu drain).
constexpr int kCompactRows = 128;
__global__ void __launch_bounds__(kScanThreads, 16) compact_paths_kernel(
    const uint32_t* __restrict__ paths, const uint32_t* __restrict__ len, ull n, ull stride,
    const ull* __restrict__ offs, uint32_t* __restrict__ flat) {
    const ull flat_base = offs[0];
    if (offs[n] - flat_base == n * stride) return;
    __shared__ ull s_off[kCompactRows];
    __shared__ uint32_t s_len[kCompactRows];
    for (ull r0 = (ull)blockIdx.x * kCompactRows; r0 < n; r0 += (ull)gridDim.x * kCompactRows) {
        const ull rows = min((ull)kCompactRows, n - r0);
        __syncthreads();
        for (int t = threadIdx.x; t < (int)rows; t += blockDim.x) {
            s_len[t] = len[r0 + t];
            s_off[t] = offs[r0 + t] - flat_base;
        }
        __syncthreads();
        const ull total = rows * stride;
        ull i = threadIdx.x / stride, j = threadIdx.x % stride;
        const uint32_t* src = paths + r0 * stride;
        for (ull k = threadIdx.x; k < total; k += blockDim.x) {
            if (j < s_len[i]) flat[s_off[i] + j] = src[k];
            j += blockDim.x;
            if (j >= stride) {
                const ull q = j / stride;
                i += q;
                j -= q * stride;
            }
        }
    }
}

cudaError_t compact_paths(const uint32_t* paths, const uint32_t* lengths, ull n, ull stride,
                          const ull* offs, uint32_t* flat, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    compact_paths_kernel<<<grid_for(n, kCompactRows), kScanThreads, 0, s>>>(paths, lengths, n,
                                                                           stride, offs, flat);
    return cudaGetLastError();
}

// ---- direct compact runs (dw_capi.cu run_direct) --------------------------------
// Predicted path length of each query: 0 for a start out of range (a query
// error, runtime.cpp:213-217), 1 for a start without neighbours (or a
// zero-step walk), target + 1 otherwise.  Exact on graphs where no edge
// leads to a vertex without neighbours and for models whose weights are
// positive by construction: no walk can then stop early.
__global__ void predict_lengths_kernel(const uint32_t* __restrict__ q, ull n,
                                       const NodeRec* __restrict__ nodes, uint32_t nv,
                                       uint32_t target, uint32_t* __restrict__ len) {
    for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (ull)gridDim.x * blockDim.x) {
        const uint32_t v = q[i];
        len[i] = v >= nv ? 0u : (target && nodes[v].degree) ? target + 1u : 1u;
    }
}

cudaError_t predict_lengths(const uint32_t* queries, ull n, const NodeRec* nodes, uint32_t nv,
                            uint32_t target, uint32_t* lengths, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    predict_lengths_kernel<<<grid_for(n, 256 * 8), 256, 0, s>>>(queries, n, nodes, nv, target,
                                                                lengths);
    return cudaGetLastError();
}

// out[c] = offs[min(c << shift, n)], c = 0..nchunks (out may be host-mapped)
__global__ void chunk_bounds_kernel(const ull* __restrict__ offs, ull n, uint32_t shift,
                                    ull nchunks, ull* out) {
    for (ull c = (ull)blockIdx.x * blockDim.x + threadIdx.x; c <= nchunks;
         c += (ull)gridDim.x * blockDim.x)
        out[c] = offs[min(c << shift, n)];
}

cudaError_t chunk_bounds(const ull* offs, ull n, uint32_t shift, ull nchunks, ull* out,
                         cudaStream_t s) {
    chunk_bounds_kernel<<<grid_for(nchunks + 1, 256), 256, 0, s>>>(offs, n, shift, nchunks, out);
    return cudaGetLastError();
}

// Walkers whose path is final before the walk (length 0: start out of range;
// 1: start without neighbours or target 0) are done here: a length-1 path's
// one id is written at its offset, and queries / query errors are counted
// (the walk kernel counts the walkers it claims).  len[i] becomes the
// walker's "walks" flag, for the scan that lists the walking ones.
__global__ void trivial_walkers_kernel(const uint32_t* __restrict__ q, ull n,
                                       uint32_t* __restrict__ len, const ull* __restrict__ offs,
                                       uint32_t* __restrict__ flat, ull* __restrict__ counters) {
    uint32_t nq = 0, ne = 0;
    for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (ull)gridDim.x * blockDim.x) {
        const uint32_t l = len[i];
        if (l == 1) flat[offs[i]] = q[i];
        nq += l <= 1;
        ne += l == 0;
        len[i] = l > 1;
    }
    __shared__ uint32_t s_c[2];
    if (threadIdx.x == 0) s_c[0] = s_c[1] = 0;
    __syncthreads();
    nq = __reduce_add_sync(0xFFFFFFFFu, nq);
    ne = __reduce_add_sync(0xFFFFFFFFu, ne);
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(&s_c[0], nq);
        atomicAdd(&s_c[1], ne);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_c[0]) atomicAdd(&counters[kCQueries], (ull)s_c[0]);
        if (s_c[1]) atomicAdd(&counters[kCQueryErrors], (ull)s_c[1]);
    }
}

cudaError_t trivial_walkers(const uint32_t* queries, ull n, uint32_t* lengths, const ull* offs,
                            uint32_t* flat, ull* counters, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    trivial_walkers_kernel<<<grid_for(n, 256 * 8), 256, 0, s>>>(queries, n, lengths, offs, flat,
                                                               counters);
    return cudaGetLastError();
}

// dw_run_device's listed walks: every walker's length (the predicted one:
// exact where listed walks are used), the whole padded row of each walker
// that does not move (its start or nothing, then 0xFFFFFFFF; a warp writes a
// row with coalesced stores), queries / query errors counted; len[i] becomes
// the "walks" flag.  The rows of the walkers that move are written whole by
// the walk (no walk ends early there), so the rows need no memset.
__global__ void trivial_rows_kernel(const uint32_t* __restrict__ q, ull n,
                                    uint32_t* __restrict__ len, uint32_t* __restrict__ paths,
                                    ull stride, uint32_t* __restrict__ lengths,
                                    ull* __restrict__ counters) {
    const int lane = threadIdx.x & 31;
    uint32_t nq = 0, ne = 0;
    const ull warps = (ull)gridDim.x * (blockDim.x >> 5);
    for (ull w = (ull)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w * 32 < n; w += warps) {
        const ull i = w * 32 + lane;
        const uint32_t l = i < n ? len[i] : 2u;
        const uint32_t v = i < n && l == 1 ? q[i] : 0xFFFFFFFFu;
        if (i < n) {
            if (lengths) lengths[i] = l;
            nq += l <= 1;
            ne += l == 0;
            len[i] = l > 1;
        }
        if (paths) {
            unsigned triv = __ballot_sync(0xFFFFFFFFu, l <= 1);
            while (triv) {
                const int b = __ffs(triv) - 1;
                triv &= triv - 1;
                const uint32_t vb = __shfl_sync(0xFFFFFFFFu, v, b);
                uint32_t* row = paths + (w * 32 + b) * stride;
                for (ull j = lane; j < stride; j += 32) row[j] = j == 0 ? vb : 0xFFFFFFFFu;
            }
        }
    }
    __shared__ uint32_t s_c[2];
    if (threadIdx.x == 0) s_c[0] = s_c[1] = 0;
    __syncthreads();
    nq = __reduce_add_sync(0xFFFFFFFFu, nq);
    ne = __reduce_add_sync(0xFFFFFFFFu, ne);
    if (lane == 0) {
        atomicAdd(&s_c[0], nq);
        atomicAdd(&s_c[1], ne);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (s_c[0]) atomicAdd(&counters[kCQueries], (ull)s_c[0]);
        if (s_c[1]) atomicAdd(&counters[kCQueryErrors], (ull)s_c[1]);
    }
}

cudaError_t trivial_rows(const uint32_t* queries, ull n, uint32_t* len, uint32_t* paths,
                         ull stride, uint32_t* lengths, ull* counters, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    trivial_rows_kernel<<<grid_for(n, 256 * 4), 256, 0, s>>>(queries, n, len, paths, stride,
                                                            lengths, counters);
    return cudaGetLastError();
}

// The walking walkers, in query order: cq / cqid / coffs[pos[i]] = query,
// global walker id (RNG key) and flat offset of every i with flag[i] set.
__global__ void walker_list_kernel(const uint32_t* __restrict__ q, const ull* __restrict__ qids,
                                   ull qid_base, ull n, const uint32_t* __restrict__ flag,
                                   const ull* __restrict__ pos, const ull* __restrict__ offs,
                                   ull stride, uint32_t* __restrict__ cq, ull* __restrict__ cqid,
                                   ull* __restrict__ coffs) {
    for (ull i = (ull)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (ull)gridDim.x * blockDim.x) {
        if (!flag[i]) continue;
        const ull j = pos[i];
        cq[j] = q[i];
        cqid[j] = qids ? qids[i] : qid_base + i;
        coffs[j] = offs ? offs[i] : i * stride;
    }
}

cudaError_t walker_list(const uint32_t* queries, const ull* qids, ull qid_base, ull n,
                        const uint32_t* flag, const ull* pos, const ull* offs, ull stride,
                        uint32_t* cq, ull* cqid, ull* coffs, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    walker_list_kernel<<<grid_for(n, 256 * 8), 256, 0, s>>>(queries, qids, qid_base, n, flag, pos,
                                                           offs, stride, cq, cqid, coffs);
    return cudaGetLastError();
}

// Copy ranges of the direct run's chunks (host-mapped out): chunk c holds
// walking walkers [c << shift, (c + 1) << shift) of the nt = *d_nt listed,
// and the flat range out[c] .. out[c + 1] (out[0] = 0, out[nch] = total;
// the paths of the walkers that do not walk are written before the walk).
// out[kMax + 1] = nt, out[kMax + 2] = nch.
__global__ void direct_bounds_kernel(const ull* __restrict__ coffs, const ull* __restrict__ d_nt,
                                     const ull* __restrict__ total, uint32_t shift, ull kmax,
                                     ull* out) {
    const ull nt = *d_nt;
    const ull nch = (nt + (1ull << shift) - 1) >> shift;
    for (ull c = (ull)blockIdx.x * blockDim.x + threadIdx.x; c <= nch;
         c += (ull)gridDim.x * blockDim.x)
        out[c] = c == nch ? *total : c == 0 ? 0ull : coffs[c << shift];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        out[kmax + 1] = nt;
        out[kmax + 2] = nch;
    }
}

cudaError_t direct_bounds(const ull* coffs, const ull* d_nt, const ull* total, uint32_t shift,
                          ull kmax, ull* out, cudaStream_t s) {
    direct_bounds_kernel<<<grid_for(kmax + 1, 256), 256, 0, s>>>(coffs, d_nt, total, shift, kmax,
                                                                out);
    return cudaGetLastError();
}

// *flag <- 1 when some edge leads to a vertex without neighbours
__global__ void sink_targets_kernel(const NodeRec* __restrict__ nodes,
                                    const EdgeRec* __restrict__ edges, ull ne,
                                    int* __restrict__ flag) {
    bool sink = false;
    for (ull e = (ull)blockIdx.x * blockDim.x + threadIdx.x; e < ne;
         e += (ull)gridDim.x * blockDim.x)
        sink |= nodes[edges[e].col].degree == 0;
    if (__any_sync(0xFFFFFFFFu, sink) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

cudaError_t sink_targets(const NodeRec* nodes, const EdgeRec* edges, ull ne, int* flag,
                         cudaStream_t s) {
    if (ne == 0) return cudaSuccess;
    sink_targets_kernel<<<grid_for(ne, 256 * 16), 256, 0, s>>>(nodes, edges, ne, flag);
    return cudaGetLastError();
}

// ---- DWG1 loads ----------------------------------------------------------------
__global__ void check_props_kernel(const float* __restrict__ prop, ull ne, int* __restrict__ bad) {
    for (ull e = blockIdx.x * (ull)blockDim.x + threadIdx.x; e < ne;
         e += (ull)gridDim.x * blockDim.x) {
        const float p = prop[e];
        if (!(p > 0.0f) || !isfinite(p)) atomicOr(bad, 1);
    }
}

// one warp per row: any descending neighbour pair marks the graph unsorted
__global__ void check_sorted_kernel(const ull* __restrict__ row, uint32_t nv,
                                    const uint32_t* __restrict__ col, int* __restrict__ unsorted) {
    const ull warp = (blockIdx.x * (ull)blockDim.x + threadIdx.x) >> 5;
    const ull nwarps = ((ull)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    for (ull v = warp; v < nv; v += nwarps) {
        const ull b = row[v], e = row[v + 1];
        bool bad = false;
        for (ull i = b + 1 + lane; i < e; i += 32) bad |= col[i - 1] > col[i];
        if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(unsorted, 1);
    }
}

__global__ void iota_kernel(uint32_t* __restrict__ out, ull n) {
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < n;
         i += (ull)gridDim.x * blockDim.x)
        out[i] = (uint32_t)i;
}

template <class T>
__global__ void gather_kernel(const T* __restrict__ in, const uint32_t* __restrict__ idx, ull n,
                              T* __restrict__ out) {
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < n;
         i += (ull)gridDim.x * blockDim.x)
        out[i] = in[idx[i]];
}

__global__ void fill_u64_kernel(ull* __restrict__ out, ull n, ull v) {
    for (ull i = blockIdx.x * (ull)blockDim.x + threadIdx.x; i < n;
         i += (ull)gridDim.x * blockDim.x)
        out[i] = v;
}

cudaError_t prepare_loaded_csr(ull** d_row, uint32_t* nv, ull ne, uint32_t* d_col, float* d_prop,
                               uint16_t* d_label, int* status, cudaStream_t s) {
    *status = 0;
    int* flags = nullptr;  // [0] bad prop, [1] unsorted
    DW_TRY(cudaMallocAsync(&flags, 2 * sizeof(int), s));
    DW_TRY(cudaMemsetAsync(flags, 0, 2 * sizeof(int), s));
    uint32_t vmax = 0;
    if (ne) {
        // Graph::build: num_vertices = max(hint, max referenced id + 1)
        uint32_t* d_max = nullptr;
        DW_TRY(cudaMallocAsync(&d_max, sizeof(uint32_t), s));
        size_t tb = 0;
        DW_TRY(cub::DeviceReduce::Max(nullptr, tb, d_col, d_max, (int64_t)ne, s));
        void* tmp = nullptr;
        DW_TRY(cudaMallocAsync(&tmp, tb, s));
        DW_TRY(cub::DeviceReduce::Max(tmp, tb, d_col, d_max, (int64_t)ne, s));
        DW_TRY(cudaMemcpyAsync(&vmax, d_max, sizeof(uint32_t), cudaMemcpyDeviceToHost, s));
        DW_TRY(cudaStreamSynchronize(s));
        DW_TRY(cudaFreeAsync(tmp, s));
        DW_TRY(cudaFreeAsync(d_max, s));
        if ((ull)vmax + 1 >= 0xFFFFFFFFull) {
            *status = 2;
            return cudaFreeAsync(flags, s);
        }
        if (vmax + 1 > *nv) {  // extend: the new vertices have no out-edges
            const uint32_t nv2 = vmax + 1;
            ull* row2 = nullptr;
            DW_TRY(cudaMallocAsync(&row2, (nv2 + 1ull) * sizeof(ull), s));
            DW_TRY(cudaMemcpyAsync(row2, *d_row, (*nv + 1ull) * sizeof(ull),
                                   cudaMemcpyDeviceToDevice, s));
            fill_u64_kernel<<<grid_for(nv2 - *nv, 256), 256, 0, s>>>(row2 + *nv + 1, nv2 - *nv, ne);
            DW_TRY(cudaFreeAsync(*d_row, s));
            *d_row = row2;
            *nv = nv2;
        }
        check_props_kernel<<<grid_for(ne, 256), 256, 0, s>>>(d_prop, ne, flags);
        check_sorted_kernel<<<grid_for((ull)*nv * 32, 256), 256, 0, s>>>(*d_row, *nv, d_col,
                                                                         flags + 1);
        DW_TRY(cudaGetLastError());
    }
    int h[2] = {0, 0};
    DW_TRY(cudaMemcpyAsync(h, flags, sizeof h, cudaMemcpyDeviceToHost, s));
    DW_TRY(cudaStreamSynchronize(s));
    DW_TRY(cudaFreeAsync(flags, s));
    if (h[0]) {
        *status = 1;
        return cudaSuccess;
    }
    if (h[1]) {  // Graph::build's per-slice stable sort by target
        if (ne > 0x7FFFFFFFull) {
            *status = 3;
            return cudaSuccess;
        }
        uint32_t *idx = nullptr, *idx2 = nullptr, *col2 = nullptr;
        DW_TRY(cudaMallocAsync(&idx, ne * sizeof(uint32_t), s));
        DW_TRY(cudaMallocAsync(&idx2, ne * sizeof(uint32_t), s));
        DW_TRY(cudaMallocAsync(&col2, ne * sizeof(uint32_t), s));
        iota_kernel<<<grid_for(ne, 256), 256, 0, s>>>(idx, ne);
        size_t tb = 0;
        DW_TRY(cub::DeviceSegmentedSort::StableSortPairs(nullptr, tb, d_col, col2, idx, idx2,
                                                         (int)ne, (int)*nv, *d_row, *d_row + 1,
                                                         s));
        void* tmp = nullptr;
        DW_TRY(cudaMallocAsync(&tmp, tb, s));
        DW_TRY(cub::DeviceSegmentedSort::StableSortPairs(tmp, tb, d_col, col2, idx, idx2, (int)ne,
                                                         (int)*nv, *d_row, *d_row + 1, s));
        DW_TRY(cudaMemcpyAsync(d_col, col2, ne * sizeof(uint32_t), cudaMemcpyDeviceToDevice, s));
        float* p2 = reinterpret_cast<float*>(col2);  // reuse as the props scratch
        gather_kernel<float><<<grid_for(ne, 256), 256, 0, s>>>(d_prop, idx2, ne, p2);
        DW_TRY(cudaMemcpyAsync(d_prop, p2, ne * sizeof(float), cudaMemcpyDeviceToDevice, s));
        if (d_label) {
            uint16_t* l2 = reinterpret_cast<uint16_t*>(idx);
            gather_kernel<uint16_t><<<grid_for(ne, 256), 256, 0, s>>>(d_label, idx2, ne, l2);
            DW_TRY(cudaMemcpyAsync(d_label, l2, ne * sizeof(uint16_t), cudaMemcpyDeviceToDevice,
                                   s));
        }
        DW_TRY(cudaGetLastError());
        DW_TRY(cudaFreeAsync(tmp, s));
        DW_TRY(cudaFreeAsync(idx, s));
        DW_TRY(cudaFreeAsync(idx2, s));
        DW_TRY(cudaFreeAsync(col2, s));
    }
    return cudaStreamSynchronize(s);
}

// ---- text sink ------------------------------------------------------------------
__device__ __forceinline__ uint32_t dec_digits(uint32_t x) {
    uint32_t d = 1;
    while (x >= 10) {
        x /= 10;
        ++d;
    }
    return d;
}

// one warp per path
__global__ void text_bytes_kernel(const uint32_t* __restrict__ paths,
                                  const uint32_t* __restrict__ len, ull n, ull stride,
                                  uint32_t* __restrict__ bytes) {
    const ull warp = (blockIdx.x * (ull)blockDim.x + threadIdx.x) >> 5;
    const ull nwarps = ((ull)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    for (ull i = warp; i < n; i += nwarps) {
        const uint32_t l = len[i];
        uint32_t b = 0;
        for (uint32_t j = lane; j < l; j += 32) b += dec_digits(paths[i * stride + j]) + 1;
        b = __reduce_add_sync(0xFFFFFFFFu, b);
        if (lane == 0) bytes[i] = l ? b : 1;  // separators + newline == l; "\n" when empty
    }
}

__global__ void text_write_kernel(const uint32_t* __restrict__ paths,
                                  const uint32_t* __restrict__ len, ull n, ull stride,
                                  const ull* __restrict__ toffs, char* __restrict__ text) {
    const ull warp = (blockIdx.x * (ull)blockDim.x + threadIdx.x) >> 5;
    const ull nwarps = ((ull)gridDim.x * blockDim.x) >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const ull base0 = toffs[0];
    for (ull i = warp; i < n; i += nwarps) {
        const uint32_t l = len[i];
        char* out = text + (toffs[i] - base0);
        if (l == 0) {
            if (lane == 0) out[0] = '\n';
            continue;
        }
        uint32_t pos = 0;  // running byte position of the chunk's first id
        for (uint32_t j0 = 0; j0 < l; j0 += 32) {
            const uint32_t j = j0 + lane;
            const uint32_t x = j < l ? paths[i * stride + j] : 0u;
            const uint32_t w = j < l ? dec_digits(x) + 1 : 0u;  // digits + separator
            uint32_t incl = w;  // inclusive warp scan of widths
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
                if (lane >= (uint32_t)o) incl += t;
            }
            if (j < l) {
                char* q = out + pos + incl - w;
                uint32_t y = x;
                for (int k = (int)w - 2; k >= 0; --k) {
                    q[k] = (char)('0' + y % 10);
                    y /= 10;
                }
                q[w - 1] = j + 1 == l ? '\n' : ' ';
            }
            pos += __shfl_sync(0xFFFFFFFFu, incl, 31);
        }
    }
}

cudaError_t path_text_bytes(const uint32_t* paths, const uint32_t* lengths, ull n, ull stride,
                            uint32_t* bytes, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    text_bytes_kernel<<<grid_for(n * 32, 256), 256, 0, s>>>(paths, lengths, n, stride, bytes);
    return cudaGetLastError();
}

cudaError_t path_text_write(const uint32_t* paths, const uint32_t* lengths, ull n, ull stride,
                            const ull* toffs, char* text, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    text_write_kernel<<<grid_for(n * 32, 256), 256, 0, s>>>(paths, lengths, n, stride, toffs,
                                                            text);
    return cudaGetLastError();
}

// ---- DSL preprocess: label aggregates ------------------------------------------
__global__ void label_agg_kernel(const NodeRec* __restrict__ nodes, uint32_t nv,
                                 const uint16_t* __restrict__ labels, double2* __restrict__ out) {
    for (ull v = blockIdx.x * (ull)blockDim.x + threadIdx.x; v < nv;
         v += (ull)gridDim.x * blockDim.x) {
        const NodeRec nr = nodes[v];
        double mx = 0.0, sum = 0.0;
        if (labels)
            for (ull e = nr.begin; e < nr.begin + nr.degree; ++e) {
                const double l = labels[e];
                if (l > mx) mx = l;
                sum += l;
            }
        out[v] = make_double2(mx, sum);
    }
}

cudaError_t build_label_aggregates(DeviceGraphBuffers& g, cudaStream_t s) {
    if (g.lagg) return cudaSuccess;
    DW_TRY(cudaMalloc(&g.lagg, std::max<uint32_t>(g.nv, 1) * sizeof(double2)));
    label_agg_kernel<<<grid_for(g.nv, 128), 128, 0, s>>>(g.nodes, g.nv, g.labels, g.lagg);
    DW_TRY(cudaGetLastError());
    return cudaStreamSynchronize(s);
}

}  // namespace dwb
