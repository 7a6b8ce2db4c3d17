// dw_common.cuh -- device data layout, Philox walker streams, bit maps.
//
// HBM layout:
//   NodeRec[nv]  32 B, one sector: {row begin u64, degree u32, -, max h f64,
//                sum h f64}.  One random sector per step serves degree(cur),
//                out_edge_begin(cur) and the cost-model aggregates
//                (graph.hpp:209-231; decide_sampler, cost_model.hpp:46-56).
//   EdgeRec[ne]   8 B: {target u32, prop f32}.  One random sector per
//                rejection trial serves edge_target(e) and edge_prop(e).
//   labels[ne]   u16, only for labelled graphs (MetaPath).
//   hslots[]     per-row membership hash sets (dw_member.cuh), 32 B buckets.
//   FatRec[ne]   48 B used of a 64 B stride (optional, "fat" layout): the edge
//                plus everything the walk needs about its target, so an
//                accepted rejection trial starts the next step with no further
//                gather.  On B200 every random miss moves a whole 128 B L2
//                line from HBM (tools/gather_probe.cu), so a record up to 64 B
//                costs the same DRAM traffic as a 16 B one; what counts is the
//                number of random requests per walker-step.
#pragma once
#ifdef __CUDACC_RTC__
// NVRTC (DSL models, dw_dsl.cu): no host headers
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef long long int64_t;
#define DBL_MAX 1.7976931348623157e+308
#else
#include <cstdint>
#include <cuda_runtime.h>
#endif

namespace dwb {

constexpr uint32_t kInvalid = 0xFFFFFFFFu;

struct alignas(32) NodeRec {
    unsigned long long begin;
    uint32_t degree;
    uint32_t hoff;  // first bucket of the row's membership hash set (dw_member.cuh)
    double hmax;
    double hsum;
};
static_assert(sizeof(NodeRec) == 32, "NodeRec must be one sector");

struct alignas(8) EdgeRec {
    uint32_t col;
    float h;
};
static_assert(sizeof(EdgeRec) == 8, "EdgeRec must be 8 bytes");

// Fat edge record for edge e = (v -> u), 64 B stride (one L2 line half):
//   w0 col = u          w1 h = edge_prop(e)
//   w2,w3 begin(u) (bits 0-39) | label(e) (bits 40-55) | label mask of u (bits 56-63:
//         bit l < 7 set iff N(u) has an edge labelled l; bit 7: N(u) has a label >= 7)
//   w4 degree(u)        w5 hoff(u)              w6 twin_lo: first index of v in N(u)
//   w7 twin_cnt: multiplicity of v in N(u) (0 for a directed edge without twin)
//   w8..11 node_prop_max(u), node_prop_sum(u) (f64, exact)
// The twin range lets eRJS reject trials without a gather: every edge of N(u)
// outside [twin_lo, twin_lo + twin_cnt) has target != v, so its weight is
// bounded by the model's non-return maximum (dw_models.cuh nonreturn_max).
struct alignas(64) FatRec {
    uint32_t col;
    float h;
    unsigned long long tbegin_label;
    uint32_t tdeg;
    uint32_t thoff;
    uint32_t twin_lo;
    uint32_t twin_cnt;
    double thmax;
    double thsum;
    uint32_t aux[4];  // reserved
};
static_assert(sizeof(FatRec) == 64, "FatRec stride must be 64 bytes");

// Compact fat record for graphs whose 64 B layout would exceed its HBM cap
// (R-MAT s27): the same fields in 32 B, one sector.  u32 words:
//   w0 col   w1 h (f32)   w2 begin bits 0-31   w3 begin bits 32-39 | degree << 8
//   w4 hoff  w5 twin: lo | cnt << 24 (cnt 255 = unknown)
//   w6 node_prop_max (f32: a maximum of f32 props, exact)
//   w7 node_prop_sum rounded to f32 -- decisions within 1e-6 of the threshold
//      fetch the exact node record instead (dw_walk_kernel.cuh)
// No labels: built only for unlabelled graphs with degrees < 2^24, and walked
// only by node2vec kernels (their decision has the one-multiply screen).
struct alignas(32) FatRec32 {
    uint32_t col;
    float h;
    uint32_t begin_lo;
    uint32_t begin_hi_deg;
    uint32_t thoff;
    uint32_t twin;
    float thmax;
    float thsum;
};
static_assert(sizeof(FatRec32) == 32, "FatRec32 must be one sector");
constexpr unsigned long long kBeginMask = (1ull << 40) - 1;
constexpr uint32_t kMaskLabels = 7;  // labels with an exact bit in the fat record's mask

struct DevGraph {
    const NodeRec* __restrict__ nodes;
    const EdgeRec* __restrict__ edges;
    const uint16_t* __restrict__ labels;  // may be null
    const uint32_t* __restrict__ hslots;  // membership hash sets, 8 slots per bucket
    const FatRec* __restrict__ fat;       // may be null (slim layout)
    const double2* __restrict__ lagg;     // per-node {label MAX, label SUM} or null (DSL)
    const uint32_t* __restrict__ twin;    // slim layout: return-edge range per edge, or null
    const FatRec32* __restrict__ fat32;   // compact fat records, or null
    // labels packed 2 bits each (16 per word) when every label is < 4, or
    // null: L2-resident at config-3 sizes (E/4 bytes), they let a MetaPath
    // trial be judged on its label before its record is gathered
    const uint32_t* __restrict__ lab2;
    uint32_t nv;
    unsigned long long ne;
};

// Error codes raised from inside kernels (first one wins).
enum DevError : int {
    kDevOk = 0,
    kDevBadWeight = 1,   // samplers.hpp:50-53
    kDevBadBound = 2,    // samplers.hpp:152-154
    kDevSchema = 3,      // models.hpp:100-101
};

__device__ __forceinline__ NodeRec load_node(const NodeRec* __restrict__ p) {
    // one 32 B sector as two 16 B non-coherent loads
    const uint4* q = reinterpret_cast<const uint4*>(p);
    const uint4 a = __ldg(q);
    const uint4 b = __ldg(q + 1);
    NodeRec r;
    r.begin = (unsigned long long)a.x | ((unsigned long long)a.y << 32);
    r.degree = a.z;
    r.hoff = a.w;
    r.hmax = __hiloint2double((int)b.y, (int)b.x);
    r.hsum = __hiloint2double((int)b.w, (int)b.z);
    return r;
}

__device__ __forceinline__ EdgeRec load_edge(const EdgeRec* __restrict__ p) {
    const uint2 v = __ldg(reinterpret_cast<const uint2*>(p));
    EdgeRec e;
    e.col = v.x;
    e.h = __uint_as_float(v.y);
    return e;
}

__device__ __forceinline__ uint32_t load_col(const EdgeRec* __restrict__ p) {
    return __ldg(reinterpret_cast<const uint32_t*>(p));
}

// Philox4x32-10 (Salmon et al. 2011; constants as curand_philox4x32_x.h:88-91).
struct U4 {
    uint32_t x, y, z, w;
};

__host__ __device__ __forceinline__ U4 philox4x32_10(U4 c, uint32_t k0, uint32_t k1) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        if (r) {
            k0 += 0x9E3779B9u;
            k1 += 0xBB67AE85u;
        }
#ifdef __CUDA_ARCH__
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
#else
        const uint64_t p0 = (uint64_t)0xD2511F53u * c.x, p1 = (uint64_t)0xCD9E8D57u * c.z;
        const uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
        const uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
#endif
        c = U4{hi1 ^ c.y ^ k0, lo1, hi0 ^ c.w ^ k1, lo0};
    }
    return c;
}

// Walker stream: key = seed, counter = (draw >> 1, step, qid lo, qid hi).
// Draw 2k = words (y:x) of block k, draw 2k+1 = words (w:z).  Same map as
// the oracle (oracle.c orc_walker_draw); one block serves one rejection trial
// (bounded(d) then uniform01, samplers.hpp:160-161).
struct WalkerKey {
    uint32_t k0, k1;      // seed
    uint32_t q0, q1;      // global walker id
    uint32_t step;
};

// Same Philox with the round keys precomputed (rk[0][r] = k0 + r*0x9E3779B9,
// rk[1][r] = k1 + r*0xBB67AE85), read straight from the kernel's constant
// parameter bank: no key-schedule registers or adds in the hot loop.
struct PhiloxKeys {
    uint32_t k[2][10];
};
__host__ __device__ __forceinline__ PhiloxKeys philox_keys(uint32_t k0, uint32_t k1) {
    PhiloxKeys r;
    for (int i = 0; i < 10; ++i) {
        r.k[0][i] = k0 + (uint32_t)i * 0x9E3779B9u;
        r.k[1][i] = k1 + (uint32_t)i * 0xBB67AE85u;
    }
    return r;
}
__device__ __forceinline__ U4 philox4x32_10_rk(U4 c, const PhiloxKeys& rk) {
#pragma unroll
    for (int r = 0; r < 10; ++r) {
        const uint32_t hi0 = __umulhi(0xD2511F53u, c.x), lo0 = 0xD2511F53u * c.x;
        const uint32_t hi1 = __umulhi(0xCD9E8D57u, c.z), lo1 = 0xCD9E8D57u * c.z;
        c = U4{hi1 ^ c.y ^ rk.k[0][r], lo1, hi0 ^ c.w ^ rk.k[1][r], lo0};
    }
    return c;
}

__device__ __forceinline__ U4 walker_block(const WalkerKey& w, uint32_t block) {
    return philox4x32_10(U4{block, w.step, w.q0, w.q1}, w.k0, w.k1);
}

__device__ __forceinline__ unsigned long long lo64(const U4& b) {
    return (unsigned long long)b.x | ((unsigned long long)b.y << 32);
}
__device__ __forceinline__ unsigned long long hi64(const U4& b) {
    return (unsigned long long)b.z | ((unsigned long long)b.w << 32);
}

// walker_draw with the seed's round keys read from the kernel parameters
// (PhiloxKeys): 40 instructions per block instead of 60, and one less key
// schedule per inlined call site
__device__ __forceinline__ unsigned long long walker_draw(const WalkerKey& w, const PhiloxKeys& rk,
                                                          unsigned long long idx) {
    const U4 b = philox4x32_10_rk(U4{(uint32_t)(idx >> 1), w.step, w.q0, w.q1}, rk);
    return (idx & 1) ? hi64(b) : lo64(b);
}

__device__ __forceinline__ unsigned long long walker_draw(const WalkerKey& w,
                                                          unsigned long long idx) {
    const U4 b = walker_block(w, (uint32_t)(idx >> 1));
    return (idx & 1) ? hi64(b) : lo64(b);
}

// Reference bit maps (rng.hpp:40-50).  Exact in IEEE double.
__device__ __forceinline__ double uniform01(unsigned long long r) {
    return __dmul_rn(__ull2double_rn(r >> 11), 0x1.0p-53);
}
__device__ __forceinline__ double open01(unsigned long long r) {
    return __dmul_rn(__dadd_rn(__ull2double_rn(r >> 11), 0.5), 0x1.0p-53);
}
__device__ __forceinline__ unsigned long long bounded(unsigned long long r,
                                                      unsigned long long n) {
    return __umul64hi(r, n);
}

// floor(log2 d) capped at 31 (runtime.cpp:42-46).
__device__ __forceinline__ int degree_bucket(uint32_t d) {
    return d ? 31 - __clz(d) : 0;
}

}  // namespace dwb
