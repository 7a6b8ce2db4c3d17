// dw_member.cuh -- Graph::has_edge (graph.cpp:114-118) as one sector probe.
//
// The reference answers "u in N(prev)?" with std::binary_search over prev's
// sorted slice: ceil(log2 d') dependent loads, 17+ on R-MAT hubs.  On the
// device every row with d > kScanMax also owns an open-addressing hash set of
// its targets: next_pow2(2d) u32 slots (load <= 1/2) grouped in 32-byte
// buckets of 8 slots, so a lookup is one sector (rarely two).  Rows with
// d <= kScanMax are scanned directly (<= 48 B, independent loads).  The answer
// is exactly the binary search's: the set holds precisely the slice's targets.
#pragma once
#include "dw_common.cuh"

namespace dwb {

// <= 6 records span at most four 16 B slots whatever the row's alignment
// (the walk kernel's MEMB phase loads them in one iteration)
constexpr uint32_t kScanMax = 6;
constexpr uint32_t kHashEmpty = 0xFFFFFFFFu;  // == kInvalid, never a target id

__host__ __device__ __forceinline__ uint32_t hash_log2_buckets(uint32_t d) {
    // slots = next_pow2(2d), >= 16; buckets = slots / 8
    uint32_t lg = 4;
    while ((1ull << lg) < 2ull * d) ++lg;
    return lg - 3;
}

__host__ __device__ __forceinline__ uint32_t hash_buckets(uint32_t d) {
    return d > kScanMax ? (1u << hash_log2_buckets(d)) : 0u;
}

__device__ __forceinline__ uint32_t hash_bucket(uint32_t u, uint32_t lg) {
    return (u * 0x9E3779B1u) >> (32 - lg);
}

__device__ __forceinline__ bool member(const DevGraph& g, unsigned long long begin, uint32_t d,
                                       uint32_t hoff, uint32_t u) {
    if (d <= kScanMax) {
        bool hit = false;
#pragma unroll
        for (uint32_t i = 0; i < kScanMax; ++i)
            if (i < d) hit |= load_col(g.edges + begin + i) == u;
        return hit;
    }
    const uint32_t lg = hash_log2_buckets(d);
    const uint32_t mask = (1u << lg) - 1u;
    uint32_t b = hash_bucket(u, lg);
    for (;;) {
        const uint4* p = reinterpret_cast<const uint4*>(g.hslots + 8ull * (hoff + b));
        const uint4 x = __ldg(p), y = __ldg(p + 1);
        if (x.x == u || x.y == u || x.z == u || x.w == u || y.x == u || y.y == u || y.z == u ||
            y.w == u)
            return true;
        if (y.w == kHashEmpty) return false;  // slots fill in order: a free slot ends the chain
        b = (b + 1) & mask;
    }
}

}  // namespace dwb
