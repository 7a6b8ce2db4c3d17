// dw_member.cuh -- Graph::has_edge (graph.cpp:114-118) as one sector probe.
//
// The reference answers "u in N(prev)?" with std::binary_search over prev's
// sorted slice: ceil(log2 d') dependent loads, 17+ on R-MAT hubs.  On the
// device every non-empty row owns an open-addressing hash set of its targets:
// max(8, next_pow2(2d)) u32 slots (load <= 1/2) grouped in 32-byte buckets of
// 8 slots, so a lookup is one random request (rarely two).  The answer is
// exactly the binary search's: the set holds precisely the slice's targets.
#pragma once
#include "dw_common.cuh"

namespace dwb {

constexpr uint32_t kHashEmpty = 0xFFFFFFFFu;  // == kInvalid, never a target id

__host__ __device__ __forceinline__ uint32_t hash_log2_buckets(uint32_t d) {
    // slots = max(8, next_pow2(2d)); buckets = slots / 8
#ifdef __CUDA_ARCH__
    return d <= 4 ? 0u : 29u - __clz(2u * d - 1u);
#else
    uint32_t lg = 3;
    while ((1ull << lg) < 2ull * d) ++lg;
    return lg - 3;
#endif
}

__host__ __device__ __forceinline__ uint32_t hash_buckets(uint32_t d) {
    return d ? (1u << hash_log2_buckets(d)) : 0u;
}

__device__ __forceinline__ uint32_t hash_bucket(uint32_t u, uint32_t lg) {
    return lg ? (u * 0x9E3779B1u) >> (32 - lg) : 0u;
}

// One probe of a bucket already in registers: 1 hit, 0 miss, -1 continue with
// the next bucket (slots fill in order, so a free last slot ends the chain).
__device__ __forceinline__ int bucket_lookup(const uint4& x, const uint4& y, uint32_t u) {
    if (x.x == u || x.y == u || x.z == u || x.w == u || y.x == u || y.y == u || y.z == u ||
        y.w == u)
        return 1;
    return y.w == kHashEmpty ? 0 : -1;
}

__device__ __forceinline__ bool member(const DevGraph& g, uint32_t d, uint32_t hoff, uint32_t u) {
    if (d == 0) return false;
    const uint32_t lg = hash_log2_buckets(d);
    const uint32_t mask = (1u << lg) - 1u;
    uint32_t b = hash_bucket(u, lg);
    for (;;) {
        const uint4* p = reinterpret_cast<const uint4*>(g.hslots + 8ull * (hoff + b));
        const int r = bucket_lookup(__ldg(p), __ldg(p + 1), u);
        if (r >= 0) return r != 0;
        b = (b + 1) & mask;
    }
}

}  // namespace dwb
