// dw_walk_kernel.cuh -- the walk hot path: K1 eRJS, K2 eRVS, K3 adaptive walker loop.
//
// Header-only so that both the library (dw_walk.cu: the builtin models) and
// NVRTC (dw_dsl.cu: DSL models compiled at run time) instantiate the same
// kernel template.
//
// One persistent kernel per run.  Each lane owns one walker at a time and
// keeps its WalkerState (walk_state.hpp:13-40) in registers for all steps;
// lanes claim walkers from a global queue with one warp-aggregated atomic
// (the run_queries scheduler, runtime.cpp:209-211).
//
// Cost model.  Every random gather on B200 moves a whole 128 B L2 line from
// HBM, whatever its size (tools/gather_probe.cu: ~3.7e10 random lines/s at
// ~4.7 TB/s of DRAM traffic).  The kernel is therefore designed around the
// NUMBER of random requests per walker-step, not their bytes:
//   * fat edge records (dw_common.cuh FatRec): an accepted trial's record
//     carries its target's row begin, degree, hash-set base, aggregates and
//     the return-edge range, so a step needs no node-record gather;
//   * free rejections: a trial whose y is >= the model's non-return maximum
//     and whose index lies outside the return-edge range is rejected without
//     gathering its edge -- about half of node2vec (0.5, 2) trials;
//   * no speculative waste beyond a ring of kRing outstanding trials.
//
// Latency structure.  A walk step is a chain of dependent random loads and
// lanes of a warp need different numbers of them, so the walker loop is a
// per-lane state machine in which every lane advances one memory phase per
// iteration:
//     A  each lane issues the gathers its phase needs as cp.async (LDGSTS)
//        into its own shared-memory landing slots
//     B  cp.async.wait_all
//     C  each lane consumes its slots and picks its next phase
// Phases:
//   NODE   one 32 B node record (the walker's first step, or every step on
//          the slim layout); cost-model decision (decide_sampler,
//          cost_model.hpp:46-56).
//   TRIAL  eRJS (samplers.hpp:145-178).  Philox is a counter RNG, so trial t's
//          (x, y) is known without running the trials before it: the lane
//          generates trials, rejects the free ones on the spot and queues
//          the others (edge record gathers) in a ring; queued trials are
//          judged in trial order.  A trial whose outcome hinges on the
//          node2vec/PR2 membership test (y between the two candidate weights)
//          parks at the ring head while one hash bucket is probed.
//   FETCH  the fat record of the edge an eRVS step chose.
//   VREC / VMEMB   eRVS on short rows (samplers.hpp:65-137), one neighbour per
//          iteration, exactly the reference's sequential jump logic.
//   COOP   rows >= kCoopMinDegree are handed to the whole warp through a
//          ballot (FlexiWalker's mixed mode): 32 lanes load a chunk and
//          resolve 32 weights in parallel, then the A-ExpJ jump scan runs
//          warp-uniformly over the chunk with shuffles.
// Paths, counters and draw counts equal the sequential reference on the same
// Philox stream (tests/test_gpu_parity.py).
#pragma once
#ifndef __CUDACC_RTC__
#include <cfloat>
#endif

#include "dw_walk.cuh"

namespace dwb {

#ifndef DW_MIN_BLOCKS
#define DW_MIN_BLOCKS 3
#endif
#ifndef DW_DONE_MODE
#define DW_DONE_MODE 0
#endif
#ifndef DW_RING
#define DW_RING 2
#endif
#ifndef DW_GEN
#define DW_GEN 4
#endif
#ifndef DW_THREADS
#define DW_THREADS 256
#endif
constexpr int kThreads = DW_THREADS;
constexpr uint32_t kRing = DW_RING;  // queued trials per lane (power of two)
constexpr uint32_t kGen = DW_GEN;    // Philox blocks per lane per iteration
static_assert((kRing & (kRing - 1)) == 0, "kRing must be a power of two");
constexpr uint32_t kCoopMinDegree = 64;
#ifndef DW_EBATCH
#define DW_EBATCH 8
#endif
#ifndef DW_EWAIT
#define DW_EWAIT 10
#endif
// short-row eRVS: rows of <= kEBatchMaxDeg neighbours collect their weights in
// the lane's first ring slot (6 doubles) and scan in batches of kEBatch lanes
constexpr uint32_t kEBatchMaxDeg = 6;
constexpr uint32_t kEBatch = DW_EBATCH;
constexpr uint32_t kEWait = DW_EWAIT;
constexpr unsigned kFull = 0xFFFFFFFFu;
typedef unsigned long long ull;

// P_DONE: the walk just ended; the next iteration's refill site books it
// (one code site for the direct compact output's chunk accounting)
enum Phase : uint32_t { P_IDLE = 0, P_NODE, P_TRIAL, P_FETCH, P_VREC, P_VMEMB, P_COOP, P_EMATH, P_CJS, P_DONE };

// Warp-cooperative eRJS for models whose bounds can be far above the typical
// weight (second-order PageRank: thousands of trials on hub rows, SURVEY
// Appendix A).  A lane whose step has run kCjsMin trials without acceptance
// hands the step to the warp: 32 consecutive trials per round, judged in
// parallel, the first accepted one (in trial order) wins -- the same trial
// the sequential loop would accept, with the same counters.  A launch is
// otherwise bound by its slowest walker: at s20, a quarter of the config-4
// walkers took 74 % of the full run's time (tools/tail_probe.py).
template <class M> struct CoopErjs { static constexpr bool value = false; };
template <bool W> struct CoopErjs<Pr2Model<W>> { static constexpr bool value = true; };
#ifndef DW_CJS_MIN
#define DW_CJS_MIN 128
#endif
constexpr uint32_t kCjsMin = DW_CJS_MIN;
// relative band around the f32 row sum of a compact record inside which the
// exact node record decides: ModelParams::fat32_band (1e-6; DW_FAT32_BAND in
// the environment widens it, which tests use to force that path)
// per-lane 64-bit counters kept in shared memory (updated per walker, per
// eRVS neighbour or per rare event): eRJS trials, single-shot eRVS trials,
// eRVS reads and draws, algorithmic bytes / 4, cap fallbacks, dead ends,
// query errors, queries.  A plain shared-memory add per update: no atomics
// and no overflow branch inside the walk loop (the 64-bit shared atomics
// those need compile to CAS loops, ~580 cold instructions that crowded the
// loop's instruction cache).  Summed per block at kernel end.
// The first LC_NUM64 grow fast (reads of hub rows, trials of loose PR2
// bounds) and are 64-bit; the rest count walkers or steps and live in 32-bit
// slots whose (practically unreachable) carry goes straight to the global
// 64-bit counter.
enum LaneCounter : int {
    LC_ETRIALS = 0, LC_EREADS, LC_EDRAWS, LC_ALG4, LC_NUM64,
    LC_ETRIALS1 = LC_NUM64, LC_FALLBACKS, LC_DEADENDS, LC_QERRORS, LC_QUERIES, LC_NUM
};

__device__ __forceinline__ bool valid_w(double w) { return !(w < 0.0) && isfinite(w); }

template <class M>
__device__ __forceinline__ uint16_t edge_label(const DevGraph& g, ull e) {
    if (!M::kUsesLabels) return 0;
    return g.labels ? __ldg(g.labels + e) : (uint16_t)0;
}

__device__ __forceinline__ void raise_error(const WalkParams& p, int code, ull q) {
    if (atomicCAS(p.error, 0, code) == 0) *p.error_info = q;
}

// ---- cp.async (LDGSTS) gathers into the lane's landing slots --------------
__device__ __forceinline__ void cp16(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp4(void* smem, const void* gmem) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(s), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_wait_all() {
    asm volatile("cp.async.wait_all;\n" ::: "memory");
}

__device__ __forceinline__ const EdgeRec* pair_of(const EdgeRec* edges, ull e) {
    return edges + (e & ~1ull);  // 16 B aligned pair holding record e
}


// ---- K2 (warp form): one row, 32 lanes; all lanes call with equal args ----
// FlexiWalker's warp reservoir (samplers.hpp:65-137) without the sequential
// chain.  A row is read in chunks of 64 neighbours, two per lane (one 16 B
// load when the row starts on an even edge, two 8 B loads otherwise), the
// next chunk in flight while this one is judged.
//
// Jump form.  The reference's jump test is a running subtraction
// `skip -= w; if (skip <= 0)`, rounded after every neighbour.  Rounding makes
// it sequential, but its sign can be decided from a parallel prefix sum:
// for the chain started at s0 over m weights, the rounded chain C_j and the
// real value S_j = s0 - (w_seg + ... + w_j) differ by at most
// gamma_m (s0 + W_j) (recursive summation of non-negative terms), and the
// warp's prefix sums (depth <= 7 roundings per chunk, carried across chunks)
// differ from S_j by a bound of the same form.  With A_j the warp's value and
// E_j = 1.1 u ((3 m + 8)(s0 + P_j) + |A_j|) (+ a subnormal floor), A_j > E_j
// proves C_j > 0 and A_j < -E_j proves C_j <= 0 (ervs_bound below).  So a
// chunk with no element inside its band costs one warp scan, and the first
// element whose band reaches 0 is the crossing whenever A_j < -E_j.  Only
// when the band straddles 0 (probability ~ m^2 u s0 / w per crossing) is the
// chain replayed exactly, sequentially, from the segment start (ervs_replay),
// and its exact value restarts the bound.  Jumps (new key, new threshold)
// are warp-uniform and rare (~ln d per row).  Draws, their order and the
// kept neighbour are the reference's; the outcome is identical, not
// approximately equal.
//
// No-jump form.  Every neighbour draws its key (draw idx0 + i; neighbours 2k
// and 2k+1 share one Philox block, because idx0 is even) and the keys merge
// with a shuffle arg-max (lower index on ties).
template <class M>
__device__ __forceinline__ double ervs_weight(const M& m, const Step& S, const DevGraph& g,
                                              uint32_t phoff, uint32_t u, float h, uint16_t lab) {
    const WeightCase wc = m.weight(S, u, h, lab);
    if (!M::kSecondOrder || !wc.needs_member) return wc.w;
    if ((double)h > S.hin) return wc.w_out;  // above the triangle bound: not in N(prev)
    return member(g, S.prev_degree, phoff, u) ? wc.w_in : wc.w_out;
}

// Membership by merging cur's sorted row with prev's sorted row
// (graph.cpp:114-118 has_edge, answered a chunk at a time).  The warp holds a
// window of 32 of prev's neighbours (one coalesced 256 B load) and slides it
// forward with the chunks: a chunk whose targets all lie below the window's
// first id needs no test; otherwise each lane binary-searches its two targets
// in the window with shuffles, and the window advances until it covers the
// chunk's last target.  Over a row scan the window reads prev's row at most
// once (plus one binary search to place it), instead of one hash-bucket
// probe per neighbour; the answers are the same.  Used when prev's row begin
// is known (the reservoir-only modes keep it per lane).
constexpr ull kNoRow = ~0ull;
struct PrevWindow {
    ull pbegin;                 // prev's row
    uint32_t pdeg;
    uint32_t pp;                // window = prev's neighbours [pp, pp + 32)
    uint32_t v;                 // this lane's entry (kInvalid past the row)
    uint32_t vfirst, vlast;     // the window's first and last entries
};
__device__ __forceinline__ void win_load(PrevWindow& w, const DevGraph& g) {
    const uint32_t lane = threadIdx.x & 31;
    w.v = w.pp + lane < w.pdeg ? load_col(g.edges + w.pbegin + w.pp + lane) : kInvalid;
    w.vfirst = __shfl_sync(kFull, w.v, 0);
    w.vlast = __shfl_sync(kFull, w.v, 31);
}
// place the window at the first of prev's neighbours >= u
__device__ __forceinline__ void win_seek(PrevWindow& w, const DevGraph& g, uint32_t u) {
    uint32_t at = 0;
    for (uint32_t len = w.pdeg; len > 1;) {  // branchless lower_bound
        const uint32_t half = len >> 1;
        if (load_col(g.edges + w.pbegin + at + half) < u) at += half;
        len -= half;
    }
    if (w.pdeg && load_col(g.edges + w.pbegin + at) < u) ++at;
    w.pp = at;
    win_load(w, g);
}
// is u one of the window's entries (sorted ascending)?
__device__ __forceinline__ bool win_has(const PrevWindow& w, uint32_t u) {
    uint32_t lo = 0;
#pragma unroll
    for (uint32_t step = 16; step; step >>= 1)
        if (__shfl_sync(kFull, w.v, lo + step - 1) < u) lo += step;
    return __shfl_sync(kFull, w.v, lo) == u;
}

// The row is read as 16 B aligned pairs: aligned position q holds neighbour
// q - off with off = begin & 1 (edge arrays are padded to even length, so the
// last pair is in bounds).  Ids of positions outside the row are kInvalid.
struct EPair {
    uint32_t u0, u1;
    float h0, h1;
    uint32_t lab;  // label(q) | label(q + 1) << 16
};
__device__ __forceinline__ EPair ervs_pair(uint4 v, uint32_t lab, uint32_t i0, uint32_t d) {
    EPair r{kInvalid, kInvalid, __uint_as_float(v.y), __uint_as_float(v.w), lab};
    if (i0 < d) r.u0 = v.x;        // i0 = q - off wraps to 2^32 - 1 before the row
    if (i0 + 1 < d) r.u1 = v.z;
    return r;
}
template <class M>
__device__ __forceinline__ EPair ervs_load_pair(const DevGraph& g, ull abase, uint32_t q,
                                                uint32_t npos, uint32_t off, uint32_t d) {
    const uint32_t i0 = q - off;
    if (q >= npos) return EPair{kInvalid, kInvalid, 0.f, 0.f, 0u};
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(g.edges + abase + q));
    uint32_t lab = 0;
    if (M::kUsesLabels && g.labels) lab = __ldg(reinterpret_cast<const uint32_t*>(g.labels + abase + q));
    return ervs_pair(v, lab, i0, d);
}

// ---- TMA (cp.async.bulk) staging of a row's chunks ------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(ull* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(ull* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
                 "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(ull* bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    } while (!done);
}
// bytes from global to this CTA's shared memory, completion counted on bar
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, ull* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// arm a stage's mbarrier with `bytes` and issue its bulk copy, with the
// shared-memory addresses already in the shared window (one asm block)
__device__ __forceinline__ void bulk_stage(uint32_t dst, uint32_t bar, const void* src,
                                           uint32_t bytes) {
    asm volatile(
        "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%1], %3;\n"
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%2], %3, [%1];\n"
        ::"r"(dst), "r"(bar), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait_u32(uint32_t bar, uint32_t parity) {
    uint32_t done = 0;
    do {
        asm volatile(
            "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
            " selp.u32 %0, 1, 0, p;\n}\n"
            : "=r"(done) : "r"(bar), "r"(parity) : "memory");
    } while (!done);
}
// order this thread's earlier generic shared-memory accesses before later
// async-proxy (bulk copy) writes to the same bytes
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

// A warp's bulk-copy ring: kTmaStages chunks of 64 neighbours (512 B) in
// flight, each landing in its own shared-memory stage and counted on its own
// mbarrier; parity bits persist across calls (the ring is reused by every
// long row the warp scans).
constexpr uint32_t kTmaStages = 3;
struct TmaRing {
    uint4* stage0;             // stage s = stage0 + s * stride (32 x 16 B each)
    uint32_t stride;           // in uint4 (no array: a dynamically indexed
                               // pointer array would live in local memory)
    ull* bar;                  // [kTmaStages]
    uint32_t* parity;          // bit s: parity of stage s's next completion
};

#ifndef DW_LAB_SCREEN
#define DW_LAB_SCREEN 1
#endif
// models whose weight is h when the edge label equals schema[step] and 0
// otherwise (MetaPath, models.hpp:95-118): their trials can be screened on
// the packed labels
template <class M> struct LabelScreen { static constexpr bool value = false; };
template <bool W> struct LabelScreen<MetaPathModel<W>> { static constexpr bool value = true; };
#ifndef DW_ERVS_TMA
#define DW_ERVS_TMA 1  // reservoir-only modes stage long rows through a bulk-copy ring
#endif
#ifndef DW_ERVS_SEQ
#define DW_ERVS_SEQ 0  // 1: the round-1 sequential shuffle chain (A/B experiments)
#endif

// The exact chain (samplers.hpp:86-90) from neighbour `seg` (whose weight is
// the first subtracted) with remaining skip s, up to neighbour `end`
// (exclusive): returns the crossing neighbour, or kInvalid with *s_out the
// chain's value after neighbour end - 1.  Weights were validated by the caller.
template <class M>
__device__ __noinline__ uint32_t ervs_replay(const ModelParams& mp, Step S, const DevGraph& g,
                                             ull begin, uint32_t phoff, uint32_t seg, double s,
                                             uint32_t end, double* s_out) {
    M m(mp);
    m.prepare(S);
    const int lane = threadIdx.x & 31;
    for (uint32_t b = seg; b < end; b += 32) {
        const uint32_t i = b + lane;
        double w = 0.0;
        if (i < end) {
            const EdgeRec er = load_edge(g.edges + begin + i);
            w = ervs_weight(m, S, g, phoff, er.col, er.h, edge_label<M>(g, begin + i));
        }
        const uint32_t n = end - b < 32u ? end - b : 32u;
        for (uint32_t j = 0; j < n; ++j) {
            const double wj = __shfl_sync(kFull, w, j);
            if (wj == 0.0) continue;
            s -= wj;
            if (s <= 0.0) return b + j;
        }
    }
    *s_out = s;
    return kInvalid;
}

// |rounded chain - warp prefix value| bound of the chunk (see above)
struct ErvsBound {
    double k;    // 1.1 u (3 m + 8)
    double lo;   // subnormal floor
};
__device__ __forceinline__ ErvsBound ervs_bound(uint32_t m, double slack) {
    const double u = 0x1.0p-53;
    return ErvsBound{1.1 * u * (3.0 * (double)m + 8.0) * slack, ((double)m + 16.0) * 0x1.0p-1060};
}

template <class M, bool NOJUMP, bool TMA>
__device__ __forceinline__ int ervs_warp(const ModelParams& mp, Step S, const WalkerKey key,
                                         const PhiloxKeys& rk,
                                         const DevGraph& g, ull begin, uint32_t phoff, ull idx0,
                                         uint32_t* next, uint32_t* nidx, ull* draws,
                                         const TmaRing& ring, ull pbegin = kNoRow) {
    M m(mp);
    m.prepare(S);
    const int lane = threadIdx.x & 31;
    const uint32_t d = S.degree;
    const uint32_t off = (uint32_t)(begin & 1);
    const ull abase = begin - off;               // 16 B aligned start of the row
    const uint32_t npos = (d + off + 1) & ~1u;   // aligned positions covering the row
    const uint32_t nch = (npos + 63) / 64;
    ull idx = idx0;                // next draw (warp-uniform)
    double bkey = -DBL_MAX;        // best log key
    uint32_t best = kInvalid, bi = 0;
    // jump chain: remaining skip s (valid when `have`), exact start value s0 at
    // neighbour seg
    bool have = false;
    double s = 0.0, s0 = 0.0;
    uint32_t seg = 0;
    ErvsBound eb{0.0, 0.0};  // the segment's rounding band (m = neighbours left in the row)
    int status = 0;
    // chunk c = aligned positions [64c, 64c + 64): bytes of its bulk copy
    auto chunk_bytes = [&](uint32_t c) { return min(64u, npos - 64u * c) * 8u; };
    // membership by merging with prev's sorted row when its begin is known
    // and prev is at most half as long as cur (about one window pass per
    // chunk at most; denser windows cost more shuffles than hash probes)
    const bool merge = M::kSecondOrder && !M::kUsesLabels && S.prev != kInvalid &&
                       pbegin != kNoRow && S.prev_degree > 0 && 2u * S.prev_degree <= d;
    PrevWindow pw{pbegin, S.prev_degree, 0u, kInvalid, kInvalid, kInvalid};
    uint32_t par = 0;
    EPair nx{};
    // the ring's shared-window addresses, formed once per row
    const uint32_t stg0 = TMA ? smem_u32(ring.stage0) : 0u, bar0 = TMA ? smem_u32(ring.bar) : 0u;
    const uint32_t stgb = ring.stride * 16u;  // bytes between stages
    if (TMA) {
        par = *ring.parity;
        if (lane == 0) {
            // earlier generic writes to the stages (other phases' landing
            // slots) before the bulk copies' async-proxy writes
            fence_proxy_async();
            for (uint32_t c = 0; c < kTmaStages && c < nch; ++c)
                bulk_stage(stg0 + c * stgb, bar0 + 8u * c, g.edges + abase + 64ull * c,
                           chunk_bytes(c));
        }
    } else {
        nx = ervs_load_pair<M>(g, abase, 2u * lane, npos, off, d);
    }
    uint32_t c = 0;
    for (; c < nch; ++c) {
        const uint32_t base = 64u * c;           // aligned position of the chunk
        const uint32_t q = base + 2u * lane;
        const uint32_t i0 = q - off;             // this lane's first neighbour
        EPair cp;
        if (TMA) {
            const uint32_t st = c % kTmaStages;
            mbar_wait_u32(bar0 + 8u * st, (par >> st) & 1u);
            par ^= 1u << st;
            const uint4 v = ring.stage0[st * ring.stride + lane];
            cp = q < npos ? ervs_pair(v, 0u, i0, d) : EPair{kInvalid, kInvalid, 0.f, 0.f, 0u};
            // every lane's read of the stage precedes its refill (the reads
            // have completed: their values are consumed above)
            __syncwarp();
            if (lane == 0 && c + kTmaStages < nch)  // refill the stage just read
                bulk_stage(stg0 + st * stgb, bar0 + 8u * st,
                           g.edges + abase + 64ull * (c + kTmaStages), chunk_bytes(c + kTmaStages));
        } else {
            cp = nx;
            if (base + 64 < npos) nx = ervs_load_pair<M>(g, abase, q + 64, npos, off, d);
        }
        double w0 = 0.0, w1 = 0.0;
        if (M::kSecondOrder && merge) {
            // the chunk's targets span [ulo, uhi] (the row is sorted)
            const uint32_t cb = base > off ? base - off : 0u;
            const uint32_t ce = base + 64 - off < d ? base + 64 - off : d;
            const uint32_t lf = (cb + off - base) >> 1, ll = (ce - 1 + off - base) >> 1;
            const uint32_t ulo = __shfl_sync(kFull, ((cb + off - base) & 1) ? cp.u1 : cp.u0, lf);
            const uint32_t uhi = __shfl_sync(kFull, ((ce - 1 + off - base) & 1) ? cp.u1 : cp.u0, ll);
            if (c == 0) win_seek(pw, g, ulo);
            while (pw.vlast < ulo && pw.pp + 32 < pw.pdeg) {
                pw.pp += 32;
                win_load(pw, g);
            }
            bool in0 = false, in1 = false;
            if (pw.vfirst <= uhi) {
                for (;;) {
                    in0 |= win_has(pw, cp.u0);
                    in1 |= win_has(pw, cp.u1);
                    if (pw.vlast >= uhi || pw.pp + 32 >= pw.pdeg) break;
                    pw.pp += 32;
                    win_load(pw, g);
                }
            }
            if (cp.u0 != kInvalid) {
                const WeightCase wc = m.weight(S, cp.u0, cp.h0, 0);
                w0 = !wc.needs_member ? wc.w : (in0 ? wc.w_in : wc.w_out);
            }
            if (cp.u1 != kInvalid) {
                const WeightCase wc = m.weight(S, cp.u1, cp.h1, 0);
                w1 = !wc.needs_member ? wc.w : (in1 ? wc.w_in : wc.w_out);
            }
        } else {
            if (cp.u0 != kInvalid) w0 = ervs_weight(m, S, g, phoff, cp.u0, cp.h0, (uint16_t)cp.lab);
            if (cp.u1 != kInvalid) w1 = ervs_weight(m, S, g, phoff, cp.u1, cp.h1, (uint16_t)(cp.lab >> 16));
        }
        // weights valid by construction (mp.pos_weights) need no vote
        if (!mp.pos_weights &&
            __any_sync(kFull, (cp.u0 != kInvalid && !valid_w(w0)) ||
                                  (cp.u1 != kInvalid && !valid_w(w1)))) {
            status = -kDevBadWeight;
            break;
        }
        if (NOJUMP) {
            double lk = -DBL_MAX;
            uint32_t src = kInvalid, cand = kInvalid;
            if (cp.u0 != kInvalid || cp.u1 != kInvalid) {
                // draws idx0 + i0 and idx0 + i0 + 1: one Philox block when
                // i0 is valid and idx0 + i0 is even (idx0 is even: rows
                // starting on an even edge); i0 wraps to 2^32 - 1 before
                // the row, so each draw index is formed from its own element
                const ull d0 = idx0 + (ull)i0, d1 = idx0 + (ull)(uint32_t)(i0 + 1u);
                ull r0 = 0, r1;
                if (cp.u0 != kInvalid && !(d0 & 1)) {
                    const U4 blk = philox4x32_10_rk(U4{(uint32_t)(d0 >> 1), key.step, key.q0, key.q1}, rk);
                    r0 = lo64(blk);
                    r1 = hi64(blk);
                } else {
                    if (cp.u0 != kInvalid) r0 = walker_draw(key, rk, d0);
                    r1 = walker_draw(key, rk, d1);
                }
                // A key can only matter if it beats the best key of the
                // earlier chunks (ties keep the earlier neighbour).  Screen
                // with a single-precision log first: log(u) <= La + dl with
                // La = ln2 * __log2f((float)u) (the float conversion and
                // MUFU.LG2 err by < 2e-5 + 1e-6 |La| in the log), so a key
                // with La + dl <= bkey * w loses for certain and skips the
                // double log and division; the keys that remain are exact.
                const double ua = open01(r0), ub = open01(r1);
                auto may_win = [&](double u, double w) {
                    if (best == kInvalid) return true;
                    const float la = 0.69314718f * __log2f((float)u);
                    const double dl = 2e-5 + 1e-6 * fabs((double)la);
                    const double bw = bkey * w;
                    return (double)la + dl > bw - 1e-12 * fabs(bw);
                };
                if (cp.u0 != kInvalid && w0 != 0.0 && may_win(ua, w0)) {
                    lk = log(ua) / w0;
                    src = i0;
                    cand = cp.u0;
                }
                if (cp.u1 != kInvalid && w1 != 0.0 && may_win(ub, w1)) {
                    const double l1 = log(ub) / w1;
                    if (src == kInvalid || l1 > lk) {
                        lk = l1;
                        src = i0 + 1;
                        cand = cp.u1;
                    }
                }
            }
            if (!__any_sync(kFull, src != kInvalid)) continue;  // nothing can beat bkey
#pragma unroll
            for (int o = 16; o; o >>= 1) {
                const double olk = __shfl_xor_sync(kFull, lk, o);
                const uint32_t osrc = __shfl_xor_sync(kFull, src, o);
                const uint32_t ocand = __shfl_xor_sync(kFull, cand, o);
                const bool take = osrc != kInvalid &&
                                  (src == kInvalid || olk > lk || (olk == lk && osrc < src));
                if (take) {
                    lk = olk;
                    src = osrc;
                    cand = ocand;
                }
            }
            if (src != kInvalid && (best == kInvalid || lk > bkey)) {
                bkey = lk;
                best = cand;
                bi = src;
            }
            continue;
        }
        // neighbours [cbeg, cend) are this chunk's
        const uint32_t cbeg = base > off ? base - off : 0u;
        const uint32_t cend = base + 64 - off < d ? base + 64 - off : d;
        // the lane that holds neighbour i, and which half
        auto owner = [&](uint32_t i) { return (int)((i + off - base) >> 1); };
        auto odd = [&](uint32_t i) { return ((i + off - base) & 1u) != 0; };
#if DW_ERVS_SEQ
        {
            for (uint32_t j = cbeg; j < cend; ++j) {
                const double wj = __shfl_sync(kFull, odd(j) ? w1 : w0, owner(j));
                const uint32_t uj = __shfl_sync(kFull, odd(j) ? cp.u1 : cp.u0, owner(j));
                if (wj == 0.0) continue;
                if (best == kInvalid) {
                    bkey = log(open01(walker_draw(key, rk, idx++))) / wj;
                    best = uj;
                    bi = j;
                    continue;
                }
                if (!have) {
                    s = log(open01(walker_draw(key, rk, idx++))) / bkey;
                    have = true;
                }
                s -= wj;
                if (s <= 0.0) {
                    const double floor_u = exp(wj * bkey);
                    const double uu = floor_u + open01(walker_draw(key, rk, idx++)) * (1.0 - floor_u);
                    const double lk = log(uu) / wj;
                    if (lk > bkey) {
                        bkey = lk;
                        best = uj;
                        bi = j;
                    }
                    have = false;
                }
            }
            continue;
        }
#endif
        uint32_t pos = cbeg;  // first neighbour of the chunk not yet consumed
        for (;;) {
            if (!have) {
                // the next positive weight: the first key, or the next threshold
                const bool nz0 = w0 != 0.0 && i0 >= pos, nz1 = w1 != 0.0 && i0 + 1 >= pos;
                const unsigned bal = __ballot_sync(kFull, nz0 || nz1);
                if (!bal) break;
                const int f = __ffs(bal) - 1;
                const uint32_t fe = __shfl_sync(kFull, nz0 ? i0 : i0 + 1, f);
                const double fw = __shfl_sync(kFull, nz0 ? w0 : w1, f);
                const uint32_t fu = __shfl_sync(kFull, nz0 ? cp.u0 : cp.u1, f);
                const double lr = log(open01(walker_draw(key, rk, idx++)));
                if (best == kInvalid) {  // samplers.hpp:82-85
                    bkey = lr / fw;
                    best = fu;
                    bi = fe;
                    pos = fe + 1;
                    continue;
                }
                s = s0 = lr / bkey;  // samplers.hpp:86-89
                eb = ervs_bound(d - fe, mp.ervs_slack);  // m <= d - seg for the whole segment
                seg = fe;
                have = true;
                pos = fe;
            }
            const double x0 = i0 >= pos ? w0 : 0.0, x1 = i0 + 1 >= pos ? w1 : 0.0;
            const double p1 = x0 + x1;
            // The chain never increases (w >= 0), so a chunk whose last value
            // is provably positive has no crossing: test that first with a
            // butterfly sum (every term through <= 6 roundings), and run the
            // per-neighbour scan only for the chunk that may cross.
            if (s > 0.0 && s < DBL_MAX) {
                double tot = p1;
#pragma unroll
                for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(kFull, tot, o);
                const double A = s - tot;
                if (A > eb.k * (s0 + tot) + 1.1 * 0x1.0p-53 * fabs(A) + eb.lo) {
                    s = A;
                    break;
                }
            }
            // prefix sums of the weights from pos on (two per lane, then a
            // Kogge-Stone warp scan)
            double inc = p1;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const double t = __shfl_up_sync(kFull, inc, o);
                if (lane >= o) inc += t;
            }
            double exc = __shfl_up_sync(kFull, inc, 1);
            if (lane == 0) exc = 0.0;
            const double P0 = exc + x0, P1 = exc + p1;
            uint32_t cross = kInvalid;
            bool decided = false;
            if (s > 0.0 && s < DBL_MAX) {
                const double A0 = s - P0, A1 = s - P1;
                const double E0 = eb.k * (s0 + P0) + 1.1 * 0x1.0p-53 * fabs(A0) + eb.lo;
                const double E1 = eb.k * (s0 + P1) + 1.1 * 0x1.0p-53 * fabs(A1) + eb.lo;
                const bool may0 = x0 != 0.0 && !(A0 > E0), may1 = x1 != 0.0 && !(A1 > E1);
                const unsigned bal = __ballot_sync(kFull, may0 || may1);
                if (!bal) {  // no crossing in this chunk
                    s = s - __shfl_sync(kFull, inc, 31);
                    break;
                }
                const int f = __ffs(bal) - 1;
                const bool sure = __shfl_sync(kFull, may0 ? (A0 < -E0) : (A1 < -E1), f);
                if (sure) {
                    cross = __shfl_sync(kFull, may0 ? i0 : i0 + 1, f);
                    decided = true;
                }
            }
            if (!decided) {
                // band straddles 0 (or s is not finite): the exact chain
                double sx = 0.0;
                cross = ervs_replay<M>(mp, S, g, begin, phoff, seg, s0, cend, &sx);
                if (cross == kInvalid) {  // exact value at the chunk end restarts the bound
                    s = s0 = sx;
                    eb = ervs_bound(d - cend, mp.ervs_slack);
                    seg = cend;
                    break;
                }
            }
            // replacement at `cross` (samplers.hpp:90-99)
            const double wj = __shfl_sync(kFull, odd(cross) ? w1 : w0, owner(cross));
            const uint32_t uj = __shfl_sync(kFull, odd(cross) ? cp.u1 : cp.u0, owner(cross));
            const double floor_u = exp(wj * bkey);
            const double uu = floor_u + open01(walker_draw(key, rk, idx++)) * (1.0 - floor_u);
            const double lk = log(uu) / wj;
            if (lk > bkey) {
                bkey = lk;
                best = uj;
                bi = cross;
            }
            have = false;
            pos = cross + 1;
        }
    }
    if (TMA) {
        // drain the copies still in flight (an early exit leaves up to
        // kTmaStages - 1 of them), so the stages and parities stay consistent
        for (uint32_t k = c + 1; k < nch && k <= c + kTmaStages; ++k) {
            const uint32_t st = k % kTmaStages;
            mbar_wait(&ring.bar[st], (par >> st) & 1u);
            par ^= 1u << st;
        }
        __syncwarp();
        if (lane == 0) *ring.parity = par;
        __syncwarp();
    }
    if (status) return status;
    *next = best;
    *nidx = bi;
    *draws = NOJUMP ? (ull)d : idx - idx0;
    return 0;
}

#ifndef DW_PR2_PAR
#define DW_PR2_PAR 1
#endif
// The parallel form out of line, for models whose adaptive runs scan hub rows
// often (PR2: cap overruns and tier-2 hand-offs), without growing their
// eRJS loop's register set
template <class M, bool NOJUMP>
__device__ __noinline__ int ervs_warp_cold(const ModelParams& mp, Step S, const WalkerKey key,
                                           const PhiloxKeys& rk, const DevGraph& g, ull begin,
                                           uint32_t phoff, ull idx0, uint32_t* next,
                                           uint32_t* nidx, ull* draws) {
    return ervs_warp<M, NOJUMP, false>(mp, S, key, rk, g, begin, phoff, idx0, next, nidx, draws,
                                       TmaRing{});
}

// Round-1 warp form: 32 neighbours per chunk and the jump chain run
// sequentially through shuffles.  Kept for the modes in which whole-row
// scans are rare (adaptive, force-erjs: cap fallbacks and adaptive eRVS
// decisions on rows of >= 64), whose loops sit at the register and
// instruction-cache limit (the parallel form adds ~14 live registers).
template <class M, bool NOJUMP>
__device__ __forceinline__ int ervs_warp_seq(const ModelParams& mp, Step S, const WalkerKey key,
                                      const PhiloxKeys& rk,
                                      const DevGraph& g, ull begin, uint32_t phoff, ull idx0,
                                      uint32_t* next, uint32_t* nidx, ull* draws) {
    M m(mp);
    m.prepare(S);
    const int lane = threadIdx.x & 31;
    ull idx = idx0;
    double best_log_key = -DBL_MAX;
    uint32_t best = kInvalid, bi = 0;
    double skip = 0.0;
    bool have = false;
    // software pipeline: chunk c+1's records load while chunk c is judged
    EdgeRec nxt{kInvalid, 0.f};
    uint16_t nlab = 0;
    if ((uint32_t)lane < S.degree) {
        nxt = load_edge(g.edges + begin + lane);
        nlab = edge_label<M>(g, begin + lane);
    }
    for (uint32_t base = 0; base < S.degree; base += 32) {
        const uint32_t i = base + lane;
        const bool in = i < S.degree;
        const EdgeRec er = nxt;
        const uint16_t lab = nlab;
        if (i + 32 < S.degree) {
            nxt = load_edge(g.edges + begin + i + 32);
            nlab = edge_label<M>(g, begin + i + 32);
        }
        double w = 0.0;
        if (in) {
            const WeightCase wc = m.weight(S, er.col, er.h, lab);
            w = (!M::kSecondOrder || !wc.needs_member)
                    ? wc.w
                    : (member(g, S.prev_degree, phoff, er.col) ? wc.w_in : wc.w_out);
        }
        if (__any_sync(kFull, in && !valid_w(w))) return -kDevBadWeight;
        if (NOJUMP) {
            // every neighbour draws its own key (draw idx0 + i), zero weights included
            double lk = -DBL_MAX;
            int has = 0;
            if (in) {
                const double u = open01(walker_draw(key, rk, idx0 + i));
                if (w != 0.0) {
                    lk = log(u) / w;
                    has = 1;
                }
            }
            int src = lane;
#pragma unroll
            for (int off = 16; off; off >>= 1) {
                const double olk = __shfl_xor_sync(kFull, lk, off);
                const int ohas = __shfl_xor_sync(kFull, has, off);
                const int osrc = __shfl_xor_sync(kFull, src, off);
                const bool take = ohas && (!has || olk > lk || (olk == lk && osrc < src));
                if (take) {
                    lk = olk;
                    has = ohas;
                    src = osrc;
                }
            }
            const uint32_t cand = __shfl_sync(kFull, er.col, src);
            if (has && (best == kInvalid || lk > best_log_key)) {
                best_log_key = lk;
                best = cand;
                bi = base + src;
            }
        } else {
            const uint32_t n = S.degree - base < 32u ? S.degree - base : 32u;
            for (uint32_t j = 0; j < n; ++j) {
                const double wj = __shfl_sync(kFull, w, j);
                const uint32_t uj = __shfl_sync(kFull, er.col, j);
                if (wj == 0.0) continue;
                if (best == kInvalid) {
                    best_log_key = log(open01(walker_draw(key, rk, idx++))) / wj;
                    best = uj;
                    bi = base + j;
                    continue;
                }
                if (!have) {
                    skip = log(open01(walker_draw(key, rk, idx++))) / best_log_key;
                    have = true;
                }
                skip -= wj;
                if (skip <= 0.0) {
                    const double floor_u = exp(wj * best_log_key);
                    const double u = floor_u + open01(walker_draw(key, rk, idx++)) * (1.0 - floor_u);
                    const double lk = log(u) / wj;
                    if (lk > best_log_key) {
                        best_log_key = lk;
                        best = uj;
                        bi = base + j;
                    }
                    have = false;
                }
            }
        }
    }
    *next = best;
    *nidx = bi;
    *draws = NOJUMP ? (ull)S.degree : idx - idx0;
    return 0;
}

// ---- K2 (lane form): one neighbour of the reservoir scan ------------------
// samplers.hpp:78-102 (jump) / 122-133 (no jump).  Kept out of line: it holds
// the log/exp code, which the hot eRJS loop never needs.
struct ErvsState {
    double best_key, skip;
    ull didx;        // next draw index of this step's stream
    uint32_t best;
    uint32_t bidx;   // relative edge index of best (bits 0-30) | threshold drawn (bit 31)
};
constexpr uint32_t kHave = 0x80000000u;

template <bool NOJUMP>
__device__ __forceinline__ ErvsState ervs_visit_impl(ErvsState s, const WalkerKey& key,
                                                     const PhiloxKeys& rk, uint32_t vi,
                                                     uint32_t u, double w) {
    if (NOJUMP) {
        const double r = open01(walker_draw(key, rk, s.didx + vi));
        if (w != 0.0) {
            const double lk = log(r) / w;
            if (s.best == kInvalid || lk > s.best_key) {
                s.best_key = lk;
                s.best = u;
                s.bidx = vi;
            }
        }
        return s;
    }
    if (w == 0.0) return s;
    if (s.best == kInvalid) {
        s.best_key = log(open01(walker_draw(key, rk, s.didx++))) / w;
        s.best = u;
        s.bidx = vi;
        return s;
    }
    if (!(s.bidx & kHave)) {
        s.skip = log(open01(walker_draw(key, rk, s.didx++))) / s.best_key;
        s.bidx |= kHave;
    }
    s.skip -= w;
    if (s.skip <= 0.0) {
        const double floor_u = exp(w * s.best_key);
        const double uu = floor_u + open01(walker_draw(key, rk, s.didx++)) * (1.0 - floor_u);
        const double lk = log(uu) / w;
        s.bidx &= ~kHave;
        if (lk > s.best_key) {
            s.best_key = lk;
            s.best = u;
            s.bidx = vi;
        }
    }
    return s;
}

template <bool NOJUMP>
__device__ __forceinline__ ErvsState ervs_visit(ErvsState s, const WalkerKey key,
                                             const PhiloxKeys& rk, uint32_t vi,
                                             uint32_t u, double w) {
    return ervs_visit_impl<NOJUMP>(s, key, rk, vi, u, w);
}

// The whole jump scan (samplers.hpp:65-107) over d <= kEBatchMaxDeg weights in
// the lane's landing slot (weight j at w[(j/2) * 2 * kThreads + j%2], i.e.
// half j%2 of uint4 j/2 of the lane); returns the draw index after the scan
// and the kept neighbour's index (kInvalid when every weight is zero).
__device__ __forceinline__ ull ervs_scan_short(const double* w, uint32_t d, const WalkerKey key,
                                            const PhiloxKeys& rk,
                                            ull didx, uint32_t* bidx) {
    ErvsState s{-DBL_MAX, 0.0, didx, kInvalid, 0};
    for (uint32_t j = 0; j < d; ++j)
        s = ervs_visit_impl<false>(s, key, rk, j, 0u, w[(j >> 1) * 2 * kThreads + (j & 1)]);
    *bidx = s.best == kInvalid ? kInvalid : (s.bidx & ~kHave);
    return s.didx;
}

__device__ __forceinline__ ull warp_sum(ull v) {
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    return v;
}

// The record's 8-bit triangle bound (dw_graph.cu tri_q) as f32 bits of an
// upper bound of the props of the edges (cur -> u), u in N(prev): 0 when
// there is none, hmax when unknown (255), else hmax (q + 1) / 256 rounded up.
__device__ __forceinline__ uint32_t tri_bound(uint32_t q, float hmax) {
    if (q == 0u) return 0u;
    if (q == 255u) return __float_as_uint(hmax);
    return __float_as_uint(__fmul_ru(hmax, (float)(q + 1u)) * 0x1.0p-8f);
}

// ---- K3: adaptive walker loop (runtime.cpp:59-153 + 192-247) --------------
// Per-lane landing slots and counters, structure-of-arrays ([.][kThreads]) so
// a warp's 16 B accesses are conflict-free.
// kLc32: rows of 32-bit lane counters (LC_NUM - LC_NUM64; the direct compact
// kernels count queries per block instead, WalkSmemFlat)
template <int kLc32>
struct WalkSmemT {
    uint4 rec[kRing][3][kThreads];   // landing: fat record / slim pair in [0]
    double y[kRing][kThreads];       // y of the queued trials
    uint32_t t[kRing][kThreads];     // trial index of the queued trials
    uint4 mb[2][kThreads];           // node record / hash bucket / eRVS pair
    ull lc[LC_NUM64][kThreads];      // per-lane RunStats counters (64-bit)
    uint32_t lc32[kLc32][kThreads];  // (bounded ones)
    // path entries staged until their 32 B sector is complete: a sector is
    // written whole (two 16 B stores) instead of eight 4 B stores, so L2 never
    // evicts a partly written sector, which HBM's ECC turns into a
    // read-modify-write (single 4 B stores cost 12 % of the s24 walk);
    // slot = (entry address / 4) mod 8
    uint32_t pst[8][kThreads];
    // walker state read once per step or per iteration, kept out of registers
    // so the loop fits the register budget of 3-4 CTAs/SM without spills
    uint32_t cur[kThreads], phoff[kThreads], plg[kThreads], hoff[kThreads], cap[kThreads],
        twlo[kThreads], twcnt[kThreads], nret[kThreads];
    double bound[kThreads], mnr[kThreads];
    uint32_t qi[kThreads];           // the lane's walker: index in this launch
    // f32 bits of the current step's triangle bound (Step::hin, rounded up):
    // props of the edges (cur -> u) with u in N(prev) are <= it
    uint32_t tq[kThreads];
    ull cnt[kCNum];
    uint32_t hist[66];
    ull lct[LC_NUM];                 // block totals of the lane counters
    // reservoir-only modes: each warp's bulk-copy ring (ervs_warp, TmaRing);
    // its stages are the warp's part of ring slot 0, idle in those modes
    ull mbar[kThreads / 32][kTmaStages];
    uint32_t tmaph[kThreads / 32];
};

using WalkSmem = WalkSmemT<LC_NUM - LC_NUM64>;
// direct compact kernels (kOutFlat): + each lane's path start in the flat
// layout (p.offs[qi]) and the chunk of the walker that ended last iteration,
// booked after this iteration's gathers are issued (0xFFFF: none); room made
// by counting queries and query errors with global atomics (one per warp
// claim, one per out-of-range start) instead of per lane
struct WalkSmemFlat : WalkSmemT<LC_QERRORS - LC_NUM64> {
    ull rowb[kThreads];
    uint16_t dchunk[kThreads];
};
// DW_MIN_BLOCKS CTAs of the narrow kernels must fit one SM's 228 KB of shared
// memory, 1 KB of which each CTA reserves (one CTA less costs ~30 %)
static_assert(DW_THREADS != 256 || DW_MIN_BLOCKS * (sizeof(WalkSmemFlat) + 1024) <= 228 * 1024,
              "WalkSmemFlat too large for DW_MIN_BLOCKS CTAs per SM");

// reservoir-only modes (force-ervs, ervs-nojump) spend their time in the
// warp-cooperative row scan, whose parallel jump chain needs ~14 more live
// registers: 2 CTAs/SM (up to 128 registers) instead of 3
#ifndef DW_ERVS_MIN_BLOCKS
#define DW_ERVS_MIN_BLOCKS 2
#endif
// PR2 (CoopErjs) kernels too: second-order PageRank on heavy-tailed weights
// spends its time in hub-row scans (cap overruns, tier-2 hand-offs), which
// then run inline instead of through an out-of-line call whose register
// saves spilled ~600 B at 80 registers
#ifndef DW_PR2_WIDE
#define DW_PR2_WIDE 1
#endif
template <class M, int MODE>
struct WideKernel {
    static constexpr bool value = MODE == kForceErvs || MODE == kErvsNoJump ||
                                  (DW_PR2_WIDE && CoopErjs<M>::value);
};
// Wide kernels (2 CTAs/SM) have shared memory to spare: each lane also keeps
// prev's row begin, so the warp reservoir merges cur's row with prev's
// instead of probing prev's hash set
struct WalkSmemWide : WalkSmem {
    ull pbeg[kThreads];
};
// OUT: where paths go.  kOutPadded: [nq][stride] rows.  kOutFlat: the flat
// layout at p.offs, with finished walkers counted per chunk and finished
// chunks flagged to the host (direct compact runs, dw_capi.cu run_direct);
// that code and its shared memory are compiled only into the kernels such
// runs use, so the padded-row kernels are exactly the ones without it
enum : int { kOutPadded = 0, kOutFlat = 1 };
template <int OUT> struct OutSmem { using type = WalkSmem; };
template <> struct OutSmem<kOutFlat> { using type = WalkSmemFlat; };
template <class M, int MODE, int OUT = kOutPadded>
constexpr size_t walk_smem_bytes() {
    return WideKernel<M, MODE>::value ? sizeof(WalkSmemWide)
                                      : sizeof(typename OutSmem<OUT>::type);
}

template <class M, int MODE, int FAT, int OUT = kOutPadded>
__global__ void __launch_bounds__(kThreads, WideKernel<M, MODE>::value ? DW_ERVS_MIN_BLOCKS
                                                                        : DW_MIN_BLOCKS)
    walk_kernel(const __grid_constant__ WalkParams p) {
    constexpr bool kNoJump = MODE == kErvsNoJump;
    // MetaPath trials judged on a packed label first (DevGraph::lab2); the
    // label batch lives in mb (count | consumed << 4), its positions in sel
    constexpr bool kLabScreen = DW_LAB_SCREEN && LabelScreen<M>::value && FAT == 1 &&
                                (MODE == kAdaptive || MODE == kForceErjs);
    constexpr uint32_t kLabBatch = 4;
    constexpr bool kSO = M::kSecondOrder;
    // dynamic shared memory (WalkSmem): may exceed the 48 KB static limit
    extern __shared__ __align__(16) unsigned char dsm[];
    using SM = typename OutSmem<OUT>::type;
    SM& sm = *reinterpret_cast<SM*>(dsm);
    // lane counters with a per-lane row (the direct kernels count queries and
    // query errors with global atomics: WalkSmemFlat)
    constexpr int kLcN = OUT == kOutFlat ? (int)LC_QERRORS : (int)LC_NUM;
    auto& s_rec = sm.rec;
    auto& s_y = sm.y;
    auto& s_t = sm.t;
    auto& s_mb = sm.mb;
    auto& s_lc = sm.lc;
    auto& s_cnt = sm.cnt;
    auto& s_hist = sm.hist;
    auto& s_lct = sm.lct;
    const int tid = threadIdx.x;
    for (int i = tid; i < kCNum; i += blockDim.x) s_cnt[i] = 0;
    if (tid < LC_NUM) s_lct[tid] = 0;
    for (int i = tid; i < 66; i += blockDim.x) s_hist[i] = 0;
#pragma unroll
    for (int c = 0; c < LC_NUM64; ++c) s_lc[c][tid] = 0;
    if constexpr (OUT != kOutPadded) sm.dchunk[tid] = 0xFFFFu;
#pragma unroll
    for (int c = 0; c < kLcN - LC_NUM64; ++c) sm.lc32[c][tid] = 0;
    constexpr bool kTma = DW_ERVS_TMA && (MODE == kForceErvs || MODE == kErvsNoJump) &&
                          !M::kUsesLabels && !M::kLabelAgg;
    if (kTma && (tid & 31) == 0) {
        for (uint32_t k = 0; k < kTmaStages; ++k) mbar_init(&sm.mbar[tid >> 5][k]);
        sm.tmaph[tid >> 5] = 0;
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
    // lane counters: LC_* accumulate per lane in shared memory
    auto lc_add = [&](int c, ull v) {
        if (c < LC_NUM64) {
            s_lc[c][tid] += v;
        } else {
            uint32_t& x = sm.lc32[c - LC_NUM64][tid];
            const uint32_t y = x + (uint32_t)v;  // v < 2^32 at every site
            x = y;
            if (y < (uint32_t)v) {
                const int gc = c == LC_ETRIALS1 ? kCTrials : c == LC_FALLBACKS ? kCFallbacks
                               : c == LC_DEADENDS ? kCDeadEnds : c == LC_QERRORS ? kCQueryErrors
                                                                                : kCQueries;
                atomicAdd(&p.counters[gc], 1ull << 32);
            }
        }
    };

    // a block's 32-bit histogram cells cannot overflow unless the launch
    // walks 2^32 steps in total
    const bool hist_wide = __umul64hi(p.nq, (ull)p.target) != 0 || p.nq * (ull)p.target >= 0xFFFFFFFFull;
    M model(p.mp);
    const int lane = tid & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const DevGraph& g = p.g;
    const bool shortcut = p.mp.shortcut != 0;

    uint32_t phase = P_IDLE;
    bool drained = false;  // warp-uniform
    uint32_t nrefill = 0;  // warp-uniform
    ull qg = 0;  // global walker id (RNG key); the launch index is sm.qi[tid]
    // walker state
    uint32_t prev = kInvalid, pdeg = 0, step = 0, deg = 0;
    uint32_t& cur = sm.cur[tid];
    uint32_t& phoff = sm.phoff[tid];  // hash set of prev
    uint32_t& plg = sm.plg[tid];      // log2 buckets of prev's hash set
    uint32_t& hoff = sm.hoff[tid];    // hash set of cur
    cur = kInvalid;
    phoff = plg = hoff = 0;
    ull begin = 0;
    // eRJS state
    double& bound = sm.bound[tid];    // rejection bound
    double& mnr = sm.mnr[tid];        // non-return maximum
    uint32_t& cap = sm.cap[tid];      // trial cap of the step (samplers.hpp:157)
    uint32_t& tw_lo = sm.twlo[tid];   // return-edge range in N(cur)
    uint32_t& tw_cnt = sm.twcnt[tid];
    uint32_t& nret = sm.nret[tid];    // judged return-edge trials
    bound = mnr = 0.0;
    cap = tw_lo = tw_cnt = nret = 0;
    uint32_t tn = 0, rh = 0, rc = 0;  // next trial, ring head, ring count
    uint32_t mb = 0, sel = 0;         // parked bucket (bit 31: parked), pair bits
    // per-walker register counters, folded into the lane counters at walk end
    uint32_t c_trials = 0, c_alg4 = 0;   // eRJS trials, algorithmic bytes / 4
    // eRVS state lives in the lane's spare ring slot (the ring is idle while a
    // lane runs eRVS), keeping the hot eRJS loop's register set small:
    //   s_rec[kRing-1][0] = {parked neighbour u, its h}   (VMEMB)
    //   s_rec[kRing-1][1..2] = ErvsState
    // tn doubles as the eRVS neighbour cursor.
    constexpr uint32_t kParked = 0x80000000u;
    static_assert(sizeof(ErvsState) == 32, "ErvsState must fill two uint4");
    auto ev_load = [&]() {
        ErvsState e;
        *reinterpret_cast<uint4*>(&e) = s_rec[kRing - 1][1][tid];
        *(reinterpret_cast<uint4*>(&e) + 1) = s_rec[kRing - 1][2][tid];
        return e;
    };
    auto ev_store = [&](const ErvsState& e) {
        s_rec[kRing - 1][1][tid] = *reinterpret_cast<const uint4*>(&e);
        s_rec[kRing - 1][2][tid] = *(reinterpret_cast<const uint4*>(&e) + 1);
    };
    auto mkstep = [&](double hmax, double hsum, double lmax = 0.0, double lsum = 0.0) {
        Step S;
        S.lmax = lmax;
        S.lsum = lsum;
        S.cur = cur;
        S.prev = prev;
        S.prev_degree = pdeg;
        S.step = step;
        S.degree = deg;
        S.hmax = hmax;
        S.hsum = hsum;
        S.hin = hmax;
        return S;
    };
    auto key_of = [&]() {
        const ull q = qg;
        return WalkerKey{p.seed_lo, p.seed_hi, (uint32_t)q, (uint32_t)(q >> 32), step};
    };
    auto fail = [&](int code) {
        raise_error(p, code, qg);
        phase = P_IDLE;
    };
    auto flush_walker = [&]() {
        lc_add(LC_ETRIALS, c_trials);
        lc_add(LC_ALG4, c_alg4);
        c_trials = c_alg4 = 0;
    };
    // a walker's path is final (direct compact output): count it in its
    // chunk; the walker that completes a chunk raises the chunk's host-mapped
    // flag, so the host copies the chunk while the launch walks on
    // (acq_rel: every path write of the chunk precedes the flag)
    auto chunk_done = [&]() {
      if constexpr (OUT != kOutPadded) {
        const uint32_t c = sm.dchunk[tid];
        if (c == 0xFFFFu) return;
        sm.dchunk[tid] = 0xFFFFu;
        unsigned old;
#if DW_DONE_MODE == 0
        asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                     : "=r"(old) : "l"(p.chunk_done + c) : "memory");
#elif DW_DONE_MODE == 1  // measurement only: no ordering
        old = atomicAdd(p.chunk_done + c, 1u);
#else
        return;
#endif
        const ull lo = (ull)c << p.chunk_shift;
        const ull n = min(p.nq - lo, 1ull << p.chunk_shift);
        if ((ull)old + 1 == n) {
            __threadfence_system();
            *(volatile unsigned*)(p.chunk_flag + c) = 1u;
        }
      }
    };
    // first entry of the lane's path: its row of the padded [nq][stride]
    // layout, or its offset in the flat layout (kOutFlat)
    auto row_start = [&]() -> uint32_t* {
        if constexpr (OUT == kOutFlat) return p.paths + sm.rowb[tid];
        else return p.paths + (ull)sm.qi[tid] * p.stride;
    };
    // path entry `step` (stage; a completed 32 B sector is written whole)
    auto put_path = [&](uint32_t v) {
        // the row start is read once (the staging stores may alias it)
        uint32_t* const rs = row_start();
        uint32_t* a = rs + step;
        const uint32_t k = (uint32_t)(reinterpret_cast<unsigned long long>(a) >> 2) & 7u;
        sm.pst[k][tid] = v;
        if (k == 7u) {
            uint32_t* s0 = a - 7;
            if (s0 >= (OUT == kOutFlat ? rs : row_start())) {  // the sector is this walker's
                reinterpret_cast<uint4*>(s0)[0] =
                    make_uint4(sm.pst[0][tid], sm.pst[1][tid], sm.pst[2][tid], sm.pst[3][tid]);
                reinterpret_cast<uint4*>(s0)[1] =
                    make_uint4(sm.pst[4][tid], sm.pst[5][tid], sm.pst[6][tid], sm.pst[7][tid]);
            } else {  // the row's first sector, shared with the previous row
                for (uint32_t* q = OUT == kOutFlat ? rs : row_start(); q <= a; ++q)
                    *q = sm.pst[(uint32_t)(reinterpret_cast<unsigned long long>(q) >> 2) & 7u][tid];
            }
        }
    };
    // the staged entries of the last, incomplete sector
    auto flush_path = [&]() {
        uint32_t* const rs0 = row_start();
        uint32_t* a = rs0 + step;
        const uint32_t k = (uint32_t)(reinterpret_cast<unsigned long long>(a) >> 2) & 7u;
        if (k == 7u) return;
        uint32_t* q = a - k;
        uint32_t* rs = OUT == kOutFlat ? rs0 : row_start();
        if (q < rs) q = rs;
        for (; q <= a; ++q)
            *q = sm.pst[(uint32_t)(reinterpret_cast<unsigned long long>(q) >> 2) & 7u][tid];
    };
    auto end_walk = [&]() {
        if (p.lengths) p.lengths[sm.qi[tid]] = step + 1;
        if (p.paths) flush_path();
        flush_walker();
        phase = OUT != kOutPadded ? P_DONE : P_IDLE;
    };
    auto start_ervs = [&](ull draw_base) {
        tn = 0;
        // §8(d): σ(8d) + 32·min(d, ⌈d'/8⌉) when membership is needed
        ull alg = ((8ull * deg + 31) / 32) * 32;
        if (kSO && prev != kInvalid) alg += 32ull * min((ull)deg, ((ull)pdeg + 7) / 8);
        c_alg4 += (uint32_t)(alg >> 2);
        if (FAT && (MODE == kAdaptive || MODE == kForceErjs) && deg == 1 && p.mp.pos_weights &&
            bound > 0.0 && isfinite(bound)) {
            // one neighbour whose weight is positive and finite by construction
            // (its h is the row's finite hmax): the reservoir keeps it after
            // its single key draw (samplers.hpp:82-85)
            lc_add(LC_EREADS, 1);
            lc_add(LC_EDRAWS, 1);
            ev_store(ErvsState{0.0, 0.0, begin, kInvalid, 0});
            phase = P_FETCH;
            return;
        }
        ev_store(ErvsState{-DBL_MAX, 0.0, draw_base, kInvalid, 0});
        phase = deg >= kCoopMinDegree ? P_COOP : P_VREC;
    };
    // trial cap of an eRJS step at cur (samplers.hpp:157), tightened by the
    // tier-2 hand-off when enabled (dw_run_opts.erjs_handoff; oracle.c erjs_cap)
    auto step_cap = [&](const Step&) -> uint32_t {
        const ull c = p.cap_per_degree * (ull)deg;
        uint32_t r = c > 0xFFFFFFFFull ? 0xFFFFFFFFu : (uint32_t)c;
        if (p.handoff > 0.0) {
            // trials worth `handoff` reservoir passes over the row (d / ratio
            // trials cost one pass under the cost model, cost_model.hpp:46-56)
            const double h = ceil(p.handoff * (double)deg / p.ratio);
            const uint32_t hc = !(h >= 32.0) ? 32u : (h >= 4294967295.0 ? 0xFFFFFFFFu : (uint32_t)h);
            if (hc < r) r = hc;
        }
        return r;
    };
    // eRJS bookkeeping for T judged trials, nret of them return edges
    auto count_erjs = [&](uint32_t T) {
        c_trials += T;
        const bool so = kSO && prev != kInvalid;
        c_alg4 += (so ? 16u : 8u) * T - (so ? 8u * nret : 0u);
        if ((c_trials | c_alg4) & 0xC0000000u) flush_walker();
    };

    // slim layout: the edge the walker took, whose twin[] word comes with the
    // next node record (s_y[1] is idle between a step's end and its node gather)
    auto twe = [&]() -> ull& { return *reinterpret_cast<ull*>(&s_y[1][tid]); };
    // wide kernels: prev's row begin (the warp reservoir merges cur's row
    // with prev's; WalkSmemWide)
    constexpr bool kPrevRow = WideKernel<M, MODE>::value && M::kSecondOrder;
    auto pbeg = [&]() -> ull& { return reinterpret_cast<WalkSmemWide&>(sm).pbeg[tid]; };

    for (;;) {
        // ---- walks that ended last iteration (end_walk)
        if constexpr (OUT != kOutPadded)
            if (phase == P_DONE) {
                // (no chunk counts: dw_run_device's listed walkers)
                if (p.chunk_done) sm.dchunk[tid] = (uint16_t)(sm.qi[tid] >> p.chunk_shift);
                phase = P_IDLE;
            }
        // ---- refill idle lanes: one atomic per warp (runtime.cpp:209-211)
        unsigned need = __ballot_sync(kFull, phase == P_IDLE);
        if (need && !drained) {
            // abandon after an error (polled on every 16th refill of the warp)
            if ((nrefill++ & 15u) == 0 && *(volatile int*)p.error != 0) drained = true;
            drained = __any_sync(kFull, drained);
            while (need && !drained) {
                const int leader = __ffs(need) - 1;
                const int n = __popc(need);
                ull base = 0;
                if (lane == leader) base = atomicAdd(p.next_walker, (ull)n);
                base = __shfl_sync(kFull, base, leader);
                if (base + (ull)n >= p.nq) drained = true;
                if (lane == leader && base < p.nq)  // one counter add per claim
                {
                    if constexpr (OUT == kOutFlat)
                        atomicAdd(&p.counters[kCQueries], min((ull)n, p.nq - base));
                    else
                        lc_add(LC_QUERIES, min((ull)n, p.nq - base));
                }
                if (phase == P_IDLE) {
                    const ull i = base + (ull)__popc(need & lt_mask);
                    if (i < p.nq) {
                        const uint32_t start = p.queries[i];
                        if constexpr (OUT == kOutFlat) {
                            // the path's flat offset loads beside the start
                            // (one load latency per claim, not two)
                            const ull rb = p.offs[i];
                            sm.qi[tid] = (uint32_t)i;
                            if (start >= g.nv) {  // runtime.cpp:213-217
                                atomicAdd(&p.counters[kCQueryErrors], 1ull);
                                if (p.lengths) p.lengths[i] = 0;
                                phase = P_DONE;  // booked next iteration
                            } else {
                                if (p.target == 0) {
                                    if (p.paths) p.paths[rb] = start;
                                    if (p.lengths) p.lengths[i] = 1;
                                    phase = P_DONE;
                                } else {
                                    phase = P_NODE;
                                    sm.rowb[tid] = rb;
                                    qg = p.qids ? p.qids[i] : p.qid_base + i;
                                    step = 0;
                                    if (p.paths) put_path(start);
                                    cur = start;
                                    prev = kInvalid;
                                    pdeg = phoff = plg = 0;
                                    step = 0;
                                }
                            }
                        } else {
                            if (start >= g.nv) {  // runtime.cpp:213-217
                                lc_add(LC_QERRORS, 1);
                                if (p.lengths) p.lengths[i] = 0;
                            } else {
                                if (p.target == 0) {
                                    if (p.paths) p.paths[i * p.stride] = start;
                                    if (p.lengths) p.lengths[i] = 1;
                                } else {
                                    phase = P_NODE;
                                    sm.qi[tid] = (uint32_t)i;
                                    qg = p.qids ? p.qids[i] : p.qid_base + i;
                                    step = 0;
                                    if (p.paths) put_path(start);
                                    cur = start;
                                    prev = kInvalid;
                                    pdeg = phoff = plg = 0;
                                    step = 0;
                                }
                            }
                        }
                    }
                }
                need = __ballot_sync(kFull, phase == P_IDLE);
            }
        }
        if (__ballot_sync(kFull, phase != P_IDLE) == 0) break;

        // ---- A: issue this iteration's gathers.  Independent blocks (not an
        // if/else chain): a divergent warp skips the blocks none of its lanes
        // need instead of serialising through a jump table (BRX)
        const uint32_t ph0 = phase;
        if (ph0 == P_TRIAL) {
            if (mb & kParked) {
                const uint32_t* b = g.hslots + 8ull * (phoff + (mb & ~kParked));
                cp16(&s_mb[0][tid], b);
                cp16(&s_mb[1][tid], b + 4);
            }
            const ull q = qg;
            // step constants into registers once per iteration: the ring's
            // shared-memory stores below would otherwise force a reload of
            // the shared-memory state on every trial
            const double bound_r = bound, mnr_r = mnr;
            const uint32_t twlo_r = tw_lo, twcnt_r = tw_cnt, cap_r = cap;
            // one trial: free rejection, or queue its record gather in the ring
            auto trial = [&](const U4& b) {
                const uint32_t x = (uint32_t)bounded(lo64(b), deg);  // draw 2t:   bounded(d)
                const double y = uniform01(hi64(b)) * bound_r;        // draw 2t+1: uniform01()*c
                if (!(y >= mnr_r && x - twlo_r >= twcnt_r)) {         // else rejected, no gather
                    const uint32_t k = (rh + rc) & (kRing - 1);
                    s_y[k][tid] = y;
                    s_t[k][tid] = tn;
                    const ull e = begin + x;
                    if (FAT == 2) {  // compact record: one sector
                        const uint4* r = reinterpret_cast<const uint4*>(g.fat32 + e);
                        cp16(&s_rec[k][0][tid], r);
                        cp16(&s_rec[k][1][tid], r + 1);
                    } else if (FAT) {
                        const uint4* r = reinterpret_cast<const uint4*>(g.fat + e);
                        cp16(&s_rec[k][0][tid], r);
                        cp16(&s_rec[k][1][tid], r + 1);
                        cp16(&s_rec[k][2][tid], r + 2);
                    } else {
                        sel = (sel & ~(1u << k)) | ((uint32_t)(e & 1) << k);
                        cp16(&s_rec[k][0][tid], pair_of(g.edges, e));
                        if (M::kUsesLabels && g.labels) cp4(&s_rec[k][1][tid], g.labels + (e & ~1ull));
                        s_rec[k][1][tid].y = x;  // the edge, for its return-edge range
                    }
                    ++rc;
                }
                ++tn;
            };
            if (kLabScreen && g.lab2) {
                // label screen (MetaPath): the previous iteration fetched the
                // packed label words of a batch of trials; a trial whose edge
                // label is not schema[step] has weight 0 (models.hpp:105-110)
                // and is rejected without gathering its record, the others
                // are regenerated and queued in trial order
                const uint32_t want = p.mp.schema[step];
                uint32_t lbn = mb & 7u, lbk = (mb >> 4) & 7u;
                const uint32_t* lw = reinterpret_cast<const uint32_t*>(&s_mb[0][tid]);
                while (lbk < lbn && rc < kRing) {
                    const uint32_t t = tn - lbn + lbk;
                    const uint32_t lab = (lw[lbk] >> (2u * ((sel >> (4u * lbk)) & 15u))) & 3u;
                    if (lab == want) {
                        const U4 b = philox4x32_10_rk(U4{t, step, (uint32_t)q, (uint32_t)(q >> 32)}, p.rk);
                        const uint32_t x = (uint32_t)bounded(lo64(b), deg);
                        const uint32_t k = (rh + rc) & (kRing - 1);
                        s_y[k][tid] = uniform01(hi64(b)) * bound_r;
                        s_t[k][tid] = t;
                        const uint4* r = reinterpret_cast<const uint4*>(g.fat + begin + x);
                        cp16(&s_rec[k][0][tid], r);
                        cp16(&s_rec[k][1][tid], r + 1);
                        cp16(&s_rec[k][2][tid], r + 2);
                        ++rc;
                    }
                    ++lbk;
                }
                if (lbk == lbn) {  // the next batch of label probes
                    lbn = lbk = 0;
                    sel = 0;
#pragma unroll 1
                    for (; lbn < kLabBatch && tn < cap_r; ++lbn, ++tn) {
                        const U4 b = philox4x32_10_rk(U4{tn, step, (uint32_t)q, (uint32_t)(q >> 32)}, p.rk);
                        const ull e = begin + (uint32_t)bounded(lo64(b), deg);
                        cp4(reinterpret_cast<uint32_t*>(&s_mb[0][tid]) + lbn, g.lab2 + (e >> 4));
                        sel |= (uint32_t)(e & 15u) << (4u * lbn);
                    }
                }
                mb = lbn | (lbk << 4);
            } else {
#pragma unroll 1
            for (uint32_t gen = 0; gen < kGen && rc < kRing && tn < cap_r; ++gen) {
                trial(philox4x32_10_rk(U4{tn, step, (uint32_t)q, (uint32_t)(q >> 32)}, p.rk));
            }
            }
        }
        if (ph0 == P_NODE) {
            const char* nr = reinterpret_cast<const char*>(g.nodes + cur);
            cp16(&s_mb[0][tid], nr);
            cp16(&s_mb[1][tid], nr + 16);
            if (!FAT && g.twin && prev != kInvalid) cp4(&s_t[0][tid], g.twin + twe());
            if (M::kLabelAgg) cp16(&s_rec[0][0][tid], g.lagg + cur);  // the ring is empty here
        }
        if (ph0 == P_FETCH) {
            const ull fe = ev_load().didx;
            if (FAT == 2) {
                const uint4* r = reinterpret_cast<const uint4*>(g.fat32 + fe);
                cp16(&s_rec[0][0][tid], r);
                cp16(&s_rec[0][1][tid], r + 1);
            } else {
                const uint4* r = reinterpret_cast<const uint4*>(g.fat + fe);
                cp16(&s_rec[0][0][tid], r);
                cp16(&s_rec[0][1][tid], r + 1);
                cp16(&s_rec[0][2][tid], r + 2);
            }
        }
        if (ph0 == P_VMEMB) {
            const uint32_t* b = g.hslots + 8ull * (phoff + mb);
            cp16(&s_mb[0][tid], b);
            cp16(&s_mb[1][tid], b + 4);
        }
        if (ph0 == P_VREC) {
            const ull e = begin + tn;
            sel = (uint32_t)(e & 1);
            cp16(&s_mb[0][tid], pair_of(g.edges, e));
            if (M::kUsesLabels && g.labels) cp4(&s_mb[1][tid], g.labels + (e & ~1ull));
        }
        // a walk that ended last iteration is final: count it in its chunk
        // (direct compact output; its release and round trip overlap the
        // gathers just issued)
        if (OUT != kOutPadded) chunk_done();
        // ---- B
        cp_wait_all();

        // ---- C: consume; a finished step leaves its outcome in `next_ev`
        // (blocks test the phase the lane had when this iteration started)
        enum : uint32_t { E_NONE = 0, E_FAT, E_ADV, E_NODE };
        uint32_t next_ev = E_NONE, next_slot = 0, next_u = 0;
        if (ph0 == P_TRIAL) {
            int acc = -1;
            const Step S = mkstep(0.0, 0.0);
            const float hin_r = __uint_as_float(sm.tq[tid]);  // triangle bound
            if (mb & kParked) {  // resolve the head's membership probe
                const uint4 v0 = s_rec[rh][0][tid];
                const uint32_t u = FAT ? v0.x : (((sel >> rh) & 1) ? v0.z : v0.x);
                const int r = bucket_lookup(s_mb[0][tid], s_mb[1][tid], u);
                if (r < 0) {
                    mb = kParked | ((mb + 1) & ((1u << plg) - 1u));
                } else {
                    const bool odd = !FAT && ((sel >> rh) & 1);
                    const float h = __uint_as_float(odd ? v0.w : v0.y);
                    uint16_t lab = 0;  // the parked record still holds its label
                    if (M::kUsesLabels)
                        lab = FAT ? (FAT == 2 ? (uint16_t)0 : (uint16_t)(v0.w >> 8))
                                  : (uint16_t)(odd ? (s_rec[rh][1][tid].x >> 16) : s_rec[rh][1][tid].x);
                    const WeightCase wc = model.weight(S, u, h, lab);
                    const double w = r ? wc.w_in : wc.w_out;
                    mb = 0;
                    if (!valid_w(w)) {
                        fail(kDevBadWeight);
                    } else if (s_y[rh][tid] < w) {
                        acc = (int)rh;
                    } else {
                        rh = (rh + 1) & (kRing - 1);
                        --rc;
                    }
                }
            }
            while (phase == P_TRIAL && acc < 0 && !(mb & kParked) && rc) {
                const uint4 v0 = s_rec[rh][0][tid];
                const bool odd = !FAT && ((sel >> rh) & 1);
                const uint32_t u = odd ? v0.z : v0.x;
                const float h = __uint_as_float(odd ? v0.w : v0.y);
                uint16_t lab = 0;
                if (M::kUsesLabels) {
                    if (FAT)
                        lab = FAT == 2 ? (uint16_t)0 : (uint16_t)(v0.w >> 8);
                    else
                        lab = (uint16_t)(odd ? (s_rec[rh][1][tid].x >> 16) : s_rec[rh][1][tid].x);
                }
                const double y = s_y[rh][tid];
                const WeightCase wc = model.weight(S, u, h, lab);
                if (kSO && u == prev) ++nret;
                if (!wc.needs_member) {
                    if (!valid_w(wc.w)) {
                        fail(kDevBadWeight);
                        break;
                    }
                    if (y < wc.w) {
                        acc = (int)rh;
                        break;
                    }
                } else {
                    const double lo = wc.w_in < wc.w_out ? wc.w_in : wc.w_out;
                    const double hi = wc.w_in < wc.w_out ? wc.w_out : wc.w_in;
                    const bool ok = valid_w(wc.w_in) && valid_w(wc.w_out);
                    if (ok && y < lo) {
                        acc = (int)rh;
                        break;
                    }
                    if (!ok || y < hi) {  // outcome hinges on u in N(prev)
                        if (h > hin_r) {
                            // a prop above the triangle bound: u is not in
                            // N(prev), no probe (weight: the "out" case)
                            if (!valid_w(wc.w_out)) {
                                fail(kDevBadWeight);
                                break;
                            }
                            if (y < wc.w_out) {
                                acc = (int)rh;
                                break;
                            }
                        } else {
                            mb = kParked | hash_bucket(u, plg);
                            break;
                        }
                    }
                }
                rh = (rh + 1) & (kRing - 1);
                --rc;
            }
            if (phase == P_TRIAL) {
                if (acc >= 0) {
                    count_erjs(s_t[acc][tid] + 1);
                    if (FAT) {
                        next_ev = E_FAT;
                        next_slot = (uint32_t)acc;
                    } else {
                        const uint4 v0 = s_rec[acc][0][tid];
                        next_ev = E_ADV;
                        next_u = ((sel >> acc) & 1) ? v0.z : v0.x;
                        twe() = begin + s_rec[acc][1][tid].y;
                    }
                } else if (!(mb & kParked) && rc == 0 && tn >= cap &&
                           (!kLabScreen || (mb & 7u) == ((mb >> 4) & 7u))) {
                    count_erjs(tn);
                    lc_add(LC_FALLBACKS, 1);  // cap overrun -> reservoir, same stream
                    start_ervs(2ull * tn);
                } else if (CoopErjs<M>::value && !(mb & kParked) && rc == 0 && tn >= kCjsMin) {
                    phase = P_CJS;  // every trial before tn judged and rejected
                }
            }
        }
        if (ph0 == P_NODE) {
            next_ev = E_NODE;
        }
        if (ph0 == P_FETCH) {
            next_ev = E_FAT;
        }
        if (ph0 == P_VMEMB || ph0 == P_VREC) {
            uint32_t u;
            float h;
            uint16_t lab = 0;
            int r = 2;  // 2: no membership needed
            if (phase == P_VMEMB) {
                const uint4 pk = s_rec[kRing - 1][0][tid];  // {u, h, label} of the parked neighbour
                u = pk.x;
                h = __uint_as_float(pk.y);
                lab = (uint16_t)pk.z;
                r = bucket_lookup(s_mb[0][tid], s_mb[1][tid], u);
                if (r < 0) mb = (mb + 1) & ((1u << plg) - 1u);
            } else {
                const uint4 v = s_mb[0][tid];
                u = sel ? v.z : v.x;
                h = __uint_as_float(sel ? v.w : v.y);
                if (M::kUsesLabels)
                    lab = (uint16_t)(sel ? (s_mb[1][tid].x >> 16) : s_mb[1][tid].x);
            }
            if (r >= 0) {
                const WeightCase wc = model.weight(mkstep(0.0, 0.0), u, h, lab);
                if (kSO && r == 2 && wc.needs_member && h > __uint_as_float(sm.tq[tid]))
                    r = 0;  // prop above the triangle bound: u is not in N(prev)
                if (kSO && r == 2 && wc.needs_member) {
                    s_rec[kRing - 1][0][tid] = make_uint4(u, __float_as_uint(h), lab, 0u);
                    mb = hash_bucket(u, plg);
                    phase = P_VMEMB;
                } else {
                    const double w = r == 2 ? wc.w : (r ? wc.w_in : wc.w_out);
                    if (!valid_w(w)) {
                        fail(kDevBadWeight);
                    } else if (FAT && deg <= kEBatchMaxDeg) {
                        // short row: collect the weights, run the reservoir
                        // scan later together with other lanes (P_EMATH)
                        // weight j in the lane's own slot-0 words: s_rec[0][j/2][tid], half j%2
                        reinterpret_cast<double*>(&s_rec[0][tn >> 1][tid])[tn & 1] = w;
                        phase = P_VREC;
                        if (++tn == deg) {
                            tn = 0;  // now counts the iterations spent waiting
                            phase = P_EMATH;
                        }
                    } else {
                        phase = P_VREC;
                        const ErvsState e0 = ev_load();
                        const ErvsState ev = ervs_visit<kNoJump>(e0, key_of(), p.rk, tn, u, w);
                        ev_store(ev);
                        lc_add(LC_EDRAWS, kNoJump ? 1ull : ev.didx - e0.didx);
                        lc_add(LC_EREADS, 1);
                        if (++tn == deg) {  // the scan is complete
                            if (ev.best == kInvalid) {  // all weights zero: dead end
                                lc_add(LC_DEADENDS, 1);
                                end_walk();
                            } else if (FAT) {
                                ErvsState e = ev;
                                e.didx = begin + (ev.bidx & ~kHave);  // its fat record starts the next step
                                ev_store(e);
                                phase = P_FETCH;
                            } else {
                                next_ev = E_ADV;
                                next_u = ev.best;
                                twe() = begin + (ev.bidx & ~kHave);
                            }
                        }
                    }
                }
            }
        }

        // ---- D: step transitions, one code site for every phase
        double hmax = 0.0, hsum = 0.0, lmax = 0.0, lsum = 0.0;
        uint32_t lmask = 0xFFu;  // labels present in N(cur) (fat record), all = unknown
        bool approx_sum = false;  // hsum from a compact record (f32)
        if (next_ev == E_FAT || next_ev == E_ADV) {
            // WalkerState::advance (walk_state.hpp:33-39)
            const uint4 v0 = s_rec[next_slot][0][tid];
            const uint32_t nx = next_ev == E_FAT ? v0.x : next_u;
            if (kPrevRow) pbeg() = begin;
            prev = cur;
            pdeg = deg;
            phoff = hoff;
            plg = hash_log2_buckets(deg);
            cur = nx;
            ++step;
            if (p.paths) put_path(nx);
            if (step >= p.target) {
                end_walk();
                next_ev = E_NONE;
            } else if (next_ev == E_FAT && FAT == 2) {
                const uint4 v1 = s_rec[next_slot][1][tid];
                begin = (ull)v0.z | ((ull)(v0.w & 0xFFu) << 32);
                deg = v0.w >> 8;
                hoff = v1.x;
                tw_lo = (v1.y >> 24) == 255u ? 0u : (v1.y & 0xFFFFFFu);
                tw_cnt = (v1.y >> 24) == 255u ? 0xFFFFFFFFu : (v1.y >> 24);
                hmax = (double)__uint_as_float(v1.z);
                // row sum truncated to 24 bits (see the decision), triangle bound
                hsum = (double)__uint_as_float(v1.w & ~0xFFu);
                sm.tq[tid] = tri_bound(v1.w & 0xFFu, __uint_as_float(v1.z));
                approx_sum = true;
            } else if (next_ev == E_FAT) {
                const uint4 v1 = s_rec[next_slot][1][tid], v2 = s_rec[next_slot][2][tid];
                begin = ((ull)v0.z | ((ull)v0.w << 32)) & kBeginMask;
                deg = v1.x;
                hoff = v1.y;
                tw_lo = v1.z;
                tw_cnt = (v1.w & 0xFFFFFFu) == 0xFFFFFFu ? 0xFFFFFFFFu : (v1.w & 0xFFFFFFu);
                hmax = __hiloint2double((int)v2.y, (int)v2.x);
                sm.tq[tid] = tri_bound(v1.w >> 24, (float)hmax);  // hmax: a max of f32 props
                hsum = __hiloint2double((int)v2.w, (int)v2.z);
                lmask = v0.w >> 24;
            } else {
                phase = P_NODE;  // slim layout: the node record comes next iteration
                next_ev = E_NONE;
            }
        } else if (next_ev == E_NODE) {
            const uint4 v0 = s_mb[0][tid], v1 = s_mb[1][tid];
            begin = (ull)v0.x | ((ull)v0.y << 32);
            deg = v0.z;
            hoff = v0.w;
            hmax = __hiloint2double((int)v1.y, (int)v1.x);
            hsum = __hiloint2double((int)v1.w, (int)v1.z);
            if (M::kLabelAgg) {
                const uint4 la = s_rec[0][0][tid];
                lmax = __hiloint2double((int)la.y, (int)la.x);
                lsum = __hiloint2double((int)la.w, (int)la.z);
            }
            // first step: no return edge; later (slim layout) the twin[] word
            // of the edge taken, or an unknown range.  A compact record whose
            // decision fell back here (need_node) keeps the range it carried.
            if (FAT != 2 || prev == kInvalid) {
                tw_lo = 0;
                tw_cnt = prev == kInvalid ? 0u : 0xFFFFFFFFu;
                sm.tq[tid] = tri_bound(255u, (float)hmax);  // no triangle bound
            }
            if (!FAT && g.twin && prev != kInvalid) {
                const uint32_t w = s_t[0][tid];
                if ((w >> 24) != 255u) {
                    tw_lo = w & 0xFFFFFFu;
                    tw_cnt = w >> 24;
                }
            }
        }
        if (next_ev != E_NONE) {
            // decide_sampler (cost_model.hpp:46-56) for the step at cur
            if (deg == 0) {  // runtime.cpp:70-71: stop without counting a step
                end_walk();
            } else {
                Step S = mkstep(hmax, hsum, lmax, lsum);
                if (FAT && prev != kInvalid) S.hin = (double)__uint_as_float(sm.tq[tid]);
                model.prepare(S);
                bool erjs = false, need_node = false;
                if (MODE == kAdaptive) {
                    if (M::kBoundable) {
                        bound = model.bound(S);
                        const double T = p.ratio * bound;
                        if (FAT == 2 && approx_sum) {
                            // compact record: decide on the estimate from the
                            // f32 sum unless T is within 1e-6 of it; then the
                            // exact node record decides (next iteration)
                            const double Wa = (M::kScreen && p.mp.screen) ? model.wsum_approx(S) : 0.0;
                            if (M::kScreen && p.mp.screen && T < Wa * (1.0 - p.mp.fat32_band))
                                erjs = true;
                            else if (M::kScreen && p.mp.screen && T > Wa * (1.0 + p.mp.fat32_band))
                                erjs = false;
                            else
                                need_node = true;
                        } else if (M::kScreen && p.mp.screen) {
                            // decide on the one-multiply estimate unless T
                            // falls in its error band (then the exact sum)
                            const double Wa = model.wsum_approx(S);
                            erjs = T < Wa * (1.0 - 1e-12)
                                       ? true
                                       : (T > Wa * (1.0 + 1e-12) ? false : T < model.wsum(S));
                        } else {
                            erjs = T < model.wsum(S);
                        }
                    }
                } else if (MODE == kForceErjs) {  // runtime.cpp:109-129
                    erjs = M::kBoundable;
                    if (erjs) bound = model.bound(S);
                }
                if (FAT == 2 && need_node) {
                    phase = P_NODE;  // the exact node record decides this step
                } else {
                {
                    const uint32_t hb = 2 * degree_bucket(deg) + (erjs ? 1 : 0);
                    if (!hist_wide) {
                        atomicAdd(&s_hist[hb], 1u);  // no result to wait for
                    } else if (atomicAdd(&s_hist[hb], 1u) == 0x7FFFFFFFu) {  // spill before overflow
                        atomicSub(&s_hist[hb], 0x80000000u);
                        atomicAdd(&s_cnt[kCHist + hb], 0x80000000ull);
                    }
                }
                // §8(d): 32 B offsets + 4 B path write (+ 32 B aggregates)
                c_alg4 += (36 + ((MODE == kAdaptive || MODE == kForceErjs) && M::kAggregates ? 32 : 0)) / 4;
                bool dead_row = false;
                if (M::kUsesLabels && FAT) {
                    // MetaPath row without an edge of label schema[step]: every
                    // weight is 0 (models.hpp:99-104).  The reference burns the
                    // 64·d trial cap, falls back to eRVS and finds no candidate;
                    // the counters of that sequence are known in closed form
                    // (samplers.hpp:156-177), so the walk ends here.
                    const uint32_t want = p.mp.schema[step];
                    dead_row = want < kMaskLabels && !(lmask & (1u << want)) &&
                               (!erjs || (bound > 0.0 && isfinite(bound)));
                }
                if (dead_row) {
                    if (erjs) {
                        nret = 0;
                        count_erjs(step_cap(S));
                        lc_add(LC_FALLBACKS, 1);
                    } else {
                        lc_add(LC_ETRIALS1, 1);  // single-shot eRVS
                    }
                    lc_add(LC_EREADS, deg);  // the reservoir pass reads every weight, draws none
                    c_alg4 += (uint32_t)(((8ull * deg + 31) / 32) * 8);
                    lc_add(LC_DEADENDS, 1);
                    end_walk();
                } else if (erjs) {
                    if (!(bound > 0.0) || !isfinite(bound)) {  // samplers.hpp:152-154
                        fail(kDevBadBound);
                    } else {
                        mnr = shortcut ? model.nonreturn_max(S) : __longlong_as_double(0x7ff0000000000000ll);
                        cap = step_cap(S);
                        tn = rh = rc = 0;
                        mb = nret = sel = 0;
                        phase = P_TRIAL;
                        if (cap == 0) {  // immediate cap overrun
                            lc_add(LC_FALLBACKS, 1);
                            start_ervs(0);
                        }
                    }
                } else {
                    lc_add(LC_ETRIALS1, 1);  // single-shot kernels report one trial (samplers.hpp:22)
                    start_ervs(0);
                }
                }  // need_node
            }
        }

        // ---- batched reservoir scans of short rows: lanes whose weights are
        // all collected wait until kEBatch of them (or one that waited
        // kEWait iterations) can run the scan in the same instruction stream
        if (FAT) {
            const unsigned ready = __ballot_sync(kFull, phase == P_EMATH);
            if (ready) {
                const bool go = __popc(ready) >= kEBatch ||
                                __any_sync(kFull, phase == P_EMATH && tn >= kEWait);
                if (phase == P_EMATH) {
                    if (go) {
                        const ull d0 = ev_load().didx;
                        uint32_t bidx = 0;
                        const ull d1 = ervs_scan_short(
                            reinterpret_cast<const double*>(&s_rec[0][0][tid]), deg, key_of(), p.rk,
                            d0, &bidx);
                        lc_add(LC_EREADS, deg);
                        lc_add(LC_EDRAWS, d1 - d0);
                        if (bidx == kInvalid) {  // all weights zero: dead end
                            lc_add(LC_DEADENDS, 1);
                            end_walk();
                        } else {
                            ErvsState e = ev_load();
                            e.didx = begin + bidx;  // its fat record starts the next step
                            ev_store(e);
                            phase = P_FETCH;
                        }
                    } else {
                        ++tn;
                    }
                }
            }
        }

        // ---- warp-cooperative eRVS for long rows (ballot hand-off)
        unsigned coop = __ballot_sync(kFull, phase == P_COOP);
        while (coop) {
            const int L = __ffs(coop) - 1;
            coop &= coop - 1;
            Step T;
            T.cur = __shfl_sync(kFull, cur, L);
            T.prev = __shfl_sync(kFull, prev, L);
            T.prev_degree = __shfl_sync(kFull, pdeg, L);
            T.step = __shfl_sync(kFull, step, L);
            T.degree = __shfl_sync(kFull, deg, L);
            T.hmax = T.hsum = 0.0;
            T.hin = (double)__uint_as_float(sm.tq[(tid & ~31) + L]);
            const uint32_t tph = __shfl_sync(kFull, phoff, L);
            const ull tb = __shfl_sync(kFull, begin, L);
            const ull q = __shfl_sync(kFull, qg, L);
            const WalkerKey K{p.seed_lo, p.seed_hi, (uint32_t)q, (uint32_t)(q >> 32), T.step};
            const ull db = __shfl_sync(kFull, lane == L ? ev_load().didx : 0ull, L);
            uint32_t nx = kInvalid, ni = 0;
            ull dr = 0;
            int st;
            if constexpr (MODE == kForceErvs || MODE == kErvsNoJump) {
                const int w = tid >> 5;
                const TmaRing ring{&sm.rec[0][0][w * 32], (uint32_t)kThreads, sm.mbar[w], &sm.tmaph[w]};
                const ull tpb = kPrevRow ? __shfl_sync(kFull, pbeg(), L) : kNoRow;
                st = ervs_warp<M, kNoJump, kTma>(p.mp, T, K, p.rk, g, tb, tph, db, &nx, &ni, &dr,
                                                 ring, T.prev != kInvalid ? tpb : kNoRow);
            }
            else if constexpr (WideKernel<M, MODE>::value) {  // PR2: cap overruns, hand-offs
                const ull tpb = kPrevRow ? __shfl_sync(kFull, pbeg(), L) : kNoRow;
                st = ervs_warp<M, kNoJump, false>(p.mp, T, K, p.rk, g, tb, tph, db, &nx, &ni, &dr,
                                                  TmaRing{}, T.prev != kInvalid ? tpb : kNoRow);
            }
            else if constexpr (DW_PR2_PAR && CoopErjs<M>::value)
                st = ervs_warp_cold<M, kNoJump>(p.mp, T, K, p.rk, g, tb, tph, db, &nx, &ni, &dr);
            else
                st = ervs_warp_seq<M, kNoJump>(p.mp, T, K, p.rk, g, tb, tph, db, &nx, &ni, &dr);
            if (lane == L) {
                if (st < 0) {
                    fail(-st);
                } else {
                    lc_add(LC_EREADS, T.degree);
                    lc_add(LC_EDRAWS, dr);
                    if (nx == kInvalid) {
                        lc_add(LC_DEADENDS, 1);
                        end_walk();
                    } else if (FAT) {
                        ErvsState e = ev_load();
                        e.didx = tb + ni;
                        ev_store(e);
                        phase = P_FETCH;
                    } else {
                        // advance here (rare path); the node record comes next iteration
                        twe() = tb + ni;
                        if (kPrevRow) pbeg() = begin;
                        prev = cur;
                        pdeg = deg;
                        phoff = hoff;
                        plg = hash_log2_buckets(deg);
                        cur = nx;
                        ++step;
                        if (p.paths) put_path(nx);
                        if (step >= p.target)
                            end_walk();
                        else
                            phase = P_NODE;
                    }
                }
            }
        }

        // ---- warp-cooperative eRJS (CoopErjs models): 32 trials per round
        if (CoopErjs<M>::value) {
            unsigned cj = __ballot_sync(kFull, phase == P_CJS);
            while (cj) {
                const int L = __ffs(cj) - 1;
                cj &= cj - 1;
                const int Lt = (tid & ~31) + L;
                Step T;
                T.cur = __shfl_sync(kFull, cur, L);
                T.prev = __shfl_sync(kFull, prev, L);
                T.prev_degree = __shfl_sync(kFull, pdeg, L);
                T.step = __shfl_sync(kFull, step, L);
                T.degree = __shfl_sync(kFull, deg, L);
                T.hmax = T.hsum = 0.0;
                T.hin = (double)__uint_as_float(sm.tq[Lt]);
                T.lmax = T.lsum = 0.0;
                M mw(p.mp);
                mw.prepare(T);
                const ull tb = __shfl_sync(kFull, begin, L);
                const uint32_t t0 = __shfl_sync(kFull, tn, L);
                const uint32_t tph = sm.phoff[Lt], tcap = sm.cap[Lt];
                const uint32_t twl = sm.twlo[Lt], twc = sm.twcnt[Lt];
                const double tbnd = sm.bound[Lt], tmnr = sm.mnr[Lt];
                const ull q = __shfl_sync(kFull, qg, L);
                int win = -1;
                bool bad = false;
                uint32_t judged = 0, rets = 0, wu = 0;
                ull we = 0;
                for (uint32_t base = t0; base < tcap && win < 0 && !bad; base += 32) {
                    const uint32_t t = base + lane;
                    bool acc = false, badw = false, isret = false;
                    ull e = 0;
                    uint32_t u = 0;
                    if (t < tcap) {
                        const U4 b = philox4x32_10_rk(U4{t, T.step, (uint32_t)q, (uint32_t)(q >> 32)}, p.rk);
                        const uint32_t x = (uint32_t)bounded(lo64(b), T.degree);
                        const double y = uniform01(hi64(b)) * tbnd;
                        if (!(y >= tmnr && x - twl >= twc)) {  // else a free rejection
                            e = tb + x;
                            float h;
                            uint16_t lab = 0;
                            if (FAT) {
                                const uint4 r0 = __ldg(FAT == 2 ? reinterpret_cast<const uint4*>(g.fat32 + e)
                                                                : reinterpret_cast<const uint4*>(g.fat + e));
                                u = r0.x;
                                h = __uint_as_float(r0.y);
                                if (M::kUsesLabels) lab = (uint16_t)(r0.w >> 8);
                            } else {
                                const EdgeRec er = load_edge(g.edges + e);
                                u = er.col;
                                h = er.h;
                                lab = edge_label<M>(g, e);
                            }
                            const WeightCase wc = mw.weight(T, u, h, lab);
                            isret = kSO && u == T.prev;
                            const double w = !wc.needs_member
                                                 ? wc.w
                                                 : ((double)h <= T.hin && member(g, T.prev_degree, tph, u)
                                                        ? wc.w_in : wc.w_out);
                            if (!valid_w(w))
                                badw = true;
                            else
                                acc = y < w;
                        }
                    }
                    const unsigned am = __ballot_sync(kFull, acc), bm = __ballot_sync(kFull, badw);
                    const unsigned rm = __ballot_sync(kFull, isret);
                    if (am | bm) {  // the first decided trial in trial order ends the step
                        const int f = __ffs(am | bm) - 1;
                        const unsigned upto = f == 31 ? kFull : ((2u << f) - 1u);
                        rets += __popc(rm & upto);
                        judged = base + f + 1 - t0;
                        if ((bm >> f) & 1) {
                            bad = true;
                        } else {
                            win = f;
                            we = __shfl_sync(kFull, e, f);
                            wu = __shfl_sync(kFull, u, f);
                        }
                    } else {
                        rets += __popc(rm);
                        judged = min(base + 32, tcap) - t0;
                    }
                }
                if (lane == L) {
                    tn = t0 + judged;
                    nret += rets;
                    if (bad) {
                        fail(kDevBadWeight);
                    } else if (win >= 0) {
                        count_erjs(tn);
                        if (FAT) {
                            ErvsState ev = ev_load();
                            ev.didx = we;  // its fat record starts the next step
                            ev_store(ev);
                            phase = P_FETCH;
                        } else {
                            twe() = we;
                            if (kPrevRow) pbeg() = begin;
                            prev = cur;
                            pdeg = deg;
                            phoff = hoff;
                            plg = hash_log2_buckets(deg);
                            cur = wu;
                            ++step;
                            if (p.paths) put_path(wu);
                            if (step >= p.target)
                                end_walk();
                            else
                                phase = P_NODE;
                        }
                    } else {  // cap overrun -> reservoir, same stream
                        count_erjs(tn);
                        lc_add(LC_FALLBACKS, 1);
                        start_ervs(2ull * tn);
                    }
                }
            }
        }
    }
    if (OUT != kOutPadded) chunk_done();  // the walks that ended in the last iteration

    // ---- flush counters: eRJS trials count as trials, reads and 2 draws each
    __syncthreads();
    if (tid < 66 && s_hist[tid]) s_cnt[kCHist + tid] += s_hist[tid];
#pragma unroll 1
    for (int c = 0; c < kLcN; ++c) {
        const ull v = warp_sum(c < LC_NUM64 ? s_lc[c][tid] : (ull)sm.lc32[c - LC_NUM64][tid]);
        if (lane == 0 && v) atomicAdd(&s_lct[c], v);
    }
    __syncthreads();
    if (tid == 0) {
        const ull t = s_lct[LC_ETRIALS];
        s_cnt[kCTrials] = t + s_lct[LC_ETRIALS1];
        s_cnt[kCWeightReads] = t + s_lct[LC_EREADS];
        s_cnt[kCRngDraws] = 2 * t + s_lct[LC_EDRAWS];
        s_cnt[kCAlgBytes] = 4 * s_lct[LC_ALG4];
        s_cnt[kCFallbacks] += s_lct[LC_FALLBACKS];
        s_cnt[kCDeadEnds] += s_lct[LC_DEADENDS];
        s_cnt[kCQueryErrors] += s_lct[LC_QERRORS];  // 0 in the direct kernels:
        s_cnt[kCQueries] += s_lct[LC_QUERIES];      // they count into p.counters
    }
    __syncthreads();
    for (int i = tid; i < kCNum; i += blockDim.x)
        if (s_cnt[i]) atomicAdd(&p.counters[i], s_cnt[i]);
}

}  // namespace dwb
