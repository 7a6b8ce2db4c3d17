// dw_walk.cu -- the walk hot path: K1 eRJS, K2 eRVS, K3 adaptive walker loop.
//
// One persistent kernel per run.  Each lane owns one walker at a time and
// keeps its WalkerState (walk_state.hpp:13-40) in registers for all steps;
// lanes claim walkers from a global queue with one warp-aggregated atomic
// (the run_queries scheduler, runtime.cpp:209-211).
//
// Latency structure.  A walk step is a chain of dependent random loads (node
// record -> rejection trials -> membership probe -> ...), and lanes of a warp
// need different numbers of them.  So the walker loop is a per-lane state
// machine in which every lane advances exactly ONE memory phase per
// iteration:
//     A  each lane computes the addresses its phase needs (ALU only)
//     B  all lanes issue their loads together (4 predicated 16 B LDGs)
//     C  each lane consumes its loads and picks its next phase (ALU only)
// so a warp iteration costs one memory latency no matter how the lanes are
// spread over phases, and no lane waits for another lane's chain.
// Phases:
//   NODE   one 32 B node record: degree, row begin, hash-set base, max/sum
//          aggregates; cost-model decision (decide_sampler,
//          cost_model.hpp:46-56).
//   TRIAL  eRJS (samplers.hpp:145-178): four trials issued at once -- Philox
//          is a counter RNG, so trial t's (x, y) is known without running the
//          trials before it -- then judged in order.  A trial whose outcome
//          hinges on the node2vec/PR2 membership test (y between the two
//          candidate weights) parks in MEMB.
//   MEMB   one 32 B hash-bucket probe (Graph::has_edge, dw_member.cuh).
//   VREC / VMEMB   eRVS on short rows (samplers.hpp:65-137), one neighbour per
//          iteration, exactly the reference's sequential jump logic.
//   COOP   rows >= kCoopMinDegree are handed to the whole warp through a
//          ballot (FlexiWalker's mixed mode): 32 lanes load a chunk and
//          resolve 32 weights in parallel, then the A-ExpJ jump scan runs
//          warp-uniformly over the chunk with shuffles.
// Paths, counters and draw counts equal the sequential reference on the same
// Philox stream (tests/test_gpu_parity.py).
#include <cfloat>

#include "dw_walk.cuh"

namespace dwb {

#ifndef DW_MIN_BLOCKS
#define DW_MIN_BLOCKS 1
#endif
constexpr int kThreads = 256;
constexpr int kSlots = 4;                 // 16 B loads per lane per iteration
constexpr uint32_t kCoopMinDegree = 64;
constexpr unsigned kFull = 0xFFFFFFFFu;
typedef unsigned long long ull;

enum Phase : uint32_t { P_IDLE = 0, P_NODE, P_TRIAL, P_MEMB, P_VREC, P_VMEMB, P_COOP };

__device__ __forceinline__ bool valid_w(double w) { return !(w < 0.0) && isfinite(w); }

template <class M>
__device__ __forceinline__ uint16_t edge_label(const DevGraph& g, ull e) {
    if (!M::kUsesLabels) return 0;
    return g.labels ? __ldg(g.labels + e) : (uint16_t)0;
}

__device__ __forceinline__ void raise_error(const WalkParams& p, int code, ull q) {
    if (atomicCAS(p.error, 0, code) == 0) *p.error_info = q;
}

__device__ __forceinline__ const uint4* slot_of(const EdgeRec* edges, ull e) {
    return reinterpret_cast<const uint4*>(edges + (e & ~1ull));
}
__device__ __forceinline__ uint32_t rec_col(const uint4& v, ull e) { return (e & 1) ? v.z : v.x; }
__device__ __forceinline__ float rec_h(const uint4& v, ull e) {
    return __uint_as_float((e & 1) ? v.w : v.y);
}
__device__ __forceinline__ bool has8(const uint4& a, const uint4& b, uint32_t u) {
    return a.x == u || a.y == u || a.z == u || a.w == u || b.x == u || b.y == u || b.z == u ||
           b.w == u;
}

// ---- K2 (warp form): one row, 32 lanes; all lanes call with equal args ----
template <class M, bool NOJUMP>
__device__ int ervs_warp(const M& m, const Step& S, const WalkerKey& key, const DevGraph& g,
                         ull idx0, uint32_t& next, ull& draws) {
    const int lane = threadIdx.x & 31;
    ull idx = idx0;
    double best_log_key = -DBL_MAX;
    uint32_t best = kInvalid;
    double skip = 0.0;
    bool have = false;
    // software pipeline: chunk c+1's records load while chunk c is judged
    EdgeRec nxt{kInvalid, 0.f};
    uint16_t nlab = 0;
    if ((uint32_t)lane < S.degree) {
        nxt = load_edge(g.edges + S.begin + lane);
        nlab = edge_label<M>(g, S.begin + lane);
    }
    for (uint32_t base = 0; base < S.degree; base += 32) {
        const uint32_t i = base + lane;
        const bool in = i < S.degree;
        const EdgeRec er = nxt;
        const uint16_t lab = nlab;
        if (i + 32 < S.degree) {
            nxt = load_edge(g.edges + S.begin + i + 32);
            nlab = edge_label<M>(g, S.begin + i + 32);
        }
        double w = 0.0;
        if (in) {
            const WeightCase wc = m.weight(S, er.col, er.h, lab);
            w = (!M::kSecondOrder || !wc.needs_member)
                    ? wc.w
                    : (member(g, S.prev_begin, S.prev_degree, S.prev_hoff, er.col) ? wc.w_in
                                                                                  : wc.w_out);
        }
        if (__any_sync(kFull, in && !valid_w(w))) return -kDevBadWeight;
        if (NOJUMP) {
            // every neighbour draws its own key (draw idx0 + i), zero weights included
            double lk = -DBL_MAX;
            int has = 0;
            if (in) {
                const double u = open01(walker_draw(key, idx0 + i));
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
            }
        } else {
            const uint32_t n = S.degree - base < 32u ? S.degree - base : 32u;
            for (uint32_t j = 0; j < n; ++j) {
                const double wj = __shfl_sync(kFull, w, j);
                const uint32_t uj = __shfl_sync(kFull, er.col, j);
                if (wj == 0.0) continue;
                if (best == kInvalid) {
                    best_log_key = log(open01(walker_draw(key, idx++))) / wj;
                    best = uj;
                    continue;
                }
                if (!have) {
                    skip = log(open01(walker_draw(key, idx++))) / best_log_key;
                    have = true;
                }
                skip -= wj;
                if (skip <= 0.0) {
                    const double floor_u = exp(wj * best_log_key);
                    const double u = floor_u + open01(walker_draw(key, idx++)) * (1.0 - floor_u);
                    const double lk = log(u) / wj;
                    if (lk > best_log_key) {
                        best_log_key = lk;
                        best = uj;
                    }
                    have = false;
                }
            }
        }
    }
    next = best;
    draws = NOJUMP ? (ull)S.degree : idx - idx0;
    return 0;
}

__device__ __forceinline__ ull warp_sum(ull v) {
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    return v;
}

// ---- K3: adaptive walker loop (runtime.cpp:59-153 + 192-247) --------------
template <class M, int MODE>
__global__ void __launch_bounds__(kThreads, DW_MIN_BLOCKS) walk_kernel(const __grid_constant__ WalkParams p) {
    constexpr bool kNoJump = MODE == kErvsNoJump;
    __shared__ ull s_cnt[kCNum];
    for (int i = threadIdx.x; i < kCNum; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();

    const M model(p.mp);
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const DevGraph& g = p.g;

    uint32_t phase = P_IDLE;
    bool drained = false;  // warp-uniform
    ull qi = 0;
    Step S;
    S.cur = S.prev = kInvalid;
    S.prev_degree = S.prev_hoff = S.step = S.degree = S.hoff = 0;
    S.prev_begin = S.begin = 0;
    S.hmax = S.hsum = 0.0;
    // eRJS state
    double bound = 0.0;
    ull t = 0, cap = 0;
    // parked membership test (TRIAL->MEMB, VREC->VMEMB)
    uint32_t pu = 0, mb = 0;
    double py = 0.0, pw_in = 0.0, pw_out = 0.0;
    // eRVS state (samplers.hpp:72-75)
    uint32_t vi = 0, best = kInvalid;
    double best_key = -DBL_MAX, skip = 0.0;
    bool have = false;
    ull didx = 0;
    // counters
    ull c_trials = 0, c_reads = 0, c_draws = 0, c_alg = 0;
    uint32_t c_queries = 0, c_qerr = 0, c_dead = 0, c_fb = 0;

    // outcome of one walk step (runtime.cpp:141-150 + walk_state.hpp:33-39)
    auto finish_step = [&](uint32_t next) {
        if (next == kInvalid) {
            ++c_dead;
            if (p.lengths) p.lengths[qi] = S.step + 1;
            phase = P_IDLE;
            return;
        }
        S.prev = S.cur;
        S.prev_degree = S.degree;
        S.prev_begin = S.begin;
        S.prev_hoff = S.hoff;
        S.cur = next;
        ++S.step;
        if (p.paths) p.paths[qi * p.stride + S.step] = next;
        if (S.step >= p.target) {
            if (p.lengths) p.lengths[qi] = S.step + 1;
            phase = P_IDLE;
        } else {
            phase = P_NODE;
        }
    };
    auto start_ervs = [&](ull draw_base) {
        vi = 0;
        best = kInvalid;
        best_key = -DBL_MAX;
        skip = 0.0;
        have = false;
        didx = draw_base;
        // §8(d): σ(8d) + 32·min(d, ⌈d'/8⌉) when membership is needed
        c_alg += ((8ull * S.degree + 31) / 32) * 32;
        if (M::kSecondOrder && S.has_prev())
            c_alg += 32ull * min((ull)S.degree, ((ull)S.prev_degree + 7) / 8);
        phase = S.degree >= kCoopMinDegree ? P_COOP : P_VREC;
    };
    auto key_of = [&]() {
        const ull q = p.qid_base + qi;
        return WalkerKey{p.seed_lo, p.seed_hi, (uint32_t)q, (uint32_t)(q >> 32), S.step};
    };
    // one neighbour of the reservoir scan (samplers.hpp:78-102 / 122-133)
    auto ervs_visit = [&](uint32_t u, double w) {
        ++c_reads;
        if (kNoJump) {
            const double r = open01(walker_draw(key_of(), didx + vi));
            ++c_draws;
            if (w != 0.0) {
                const double lk = log(r) / w;
                if (best == kInvalid || lk > best_key) {
                    best_key = lk;
                    best = u;
                }
            }
        } else if (w != 0.0) {
            const WalkerKey key = key_of();
            if (best == kInvalid) {
                best_key = log(open01(walker_draw(key, didx++))) / w;
                ++c_draws;
                best = u;
            } else {
                if (!have) {
                    skip = log(open01(walker_draw(key, didx++))) / best_key;
                    ++c_draws;
                    have = true;
                }
                skip -= w;
                if (skip <= 0.0) {
                    const double floor_u = exp(w * best_key);
                    const double uu = floor_u + open01(walker_draw(key, didx++)) * (1.0 - floor_u);
                    ++c_draws;
                    const double lk = log(uu) / w;
                    if (lk > best_key) {
                        best_key = lk;
                        best = u;
                    }
                    have = false;
                }
            }
        }
        if (++vi == S.degree) finish_step(best);
    };
    auto park = [&](uint32_t u, double y, double w_in, double w_out, uint32_t next_phase) {
        pu = u;
        py = y;
        pw_in = w_in;
        pw_out = w_out;
        mb = S.prev_degree > kScanMax ? hash_bucket(u, hash_log2_buckets(S.prev_degree)) : 0;
        phase = next_phase;
    };
    auto fail = [&](int code) {
        raise_error(p, code, p.qid_base + qi);
        phase = P_IDLE;
    };

    for (;;) {
        // ---- refill idle lanes: one atomic per warp (runtime.cpp:209-211)
        if (!drained) {
            if (__any_sync(kFull, *(volatile int*)p.error != 0)) drained = true;
            unsigned need = __ballot_sync(kFull, phase == P_IDLE);
            while (need && !drained) {
                const int leader = __ffs(need) - 1;
                const int n = __popc(need);
                ull base = 0;
                if (lane == leader) base = atomicAdd(p.next_walker, (ull)n);
                base = __shfl_sync(kFull, base, leader);
                if (base + (ull)n >= p.nq) drained = true;
                if (phase == P_IDLE) {
                    const ull i = base + (ull)__popc(need & lt_mask);
                    if (i < p.nq) {
                        ++c_queries;
                        const uint32_t start = p.queries[i];
                        if (start >= g.nv) {  // runtime.cpp:213-217
                            ++c_qerr;
                            if (p.lengths) p.lengths[i] = 0;
                        } else {
                            if (p.paths) p.paths[i * p.stride] = start;
                            if (p.target == 0) {
                                if (p.lengths) p.lengths[i] = 1;
                            } else {
                                phase = P_NODE;
                                qi = i;
                                S.cur = start;
                                S.prev = kInvalid;
                                S.prev_degree = S.prev_hoff = 0;
                                S.prev_begin = 0;
                                S.step = 0;
                            }
                        }
                    }
                }
                need = __ballot_sync(kFull, phase == P_IDLE);
            }
        } else if (*(volatile int*)p.error != 0) {
            phase = P_IDLE;  // abandon the run after the first error
        }
        if (__ballot_sync(kFull, phase != P_IDLE) == 0) break;

        // ---- A: addresses of this iteration's loads
        const uint4* a[kSlots] = {nullptr, nullptr, nullptr, nullptr};
        const uint16_t* la[kSlots] = {nullptr, nullptr, nullptr, nullptr};
        double ty[kSlots];
        ull te[kSlots];
        int kk = 0;
        if (phase == P_NODE) {
            a[0] = reinterpret_cast<const uint4*>(g.nodes + S.cur);
            a[1] = a[0] + 1;
        } else if (phase == P_TRIAL) {
            const WalkerKey key = key_of();
            kk = (cap - t) < (ull)kSlots ? (int)(cap - t) : kSlots;
#pragma unroll
            for (int k = 0; k < kSlots; ++k) {
                if (k < kk) {
                    const U4 b = walker_block(key, (uint32_t)(t + k));
                    te[k] = S.begin + bounded(lo64(b), S.degree);  // draw 2t:   bounded(d)
                    ty[k] = uniform01(hi64(b)) * bound;            // draw 2t+1: uniform01()*c
                    a[k] = slot_of(g.edges, te[k]);
                    if (M::kUsesLabels && g.labels) la[k] = g.labels + te[k];
                }
            }
        } else if (phase == P_MEMB || phase == P_VMEMB) {
            if (S.prev_degree <= kScanMax) {
                const ull e0 = S.prev_begin & ~1ull;
                const ull n = S.prev_begin + S.prev_degree - e0;
#pragma unroll
                for (int k = 0; k < kSlots; ++k)
                    if ((ull)(2 * k) < n) a[k] = slot_of(g.edges, e0 + 2 * k);
            } else {
                a[0] = reinterpret_cast<const uint4*>(g.hslots + 8ull * (S.prev_hoff + mb));
                a[1] = a[0] + 1;
            }
        } else if (phase == P_VREC) {
            te[0] = S.begin + vi;
            a[0] = slot_of(g.edges, te[0]);
            if (M::kUsesLabels && g.labels) la[0] = g.labels + te[0];
        }

        // ---- B: issue every lane's loads together
        uint4 v[kSlots];
        uint16_t lb[kSlots];
#pragma unroll
        for (int k = 0; k < kSlots; ++k) {
            v[k] = a[k] ? __ldg(a[k]) : make_uint4(0, 0, 0, 0);
            lb[k] = la[k] ? __ldg(la[k]) : (uint16_t)0;
        }

        // ---- C: consume
        if (phase == P_NODE) {
            S.begin = (ull)v[0].x | ((ull)v[0].y << 32);
            S.degree = v[0].z;
            S.hoff = v[0].w;
            S.hmax = __hiloint2double((int)v[1].y, (int)v[1].x);
            S.hsum = __hiloint2double((int)v[1].w, (int)v[1].z);
            if (S.degree == 0) {  // runtime.cpp:70-71
                if (p.lengths) p.lengths[qi] = S.step + 1;
                phase = P_IDLE;
            } else {
                bool erjs = false;
                if (MODE == kAdaptive) {  // decide_sampler, cost_model.hpp:46-56
                    if (M::kBoundable) {
                        bound = model.bound(S);
                        erjs = p.ratio * bound < model.wsum(S);
                    }
                } else if (MODE == kForceErjs) {  // runtime.cpp:109-129
                    erjs = M::kBoundable;
                    if (erjs) bound = model.bound(S);
                }
                atomicAdd(&s_cnt[kCHist + 2 * degree_bucket(S.degree) + (erjs ? 1 : 0)], 1ull);
                // §8(d): 32 B offsets + 4 B path write (+ 32 B aggregates)
                c_alg += 36 + ((MODE == kAdaptive || MODE == kForceErjs) && M::kAggregates ? 32 : 0);
                if (erjs) {
                    if (!(bound > 0.0) || !isfinite(bound)) {  // samplers.hpp:152-154
                        fail(kDevBadBound);
                    } else {
                        t = 0;
                        cap = p.cap_per_degree * S.degree;
                        phase = P_TRIAL;
                        if (cap == 0) {  // immediate cap overrun
                            ++c_fb;
                            start_ervs(0);
                        }
                    }
                } else {
                    ++c_trials;  // single-shot kernels report one trial (samplers.hpp:22)
                    start_ervs(0);
                }
            }
        } else if (phase == P_TRIAL) {
            bool done = false;
#pragma unroll
            for (int k = 0; k < kSlots; ++k) {
                if (k < kk && !done) {
                    const uint32_t u = rec_col(v[k], te[k]);
                    const WeightCase wc = model.weight(S, u, rec_h(v[k], te[k]), lb[k]);
                    // 32 B edge record + 32 B membership sector when u != prev (§8(d))
                    c_alg += (M::kSecondOrder && S.has_prev() && u != S.prev) ? 64 : 32;
                    ++c_trials;
                    ++c_reads;
                    c_draws += 2;
                    if (!wc.needs_member) {
                        if (!valid_w(wc.w)) {
                            fail(kDevBadWeight);
                            done = true;
                        } else if (ty[k] < wc.w) {
                            done = true;
                            finish_step(u);
                        }
                    } else {
                        const double lo = wc.w_in < wc.w_out ? wc.w_in : wc.w_out;
                        const double hi = wc.w_in < wc.w_out ? wc.w_out : wc.w_in;
                        const bool ok = valid_w(wc.w_in) && valid_w(wc.w_out);
                        if (ok && ty[k] < lo) {
                            done = true;
                            finish_step(u);
                        } else if (!ok || ty[k] < hi) {  // outcome hinges on u in N(prev)
                            done = true;
                            t += k + 1;
                            park(u, ty[k], wc.w_in, wc.w_out, P_MEMB);
                        }
                    }
                }
            }
            if (!done) {
                t += kk;
                if (t >= cap) {  // cap overrun -> reservoir with the same stream
                    ++c_fb;
                    start_ervs(2 * t);
                }
            }
        } else if (phase == P_MEMB || phase == P_VMEMB) {
            int hit = -1;  // -1: probe the next bucket
            if (S.prev_degree <= kScanMax) {
                const ull e0 = S.prev_begin & ~1ull;
                const uint32_t off = (uint32_t)(S.prev_begin - e0);
                bool f = false;
#pragma unroll
                for (int k = 0; k < kSlots; ++k) {
                    const uint32_t j0 = 2 * k, j1 = 2 * k + 1;
                    f |= (j0 >= off && j0 < off + S.prev_degree && v[k].x == pu);
                    f |= (j1 >= off && j1 < off + S.prev_degree && v[k].z == pu);
                }
                hit = f ? 1 : 0;
            } else if (has8(v[0], v[1], pu)) {
                hit = 1;
            } else if (v[1].w == kHashEmpty) {
                hit = 0;
            } else {
                mb = (mb + 1) & ((1u << hash_log2_buckets(S.prev_degree)) - 1u);
            }
            if (hit >= 0) {
                const double w = hit ? pw_in : pw_out;
                if (!valid_w(w)) {
                    fail(kDevBadWeight);
                } else if (phase == P_MEMB) {
                    if (py < w) {
                        finish_step(pu);
                    } else if (t >= cap) {
                        ++c_fb;
                        start_ervs(2 * t);
                    } else {
                        phase = P_TRIAL;
                    }
                } else {
                    phase = P_VREC;
                    ervs_visit(pu, w);
                }
            }
        } else if (phase == P_VREC) {
            const uint32_t u = rec_col(v[0], te[0]);
            const WeightCase wc = model.weight(S, u, rec_h(v[0], te[0]), lb[0]);
            if (M::kSecondOrder && wc.needs_member) {
                park(u, 0.0, wc.w_in, wc.w_out, P_VMEMB);
            } else if (!valid_w(wc.w)) {
                fail(kDevBadWeight);
            } else {
                ervs_visit(u, wc.w);
            }
        }

        // ---- warp-cooperative eRVS for long rows (ballot hand-off)
        unsigned coop = __ballot_sync(kFull, phase == P_COOP);
        while (coop) {
            const int L = __ffs(coop) - 1;
            coop &= coop - 1;
            Step T;
            T.cur = __shfl_sync(kFull, S.cur, L);
            T.prev = __shfl_sync(kFull, S.prev, L);
            T.prev_degree = __shfl_sync(kFull, S.prev_degree, L);
            T.prev_begin = __shfl_sync(kFull, S.prev_begin, L);
            T.prev_hoff = __shfl_sync(kFull, S.prev_hoff, L);
            T.step = __shfl_sync(kFull, S.step, L);
            T.degree = __shfl_sync(kFull, S.degree, L);
            T.hoff = __shfl_sync(kFull, S.hoff, L);
            T.begin = __shfl_sync(kFull, S.begin, L);
            T.hmax = __shfl_sync(kFull, S.hmax, L);
            T.hsum = __shfl_sync(kFull, S.hsum, L);
            const ull q = p.qid_base + __shfl_sync(kFull, qi, L);
            const WalkerKey K{p.seed_lo, p.seed_hi, (uint32_t)q, (uint32_t)(q >> 32), T.step};
            const ull db = __shfl_sync(kFull, didx, L);
            uint32_t nx = kInvalid;
            ull dr = 0;
            const int st = ervs_warp<M, kNoJump>(model, T, K, g, db, nx, dr);
            if (lane == L) {
                if (st < 0) {
                    fail(-st);
                } else {
                    c_reads += T.degree;
                    c_draws += dr;
                    finish_step(nx);
                }
            }
        }
    }

    // ---- flush counters
    const ull cv[8] = {c_queries, c_qerr, c_dead, c_trials, c_reads, c_draws, c_fb, c_alg};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const ull s = warp_sum(cv[k]);
        if (lane == 0 && s) atomicAdd(&s_cnt[k], s);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < kCNum; i += blockDim.x)
        if (s_cnt[i]) atomicAdd(&p.counters[i], s_cnt[i]);
}

template <class M, int MODE>
static cudaError_t launch_t(const WalkParams& p, int num_sms, cudaStream_t stream) {
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, walk_kernel<M, MODE>,
                                                                  kThreads, 0);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) per_sm = 1;
    unsigned long long blocks = (unsigned long long)num_sms * per_sm;
    const unsigned long long need = (p.nq + kThreads - 1) / kThreads;
    if (need < blocks) blocks = need ? need : 1;
    walk_kernel<M, MODE><<<(unsigned)blocks, kThreads, 0, stream>>>(p);
    return cudaGetLastError();
}

template <class M>
static cudaError_t launch_m(int mode, const WalkParams& p, int num_sms, cudaStream_t s) {
    switch (mode) {
    case kAdaptive: return launch_t<M, kAdaptive>(p, num_sms, s);
    case kForceErvs: return launch_t<M, kForceErvs>(p, num_sms, s);
    case kForceErjs: return launch_t<M, kForceErjs>(p, num_sms, s);
    case kErvsNoJump: return launch_t<M, kErvsNoJump>(p, num_sms, s);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_walk(int kind, bool weighted, int mode, const WalkParams& p, int num_sms,
                        cudaStream_t s) {
    switch (kind) {
    case 0: return weighted ? launch_m<StaticModel<true>>(mode, p, num_sms, s)
                            : launch_m<StaticModel<false>>(mode, p, num_sms, s);
    case 1: return weighted ? launch_m<Node2VecModel<true>>(mode, p, num_sms, s)
                            : launch_m<Node2VecModel<false>>(mode, p, num_sms, s);
    case 2: return weighted ? launch_m<MetaPathModel<true>>(mode, p, num_sms, s)
                            : launch_m<MetaPathModel<false>>(mode, p, num_sms, s);
    case 3: return weighted ? launch_m<Pr2Model<true>>(mode, p, num_sms, s)
                            : launch_m<Pr2Model<false>>(mode, p, num_sms, s);
    }
    return cudaErrorInvalidValue;
}

}  // namespace dwb
