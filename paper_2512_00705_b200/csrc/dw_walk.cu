// dw_walk.cu -- the walk hot path: K1 eRJS, K2 eRVS, K3 adaptive walker loop.
//
// One persistent kernel per run.  Each lane owns one walker at a time and
// keeps its WalkerState (walk_state.hpp:13-40) in registers for all steps;
// lanes claim walkers from a global queue with one warp-aggregated atomic
// (the run_queries scheduler, runtime.cpp:209-211).  Per step a lane reads
// one 32 B node record, makes the cost-model decision (cost_model.hpp:46-56)
// and samples:
//   * eRJS  (samplers.hpp:145-178): K trials are issued speculatively per
//     round -- Philox is a counter RNG, so trial t's (x, y) is known without
//     running trials < t -- their edge records load in parallel, and the
//     trials are then judged in order, stopping at the first accept.  The
//     node2vec / PR2 membership probe runs only when y falls between the two
//     candidate weights.  Paths, counters and draw counts are those of the
//     sequential reference.
//   * eRVS  (samplers.hpp:65-107, 112-137): rows below kCoopMinDegree run
//     serially in the lane; longer rows (and every eRJS cap fallback on them)
//     are handed to the whole warp through a ballot (FlexiWalker's mixed
//     mode): 32 lanes load a chunk of the row and resolve the 32 weights
//     (membership probes included) in parallel, then the A-ExpJ jump scan --
//     a short sequential chain of double subtractions -- runs warp-uniformly
//     over the chunk with shuffles.  ervs-nojump keys are independent per
//     neighbour and merge with a shuffle arg-max.
// Counters follow RunStats exactly (runtime.cpp:141-149).
#include <cfloat>

#include "dw_walk.cuh"

namespace dwb {

constexpr int kThreads = 256;
constexpr int kTrialBatch = 4;
constexpr uint32_t kCoopMinDegree = 32;
constexpr unsigned kFull = 0xFFFFFFFFu;
typedef unsigned long long ull;

__device__ __forceinline__ bool valid_w(double w) { return !(w < 0.0) && isfinite(w); }

// Graph::has_edge (graph.cpp:114-118): u in the sorted slice [begin, begin+d).
__device__ __forceinline__ bool has_edge(const EdgeRec* __restrict__ edges, ull begin, uint32_t d,
                                         uint32_t u) {
    if (d == 0) return false;
    ull base = begin;
    uint32_t n = d;
    while (n > 1) {
        const uint32_t half = n >> 1;
        if (load_col(edges + base + half) <= u) base += half;
        n -= half;
    }
    return load_col(edges + base) == u;
}

template <class M>
__device__ __forceinline__ uint16_t edge_label(const DevGraph& g, ull e) {
    if (!M::kUsesLabels) return 0;
    return g.labels ? __ldg(g.labels + e) : (uint16_t)0;
}

template <class M>
__device__ __forceinline__ double resolve(const WeightCase& wc, const Step& S, const DevGraph& g,
                                          uint32_t u) {
    if (!M::kSecondOrder || !wc.needs_member) return wc.w;
    return has_edge(g.edges, S.prev_begin, S.prev_degree, u) ? wc.w_in : wc.w_out;
}

__device__ __forceinline__ void raise_error(const WalkParams& p, int code, ull q) {
    if (atomicCAS(p.error, 0, code) == 0) *p.error_info = q;
}

// ---- K1: rejection trials (samplers.hpp:159-171) -------------------------
// status: 0 accepted, 1 cap exhausted (caller falls back to eRVS), <0 error
template <class M>
__device__ __forceinline__ int erjs_trials(const M& m, const Step& S, const WalkerKey& key,
                                           const DevGraph& g, double bound, ull cap,
                                           uint32_t& next, ull& trials, ull& alg_bytes) {
    ull t = 0;
    while (t < cap) {
        const int kk = (cap - t) < (ull)kTrialBatch ? (int)(cap - t) : kTrialBatch;
        EdgeRec er[kTrialBatch];
        uint16_t lab[kTrialBatch];
        double y[kTrialBatch];
#pragma unroll
        for (int k = 0; k < kTrialBatch; ++k) {
            if (k < kk) {
                const U4 b = walker_block(key, (uint32_t)(t + k));
                const ull x = bounded(lo64(b), S.degree);      // draw 2t:   bounded(d)
                y[k] = uniform01(hi64(b)) * bound;             // draw 2t+1: uniform01()*c
                er[k] = load_edge(g.edges + S.begin + x);
                lab[k] = edge_label<M>(g, S.begin + x);
            }
        }
#pragma unroll
        for (int k = 0; k < kTrialBatch; ++k) {
            if (k < kk) {
                const WeightCase wc = m.weight(S, er[k].col, er[k].h, lab[k]);
                // 32 B edge record + 32 B membership sector when u != prev (§8(d))
                alg_bytes += (M::kSecondOrder && S.has_prev() && er[k].col != S.prev) ? 64 : 32;
                bool acc;
                if (!wc.needs_member) {
                    if (!valid_w(wc.w)) {
                        trials = t + k;
                        return -kDevBadWeight;
                    }
                    acc = y[k] < wc.w;
                } else if (valid_w(wc.w_in) && valid_w(wc.w_out)) {
                    const double lo = wc.w_in < wc.w_out ? wc.w_in : wc.w_out;
                    const double hi = wc.w_in < wc.w_out ? wc.w_out : wc.w_in;
                    if (y[k] < lo)
                        acc = true;
                    else if (!(y[k] < hi))
                        acc = false;
                    else
                        acc = y[k] < resolve<M>(wc, S, g, er[k].col);
                } else {
                    const double w = resolve<M>(wc, S, g, er[k].col);
                    if (!valid_w(w)) {
                        trials = t + k;
                        return -kDevBadWeight;
                    }
                    acc = y[k] < w;
                }
                if (acc) {
                    next = er[k].col;
                    trials = t + k + 1;
                    return 0;
                }
            }
        }
        t += kk;
    }
    trials = cap;
    return 1;
}

// ---- K2 (lane form): eRVS with jumps, samplers.hpp:65-107 -----------------
template <class M>
__device__ int ervs_serial(const M& m, const Step& S, const WalkerKey& key, const DevGraph& g,
                           ull idx, uint32_t& next, ull& draws) {
    const ull idx0 = idx;
    double best_log_key = -DBL_MAX;
    uint32_t best = kInvalid;
    double skip = 0.0;
    bool have = false;
    for (uint32_t i = 0; i < S.degree; ++i) {
        const EdgeRec er = load_edge(g.edges + S.begin + i);
        const WeightCase wc = m.weight(S, er.col, er.h, edge_label<M>(g, S.begin + i));
        const double w = resolve<M>(wc, S, g, er.col);
        if (!valid_w(w)) return -kDevBadWeight;
        if (w == 0.0) continue;
        if (best == kInvalid) {
            best_log_key = log(open01(walker_draw(key, idx++))) / w;
            best = er.col;
            continue;
        }
        if (!have) {
            skip = log(open01(walker_draw(key, idx++))) / best_log_key;
            have = true;
        }
        skip -= w;
        if (skip <= 0.0) {
            const double floor_u = exp(w * best_log_key);
            const double u = floor_u + open01(walker_draw(key, idx++)) * (1.0 - floor_u);
            const double lk = log(u) / w;
            if (lk > best_log_key) {
                best_log_key = lk;
                best = er.col;
            }
            have = false;
        }
    }
    next = best;
    draws = idx - idx0;
    return 0;
}

// ---- eRVS without jumps, samplers.hpp:112-137 -----------------------------
template <class M>
__device__ int ervs_nojump_serial(const M& m, const Step& S, const WalkerKey& key,
                                  const DevGraph& g, ull idx0, uint32_t& next, ull& draws) {
    double best_log_key = -DBL_MAX;
    uint32_t best = kInvalid;
    for (uint32_t i = 0; i < S.degree; ++i) {
        const EdgeRec er = load_edge(g.edges + S.begin + i);
        const WeightCase wc = m.weight(S, er.col, er.h, edge_label<M>(g, S.begin + i));
        const double w = resolve<M>(wc, S, g, er.col);
        if (!valid_w(w)) return -kDevBadWeight;
        const double u = open01(walker_draw(key, idx0 + i));
        if (w == 0.0) continue;
        const double lk = log(u) / w;
        if (best == kInvalid || lk > best_log_key) {
            best_log_key = lk;
            best = er.col;
        }
    }
    next = best;
    draws = S.degree;
    return 0;
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
        if (in) w = resolve<M>(m.weight(S, er.col, er.h, lab), S, g, er.col);
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
__global__ void __launch_bounds__(kThreads) walk_kernel(const __grid_constant__ WalkParams p) {
    __shared__ ull s_cnt[kCNum];
    for (int i = threadIdx.x; i < kCNum; i += blockDim.x) s_cnt[i] = 0;
    __syncthreads();

    const M model(p.mp);
    const int lane = threadIdx.x & 31;
    const unsigned lt_mask = (1u << lane) - 1u;
    const DevGraph& g = p.g;

    bool active = false;
    bool drained = false;  // warp-uniform
    ull qi = 0;
    Step S;
    S.cur = S.prev = kInvalid;
    S.prev_degree = 0;
    S.prev_begin = 0;
    S.step = 0;
    S.degree = 0;
    S.begin = 0;
    S.hmax = S.hsum = 0.0;
    ull c_trials = 0, c_reads = 0, c_draws = 0, c_alg = 0;
    uint32_t c_queries = 0, c_qerr = 0, c_dead = 0, c_fb = 0;

    for (;;) {
        // ---- refill idle lanes: one atomic per warp (runtime.cpp:209-211)
        if (!drained) {
            if (__any_sync(kFull, *(volatile int*)p.error != 0)) drained = true;
            unsigned need = __ballot_sync(kFull, !active);
            while (need && !drained) {
                const int leader = __ffs(need) - 1;
                const int n = __popc(need);
                ull base = 0;
                if (lane == leader) base = atomicAdd(p.next_walker, (ull)n);
                base = __shfl_sync(kFull, base, leader);
                if (base + (ull)n >= p.nq) drained = true;
                if (!active) {
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
                                active = true;
                                qi = i;
                                S.cur = start;
                                S.prev = kInvalid;
                                S.prev_degree = 0;
                                S.prev_begin = 0;
                                S.step = 0;
                            }
                        }
                    }
                }
                need = __ballot_sync(kFull, !active);
            }
        }
        if (__ballot_sync(kFull, active) == 0) break;

        // ---- one step per active lane
        uint32_t next = kInvalid;
        bool stepping = false, need_warp = false, fell_back = false;
        ull trials = 1, reads = 0, draws = 0, draw_base = 0, alg = 0;
        const ull q = p.qid_base + qi;
        WalkerKey key{p.seed_lo, p.seed_hi, (uint32_t)q, (uint32_t)(q >> 32), S.step};
        if (active) {
            const NodeRec nr = load_node(g.nodes + S.cur);
            S.degree = nr.degree;
            S.begin = nr.begin;
            S.hmax = nr.hmax;
            S.hsum = nr.hsum;
            // §8(d): 32 B offsets + 4 B path write (+ 32 B aggregates when the
            // bound / cost model reads them)
            alg = 36 + ((MODE == kAdaptive || MODE == kForceErjs) && M::kAggregates ? 32 : 0);
            if (S.degree == 0) {  // runtime.cpp:70-71
                if (p.lengths) p.lengths[qi] = S.step + 1;
                active = false;
            } else {
                stepping = true;
                bool erjs = false;
                double bound = 0.0;
                if (MODE == kAdaptive) {  // decide_sampler, cost_model.hpp:46-56
                    if (M::kBoundable) {
                        bound = model.bound(S);
                        const double sum = model.wsum(S);
                        erjs = p.ratio * bound < sum;
                    }
                } else if (MODE == kForceErjs) {  // runtime.cpp:109-129
                    erjs = M::kBoundable;
                    if (erjs) bound = model.bound(S);
                }
                atomicAdd(&s_cnt[kCHist + 2 * degree_bucket(S.degree) + (erjs ? 1 : 0)], 1ull);
                bool ervs = !erjs;
                if (erjs) {
                    if (!(bound > 0.0) || !isfinite(bound)) {  // samplers.hpp:152-154
                        raise_error(p, kDevBadBound, q);
                        active = stepping = false;
                    } else {
                        const int st = erjs_trials(model, S, key, g, bound,
                                                   p.cap_per_degree * S.degree, next, trials, alg);
                        if (st < 0) {
                            raise_error(p, -st, q);
                            active = stepping = false;
                        } else {
                            reads = trials;
                            draws = 2 * trials;
                            if (st == 1) {  // cap overrun -> reservoir (samplers.hpp:172-177)
                                fell_back = true;
                                ervs = true;
                                draw_base = draws;
                            }
                        }
                    }
                }
                if (ervs && stepping) {
                    // σ(8d) + 32·min(d, ⌈d'/8⌉) when membership is needed (§8(d))
                    alg += ((8ull * S.degree + 31) / 32) * 32;
                    if (M::kSecondOrder && S.has_prev())
                        alg += 32ull * min((ull)S.degree, ((ull)S.prev_degree + 7) / 8);
                    if (S.degree >= kCoopMinDegree) {
                        need_warp = true;
                    } else {
                        ull dr = 0;
                        const int st = MODE == kErvsNoJump
                                           ? ervs_nojump_serial(model, S, key, g, draw_base, next, dr)
                                           : ervs_serial(model, S, key, g, draw_base, next, dr);
                        if (st < 0) {
                            raise_error(p, -st, q);
                            active = stepping = false;
                        }
                        reads += S.degree;
                        draws += dr;
                    }
                }
            }
        }

        // ---- warp-cooperative eRVS for long rows (ballot hand-off)
        unsigned coop = __ballot_sync(kFull, need_warp);
        while (coop) {
            const int L = __ffs(coop) - 1;
            coop &= coop - 1;
            Step T;
            T.cur = __shfl_sync(kFull, S.cur, L);
            T.prev = __shfl_sync(kFull, S.prev, L);
            T.prev_degree = __shfl_sync(kFull, S.prev_degree, L);
            T.prev_begin = __shfl_sync(kFull, S.prev_begin, L);
            T.step = __shfl_sync(kFull, S.step, L);
            T.degree = __shfl_sync(kFull, S.degree, L);
            T.begin = __shfl_sync(kFull, S.begin, L);
            T.hmax = __shfl_sync(kFull, S.hmax, L);
            T.hsum = __shfl_sync(kFull, S.hsum, L);
            WalkerKey K{p.seed_lo, p.seed_hi, __shfl_sync(kFull, key.q0, L),
                        __shfl_sync(kFull, key.q1, L), T.step};
            const ull db = __shfl_sync(kFull, draw_base, L);
            uint32_t nx = kInvalid;
            ull dr = 0;
            const int st = ervs_warp<M, MODE == kErvsNoJump>(model, T, K, g, db, nx, dr);
            if (lane == L) {
                if (st < 0) {
                    raise_error(p, -st, q);
                    active = stepping = false;
                }
                next = nx;
                reads += T.degree;
                draws += dr;
            }
        }

        // ---- counters + WalkerState::advance (runtime.cpp:141-150)
        if (stepping) {
            c_trials += trials;
            c_reads += reads;
            c_draws += draws;
            c_fb += fell_back ? 1u : 0u;
            c_alg += alg;
            if (next == kInvalid) {
                ++c_dead;
                if (p.lengths) p.lengths[qi] = S.step + 1;
                active = false;
            } else {
                S.prev = S.cur;
                S.prev_degree = S.degree;
                S.prev_begin = S.begin;
                S.cur = next;
                ++S.step;
                if (p.paths) p.paths[qi * p.stride + S.step] = next;
                if (S.step >= p.target) {
                    if (p.lengths) p.lengths[qi] = S.step + 1;
                    active = false;
                }
            }
        }
    }

    // ---- flush counters
    const ull v[8] = {c_queries, c_qerr, c_dead, c_trials, c_reads, c_draws, c_fb, c_alg};
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const ull s = warp_sum(v[k]);
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
