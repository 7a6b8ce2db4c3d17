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
//     A  each lane issues the 16 B gathers its phase needs as cp.async
//        (LDGSTS) into its own shared-memory landing slots -- no registers
//        are tied up by loads in flight, so many gathers overlap per lane
//     B  cp.async.wait_all
//     C  each lane consumes its slots and picks its next phase
// so a warp iteration costs one memory latency no matter how the lanes are
// spread over phases, and no lane waits for another lane's chain.
// Phases:
//   NODE   one 32 B node record: degree, row begin, hash-set base, max/sum
//          aggregates; cost-model decision (decide_sampler,
//          cost_model.hpp:46-56).
//   TRIAL  eRJS (samplers.hpp:145-178): kSlots trials issued at once --
//          Philox is a counter RNG, so trial t's (x, y) is known without
//          running the trials before it -- then judged in order.  A trial
//          whose outcome hinges on the node2vec/PR2 membership test (y between
//          the two candidate weights) parks in MEMB.
//   MEMB   one 32 B hash-bucket probe (Graph::has_edge, dw_member.cuh), or a
//          scan of a <= 6-record row.
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
#define DW_MIN_BLOCKS 3
#endif
#ifndef DW_SLOTS
#define DW_SLOTS 4
#endif
constexpr int kThreads = 256;
constexpr int kSlots = DW_SLOTS;          // 16 B gathers per lane per iteration
constexpr uint32_t kCoopMinDegree = 64;
constexpr unsigned kFull = 0xFFFFFFFFu;
typedef unsigned long long ull;

enum Phase : uint32_t { P_IDLE = 0, P_NODE, P_TRIAL, P_MEMB, P_VREC, P_VMEMB, P_COOP };
// per-lane counters kept in shared memory (runtime.cpp:141-145)
enum LaneCounter : int { LC_QUERIES = 0, LC_QERR, LC_DEAD, LC_TRIALS, LC_READS, LC_DRAWS, LC_FB,
                         LC_ALG, LC_NUM };

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
__device__ __forceinline__ bool has8(const uint4& a, const uint4& b, uint32_t u) {
    return a.x == u || a.y == u || a.z == u || a.w == u || b.x == u || b.y == u || b.z == u ||
           b.w == u;
}

// ---- K2 (warp form): one row, 32 lanes; all lanes call with equal args ----
template <class M, bool NOJUMP>
__device__ __noinline__ int ervs_warp(const M& m, const Step& S, const WalkerKey& key,
                                      const DevGraph& g, ull idx0, uint32_t& next, ull& draws) {
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

// ---- K2 (lane form): one neighbour of the reservoir scan ------------------
// samplers.hpp:78-102 (jump) / 122-133 (no jump).  Kept out of line: it holds
// the log/exp code, which the hot eRJS loop never needs.
struct ErvsState {
    double best_key, skip;
    ull didx;       // next draw index of this step's stream
    uint32_t best;
    uint32_t have;  // threshold drawn
    uint32_t draws; // draws made by this call
};

template <bool NOJUMP>
__device__ __noinline__ ErvsState ervs_visit(ErvsState s, const WalkerKey key, uint32_t vi,
                                             uint32_t u, double w) {
    s.draws = 0;
    if (NOJUMP) {
        const double r = open01(walker_draw(key, s.didx + vi));
        s.draws = 1;
        if (w != 0.0) {
            const double lk = log(r) / w;
            if (s.best == kInvalid || lk > s.best_key) {
                s.best_key = lk;
                s.best = u;
            }
        }
        return s;
    }
    if (w == 0.0) return s;
    if (s.best == kInvalid) {
        s.best_key = log(open01(walker_draw(key, s.didx++))) / w;
        s.draws = 1;
        s.best = u;
        return s;
    }
    if (!s.have) {
        s.skip = log(open01(walker_draw(key, s.didx++))) / s.best_key;
        s.draws = 1;
        s.have = 1;
    }
    s.skip -= w;
    if (s.skip <= 0.0) {
        const double floor_u = exp(w * s.best_key);
        const double uu = floor_u + open01(walker_draw(key, s.didx++)) * (1.0 - floor_u);
        ++s.draws;
        const double lk = log(uu) / w;
        if (lk > s.best_key) {
            s.best_key = lk;
            s.best = u;
        }
        s.have = 0;
    }
    return s;
}

__device__ __forceinline__ ull warp_sum(ull v) {
#pragma unroll
    for (int off = 16; off; off >>= 1) v += __shfl_xor_sync(kFull, v, off);
    return v;
}

// ---- K3: adaptive walker loop (runtime.cpp:59-153 + 192-247) --------------
template <class M, int MODE>
__global__ void __launch_bounds__(kThreads, DW_MIN_BLOCKS)
    walk_kernel(const __grid_constant__ WalkParams p) {
    constexpr bool kNoJump = MODE == kErvsNoJump;
    __shared__ uint4 s_slot[kSlots][kThreads];   // cp.async landing zone, [slot][lane]
    __shared__ double s_y[kSlots][kThreads];     // y of the trials in flight
    __shared__ uint32_t s_lab[kSlots][kThreads]; // label words (MetaPath)
    __shared__ ull s_lc[LC_NUM][kThreads];       // per-lane RunStats counters
    __shared__ ull s_cnt[kCNum];
    const int tid = threadIdx.x;
    for (int i = tid; i < kCNum; i += blockDim.x) s_cnt[i] = 0;
#pragma unroll
    for (int c = 0; c < LC_NUM; ++c) s_lc[c][tid] = 0;
    __syncthreads();
#define LC(c) s_lc[c][tid]

    const M model(p.mp);
    const int lane = tid & 31;
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
    // TRIAL/MEMB: t trials judged, bound, parked y.  VREC/VMEMB: eRVS state.
    ull t = 0;
    double bound = 0.0, py = 0.0;
    ErvsState ev{0.0, 0.0, 0, kInvalid, 0, 0};
    uint32_t vi = 0;
    // parked membership test (TRIAL->MEMB, VREC->VMEMB)
    uint32_t pu = 0, mb = 0;
    float ph = 0.f;
    uint32_t kk = 0, sel = 0;

    // outcome of one walk step (runtime.cpp:141-150 + walk_state.hpp:33-39)
    auto finish_step = [&](uint32_t next) {
        if (next == kInvalid) {
            ++LC(LC_DEAD);
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
        ev.best = kInvalid;
        ev.best_key = -DBL_MAX;
        ev.skip = 0.0;
        ev.have = 0;
        ev.didx = draw_base;
        // §8(d): σ(8d) + 32·min(d, ⌈d'/8⌉) when membership is needed
        ull alg = ((8ull * S.degree + 31) / 32) * 32;
        if (M::kSecondOrder && S.has_prev())
            alg += 32ull * min((ull)S.degree, ((ull)S.prev_degree + 7) / 8);
        LC(LC_ALG) += alg;
        phase = S.degree >= kCoopMinDegree ? P_COOP : P_VREC;
    };
    auto key_of = [&]() {
        const ull q = p.qid_base + qi;
        return WalkerKey{p.seed_lo, p.seed_hi, (uint32_t)q, (uint32_t)(q >> 32), S.step};
    };
    auto visit = [&](uint32_t u, double w) {
        ev = ervs_visit<kNoJump>(ev, key_of(), vi, u, w);
        LC(LC_DRAWS) += ev.draws;
        ++LC(LC_READS);
        if (++vi == S.degree) finish_step(ev.best);
    };
    auto park = [&](uint32_t u, float h, double y, uint32_t next_phase) {
        pu = u;
        ph = h;
        py = y;
        mb = S.prev_degree > kScanMax ? hash_bucket(u, hash_log2_buckets(S.prev_degree)) : 0;
        phase = next_phase;
    };
    auto fail = [&](int code) {
        raise_error(p, code, p.qid_base + qi);
        phase = P_IDLE;
    };

    for (;;) {
        // ---- refill idle lanes: one atomic per warp (runtime.cpp:209-211)
        unsigned need = __ballot_sync(kFull, phase == P_IDLE);
        if (need && !drained) {
            if (*(volatile int*)p.error != 0) drained = true;  // abandon after an error
            drained = __any_sync(kFull, drained);
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
                        ++LC(LC_QUERIES);
                        const uint32_t start = p.queries[i];
                        if (start >= g.nv) {  // runtime.cpp:213-217
                            ++LC(LC_QERR);
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
        }
        if (__ballot_sync(kFull, phase != P_IDLE) == 0) break;

        // ---- A: issue this iteration's gathers
        if (phase == P_NODE) {
            const char* nr = reinterpret_cast<const char*>(g.nodes + S.cur);
            cp16(&s_slot[0][tid], nr);
            cp16(&s_slot[1][tid], nr + 16);
        } else if (phase == P_TRIAL) {
            const WalkerKey key = key_of();
            const ull cap = p.cap_per_degree * S.degree;
            kk = (cap - t) < (ull)kSlots ? (uint32_t)(cap - t) : (uint32_t)kSlots;
            sel = 0;
#pragma unroll 1
            for (uint32_t k = 0; k < kk; ++k) {
                const U4 b = walker_block(key, (uint32_t)(t + k));
                const ull e = S.begin + bounded(lo64(b), S.degree);  // draw 2t:   bounded(d)
                s_y[k][tid] = uniform01(hi64(b)) * bound;             // draw 2t+1: uniform01()*c
                sel |= (uint32_t)(e & 1) << k;
                cp16(&s_slot[k][tid], pair_of(g.edges, e));
                if (M::kUsesLabels && g.labels) cp4(&s_lab[k][tid], g.labels + (e & ~1ull));
            }
        } else if (phase == P_MEMB || phase == P_VMEMB) {
            if (S.prev_degree <= kScanMax) {
                const ull e0 = S.prev_begin & ~1ull;
                const ull n = S.prev_begin + S.prev_degree - e0;
#pragma unroll
                for (int k = 0; k < 4; ++k)
                    if ((ull)(2 * k) < n) cp16(&s_slot[k][tid], g.edges + e0 + 2 * k);
            } else {
                const uint32_t* b = g.hslots + 8ull * (S.prev_hoff + mb);
                cp16(&s_slot[0][tid], b);
                cp16(&s_slot[1][tid], b + 4);
            }
        } else if (phase == P_VREC) {
            const ull e = S.begin + vi;
            sel = (uint32_t)(e & 1);
            cp16(&s_slot[0][tid], pair_of(g.edges, e));
            if (M::kUsesLabels && g.labels) cp4(&s_lab[0][tid], g.labels + (e & ~1ull));
        }
        // ---- B
        cp_wait_all();

        // ---- C: consume
        if (phase == P_NODE) {
            const uint4 v0 = s_slot[0][tid], v1 = s_slot[1][tid];
            S.begin = (ull)v0.x | ((ull)v0.y << 32);
            S.degree = v0.z;
            S.hoff = v0.w;
            S.hmax = __hiloint2double((int)v1.y, (int)v1.x);
            S.hsum = __hiloint2double((int)v1.w, (int)v1.z);
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
                LC(LC_ALG) +=
                    36 + ((MODE == kAdaptive || MODE == kForceErjs) && M::kAggregates ? 32 : 0);
                if (erjs) {
                    if (!(bound > 0.0) || !isfinite(bound)) {  // samplers.hpp:152-154
                        fail(kDevBadBound);
                    } else {
                        t = 0;
                        phase = P_TRIAL;
                        if (p.cap_per_degree == 0) {  // immediate cap overrun
                            ++LC(LC_FB);
                            start_ervs(0);
                        }
                    }
                } else {
                    ++LC(LC_TRIALS);  // single-shot kernels report one trial (samplers.hpp:22)
                    start_ervs(0);
                }
            }
        } else if (phase == P_TRIAL) {
            uint32_t k = 0;
            for (; k < kk; ++k) {
                const uint4 v = s_slot[k][tid];
                const bool odd = (sel >> k) & 1;
                const uint32_t u = odd ? v.z : v.x;
                const float h = __uint_as_float(odd ? v.w : v.y);
                const uint16_t lab =
                    M::kUsesLabels ? (uint16_t)(odd ? (s_lab[k][tid] >> 16) : s_lab[k][tid]) : 0;
                const double y = s_y[k][tid];
                const WeightCase wc = model.weight(S, u, h, lab);
                // 32 B edge record + 32 B membership sector when u != prev (§8(d))
                LC(LC_ALG) += (M::kSecondOrder && S.has_prev() && u != S.prev) ? 64 : 32;
                if (!wc.needs_member) {
                    if (!valid_w(wc.w)) {
                        fail(kDevBadWeight);
                        break;
                    }
                    if (y < wc.w) {
                        finish_step(u);
                        break;
                    }
                } else {
                    const double lo = wc.w_in < wc.w_out ? wc.w_in : wc.w_out;
                    const double hi = wc.w_in < wc.w_out ? wc.w_out : wc.w_in;
                    const bool ok = valid_w(wc.w_in) && valid_w(wc.w_out);
                    if (ok && y < lo) {
                        finish_step(u);
                        break;
                    }
                    if (!ok || y < hi) {  // outcome hinges on u in N(prev)
                        park(u, h, y, P_MEMB);
                        break;
                    }
                }
            }
            const uint32_t judged = k < kk ? k + 1 : kk;
            t += judged;
            LC(LC_TRIALS) += judged;
            LC(LC_READS) += judged;
            LC(LC_DRAWS) += 2 * judged;
            if (phase == P_TRIAL && t >= p.cap_per_degree * S.degree) {
                ++LC(LC_FB);  // cap overrun -> reservoir with the same stream
                start_ervs(2 * t);
            }
        } else if (phase == P_MEMB || phase == P_VMEMB) {
            int hit = -1;  // -1: probe the next bucket
            if (S.prev_degree <= kScanMax) {
                const uint32_t off = (uint32_t)(S.prev_begin & 1ull);
                bool f = false;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const uint4 v = s_slot[k][tid];
                    const uint32_t j0 = 2 * k, j1 = 2 * k + 1;
                    f |= (j0 >= off && j0 < off + S.prev_degree && v.x == pu);
                    f |= (j1 >= off && j1 < off + S.prev_degree && v.z == pu);
                }
                hit = f ? 1 : 0;
            } else {
                const uint4 v0 = s_slot[0][tid], v1 = s_slot[1][tid];
                if (has8(v0, v1, pu))
                    hit = 1;
                else if (v1.w == kHashEmpty)
                    hit = 0;
                else
                    mb = (mb + 1) & ((1u << hash_log2_buckets(S.prev_degree)) - 1u);
            }
            if (hit >= 0) {
                const WeightCase wc = model.weight(S, pu, ph, 0);
                const double w = hit ? wc.w_in : wc.w_out;
                if (!valid_w(w)) {
                    fail(kDevBadWeight);
                } else if (phase == P_MEMB) {
                    if (py < w) {
                        finish_step(pu);
                    } else if (t >= p.cap_per_degree * S.degree) {
                        ++LC(LC_FB);
                        start_ervs(2 * t);
                    } else {
                        phase = P_TRIAL;
                    }
                } else {
                    phase = P_VREC;
                    visit(pu, w);
                }
            }
        } else if (phase == P_VREC) {
            const uint4 v = s_slot[0][tid];
            const uint32_t u = sel ? v.z : v.x;
            const float h = __uint_as_float(sel ? v.w : v.y);
            const uint16_t lab =
                M::kUsesLabels ? (uint16_t)(sel ? (s_lab[0][tid] >> 16) : s_lab[0][tid]) : 0;
            const WeightCase wc = model.weight(S, u, h, lab);
            if (M::kSecondOrder && wc.needs_member) {
                park(u, h, 0.0, P_VMEMB);
            } else if (!valid_w(wc.w)) {
                fail(kDevBadWeight);
            } else {
                visit(u, wc.w);
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
            const ull db = __shfl_sync(kFull, ev.didx, L);
            uint32_t nx = kInvalid;
            ull dr = 0;
            const int st = ervs_warp<M, kNoJump>(model, T, K, g, db, nx, dr);
            if (lane == L) {
                if (st < 0) {
                    fail(-st);
                } else {
                    LC(LC_READS) += T.degree;
                    LC(LC_DRAWS) += dr;
                    finish_step(nx);
                }
            }
        }
    }

    // ---- flush counters (Counter order == LaneCounter order)
#pragma unroll
    for (int k = 0; k < LC_NUM; ++k) {
        const ull s = warp_sum(s_lc[k][tid]);
        if (lane == 0 && s) atomicAdd(&s_cnt[k], s);
    }
#undef LC
    __syncthreads();
    for (int i = tid; i < kCNum; i += blockDim.x)
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
