// dw_models.cuh -- the user walk-logic plugin, compiled into the kernels.
//
// Device form of the reference Model concept (models.hpp:20-30):
//   weight(g, st, e)          -> weight(S, u, h, label) returning a WeightCase:
//                                the exact weight, or the two candidates
//                                {u in N(prev), u not in N(prev)} when the
//                                value hinges on Graph::has_edge
//                                (graph.cpp:114-118).  The sampler resolves the
//                                membership test only when the accept/reject
//                                outcome depends on it, so the result is the
//                                same as evaluating weight() eagerly.
//   estimation_flag()         -> kBoundable (PER_STEP / PER_KERNEL vs NONE)
//   estimate_bound(g, st)     -> bound(S)
//   estimate_weight_sum(g,st) -> wsum(S)
//   max_steps()               -> max_steps()
// A user model is a struct with these members passed as the template
// argument of walk_kernel (dw_walk.cu); there is no virtual dispatch and no
// interpretation.  Arithmetic follows the reference operation order; the
// library builds with --fmad=false so no multiply-add is ever contracted.
#pragma once
#include "dw_member.cuh"

namespace dwb {

// WalkerState (walk_state.hpp:13-40) plus the cur/prev node records the
// models read (degree(cur), node_prop_max/sum(cur), prev_degree).
struct Step {
    uint32_t cur, prev;  // prev == kInvalid: first step
    uint32_t prev_degree;
    uint32_t prev_hoff;  // prev's membership hash set (dw_member.cuh)
    unsigned long long prev_begin;
    uint32_t step;
    uint32_t degree;  // d(cur)
    uint32_t hoff;
    unsigned long long begin;
    double hmax, hsum;
    __device__ __forceinline__ bool has_prev() const { return prev != kInvalid; }
};

struct WeightCase {
    double w;             // exact weight when !needs_member
    double w_in, w_out;   // weight if u in N(prev) / not in N(prev)
    bool needs_member;
};

__device__ __forceinline__ WeightCase exact(double w) { return WeightCase{w, w, w, false}; }

struct ModelParams {
    double a, b, gamma;
    uint32_t schema_len;
    uint16_t schema[128];
};

__device__ __forceinline__ double dmax3(double x, double y, double z) {
    double m = x;
    if (m < y) m = y;
    if (m < z) m = z;
    return m;
}

// StaticWalk (models.hpp:33-51)
template <bool W>
struct StaticModel {
    static constexpr bool kUsesLabels = false;
    static constexpr bool kSecondOrder = false;
    static constexpr bool kBoundable = true;
    static constexpr bool kAggregates = W;  // PER_STEP bound reads node max/sum
    __device__ explicit StaticModel(const ModelParams&) {}
    __device__ uint32_t max_steps() const { return 0xFFFFFFFFu; }
    __device__ double bound(const Step& s) const { return W ? s.hmax : 1.0; }
    __device__ double wsum(const Step& s) const { return W ? s.hsum : (double)s.degree; }
    __device__ WeightCase weight(const Step&, uint32_t, float h, uint16_t) const {
        return exact(W ? (double)h : 1.0);
    }
    __device__ bool step_ok(const Step&) const { return true; }
};

// Node2Vec (models.hpp:57-90)
template <bool W>
struct Node2VecModel {
    static constexpr bool kUsesLabels = false;
    static constexpr bool kSecondOrder = true;
    static constexpr bool kBoundable = true;
    static constexpr bool kAggregates = W;  // PER_STEP bound reads node max/sum
    double a, b;
    __device__ explicit Node2VecModel(const ModelParams& p) : a(p.a), b(p.b) {}
    __device__ uint32_t max_steps() const { return 0xFFFFFFFFu; }
    __device__ double bound(const Step& s) const {  // models.hpp:74-79
        const double hmax = W ? s.hmax : 1.0;
        return dmax3(hmax / a, hmax, hmax / b);
    }
    __device__ double wsum(const Step& s) const {  // models.hpp:80-87
        if (W) {
            const double x = s.hsum;
            return (x / a + x + x / b) / 3.0;
        }
        return ((1.0 / a + 1.0 + 1.0 / b) / 3.0) * (double)s.degree;
    }
    __device__ WeightCase weight(const Step& s, uint32_t u, float hf, uint16_t) const {
        const double h = W ? (double)hf : 1.0;  // models.hpp:62-69
        if (!s.has_prev()) return exact(h);
        if (u == s.prev) return exact(h / a);
        return WeightCase{0.0, h, h / b, true};
    }
    __device__ bool step_ok(const Step&) const { return true; }
};

// MetaPath (models.hpp:95-118)
template <bool W>
struct MetaPathModel {
    static constexpr bool kUsesLabels = true;
    static constexpr bool kSecondOrder = false;
    static constexpr bool kBoundable = true;
    static constexpr bool kAggregates = W;  // PER_STEP bound reads node max/sum
    const ModelParams* p;
    __device__ explicit MetaPathModel(const ModelParams& mp) : p(&mp) {}
    __device__ uint32_t max_steps() const { return p->schema_len; }
    __device__ double bound(const Step& s) const { return W ? s.hmax : 1.0; }
    __device__ double wsum(const Step& s) const {
        if (W) return (s.hsum + 0.0) / 2.0;
        return ((1.0 + 0.0) / 2.0) * (double)s.degree;
    }
    __device__ WeightCase weight(const Step& s, uint32_t, float hf, uint16_t label) const {
        const double h = W ? (double)hf : 1.0;
        return exact(label == p->schema[s.step] ? h : 0.0);
    }
    __device__ bool step_ok(const Step& s) const { return s.step < p->schema_len; }
};

// SecondOrderPr (models.hpp:124-164)
template <bool W>
struct Pr2Model {
    static constexpr bool kUsesLabels = false;
    static constexpr bool kSecondOrder = true;
    static constexpr bool kBoundable = true;
    static constexpr bool kAggregates = W;  // PER_STEP bound reads node max/sum
    double gamma;
    __device__ explicit Pr2Model(const ModelParams& p) : gamma(p.gamma) {}
    __device__ uint32_t max_steps() const { return 0xFFFFFFFFu; }
    __device__ double bound(const Step& s) const {  // models.hpp:142-151
        const double hmax = W ? s.hmax : 1.0;
        const double dcur = (double)s.degree;
        const double dprev = s.has_prev() ? (double)s.prev_degree : dcur;
        const double maxd = dcur < dprev ? dprev : dcur;
        const double boosted = hmax * ((1.0 - gamma) / dcur + gamma / dprev) * maxd;
        const double plain = hmax * ((1.0 - gamma) / dcur) * maxd;
        return dmax3(hmax, boosted, plain);
    }
    __device__ double wsum(const Step& s) const {  // models.hpp:152-161
        const double dcur = (double)s.degree;
        const double dprev = s.has_prev() ? (double)s.prev_degree : dcur;
        const double maxd = dcur < dprev ? dprev : dcur;
        const double x = W ? s.hsum : 1.0;
        const double boosted = x * ((1.0 - gamma) / dcur + gamma / dprev) * maxd;
        const double plain = x * ((1.0 - gamma) / dcur) * maxd;
        const double avg = (x + boosted + plain) / 3.0;
        return W ? avg : avg * dcur;
    }
    __device__ WeightCase weight(const Step& s, uint32_t u, float hf, uint16_t) const {
        const double h = W ? (double)hf : 1.0;  // models.hpp:128-138
        if (!s.has_prev()) return exact(h);
        const double dcur = (double)s.degree;
        const double dprev = (double)s.prev_degree;
        const double maxd = dcur < dprev ? dprev : dcur;
        const double plain = h * ((1.0 - gamma) / dcur) * maxd;
        if (u == s.prev) return exact(plain);
        const double boosted = h * ((1.0 - gamma) / dcur + gamma / dprev) * maxd;
        return WeightCase{0.0, boosted, plain, true};
    }
    __device__ bool step_ok(const Step&) const { return true; }
};

}  // namespace dwb
