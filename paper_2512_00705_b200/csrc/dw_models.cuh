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
// plus one device-only member that the reference derives implicitly:
//   nonreturn_max(S)          -> an upper bound on weight(e) over every edge
//                                whose target is not prev (every edge on the
//                                first step), in the same rounding as
//                                weight().  eRJS rejects a trial with
//                                y >= nonreturn_max whose index is outside the
//                                return-edge range without gathering the edge
//                                (dw_walk.cu); the outcome is unchanged.
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
    uint32_t step;
    uint32_t degree;  // d(cur)
    double hmax, hsum;
    double lmax, lsum;  // per-node label MAX/SUM (DSL models whose estimators read labels)
    // upper bound of h(cur -> u) over u in N(prev), u != prev (the record's
    // triangle bound, dw_graph.cu tri_q): 0 when there is no such edge,
    // hmax when unknown.  Only nonreturn_max reads it.
    double hin;
    __device__ __forceinline__ bool has_prev() const { return prev != kInvalid; }
};

struct WeightCase {
    double w;             // exact weight when !needs_member
    double w_in, w_out;   // weight if u in N(prev) / not in N(prev)
    bool needs_member;
};

__device__ __forceinline__ WeightCase exact(double w) { return WeightCase{w, w, w, false}; }

// Host-filled run constants.  inv_* are the correctly rounded reciprocals
// 1.0/a, 1.0/b, 1.0/3.0 (IEEE division on the host); the host requires a and
// b in [2^-500, 2^500] for node2vec (dw_capi.cu check_model), so every
// quotient the models form stays in the normal range and ddiv() is exact.
// fast_div is kept for the record.  shortcut is set when the model's weights are provably valid
// (node2vec a, b > 0; pr2 0 <= gamma <= 1), so skipping the evaluation of a
// rejected trial cannot hide a weight error the reference would raise.
struct ModelParams {
    double a, b, gamma;
    double inv_a, inv_b, inv_3;
    uint32_t fast_div, shortcut;
    uint32_t pos_weights;     // every weight is > 0 and finite by construction
    uint32_t screen;          // wsum_approx is within 1e-15 (relative) of wsum
    double wsum_coef;         // node2vec: RN((1/a + 1 + 1/b) / 3)
    double fat32_band;        // relative band of the compact records' f32 row sum
    double ervs_slack;        // widens the warp reservoir's rounding band (1; tests force the exact replay)
    uint32_t schema_len;
    uint16_t schema[128];
};

// Correctly rounded x / d from inv = RN(1/d) (Markstein; exact whenever x,
// the quotient and the residual are normal doubles, which the parameter range
// guarantees for every operand the models form: x is an f32 weight or a sum
// of them).  Avoids the DDIV slow-path call (and its register spills) in the
// hot loop; --fmad=false does not affect the explicit fma.
__device__ __forceinline__ double ddiv(double x, double d, double inv) {
    const double q = __dmul_rn(x, inv);
    const double r = __fma_rn(-q, d, x);
    return __fma_rn(r, inv, q);
}

__device__ __forceinline__ double dmax3(double x, double y, double z) {
    double m = x;
    if (m < y) m = y;
    if (m < z) m = z;
    return m;
}

// StaticWalk (models.hpp:33-51)
template <bool W>
struct StaticModel {
    static constexpr bool kScreen = false;
    static constexpr bool kLabelAgg = false;
    static constexpr bool kUsesLabels = false;
    static constexpr bool kSecondOrder = false;
    static constexpr bool kBoundable = true;
    static constexpr bool kAggregates = W;  // PER_STEP bound reads node max/sum
    __device__ explicit StaticModel(const ModelParams&) {}
    __device__ uint32_t max_steps() const { return 0xFFFFFFFFu; }
    __device__ double bound(const Step& s) const { return W ? s.hmax : 1.0; }
    __device__ double wsum(const Step& s) const { return W ? s.hsum : (double)s.degree; }
    __device__ double nonreturn_max(const Step& s) const { return bound(s); }
    __device__ void prepare(const Step&) const {}
    __device__ double wsum_approx(const Step& s) const { return wsum(s); }
    __device__ WeightCase weight(const Step&, uint32_t, float h, uint16_t) const {
        return exact(W ? (double)h : 1.0);
    }
};

// Node2Vec (models.hpp:57-90)
template <bool W>
struct Node2VecModel {
    static constexpr bool kUsesLabels = false;
    static constexpr bool kSecondOrder = true;
    static constexpr bool kBoundable = true;
    static constexpr bool kAggregates = W;  // PER_STEP bound reads node max/sum
    static constexpr bool kScreen = true;
    static constexpr bool kLabelAgg = false;
    double a, b, ia, ib, i3, wc;
    __device__ explicit Node2VecModel(const ModelParams& p)
        : a(p.a), b(p.b), ia(p.inv_a), ib(p.inv_b), i3(p.inv_3), wc(p.wsum_coef) {}
    // x * (1/a + 1 + 1/b) / 3 in one multiply: relative error <= ~8 ulp
    // against wsum() when a, b > 0 (all terms positive), so the decision
    // ratio * bound < wsum only needs wsum() within a 1e-12 band
    __device__ double wsum_approx(const Step& s) const {
        return W ? s.hsum * wc : wc * (double)s.degree;
    }
    // Markstein division, exact for power-of-two divisors as well (zero
    // residual): one code path, no select between a multiply and a division
    // (measured +1 % over the select)
    __device__ double da(double x) const { return ddiv(x, a, ia); }
    __device__ double db(double x) const { return ddiv(x, b, ib); }
    __device__ uint32_t max_steps() const { return 0xFFFFFFFFu; }
    __device__ double bound(const Step& s) const {  // models.hpp:74-79
        const double hmax = W ? s.hmax : 1.0;
        return dmax3(da(hmax), hmax, db(hmax));
    }
    __device__ double wsum(const Step& s) const {  // models.hpp:80-87
        if (W) {
            const double x = s.hsum;
            return ddiv(da(x) + x + db(x), 3.0, i3);
        }
        return ddiv(da(1.0) + 1.0 + db(1.0), 3.0, i3) * (double)s.degree;
    }
    // u != prev: weight is h (u in N(prev): h <= hin, the triangle bound)
    // or h/b (h <= hmax); RN is monotone and b > 0
    __device__ double nonreturn_max(const Step& s) const {
        const double hmax = W ? s.hmax : 1.0;
        if (!s.has_prev()) return hmax;
        const double hin = W ? s.hin : (s.hin > 0.0 ? 1.0 : 0.0);
        const double hb = db(hmax);
        return hb > hin ? hb : hin;
    }
    __device__ void prepare(const Step&) const {}
    __device__ WeightCase weight(const Step& s, uint32_t u, float hf, uint16_t) const {
        const double h = W ? (double)hf : 1.0;  // models.hpp:62-69
        if (!s.has_prev()) return exact(h);
        if (u == s.prev) return exact(da(h));
        return WeightCase{0.0, h, db(h), true};
    }
};

// MetaPath (models.hpp:95-118)
template <bool W>
struct MetaPathModel {
    static constexpr bool kScreen = false;
    static constexpr bool kLabelAgg = false;
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
    __device__ double nonreturn_max(const Step& s) const { return bound(s); }
    __device__ void prepare(const Step&) const {}
    __device__ double wsum_approx(const Step& s) const { return wsum(s); }
    __device__ WeightCase weight(const Step& s, uint32_t, float hf, uint16_t label) const {
        const double h = W ? (double)hf : 1.0;
        return exact(label == p->schema[s.step] ? h : 0.0);
    }
};

// SecondOrderPr (models.hpp:124-164).  The per-step factors
// (1-gamma)/dcur and (1-gamma)/dcur + gamma/dprev are formed once per step
// (prepare) with the reference's operation order; weight() then multiplies.
template <bool W>
struct Pr2Model {
    static constexpr bool kScreen = false;
    static constexpr bool kLabelAgg = false;
    static constexpr bool kUsesLabels = false;
    static constexpr bool kSecondOrder = true;
    static constexpr bool kBoundable = true;
    static constexpr bool kAggregates = W;  // PER_STEP bound reads node max/sum
    double gamma;
    // per-step state (prepare)
    double c_plain, c_boost, maxd;
    __device__ explicit Pr2Model(const ModelParams& p)
        : gamma(p.gamma), c_plain(0.0), c_boost(0.0), maxd(0.0) {}
    __device__ uint32_t max_steps() const { return 0xFFFFFFFFu; }
    __device__ void factors(const Step& s, double& cp, double& cb, double& md) const {
        const double dcur = (double)s.degree;
        const double dprev = s.has_prev() ? (double)s.prev_degree : dcur;
        md = dcur < dprev ? dprev : dcur;
        cp = (1.0 - gamma) / dcur;
        cb = (1.0 - gamma) / dcur + gamma / dprev;
    }
    __device__ double bound(const Step& s) const {  // models.hpp:142-151
        const double hmax = W ? s.hmax : 1.0;
        double cp, cb, md;
        factors(s, cp, cb, md);
        return dmax3(hmax, hmax * cb * md, hmax * cp * md);
    }
    __device__ double wsum(const Step& s) const {  // models.hpp:152-161
        double cp, cb, md;
        factors(s, cp, cb, md);
        const double x = W ? s.hsum : 1.0;
        const double avg = (x + x * cb * md + x * cp * md) / 3.0;
        return W ? avg : avg * (double)s.degree;
    }
    // u != prev: boosted h * cb * md when u in N(prev) (h <= hin, the
    // triangle bound), plain h * cp * md otherwise (h <= hmax)
    __device__ double nonreturn_max(const Step& s) const {
        const double hmax = W ? s.hmax : 1.0;
        if (!s.has_prev()) return hmax;
        const double hin = W ? s.hin : (s.hin > 0.0 ? 1.0 : 0.0);
        double cp, cb, md;
        factors(s, cp, cb, md);
        const double x = hin * cb * md, y = hmax * cp * md;
        return x > y ? x : y;
    }
    __device__ void prepare(const Step& s) {
        if (s.has_prev()) factors(s, c_plain, c_boost, maxd);
    }
    __device__ double wsum_approx(const Step& s) const { return wsum(s); }
    __device__ WeightCase weight(const Step& s, uint32_t u, float hf, uint16_t) const {
        const double h = W ? (double)hf : 1.0;  // models.hpp:128-138
        if (!s.has_prev()) return exact(h);
        const double plain = h * c_plain * maxd;
        if (u == s.prev) return exact(plain);
        return WeightCase{0.0, h * c_boost * maxd, plain, true};
    }
};

}  // namespace dwb
