// dw_dsl_rt.cuh -- device runtime for DSL weight functions compiled to CUDA.
//
// host/dsl_codegen.hpp translates a DslWalk program (the reference's DSL:
// ast.hpp, interp.cpp, estimator.cpp) into a model functor that includes this
// header; NVRTC compiles it into the walk kernel (dw_dsl.cu).  Nothing here
// interprets: every helper is the device form of one operation of the
// reference's evaluator, with its exact rounding and edge semantics.
//   * weight evaluation (dsl_interp.cpp:45-100): doubles; a runtime error
//     (division by zero, index out of range, loop budget, no return) sets
//     `err`, and the weight then comes back NaN, which the walk kernel
//     rejects as an invalid weight;
//   * estimators (dsl_estimator.cpp:10-147, 197-221): interval arithmetic on
//     the analyzer's unique leaves, the same corner rules and min/max order.
#pragma once
#include "dw_common.cuh"

namespace dwb {
namespace dsl {

constexpr unsigned long long kLoopBudget = 100000;  // dsl_interp.cpp:11

__device__ __forceinline__ double nan_value() { return __longlong_as_double(0x7ff8000000000000ll); }
__device__ __forceinline__ double inf_value() { return __longlong_as_double(0x7ff0000000000000ll); }

// std::min / std::max argument order (the interpreter calls them directly)
__device__ __forceinline__ double smin(double a, double b) { return (b < a) ? b : a; }
__device__ __forceinline__ double smax(double a, double b) { return (a < b) ? b : a; }

__device__ __forceinline__ double div_checked(double l, double r, int& err) {
    if (r == 0.0) {
        err = 1;  // "weight function divided by zero"
        return 0.0;
    }
    return l / r;
}

// hyperparameter array lookup: nearest integer within 1e-9, in range
__device__ __forceinline__ double index_checked(const double* v, int n, double raw, int& err) {
    const double r = rint(raw);  // std::nearbyint in the default rounding mode
    if (fabs(raw - r) > 1e-9 || r < 0.0 || r >= (double)n) {
        err = 1;  // "index into '<name>' out of range"
        return 0.0;
    }
    return v[(int)r];
}

// ---- interval arithmetic (dsl_estimator.cpp) --------------------------------
struct Interval {
    double lo, hi;
};
__device__ __forceinline__ Interval ipoint(double v) { return Interval{v, v}; }
__device__ __forceinline__ bool is_point(const Interval& a) { return a.lo == a.hi; }

__device__ __forceinline__ double safe_mul(double a, double b) {
    if (a == 0.0 || b == 0.0) return 0.0;
    return a * b;
}
__device__ __forceinline__ double min4(double a, double b, double c, double d) {
    return smin(smin(smin(a, b), c), d);
}
__device__ __forceinline__ double max4(double a, double b, double c, double d) {
    return smax(smax(smax(a, b), c), d);
}
__device__ __forceinline__ Interval imul(Interval a, Interval b) {
    const double c0 = safe_mul(a.lo, b.lo), c1 = safe_mul(a.lo, b.hi), c2 = safe_mul(a.hi, b.lo),
                 c3 = safe_mul(a.hi, b.hi);
    return Interval{min4(c0, c1, c2, c3), max4(c0, c1, c2, c3)};
}
__device__ __forceinline__ double safe_div(double a, double b) {
    if (a == 0.0) return 0.0;
    return a / b;
}
// a divisor interval containing zero is an estimator error: the bound becomes
// NaN and the walk reports an invalid rejection bound
__device__ __forceinline__ Interval idiv(Interval a, Interval b, int& err) {
    if (b.lo <= 0.0 && b.hi >= 0.0) {
        err = 1;
        return Interval{nan_value(), nan_value()};
    }
    const double c0 = safe_div(a.lo, b.lo), c1 = safe_div(a.lo, b.hi), c2 = safe_div(a.hi, b.lo),
                 c3 = safe_div(a.hi, b.hi);
    return Interval{min4(c0, c1, c2, c3), max4(c0, c1, c2, c3)};
}
__device__ __forceinline__ Interval iadd(Interval a, Interval b) {
    return Interval{a.lo + b.lo, a.hi + b.hi};
}
__device__ __forceinline__ Interval isub(Interval a, Interval b) {
    return Interval{a.lo - b.hi, a.hi - b.lo};
}
__device__ __forceinline__ Interval imin(Interval a, Interval b) {
    return Interval{smin(a.lo, b.lo), smin(a.hi, b.hi)};
}
__device__ __forceinline__ Interval imax(Interval a, Interval b) {
    return Interval{smax(a.lo, b.lo), smax(a.hi, b.hi)};
}
__device__ __forceinline__ Interval ineg(Interval a) { return Interval{-a.hi, -a.lo}; }
__device__ __forceinline__ Interval inot(Interval x) {
    if (is_point(x)) return ipoint(x.lo == 0.0 ? 1.0 : 0.0);
    if (x.lo > 0.0 || x.hi < 0.0) return ipoint(0.0);
    return Interval{0.0, 1.0};
}
__device__ __forceinline__ bool overlap(Interval l, Interval r) { return l.lo <= r.hi && r.lo <= l.hi; }
__device__ __forceinline__ Interval ieq(Interval l, Interval r) {
    if (is_point(l) && is_point(r)) return ipoint(l.lo == r.lo ? 1.0 : 0.0);
    return overlap(l, r) ? Interval{0.0, 1.0} : ipoint(0.0);
}
__device__ __forceinline__ Interval ine(Interval l, Interval r) {
    if (is_point(l) && is_point(r)) return ipoint(l.lo != r.lo ? 1.0 : 0.0);
    return overlap(l, r) ? Interval{0.0, 1.0} : ipoint(1.0);
}
__device__ __forceinline__ Interval ilt(Interval l, Interval r) {
    if (l.hi < r.lo) return ipoint(1.0);
    if (l.lo >= r.hi) return ipoint(0.0);
    return Interval{0.0, 1.0};
}
__device__ __forceinline__ Interval ile(Interval l, Interval r) {
    if (l.hi <= r.lo) return ipoint(1.0);
    if (l.lo > r.hi) return ipoint(0.0);
    return Interval{0.0, 1.0};
}
__device__ __forceinline__ Interval igt(Interval l, Interval r) {
    if (l.lo > r.hi) return ipoint(1.0);
    if (l.hi <= r.lo) return ipoint(0.0);
    return Interval{0.0, 1.0};
}
__device__ __forceinline__ Interval ige(Interval l, Interval r) {
    if (l.lo >= r.hi) return ipoint(1.0);
    if (l.hi < r.lo) return ipoint(0.0);
    return Interval{0.0, 1.0};
}
__device__ __forceinline__ bool has_zero(Interval a) { return a.lo <= 0.0 && a.hi >= 0.0; }
__device__ __forceinline__ Interval iand(Interval l, Interval r) {
    const bool false_sure = (is_point(l) && l.lo == 0.0) || (is_point(r) && r.lo == 0.0);
    if (false_sure) return ipoint(0.0);
    const bool true_sure = !has_zero(l) && !has_zero(r);
    return true_sure ? ipoint(1.0) : Interval{0.0, 1.0};
}
__device__ __forceinline__ Interval ior(Interval l, Interval r) {
    const bool true_sure = (is_point(l) && l.lo != 0.0) || (is_point(r) && r.lo != 0.0) ||
                           !has_zero(l) || !has_zero(r);
    const bool false_sure = is_point(l) && l.lo == 0.0 && is_point(r) && r.lo == 0.0;
    if (false_sure) return ipoint(0.0);
    return true_sure ? ipoint(1.0) : Interval{0.0, 1.0};
}
// array indexed by an interval: the element when the index is an in-range
// integer point, else the hull of the whole array
__device__ __forceinline__ Interval iindex(const double* v, int n, Interval idx) {
    if (is_point(idx)) {
        const double r = rint(idx.lo);
        if (fabs(idx.lo - r) <= 1e-9 && r >= 0.0 && r < (double)n) return ipoint(v[(int)r]);
    }
    double lo = inf_value(), hi = -inf_value();
    for (int i = 0; i < n; ++i) {
        lo = smin(lo, v[i]);
        hi = smax(hi, v[i]);
    }
    return Interval{lo, hi};
}

}  // namespace dsl
}  // namespace dwb
