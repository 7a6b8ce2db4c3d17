// dsl_codegen.hpp -- DslWalk programs compiled to CUDA model functors.
//
// the user's weight function is specialised into the walk
// kernel at compile time, with no interpretation on the device.  This header
// sits on the reference side of the boundary (it reads the reference's own
// parsed dsl::Program and dsl::AnalysisResult, ast.hpp / analyzer.hpp) and
// emits CUDA C++ for a model functor with the device Model interface
// (csrc/dw_models.cuh).  dw_model_compile() builds it with NVRTC into the walk
// kernel template (csrc/dw_walk_kernel.cuh).
//   weight()       the program's statements, one C++ statement each; the
//                  interpreter's semantics (dsl_interp.cpp:45-100): doubles,
//                  short-circuit and/or, std::min/max argument order, checked
//                  division and array indexing, the 100000-iteration loop
//                  budget.  `dist` becomes a parameter: the functor returns the
//                  two candidates {dist = 1, dist = 2} and the kernel resolves
//                  the membership test only when they differ.
//   bound()/wsum() the analyzer's unique leaves in interval arithmetic, leaf
//                  by leaf (dsl_estimator.cpp:197-221).
#pragma once

#include <cstdint>
#include <cstdio>
#include <limits>
#include <sstream>
#include <string>
#include <vector>

#include "dynwalk/dsl/analyzer.hpp"
#include "dynwalk/dsl/ast.hpp"
#include "dynwalk/types.hpp"

namespace dynwalk::gpu::detail {

struct DslCode {
    std::string source;           // CUDA C++ defining dwb::DslModel
    bool uses_label = false;      // reads the edge label
    bool label_aggregates = false;  // estimators read per-node label MAX/SUM
    bool second_order = false;    // reads dist
};

class DslCodegen {
public:
    DslCodegen(const dsl::Program& prog, const dsl::AnalysisResult& res, std::uint32_t max_steps)
        : prog_(prog), res_(res), max_steps_(max_steps) {}

    DslCode run() {
        DslCode out;
        scan_body(prog_.body);
        for (const auto& leaf : res_.unique_leaves) scan_expr(leaf);
        out.uses_label = uses_label_;
        out.second_order = uses_dist_;
        out.label_aggregates = res_.uses_label;
        std::ostringstream s;
        s << "// generated from DSL program '" << prog_.source_name << "'\n";
        s << "#include \"dw_walk_kernel.cuh\"\n#include \"dw_dsl_rt.cuh\"\nnamespace dwb {\n";
        for (std::size_t i = 0; i < prog_.array_params.size(); ++i) {
            const auto& vals = prog_.array_params[i].second;
            s << "__device__ const double dsl_arr_" << i << "[" << std::max<std::size_t>(vals.size(), 1)
              << "] = {";
            for (std::size_t k = 0; k < vals.size(); ++k) s << (k ? ", " : "") << lit(vals[k]);
            if (vals.empty()) s << "0.0";
            s << "};\n";
        }
        // weight function (dsl_interp.cpp)
        s << "__device__ __forceinline__ double dsl_weight(double h, double lab, double degc, "
             "double degp, double step, double dist, int& err) {\n";
        s << "    (void)h; (void)lab; (void)degc; (void)degp; (void)step; (void)dist;\n";
        for (int v = 0; v < prog_.slot_count; ++v) s << "    double v" << v << " = 0.0;\n";
        s << "    unsigned long long budget = dsl::kLoopBudget;\n    (void)budget;\n";
        emit_body(s, prog_.body, 1);
        s << "    err = 1;  // fell off the end without returning\n    return 0.0;\n}\n";
        // model functor
        const bool boundable = res_.flag != EstimationFlag::None;
        s << "struct DslModel {\n";
        s << "    static constexpr bool kScreen = false;\n";
        s << "    static constexpr bool kLabelAgg = " << (res_.uses_label ? "true" : "false") << ";\n";
        s << "    static constexpr bool kUsesLabels = " << (uses_label_ ? "true" : "false") << ";\n";
        s << "    static constexpr bool kSecondOrder = " << (uses_dist_ ? "true" : "false") << ";\n";
        s << "    static constexpr bool kBoundable = " << (boundable ? "true" : "false") << ";\n";
        s << "    static constexpr bool kAggregates = "
          << (res_.flag == EstimationFlag::PerStep ? "true" : "false") << ";\n";
        s << "    __device__ explicit DslModel(const ModelParams&) {}\n";
        s << "    __device__ uint32_t max_steps() const { return " << max_steps_ << "u; }\n";
        s << "    __device__ void prepare(const Step&) const {}\n";
        s << "    __device__ double wsum_approx(const Step& s) const { return wsum(s); }\n";
        s << "    __device__ double nonreturn_max(const Step& s) const { return bound(s); }\n";
        emit_estimators(s, boundable);
        s << "    __device__ WeightCase weight(const Step& s, uint32_t u, float hf, uint16_t label) "
             "const {\n";
        s << "        const double h = (double)hf, lab = (double)label, degc = (double)s.degree;\n";
        s << "        const double degp = s.has_prev() ? (double)s.prev_degree : degc;\n";
        s << "        const double st = (double)s.step;\n";
        s << "        int e1 = 0;\n";
        if (!uses_dist_) {
            s << "        const double w = dsl_weight(h, lab, degc, degp, st, 1.0, e1);\n";
            s << "        return exact(e1 ? dsl::nan_value() : w);\n";
        } else {
            // dist: 1 on the first step, 0 for the previous node, else by membership
            s << "        if (!s.has_prev()) { const double w = dsl_weight(h, lab, degc, degp, st, "
                 "1.0, e1); return exact(e1 ? dsl::nan_value() : w); }\n";
            s << "        if (u == s.prev) { const double w = dsl_weight(h, lab, degc, degp, st, 0.0, "
                 "e1); return exact(e1 ? dsl::nan_value() : w); }\n";
            s << "        int e2 = 0;\n";
            s << "        double wi = dsl_weight(h, lab, degc, degp, st, 1.0, e1);\n";
            s << "        double wo = dsl_weight(h, lab, degc, degp, st, 2.0, e2);\n";
            s << "        if (e1) wi = dsl::nan_value();\n        if (e2) wo = dsl::nan_value();\n";
            s << "        if (!e1 && !e2 && wi == wo) return exact(wi);\n";
            s << "        return WeightCase{0.0, wi, wo, true};\n";
        }
        s << "    }\n};\n}  // namespace dwb\n";
        out.source = s.str();
        return out;
    }

private:
    const dsl::Program& prog_;
    const dsl::AnalysisResult& res_;
    std::uint32_t max_steps_;
    bool uses_label_ = false, uses_dist_ = false;

    static std::string lit(double v) {
        char buf[64];
        if (v != v) return "dsl::nan_value()";
        if (v == std::numeric_limits<double>::infinity()) return "dsl::inf_value()";
        if (v == -std::numeric_limits<double>::infinity()) return "(-dsl::inf_value())";
        std::snprintf(buf, sizeof buf, "%a", v);  // exact
        return std::string("(") + buf + ")";
    }

    int array_index(const std::string& name) const {
        for (std::size_t i = 0; i < prog_.array_params.size(); ++i)
            if (prog_.array_params[i].first == name) return (int)i;
        throw Error("internal: unknown array parameter '" + name + "'");
    }

    void scan_expr(const dsl::ExprPtr& e) {
        using E = dsl::Expr;
        if (const auto* st = std::get_if<E::State>(&e->node)) {
            if (st->ref == dsl::StateRef::Lab) uses_label_ = true;
            if (st->ref == dsl::StateRef::Dist) uses_dist_ = true;
        } else if (const auto* pi = std::get_if<E::ParamIndex>(&e->node)) {
            scan_expr(pi->index);
        } else if (const auto* u = std::get_if<E::Unary>(&e->node)) {
            scan_expr(u->operand);
        } else if (const auto* b = std::get_if<E::Binary>(&e->node)) {
            scan_expr(b->lhs);
            scan_expr(b->rhs);
        }
    }
    void scan_body(const std::vector<dsl::Stmt>& body) {
        using S = dsl::Stmt;
        for (const auto& st : body) {
            if (const auto* r = std::get_if<S::Return>(&st.node)) scan_expr(r->value);
            else if (const auto* l = std::get_if<S::Let>(&st.node)) scan_expr(l->value);
            else if (const auto* a = std::get_if<S::Assign>(&st.node)) scan_expr(a->value);
            else if (const auto* i = std::get_if<S::If>(&st.node)) {
                scan_expr(i->cond);
                scan_body(i->then_body);
                scan_body(i->else_body);
            } else if (const auto* w = std::get_if<S::While>(&st.node)) {
                scan_expr(w->cond);
                scan_body(w->body);
            }
        }
    }

    // ---- weight expressions (dsl_interp.cpp:45-100)
    std::string expr(const dsl::ExprPtr& e) {
        using E = dsl::Expr;
        if (const auto* n = std::get_if<E::Number>(&e->node)) return lit(n->value);
        if (const auto* p = std::get_if<E::Param>(&e->node)) return lit(p->value);
        if (const auto* pi = std::get_if<E::ParamIndex>(&e->node)) {
            const int a = array_index(pi->name);
            return "dsl::index_checked(dsl_arr_" + std::to_string(a) + ", " +
                   std::to_string(pi->values->size()) + ", " + expr(pi->index) + ", err)";
        }
        if (const auto* st = std::get_if<E::State>(&e->node)) {
            switch (st->ref) {
            case dsl::StateRef::Prop: return "h";
            case dsl::StateRef::Lab: return "lab";
            case dsl::StateRef::DegCur: return "degc";
            case dsl::StateRef::DegPrev: return "degp";
            case dsl::StateRef::Step: return "step";
            case dsl::StateRef::Dist: return "dist";
            }
        }
        if (const auto* v = std::get_if<E::Var>(&e->node)) return "v" + std::to_string(v->slot);
        if (const auto* u = std::get_if<E::Unary>(&e->node)) {
            const std::string x = expr(u->operand);
            if (u->op == dsl::UnOp::Neg) return "(-" + x + ")";
            return "((" + x + ") == 0.0 ? 1.0 : 0.0)";
        }
        const auto& b = std::get<E::Binary>(e->node);
        const std::string l = expr(b.lhs), r = expr(b.rhs);
        switch (b.op) {
        case dsl::BinOp::Add: return "(" + l + " + " + r + ")";
        case dsl::BinOp::Sub: return "(" + l + " - " + r + ")";
        case dsl::BinOp::Mul: return "(" + l + " * " + r + ")";
        case dsl::BinOp::Div: return "dsl::div_checked(" + l + ", " + r + ", err)";
        case dsl::BinOp::Eq: return "((" + l + ") == (" + r + ") ? 1.0 : 0.0)";
        case dsl::BinOp::Ne: return "((" + l + ") != (" + r + ") ? 1.0 : 0.0)";
        case dsl::BinOp::Lt: return "((" + l + ") < (" + r + ") ? 1.0 : 0.0)";
        case dsl::BinOp::Le: return "((" + l + ") <= (" + r + ") ? 1.0 : 0.0)";
        case dsl::BinOp::Gt: return "((" + l + ") > (" + r + ") ? 1.0 : 0.0)";
        case dsl::BinOp::Ge: return "((" + l + ") >= (" + r + ") ? 1.0 : 0.0)";
        case dsl::BinOp::And: return "(((" + l + ") != 0.0 && (" + r + ") != 0.0) ? 1.0 : 0.0)";
        case dsl::BinOp::Or: return "(((" + l + ") != 0.0 || (" + r + ") != 0.0) ? 1.0 : 0.0)";
        case dsl::BinOp::Min: return "dsl::smin(" + l + ", " + r + ")";
        case dsl::BinOp::Max: return "dsl::smax(" + l + ", " + r + ")";
        }
        return "0.0";
    }

    void emit_body(std::ostringstream& s, const std::vector<dsl::Stmt>& body, int depth) {
        using S = dsl::Stmt;
        const std::string ind(4 * depth, ' ');
        for (const auto& st : body) {
            if (const auto* r = std::get_if<S::Return>(&st.node)) {
                s << ind << "return " << expr(r->value) << ";\n";
            } else if (const auto* l = std::get_if<S::Let>(&st.node)) {
                s << ind << "v" << l->slot << " = " << expr(l->value) << ";\n";
            } else if (const auto* a = std::get_if<S::Assign>(&st.node)) {
                s << ind << "v" << a->slot << " = " << expr(a->value) << ";\n";
            } else if (const auto* i = std::get_if<S::If>(&st.node)) {
                s << ind << "if ((" << expr(i->cond) << ") != 0.0) {\n";
                emit_body(s, i->then_body, depth + 1);
                s << ind << "} else {\n";
                emit_body(s, i->else_body, depth + 1);
                s << ind << "}\n";
            } else if (const auto* w = std::get_if<S::While>(&st.node)) {
                s << ind << "while ((" << expr(w->cond) << ") != 0.0) {\n";
                s << ind << "    if (budget-- == 0) { err = 1; return 0.0; }\n";
                emit_body(s, w->body, depth + 1);
                s << ind << "}\n";
            }
            // a runtime error stops the program where the interpreter throws
            s << ind << "if (err) return 0.0;\n";
        }
    }

    // ---- estimators (dsl_estimator.cpp:10-147): interval expressions
    std::string iexpr(const dsl::ExprPtr& e) {
        using E = dsl::Expr;
        if (const auto* n = std::get_if<E::Number>(&e->node)) return "dsl::ipoint(" + lit(n->value) + ")";
        if (const auto* p = std::get_if<E::Param>(&e->node)) return "dsl::ipoint(" + lit(p->value) + ")";
        if (const auto* pi = std::get_if<E::ParamIndex>(&e->node)) {
            const int a = array_index(pi->name);
            return "dsl::iindex(dsl_arr_" + std::to_string(a) + ", " +
                   std::to_string(pi->values->size()) + ", " + iexpr(pi->index) + ")";
        }
        if (const auto* st = std::get_if<E::State>(&e->node)) {
            switch (st->ref) {
            case dsl::StateRef::Prop: return "env_prop";
            case dsl::StateRef::Lab: return "env_label";
            case dsl::StateRef::DegCur: return "dsl::ipoint(degc)";
            case dsl::StateRef::DegPrev: return "dsl::ipoint(degp)";
            case dsl::StateRef::Step: return "dsl::ipoint(st)";
            case dsl::StateRef::Dist: return "env_dist";
            }
        }
        if (std::get_if<E::Var>(&e->node)) throw Error("internal: unsubstituted variable in estimator");
        if (const auto* u = std::get_if<E::Unary>(&e->node)) {
            return std::string(u->op == dsl::UnOp::Neg ? "dsl::ineg(" : "dsl::inot(") +
                   iexpr(u->operand) + ")";
        }
        const auto& b = std::get<E::Binary>(e->node);
        const std::string l = iexpr(b.lhs), r = iexpr(b.rhs);
        const char* f = "";
        switch (b.op) {
        case dsl::BinOp::Add: f = "dsl::iadd"; break;
        case dsl::BinOp::Sub: f = "dsl::isub"; break;
        case dsl::BinOp::Mul: f = "dsl::imul"; break;
        case dsl::BinOp::Div: return "dsl::idiv(" + l + ", " + r + ", err)";
        case dsl::BinOp::Min: f = "dsl::imin"; break;
        case dsl::BinOp::Max: f = "dsl::imax"; break;
        case dsl::BinOp::Eq: f = "dsl::ieq"; break;
        case dsl::BinOp::Ne: f = "dsl::ine"; break;
        case dsl::BinOp::Lt: f = "dsl::ilt"; break;
        case dsl::BinOp::Le: f = "dsl::ile"; break;
        case dsl::BinOp::Gt: f = "dsl::igt"; break;
        case dsl::BinOp::Ge: f = "dsl::ige"; break;
        case dsl::BinOp::And: f = "dsl::iand"; break;
        case dsl::BinOp::Or: f = "dsl::ior"; break;
        }
        return std::string(f) + "(" + l + ", " + r + ")";
    }

    void emit_estimators(std::ostringstream& s, bool boundable) {
        const char* head =
            "        const double degc = (double)s.degree;\n"
            "        const double degp = s.has_prev() ? (double)s.prev_degree : degc;\n"
            "        const double st = (double)s.step;\n"
            "        (void)degc; (void)degp; (void)st;\n"
            "        int err = 0;\n"
            "        const dsl::Interval env_dist{0.0, 2.0};\n"
            "        (void)env_dist;\n";
        s << "    __device__ double bound(const Step& s) const {\n";
        if (!boundable) {
            s << "        return dsl::nan_value();\n    }\n";
            s << "    __device__ double wsum(const Step& s) const { return dsl::nan_value(); }\n";
            return;
        }
        s << head;
        s << "        const dsl::Interval env_prop{0.0, s.hmax}, env_label{0.0, s.lmax};\n";
        s << "        (void)env_prop; (void)env_label;\n";
        s << "        double best = -dsl::inf_value();\n";
        for (const auto& leaf : res_.unique_leaves)
            s << "        best = dsl::smax(best, " << iexpr(leaf) << ".hi);\n";
        s << "        return err ? dsl::nan_value() : best;\n    }\n";
        s << "    __device__ double wsum(const Step& s) const {\n" << head;
        s << "        const dsl::Interval env_prop = dsl::ipoint(s.hsum), env_label = "
             "dsl::ipoint(s.lsum);\n";
        s << "        (void)env_prop; (void)env_label;\n";
        s << "        double acc = 0.0;\n";
        for (const auto& leaf : res_.unique_leaves)
            s << "        acc += " << iexpr(leaf) << ".hi;\n";
        s << "        const double avg = acc / " << lit((double)res_.unique_leaves.size()) << ";\n";
        s << "        if (err) return dsl::nan_value();\n";
        s << "        return " << (res_.flag == EstimationFlag::PerKernel ? "avg * degc" : "avg")
          << ";\n    }\n";
    }
};

inline DslCode dsl_codegen(const dsl::Program& prog, const dsl::AnalysisResult& res,
                           std::uint32_t max_steps) {
    return DslCodegen(prog, res, max_steps).run();
}

}  // namespace dynwalk::gpu::detail
