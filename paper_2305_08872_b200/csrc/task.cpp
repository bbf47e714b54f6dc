// task.cpp — task text -> amlt_body_desc (the compile_task boundary).
//
// The reference compiles a task with parse_task -> recognize -> build_dag
// (src/engine.cpp:86-102). The B200 backend needs only the outcome: is the
// statement one of the bodies it has a fused kernel for, what are its
// operands' roles and orientations. This is a small recursive-descent parser
// for the reference grammar (README.md:37-60, parser.cpp:142-365; `//` and
// `#` comments), the recognition conditions 2-4 (recognize.cpp:84-166), and
// a match of the statement tree against the bodies' canonical trees
// (presets.cpp:52-94 + the sqdiff / eqcount statements) after normalising
// comparisons (t < p -> p > t) and matching products and sums as factor /
// term lists in any order, and the op counts of the reference's compiled
// program for the statement (SURVEY §8(d) measure (B)). The Python front
// end (task.py) calls this through amlt_gpu_recognize.
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "task.h"

namespace amltk {

namespace {

struct Node {
    enum Kind { Num, Ref, Bin, Role, Aux } kind = Num;
    double num = 0;
    std::string name;               // Ref / Aux
    std::vector<std::string> idx;   // Ref subscripts
    std::string op;                 // Bin
    std::string cls;                // Aux: "c", "i", "j", "ij"; Role: "A"/"B"
    std::shared_ptr<Node> l, r;
};
using P = std::shared_ptr<Node>;

struct Lexer {
    std::vector<std::string> toks;
    explicit Lexer(const std::string& s) {
        size_t i = 0;
        while (i < s.size()) {
            char c = s[i];
            if (std::isspace(static_cast<unsigned char>(c))) { ++i; continue; }
            if (c == '#' || (c == '/' && i + 1 < s.size() && s[i + 1] == '/')) {
                while (i < s.size() && s[i] != '\n') ++i;
                continue;
            }
            if (std::isdigit(static_cast<unsigned char>(c))) {
                size_t j = i;
                while (j < s.size() && std::isdigit(static_cast<unsigned char>(s[j]))) ++j;
                if (j + 1 < s.size() && s[j] == '.' && std::isdigit(static_cast<unsigned char>(s[j + 1]))) {
                    ++j;
                    while (j < s.size() && std::isdigit(static_cast<unsigned char>(s[j]))) ++j;
                }
                toks.push_back(s.substr(i, j - i));
                i = j;
                continue;
            }
            if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
                size_t j = i;
                while (j < s.size() && (std::isalnum(static_cast<unsigned char>(s[j])) || s[j] == '_')) ++j;
                toks.push_back(s.substr(i, j - i));
                i = j;
                continue;
            }
            static const char* two[] = {"+=", "==", ">=", "<=", ".."};
            bool got = false;
            for (const char* t : two)
                if (s.compare(i, 2, t) == 0) {
                    toks.push_back(t);
                    i += 2;
                    got = true;
                    break;
                }
            if (got) continue;
            if (std::strchr("-+*/<>=()[]{};", c)) {
                toks.push_back(std::string(1, c));
                ++i;
                continue;
            }
            throw TaskError(AMLT_ERR_ENGINE, std::string("parse error near '") + s.substr(i, 10) + "'");
        }
    }
};

struct Parser {
    std::vector<std::string> t;
    size_t p = 0;
    const std::string* peek() const { return p < t.size() ? &t[p] : nullptr; }
    bool is(const char* s) const { return peek() && *peek() == s; }
    std::string take(const char* want = nullptr) {
        if (!peek() || (want && *peek() != want))
            throw TaskError(AMLT_ERR_ENGINE, std::string("parse error: expected '") + (want ? want : "token") +
                                                 "', got '" + (peek() ? *peek() : "end") + "'");
        return t[p++];
    }
    std::string ident() {
        std::string s = take();
        if (!(std::isalpha(static_cast<unsigned char>(s[0])) || s[0] == '_'))
            throw TaskError(AMLT_ERR_ENGINE, "parse error: expected identifier, got '" + s + "'");
        return s;
    }
    P expr() {
        P l = sum();
        for (const char* op : {">", ">=", "<", "<=", "=="})
            if (is(op)) {
                take();
                auto n = std::make_shared<Node>();
                n->kind = Node::Bin;
                n->op = op;
                n->l = l;
                n->r = sum();
                return n;
            }
        return l;
    }
    P sum() {
        P n = term();
        while (is("+") || is("-")) {
            auto b = std::make_shared<Node>();
            b->kind = Node::Bin;
            b->op = take();
            b->l = n;
            b->r = term();
            n = b;
        }
        return n;
    }
    P term() {
        P n = factor();
        while (is("*") || is("/")) {
            auto b = std::make_shared<Node>();
            b->kind = Node::Bin;
            b->op = take();
            b->l = n;
            b->r = factor();
            n = b;
        }
        return n;
    }
    P factor() {
        if (is("(")) {
            take();
            P e = expr();
            take(")");
            return e;
        }
        if (peek() && std::isdigit(static_cast<unsigned char>((*peek())[0]))) {
            auto n = std::make_shared<Node>();
            n->kind = Node::Num;
            n->num = std::stod(take());
            return n;
        }
        auto n = std::make_shared<Node>();
        n->kind = Node::Ref;
        n->name = ident();
        while (is("[")) {
            take();
            n->idx.push_back(ident());
            take("]");
        }
        return n;
    }
};

bool same(const P& a, const P& b) {
    if (a->kind != b->kind) return false;
    switch (a->kind) {
        case Node::Num: return a->num == b->num;
        case Node::Role: return a->cls == b->cls;
        case Node::Aux: return a->name == b->name && a->cls == b->cls;
        case Node::Ref: return a->name == b->name && a->idx == b->idx;
        case Node::Bin: return a->op == b->op && same(a->l, b->l) && same(a->r, b->r);
    }
    return false;
}

using Env = std::map<std::string, P>;

// Canonical form for matching (the reference DAG's own normalisations,
// expr_dag.cpp:182-245, plus the IEEE identities that hold exactly):
//   x < y  ->  y > x,   x <= y  ->  y >= x   (same truth value, NaN included)
// and products / sums are matched as flattened factor / term lists in any
// order (a commuted or re-associated product of the same factors differs by
// rounding only, inside the bodies' stated tolerance, and not at all on
// integer-valued data).
P canon(const P& n) {
    if (n->kind != Node::Bin) return n;
    auto b = std::make_shared<Node>(*n);
    b->l = canon(n->l);
    b->r = canon(n->r);
    if (b->op == "<" || b->op == "<=") {
        std::swap(b->l, b->r);
        b->op = b->op == "<" ? ">" : ">=";
    }
    return b;
}

void flatten(const P& n, const std::string& op, std::vector<P>& out) {
    if (n->kind == Node::Bin && n->op == op) {
        flatten(n->l, op, out);
        flatten(n->r, op, out);
    } else {
        out.push_back(n);
    }
}

bool match(const P& tpl, const P& n, Env& env);

// Template factors tf[i..] against tree factors nf (a permutation), with
// backtracking over the placeholder bindings.
bool match_perm(const std::vector<P>& tf, size_t i, const std::vector<P>& nf, std::vector<bool>& used, Env& env) {
    if (i == tf.size()) return true;
    for (size_t j = 0; j < nf.size(); ++j) {
        if (used[j]) continue;
        Env saved = env;
        if (match(tf[i], nf[j], env)) {
            used[j] = true;
            if (match_perm(tf, i + 1, nf, used, env)) return true;
            used[j] = false;
        }
        env = saved;
    }
    return false;
}

bool match(const P& tpl, const P& n, Env& env) {
    if (tpl->kind == Node::Ref) {  // placeholder A, B, T, D
        const std::string& ph = tpl->name;
        if (ph == "A" || ph == "B") return n->kind == Node::Role && n->cls == ph;
        if (ph == "T" && !(n->kind == Node::Aux || n->kind == Node::Num)) return false;
        if (ph == "D" && !(n->kind == Node::Aux && n->cls == "j")) return false;
        auto it = env.find(ph);
        if (it != env.end()) return same(it->second, n);
        env[ph] = n;
        return true;
    }
    if (tpl->kind == Node::Num) return n->kind == Node::Num && n->num == tpl->num;
    if (n->kind != Node::Bin || n->op != tpl->op) return false;
    if (tpl->op == "*" || tpl->op == "+") {
        std::vector<P> tf, nf;
        flatten(tpl, tpl->op, tf);
        flatten(n, tpl->op, nf);
        if (tf.size() != nf.size()) return false;
        std::vector<bool> used(nf.size(), false);
        return match_perm(tf, 0, nf, used, env);
    }
    Env saved = env;
    if (match(tpl->l, n->l, env) && match(tpl->r, n->r, env)) return true;
    env = saved;
    if (tpl->op == "==" && match(tpl->l, n->r, env) && match(tpl->r, n->l, env)) return true;
    env = saved;
    return false;
}

// ---------------------------------------------------------------------------
// The reference's compiled program for a statement (build_dag +
// schedule_labelfs, expr_dag.cpp:63-245, schedule.cpp:265-273): one pseudo-
// instruction per DAG op node (equal subexpressions shared), then the final
// accumulate (or move, for "="). Restated here only to COUNT the program's
// operations per opcode: the body-op flops of SURVEY §8(d) measure (B).
// Mask rewrites: in an additive chain a product with a comparison factor
// becomes masksub / maskadd(lhs, cond, product of the other factors); any
// other comparison used as a number becomes maskadd(0, cond, 1).
struct ProgramCounter {
    std::map<std::string, int> ids;  // structural key -> node id (CSE)
    int counts[AMLT_PROG_NOPS] = {};

    std::string key_of(const P& n) const {
        switch (n->kind) {
            case Node::Num: {
                char buf[64];
                std::snprintf(buf, sizeof(buf), "#%a", n->num);
                return buf;
            }
            case Node::Role: return "@" + n->cls;
            case Node::Aux: return "$" + n->name;
            default: return "?";
        }
    }
    std::string leaf(const P& n) { return key_of(n); }
    std::string lit(double v) {
        char buf[64];
        std::snprintf(buf, sizeof(buf), "#%a", v);
        return buf;
    }
    std::string op(int opc, const std::string& a, const std::string& b, const std::string& c = "") {
        const std::string k = "(" + std::to_string(opc) + " " + a + " " + b + " " + c + ")";
        if (!ids.count(k)) {
            ids[k] = static_cast<int>(ids.size());
            ++counts[opc];
        }
        return k;
    }
    static bool is_cmp(const P& n) {
        return n->kind == Node::Bin && (n->op == ">" || n->op == ">=" || n->op == "<" || n->op == "<=" || n->op == "==");
    }
    static int cmp_code(const std::string& o) {
        return o == ">" ? AMLT_PROG_GTCMP : o == ">=" ? AMLT_PROG_GECMP : o == "<" ? AMLT_PROG_LTCMP
               : o == "<=" ? AMLT_PROG_LECMP : AMLT_PROG_EQCMP;
    }
    void factors(const P& n, std::vector<P>& out) const {  // Mul spine only; Div is opaque
        if (n->kind == Node::Bin && n->op == "*") {
            factors(n->l, out);
            out.push_back(n->r);
        } else {
            out.push_back(n);
        }
    }
    std::string cmp(const P& n) { return op(cmp_code(n->op), numeric(n->l), numeric(n->r)); }
    // a product term with a comparison factor: (cond, value)
    bool masked(const P& n, std::string* cond, std::string* value) {
        if (is_cmp(n)) {
            *cond = cmp(n);
            *value = lit(1.0);
            return true;
        }
        if (!(n->kind == Node::Bin && n->op == "*")) return false;
        std::vector<P> f;
        factors(n, f);
        size_t at = f.size();
        for (size_t i = 0; i < f.size() && at == f.size(); ++i)
            if (is_cmp(f[i])) at = i;
        if (at == f.size()) return false;
        *cond = cmp(f[at]);
        std::string v;
        for (size_t i = 0; i < f.size(); ++i) {
            if (i == at) continue;
            const std::string x = numeric(f[i]);
            v = v.empty() ? x : op(AMLT_PROG_MUL, v, x);
        }
        *value = v.empty() ? lit(1.0) : v;
        return true;
    }
    std::string sum(const P& n) {
        if (n->kind == Node::Bin && (n->op == "+" || n->op == "-")) {
            const std::string l = sum(n->l);
            std::string c, v;
            if (masked(n->r, &c, &v)) return op(n->op == "-" ? AMLT_PROG_MASKSUB : AMLT_PROG_MASKADD, l, c, v);
            return op(n->op == "-" ? AMLT_PROG_SUB : AMLT_PROG_ADD, l, numeric(n->r));
        }
        std::string c, v;
        if (masked(n, &c, &v)) return op(AMLT_PROG_MASKADD, lit(0.0), c, v);
        return plain(n);
    }
    std::string numeric(const P& n) {
        if (is_cmp(n)) return op(AMLT_PROG_MASKADD, lit(0.0), cmp(n), lit(1.0));
        if (n->kind == Node::Bin && (n->op == "+" || n->op == "-")) return sum(n);
        std::string c, v;
        if (masked(n, &c, &v)) return op(AMLT_PROG_MASKADD, lit(0.0), c, v);
        return plain(n);
    }
    std::string plain(const P& n) {
        if (n->kind != Node::Bin) return leaf(n);
        if (n->op == "+" || n->op == "-") return sum(n);
        if (n->op == "*") return op(AMLT_PROG_MUL, numeric(n->l), numeric(n->r));
        if (n->op == "/") return op(AMLT_PROG_DIV, numeric(n->l), numeric(n->r));
        return op(AMLT_PROG_MASKADD, lit(0.0), cmp(n), lit(1.0));
    }
};

P parse_expr(const char* text) {
    Parser ps;
    ps.t = Lexer(text).toks;
    return ps.expr();
}

}  // namespace

RecognizedTask recognize_task(const std::string& source) {
    Parser ps;
    ps.t = Lexer(source).toks;
    ps.take("where");
    ps.take("(");
    struct Loop { std::string v, lo, hi; };
    std::vector<Loop> loops;
    auto clause = [&] {
        Loop l;
        l.v = ps.ident();
        ps.take("in");
        ps.take("[");
        l.lo = ps.take();
        ps.take("..");
        l.hi = ps.take();
        ps.take("]");
        loops.push_back(l);
    };
    clause();
    while (ps.is("and")) {
        ps.take();
        clause();
    }
    ps.take(")");
    ps.take("{");
    std::string target = ps.ident();
    std::vector<std::string> subs;
    while (ps.is("[")) {
        ps.take();
        subs.push_back(ps.ident());
        ps.take("]");
    }
    std::string op = ps.take();
    if (op != "=" && op != "+=") throw TaskError(AMLT_ERR_ENGINE, "statement must be '=' or '+='");
    P rhs = ps.expr();
    ps.take(";");
    ps.take("}");
    if (ps.peek()) throw TaskError(AMLT_ERR_ENGINE, "trailing input after the task");

    auto unsup = [](const std::string& m) { return TaskError(AMLT_ERR_UNSUPPORTED, m); };
    if (loops.size() != 3) throw unsup("not an MMLT: needs exactly three loop variables");
    auto is_var = [&](const std::string& s) {
        for (auto& l : loops)
            if (l.v == s) return true;
        return false;
    };
    if (subs.size() != 2 || subs[0] == subs[1] || !is_var(subs[0]) || !is_var(subs[1]))
        throw unsup("not an MMLT: target must be 2-D over two distinct loop variables");
    for (auto& l : loops)
        if (l.lo != "0") throw unsup("loop ranges must start at 0 for the GPU backend");
    const std::string vi = subs[0], vj = subs[1];
    std::string vk;
    for (auto& l : loops)
        if (l.v != vi && l.v != vj) vk = l.v;

    RecognizedTask rt;
    rt.r = target;
    std::map<std::string, std::string> role;  // name -> "A0","A1","B0","B1","c","i","j","ij"
    std::function<P(const P&)> classify = [&](const P& n) -> P {
        if (n->kind == Node::Num) return n;
        if (n->kind == Node::Bin) {
            auto b = std::make_shared<Node>(*n);
            b->l = classify(n->l);
            b->r = classify(n->r);
            return b;
        }
        if (n->name == target) throw unsup("target appears on the right-hand side");
        std::string r;
        const auto& ix = n->idx;
        if (ix.empty()) {
            if (is_var(n->name)) throw unsup("loop variable used as a value");
            r = "c";
        } else {
            for (auto& s : ix)
                if (!is_var(s)) throw unsup("subscripts must be loop variables");
            if (ix.size() == 2 && ix[0] == vi && ix[1] == vk) r = "A0";
            else if (ix.size() == 2 && ix[0] == vk && ix[1] == vi) r = "A1";
            else if (ix.size() == 2 && ix[0] == vk && ix[1] == vj) r = "B0";
            else if (ix.size() == 2 && ix[0] == vj && ix[1] == vk) r = "B1";
            else if (ix.size() == 1 && ix[0] == vi) r = "i";
            else if (ix.size() == 1 && ix[0] == vj) r = "j";
            else if (ix.size() == 2 && ix[0] == vi && ix[1] == vj) r = "ij";
            else throw unsup("operand " + n->name + " does not fit the MMLT pattern");
        }
        auto it = role.find(n->name);
        if (it != role.end() && it->second != r) throw unsup("array " + n->name + " used with two index patterns");
        role[n->name] = r;
        auto out = std::make_shared<Node>();
        if (r[0] == 'A' || r[0] == 'B') {
            out->kind = Node::Role;
            out->cls = r.substr(0, 1);
        } else {
            out->kind = Node::Aux;
            out->name = n->name;
            out->cls = r;
        }
        return out;
    };
    P tree = classify(rhs);
    {
        ProgramCounter pc;
        pc.numeric(tree);
        pc.counts[op == "+=" ? AMLT_PROG_ADD : AMLT_PROG_MOV] += 1;  // the final accumulate / move
        int instrs = 0, flops = 0;
        for (int c = 0; c < AMLT_PROG_NOPS; ++c) {
            rt.prog_counts[c] = pc.counts[c];
            instrs += pc.counts[c];
            // (B): add / sub / mul / div / compare 1, masksub / maskadd 2 (x -+ m*y), mov 0
            flops += pc.counts[c] * (c == AMLT_PROG_MOV ? 0 : (c == AMLT_PROG_MASKSUB || c == AMLT_PROG_MASKADD) ? 2 : 1);
        }
        rt.prog_instrs = instrs;
        rt.prog_flops = flops;
    }
    const P ctree = canon(tree);
    int na = 0, nb = 0;
    for (auto& kv : role) {
        if (kv.second[0] == 'A') {
            ++na;
            rt.a = kv.first;
            rt.desc.layout_a = kv.second == "A1" ? AMLT_LAYOUT_TRANSPOSED : AMLT_LAYOUT_NORMAL;
        }
        if (kv.second[0] == 'B') {
            ++nb;
            rt.b = kv.first;
            rt.desc.layout_b = kv.second == "B1" ? AMLT_LAYOUT_TRANSPOSED : AMLT_LAYOUT_NORMAL;
        }
    }
    if (na != 1 || nb != 1) throw unsup("not an MMLT: needs exactly one A[i][k] and one B[k][j] array");

    static const struct { const char* text; int body; } kTemplates[] = {
        {"A*B", AMLT_BODY_GEMM},
        {"A*B - (A*B > T)*A*B*D", AMLT_BODY_DISCOUNT},
        {"A*B + (A*B > T)*(A*B - T)", AMLT_BODY_BOOST},
        {"(A - B)*(A - B)", AMLT_BODY_SQDIFF},
        {"A == B", AMLT_BODY_EQCOUNT},
        {"A*B > T", AMLT_BODY_THRCOUNT},
    };
    for (const auto& tp : kTemplates) {
        Env env;
        if (!match(canon(parse_expr(tp.text)), ctree, env)) continue;
        rt.desc.body = tp.body;
        rt.desc.accumulate = op == "+=" ? 1 : 0;
        rt.desc.thres_class = AMLT_LEAF_CONSTANT;
        rt.desc.thres_value = 0.0;
        auto t = env.find("T");
        if (t != env.end()) {
            if (t->second->kind == Node::Num) {
                rt.desc.thres_value = t->second->num;
            } else {
                rt.thres = t->second->name;
                const std::string& c = t->second->cls;
                rt.desc.thres_class = c == "c" ? AMLT_LEAF_CONSTANT
                                      : c == "i" ? AMLT_LEAF_VEC_I
                                      : c == "j" ? AMLT_LEAF_VEC_J
                                                 : AMLT_LEAF_MAT_IJ;
            }
        }
        auto d = env.find("D");
        if (d != env.end()) rt.dis = d->second->name;
        return rt;
    }
    // Any other recognised statement: a generated body (csrc/jit.cu compiles
    // it into the same tile kernels at plan time).
    rt.desc.body = AMLT_BODY_GENERIC;
    rt.desc.accumulate = op == "+=" ? 1 : 0;
    rt.desc.thres_class = AMLT_LEAF_CONSTANT;
    rt.desc.thres_value = 0.0;
    std::function<std::string(const P&)> gen = [&](const P& n) -> std::string {
        switch (n->kind) {
            case Node::Num: {
                char buf[64];
                std::snprintf(buf, sizeof(buf), "T(%a)", n->num);
                return buf;
            }
            case Node::Role:
                return n->cls == "A" ? "a" : "b";
            case Node::Aux: {
                size_t q = 0;
                while (q < rt.aux_names.size() && rt.aux_names[q] != n->name) ++q;
                if (q == rt.aux_names.size()) {
                    if (q >= AMLT_MAX_AUX)
                        throw unsup("more than " + std::to_string(AMLT_MAX_AUX) +
                                    " auxiliary arrays in one statement");
                    rt.aux_names.push_back(n->name);
                    rt.aux_class.push_back(n->cls == "c"   ? AMLT_LEAF_CONSTANT
                                           : n->cls == "i" ? AMLT_LEAF_VEC_I
                                           : n->cls == "j" ? AMLT_LEAF_VEC_J
                                                           : AMLT_LEAF_MAT_IJ);
                }
                return "c.v[" + std::to_string(q) + "]";
            }
            case Node::Bin: {
                const std::string l = gen(n->l), r = gen(n->r);
                if (n->op == "+") return "add_rn(" + l + ", " + r + ")";
                if (n->op == "-") return "sub_rn(" + l + ", " + r + ")";
                if (n->op == "*") return "mul_rn(" + l + ", " + r + ")";
                if (n->op == "/") {
                    // x / 2^e == x * 2^-e exactly (both are the correctly
                    // rounded x * 2^-e): a multiply instead of a division
                    int e2 = 0;
                    if (n->r->kind == Node::Num && n->r->num > 0 &&
                        std::frexp(n->r->num, &e2) == 0.5 && e2 - 1 < 120 && e2 - 1 > -120) {
                        char buf[64];
                        std::snprintf(buf, sizeof(buf), "T(%a)", std::ldexp(1.0, -(e2 - 1)));
                        return "mul_rn(" + l + ", " + buf + ")";
                    }
                    return "div_rn(" + l + ", " + r + ")";
                }
                return "((" + l + ") " + n->op + " (" + r + ") ? T(1) : T(0))";
            }
            default:
                throw unsup("unexpected node in the statement");
        }
    };
    rt.expr = gen(tree);
    return rt;
}

}  // namespace amltk
