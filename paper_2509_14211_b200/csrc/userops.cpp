// userops.cpp -- user-defined operators.
//
// The paper's multi-stage programming splices the user's Julia function into the generated loop
// ("the lambda inlined", Fig. 2; methods specialised on "the concrete operations",
// PAPER.md:227; SuiteSparse's JIT of user operators).  The GPU form: the caller gives
// a CUDA C++ expression over the operand(s) `x` (`y`) and the constants `c0`, `c1`; it is spliced
// into every generated kernel that uses it as a typed lambda evaluated in the operation's compute
// type (the rule of the built-in operators, R1), compiled by NVRTC with the region.  The
// expression text is part of the generated source, hence of the persistent cubin cache key; the
// operator code is part of the region signature (plan cache), codes are unique per process.
#include <nvrtc.h>

#include <deque>
#include <mutex>

#include "nbg_internal.hpp"

namespace nbg {

extern const char *NBG_PRELUDE_SRC;

namespace {
std::mutex g_mu;
std::deque<UserOp> g_ops;    // code = NBG_USER_OP_BASE + index (deque: stable element addresses)
}  // namespace

const UserOp *user_op(int code) {
    if (code < NBG_USER_OP_BASE) return nullptr;
    std::lock_guard<std::mutex> lk(g_mu);
    const size_t i = (size_t)(code - NBG_USER_OP_BASE);
    return i < g_ops.size() ? &g_ops[i] : nullptr;
}

// `([&]() -> C { const C x = X; [const C y = Y;] const C c0 = K0; const C c1 = K1; return (C)(EXPR); }())`
std::string user_op_call(const UserOp &op, const std::string &C, const std::string &x, const std::string &y,
                         const std::string &k0, const std::string &k1) {
    std::string s = "([&]() -> " + C + " { const " + C + " x = (" + C + ")(" + x + "); ";
    if (op.arity == 2) s += "const " + C + " y = (" + C + ")(" + y + "); ";
    s += "const " + C + " c0 = (" + C + ")(" + k0 + "); const " + C + " c1 = (" + C + ")(" + k1 + "); ";
    s += "(void)c0; (void)c1; return (" + C + ")(" + op.expr + "); }())";
    return s;
}

// compile the expression for every compute type a kernel may use (NVRTC, no device needed)
static std::string validate(const UserOp &op) {
    std::string src = std::string(NBG_PRELUDE_SRC) + "\n";
    const char *types[] = {"float", "double", "int", "long long"};
    src += "extern \"C\" __global__ void nbg_userop_validate(void *p) {\n";
    int k = 0;
    for (const char *T : types) {
        const std::string C = T;
        src += "  { " + C + " *q = (" + C + " *)p + " + std::to_string(8 * k++) + "; q[0] = " +
               user_op_call(op, C, "q[1]", "q[2]", "q[3]", "q[4]") + "; }\n";
    }
    src += "}\n";
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, src.c_str(), "userop.cu", 0, nullptr, nullptr) != NVRTC_SUCCESS) return "nvrtcCreateProgram failed";
    const char *opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "-std=c++17", "-default-device", "--device-int128"};
    nvrtcResult r = nvrtcCompileProgram(prog, (int)(sizeof opts / sizeof opts[0]), opts);
    std::string log;
    if (r != NVRTC_SUCCESS) {
        size_t ls = 0;
        nvrtcGetProgramLogSize(prog, &ls);
        log.assign(ls, '\0');
        nvrtcGetProgramLog(prog, &log[0]);
        log = std::string(nvrtcGetErrorString(r)) + "\n" + log.substr(0, 2000);
    }
    nvrtcDestroyProgram(&prog);
    return log;
}

int user_op_define(int arity, const std::string &name, const std::string &expr, std::string *err) {
    if (expr.empty() || expr.size() > 4096) {
        if (err) *err = "empty or oversized expression";
        return -1;
    }
    // the expression is spliced inside a lambda body's return statement: reject text that could
    // close it early (a ';' or an unbalanced brace / parenthesis)
    int par = 0, br = 0;
    for (char ch : expr) {
        if (ch == ';' || ch == '`') { if (err) *err = "';' not allowed in an operator expression"; return -1; }
        par += ch == '(' ? 1 : (ch == ')' ? -1 : 0);
        br += ch == '{' ? 1 : (ch == '}' ? -1 : 0);
        if (par < 0 || br < 0) { if (err) *err = "unbalanced parentheses or braces"; return -1; }
    }
    if (par || br) { if (err) *err = "unbalanced parentheses or braces"; return -1; }
    UserOp op;
    op.arity = arity;
    op.name = name;
    op.expr = expr;
    std::string log = validate(op);
    if (!log.empty()) {
        if (err) *err = "operator expression does not compile: " + log;
        return -1;
    }
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_ops.size() >= 100000) {
        if (err) *err = "too many user operators";
        return -1;
    }
    g_ops.push_back(op);
    return NBG_USER_OP_BASE + (int)g_ops.size() - 1;
}

}  // namespace nbg

using namespace nbg;

extern "C" {

static nbg_status define(int arity, const char *name, const char *expr, int *code) {
    if (!expr || !code) return NBG_NULL_POINTER;
    std::string err;
    const int c = user_op_define(arity, name ? name : "", expr, &err);
    if (c < 0) {
        fprintf(stderr, "[nbg] %s\n", err.c_str());
        return NBG_INVALID_VALUE;
    }
    *code = c;
    return NBG_SUCCESS;
}

nbg_status nbg_unop_define(const char *name, const char *expr, int *code) { return define(1, name, expr, code); }
nbg_status nbg_binop_define(const char *name, const char *expr, int *code) { return define(2, name, expr, code); }

}  // extern "C"
