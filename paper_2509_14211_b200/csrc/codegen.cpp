// codegen.cpp -- region IR -> CUDA C++ source for NVRTC (sm_100a).
//
// This is the GPU form of the paper's multi-stage programming (Figs. 1,2,4,5):
// the planner hands over a region of the DAG as a small SSA program (Prog); we splice the
// operators inline into ONE loop over the output index space -- "one or two outer loops per
// wait, nested methods fused into that loop" -- and, when the region contains
// an mxv, into the epilogue of the SpMV tile loop.  Constants and iso values are runtime
// arguments (a.imm[]), so a kernel depends only on the signature, not on values.
//
// Two skeletons:
//   ewise : grid-stride loop, 4 elements per thread per step with 16-byte vector loads/stores
//           (float4 / int4 / 2x double2 / uchar4), reductions -> fp64 per-thread partial ->
//           fixed shuffle tree -> warp partials in order -> exact limb atomics (prelude).
//   spmv  : persistent CTAs walk work items (long-row chunks first, then row tiles):
//           tile:  rowptr slice -> smem offsets; gather MUL(A(i,j), x(j)) for all nonzeros of the
//                  tile into smem with lanes on consecutive nonzeros (coalesced colidx stream,
//                  neighbouring columns of a row share sectors); rows with > 32 entries are
//                  reduced by a warp (lane-strided + shuffle tree), the rest sequentially by one
//                  thread; then the epilogue program runs once per row, one thread per row.
//           chunk: CHUNK nonzeros of one long row reduced by the CTA; the CTA that completes the
//                  row's last chunk (atomic ticket) sums the chunk partials in chunk order and
//                  runs the epilogue.
//          The summation order of a row depends only on its length, so the
//          fused and the blocking mxv -- and every row partition -- produce identical row sums.
#include <algorithm>
#include <charconv>
#include <sstream>

#include "nbg_internal.hpp"

namespace nbg {

static const char *ctype(int t) {
    switch (t) {
        case NBG_BOOL: return "unsigned char";
        case NBG_INT32: return "int";
        case NBG_INT64: return "long long";
        case NBG_FP32: return "float";
        case NBG_FP64: return "double";
    }
    return "?";
}
// type in which an operator with output type t is evaluated
static const char *ctype_compute(int t) { return t == NBG_BOOL ? "long long" : ctype(t); }

// The signature is emitted into a sink: a string (the plan-cache key, exact) or a 64-bit FNV-1a
// hash of the same token stream (the region identity for learned hints, computed at every wait
// without building the string).
struct SigStr {
    std::string &s;
    void put(long long v, char sep) {
        char buf[24];
        auto r = std::to_chars(buf, buf + sizeof buf, v);
        s.append(buf, r.ptr);
        s.push_back(sep);
    }
    void ch(char c) { s.push_back(c); }
};
struct SigHash {
    uint64_t h = 1469598103934665603ull;
    void put(long long v, char sep) {
        uint64_t u = (uint64_t)v;
        for (int k = 0; k < 8; k++) {
            h ^= (u >> (8 * k)) & 0xff;
            h *= 1099511628211ull;
        }
        ch(sep);
    }
    void ch(char c) {
        h ^= (unsigned char)c;
        h *= 1099511628211ull;
    }
};
template <class S>
static void sig_emit(const Prog &p, S &s) {
    s.ch(p.spmv ? (p.tp ? 'T' : (p.lpr ? 'L' : (p.rb ? (p.rb_inline ? 'I' : (p.rb_pipe ? 'P' : 'R')) : 'S'))) : 'E');
    s.ch(p.vec ? 'v' : 's');
    s.ch(p.tma ? 'T' : 'n');
    s.put(p.nt, ',');
    s.put(p.hot_kb, '|');
    if (p.spmv) {
        s.put(p.sp.add, ','); s.put(p.sp.mul, ','); s.put(p.sp.T, ','); s.put(p.sp.xt, ',');
        s.put(p.sp.at, ','); s.put(p.sp.has_vals, '|');
    }
    for (const Ins &i : p.ins) {
        s.put((int)i.k, ':'); s.put(i.t, ':'); s.put(i.code, ':'); s.put(i.a, ':'); s.put(i.b, ':');
        s.put(i.imm0, ':'); s.put(i.imm1, ':'); s.put(i.slot, ':'); s.put((int)i.fmt, ';');
    }
    s.ch('|');
    for (const OutV &o : p.outs) {
        s.put(o.ins, '>');
        s.put(o.out, o.affine ? (o.multi ? 'A' : 'a') : (o.multi ? 'm' : (o.scatter ? 's' : ';')));
    }
    s.ch('|');
    for (const RedOut &r : p.reds) {
        s.put(r.ins, '>'); s.put(r.monoid, ':'); s.put(r.racc, ':'); s.put((int)r.fmt, ';');
    }
    s.ch('|');
    s.put(p.n_in, ','); s.put(p.n_out, ','); s.put(p.n_imm, ','); s.put(p.n_sin, ','); s.put(p.n_red, '.');
}
std::string Prog::signature() const {
    std::string str;
    str.reserve(32 + 48 * ins.size() + 12 * (outs.size() + reds.size()));
    SigStr s{str};
    sig_emit(*this, s);
    return str;
}
uint64_t Prog::sig_hash() const {
    SigHash h;
    sig_emit(*this, h);
    return h.h;
}

namespace {

struct Gen {
    const Prog &p;
    std::ostringstream o;
    explicit Gen(const Prog &pp) : p(pp) {}

    std::string v(int i) const { return "v" + std::to_string(i); }

    // store of output ov at element index `idx` (plain, or scattered through a.oscat)
    std::string scat(const OutV &ov, const std::string &idx) const {
        const std::string o = std::to_string(ov.out), T = ctype(p.ins[ov.ins].t);
        if (ov.affine) return aff(ov, idx);
        if (ov.multi)   // the exchange: the same element stored into every rank's buffer (P2P over NVLink)
            return std::string("{ const int d_ = a.oscat[") + o + "][" + idx + "]; if (d_ >= 0) { const " + T + " v_ = " + v(ov.ins) +
                   "; for (int q_ = 0; q_ < a.npeer; q_++) ((" + T + "*)a.peer[q_])[d_] = v_; } }";
        return std::string("{ const int d_ = a.oscat[") + o + "][" + idx + "]; if (d_ >= 0) ((" + T +
               "*)a.out[" + o + "])[d_] = " + v(ov.ins) + "; }";
    }
    // vector skeletons: the scatter map of 4 consecutive elements loaded once, before any store of
    // the trip (a per-element map load after the previous element's store cannot be hoisted above
    // it -- the compiler must assume they alias -- so each element would cost a round trip)
    // affine target (contiguous slice of an exchange buffer): out[ooff + i] for i < olim, no map
    std::string aff(const OutV &ov, const std::string &idx) const {
        const std::string o = std::to_string(ov.out), T = ctype(p.ins[ov.ins].t);
        const std::string d = "a.ooff[" + o + "] + (" + idx + ")";
        if (ov.multi)
            return "{ if ((" + idx + ") < a.olim[" + o + "]) { const " + T + " v_ = " + v(ov.ins) + "; for (int q_ = 0; q_ < a.npeer; q_++) ((" + T +
                   "*)a.peer[q_])[" + d + "] = v_; } }";
        return "{ if ((" + idx + ") < a.olim[" + o + "]) ((" + T + "*)a.out[" + o + "])[" + d + "] = " + v(ov.ins) + "; }";
    }
    std::string scat_preload(const OutV &ov, const std::string &vi) const {
        const std::string o = std::to_string(ov.out);
        if (ov.affine) return "";
        return "const int4 M" + o + "_ = __ldg(((const int4*)a.oscat[" + o + "]) + " + vi + ");";
    }
    std::string scat_pre(const OutV &ov, const std::string &e, const std::string &idx) const {
        const std::string o = std::to_string(ov.out), T = ctype(p.ins[ov.ins].t);
        if (ov.affine) return aff(ov, idx);
        const std::string d = "(" + e + " == 0 ? M" + o + "_.x : (" + e + " == 1 ? M" + o + "_.y : (" + e + " == 2 ? M" + o + "_.z : M" + o + "_.w)))";
        if (ov.multi)
            return std::string("{ const int d_ = ") + d + "; if (d_ >= 0) { const " + T + " v_ = " + v(ov.ins) +
                   "; for (int q_ = 0; q_ < a.npeer; q_++) ((" + T + "*)a.peer[q_])[d_] = v_; } }";
        return std::string("{ const int d_ = ") + d + "; if (d_ >= 0) ((" + T + "*)a.out[" + o + "])[d_] = " + v(ov.ins) + "; }";
    }
    std::string store(const OutV &ov, const std::string &idx) const {
        if (ov.scatter) return scat(ov, idx);
        return std::string("((") + ctype(p.ins[ov.ins].t) + "*)a.out[" + std::to_string(ov.out) + "])[" + idx + "] = " + v(ov.ins) + ";";
    }

    std::string cvt(int to, const std::string &x) const {
        if (to == NBG_BOOL) return "((unsigned char)((" + x + ") != 0))";
        return "((" + std::string(ctype(to)) + ")(" + x + "))";
    }

    // expression computing instruction i (operands are already-declared variables)
    std::string expr(const Ins &in, const std::string &accname) const {
        const std::string C = ctype_compute(in.t);
        auto opnd = [&](int j) { return "((" + C + ")(" + v(j) + "))"; };
        auto k0 = [&]() { return "((" + C + ")(a.imm[" + std::to_string(in.imm0) + "]))"; };
        auto k1 = [&]() { return "((" + C + ")(a.imm[" + std::to_string(in.imm1) + "]))"; };
        std::string r;
        switch (in.k) {
            case Ins::LD_VEC:
                return "";   // handled by the skeleton
            case Ins::LD_ISO:
            case Ins::LD_SHOST:
                return cvt(in.t, "a.imm[" + std::to_string(in.slot) + "]");
            case Ins::LD_SDEV:
                if (is_float(in.t))
                    return cvt(in.t, "nbg_sval(a.sin[" + std::to_string(in.slot) + "], " + std::to_string(in.fmt) + ")");
                return cvt(in.t, "nbg_sval_i(a.sin[" + std::to_string(in.slot) + "], " + std::to_string(in.fmt) + ")");
            case Ins::MXV_ACC:
                return cvt(in.t, accname);
            case Ins::CVT:
                return cvt(in.t, v(in.a));
            case Ins::UN: {
                std::string x = opnd(in.a);
                switch (in.code) {
                    case NBG_IDENTITY: r = x; break;
                    case NBG_AINV: r = "(-" + x + ")"; break;
                    case NBG_ABS: r = "nbg_abs(" + x + ")"; break;
                    case NBG_MINV: r = "nbg_div((" + C + ")1, " + x + ")"; break;
                    case NBG_ADD_C: r = "(" + x + " + " + k0() + ")"; break;
                    case NBG_MUL_C: r = "(" + x + " * " + k0() + ")"; break;
                    case NBG_AXPB: r = "((" + k0() + " * " + x + ") + " + k1() + ")"; break;
                    case NBG_ABS_SUB_C: r = "nbg_abs(" + x + " - " + k0() + ")"; break;
                    case NBG_RECIP_SCALED:
                        r = "((" + x + " != (" + C + ")0) ? nbg_div(" + k0() + ", " + x + ") : (" + C + ")0)";
                        break;
                    case NBG_ISZERO: r = "((" + x + " == (" + C + ")0) ? (" + C + ")1 : (" + C + ")0)"; break;
                    default: {
                        const UserOp *u = user_op(in.code);
                        if (!u || u->arity != 1) fail(NBG_INVALID_VALUE, "codegen: unop code");
                        r = user_op_call(*u, C, x, "", "a.imm[" + std::to_string(in.imm0) + "]",
                                         "a.imm[" + std::to_string(in.imm1) + "]");
                    }
                }
                break;
            }
            case Ins::BIN: {
                std::string x = opnd(in.a), y = opnd(in.b);
                switch (in.code) {
                    case NBG_PLUS: r = "(" + x + " + " + y + ")"; break;
                    case NBG_MINUS: r = "(" + x + " - " + y + ")"; break;
                    case NBG_TIMES: r = "(" + x + " * " + y + ")"; break;
                    case NBG_DIV: r = "nbg_div(" + x + ", " + y + ")"; break;
                    case NBG_MIN: r = "nbg_min(" + x + ", " + y + ")"; break;
                    case NBG_MAX: r = "nbg_max(" + x + ", " + y + ")"; break;
                    case NBG_FIRST: r = x; break;
                    case NBG_SECOND: r = y; break;
                    case NBG_ABSDIFF: r = "nbg_abs(" + x + " - " + y + ")"; break;
                    case NBG_MAX_DIVX_C: r = "nbg_max(nbg_div(" + x + ", " + k0() + "), " + y + ")"; break;
                    default: {
                        const UserOp *u = user_op(in.code);
                        if (!u || u->arity != 2) fail(NBG_INVALID_VALUE, "codegen: binop code");
                        r = user_op_call(*u, C, x, y, in.imm0 >= 0 ? "a.imm[" + std::to_string(in.imm0) + "]" : "0", "0");
                    }
                }
                break;
            }
        }
        if (in.t == NBG_BOOL) return "((unsigned char)((" + r + ") != 0))";
        return r;
    }

    // --- reductions
    struct RedKind { std::string acct, ident, comb; int kind; };
    // index of a float PLUS reduction over fp64 terms among the region's exact reductions (-1: none)
    int xidx(const RedOut &r) const {
        int k = 0;
        for (const RedOut &q : p.reds) {
            if (&q == &r) return exact_red(q) ? k : -1;
            if (exact_red(q)) k++;
        }
        return -1;
    }
    int n_exact() const {
        int k = 0;
        for (const RedOut &q : p.reds) k += exact_red(q) ? 1 : 0;
        return k;
    }
    // PLUS over fp64 TERMS (the value before the conversion to the reduce type): summed exactly per
    // thread (prelude nbg_xt), so the value does not depend on the grouping (DESIGN.md §4 P9).  fp32
    // terms keep the fp64 running sum (exact for the value ranges of the hot path).
    bool exact_red(const RedOut &r) const {
        if (r.monoid != NBG_PLUS || !is_float(p.ins[r.ins].t)) return false;
        const Ins &in = p.ins[r.ins];
        const int src = (in.k == Ins::CVT && in.a >= 0) ? p.ins[in.a].t : in.t;
        return src == NBG_FP64;
    }
    RedKind redkind(const RedOut &r) const {
        int t = p.ins[r.ins].t;
        bool f = is_float(t);
        // monoid evaluated on the term converted to the reduce output type (already done by the
        // planner with a CVT instruction), accumulated in fp64 (floats) or int64 (ints)
        if (r.monoid == NBG_PLUS) {
            if (f && exact_red(r)) return {"nbg_xt", "nbg_xt_zero()", "xt", 6};
            if (f) return {"double", "0.0", "+", 0};
            return {"long long", "0ll", "+", 1};
        }
        if (r.monoid == NBG_MAX) {
            if (f) return {"double", "(-__longlong_as_double(0x7ff0000000000000ll))", "max", 2};
            return {"long long", "((long long)0x8000000000000000ull)", "max", 4};
        }
        if (f) return {"double", "(__longlong_as_double(0x7ff0000000000000ll))", "min", 3};
        return {"long long", "0x7fffffffffffffffll", "min", 5};
    }
    std::string red_update(const RedOut &r, const std::string &acc, const std::string &val) const {
        RedKind k = redkind(r);
        if (k.kind == 6) return "nbg_xt_add(" + acc + ", (double)(" + val + "), &nbg_xl[" + std::to_string(xidx(r)) + "][0]);";
        std::string x = "((" + k.acct + ")(" + val + "))";
        if (k.comb == "+") return acc + " += " + x + ";";
        if (k.comb == "max") return acc + " = nbg_max(" + acc + ", " + x + ");";
        return acc + " = nbg_min(" + acc + ", " + x + ");";
    }
    // a single term straight to the global combine (long-row epilogue)
    std::string red_direct(const RedOut &r, const std::string &val) const {
        RedKind k = redkind(r);
        std::string acc = "a.racc[" + std::to_string(r.racc) + "]";
        std::string x = "((" + (k.kind == 6 ? std::string("double") : k.acct) + ")(" + val + "))";
        switch (k.kind) {
            case 0:
            case 6: return "nbg_xacc_add(" + acc + ", " + x + ");";
            case 1: return "atomicAdd(&" + acc + "[11], (u64)" + x + ");";
            case 2: return "atomicMax(&" + acc + "[11], nbg_fkey(" + x + "));";
            case 3: return "atomicMax(&" + acc + "[11], ~nbg_fkey(" + x + "));";
            case 4: return "atomicMax(&" + acc + "[11], nbg_ikey(" + x + "));";
            default: return "atomicMax(&" + acc + "[11], ~nbg_ikey(" + x + "));";
        }
    }

    void emit_uniform() {
        for (size_t i = 0; i < p.ins.size(); i++) {
            const Ins &in = p.ins[i];
            if (!in.uniform) continue;
            o << "  const " << ctype(in.t) << " " << v((int)i) << " = " << expr(in, "") << ";\n";
        }
    }
    // uniform values computed once per CTA into shared memory (spmv: keeps them out of registers
    // across the step loop) and re-read where the epilogue needs them
    int n_uniform() const {
        int k = 0;
        for (const Ins &in : p.ins) k += in.uniform ? 1 : 0;
        return k;
    }
    void emit_uniform_to_smem(const std::string &arr) {
        o << "  if (threadIdx.x == 0) {\n";
        int k = 0;
        for (size_t i = 0; i < p.ins.size(); i++) {
            const Ins &in = p.ins[i];
            if (!in.uniform) continue;
            o << "    const " << ctype(in.t) << " " << v((int)i) << " = " << expr(in, "") << ";\n";
            o << "    *(" << ctype(in.t) << "*)&" << arr << "[" << k++ << "] = " << v((int)i) << ";\n";
        }
        o << "  }\n";
    }
    void emit_uniform_reload(const std::string &ind, const std::string &arr) {
        int k = 0;
        for (size_t i = 0; i < p.ins.size(); i++) {
            const Ins &in = p.ins[i];
            if (!in.uniform) continue;
            o << ind << "const " << ctype(in.t) << " " << v((int)i) << " = *(const " << ctype(in.t) << "*)&" << arr << "[" << k++ << "];\n";
        }
    }
    // every thread must reach this (top level of the kernel): it may contain a __syncthreads
    void emit_red_decl() {
        const int nx = n_exact();
        if (nx) {
            o << "  __shared__ u64 nbg_xl[" << nx << "][16];\n";
            o << "  for (int k_ = threadIdx.x; k_ < " << 16 * nx << "; k_ += blockDim.x) (&nbg_xl[0][0])[k_] = 0ull;\n";
            o << "  __syncthreads();\n";
        }
        for (size_t j = 0; j < p.reds.size(); j++) {
            RedKind k = redkind(p.reds[j]);
            o << "  " << k.acct << " r" << j << " = " << k.ident << ";\n";
        }
    }
    std::string red_finish_xt(size_t j) const {
        return "  nbg_block_finish_xt(r" + std::to_string(j) + ", &nbg_xl[" + std::to_string(xidx(p.reds[j])) + "][0], a.racc[" +
               std::to_string(p.reds[j].racc) + "]);\n";
    }
    void emit_red_finish() {
        for (size_t j = 0; j < p.reds.size(); j++) {
            RedKind k = redkind(p.reds[j]);
            if (k.kind == 6) { o << red_finish_xt(j); continue; }
            if (k.acct == "double")
                o << "  nbg_block_finish_f(r" << j << ", " << k.kind << ", a.racc[" << p.reds[j].racc << "], nbg_sh);\n";
            else
                o << "  nbg_block_finish_i(r" << j << ", " << k.kind << ", a.racc[" << p.reds[j].racc << "], nbg_sh);\n";
        }
    }

    // LD_VEC values of the body loaded ahead of time (declared, loaded when `cond` holds)
    template <class LD>
    void emit_hoisted_loads(const std::string &ind, LD ld, const std::string &cond) {
        for (size_t i = 0; i < p.ins.size(); i++) {
            const Ins &in = p.ins[i];
            if (in.uniform || in.k != Ins::LD_VEC) continue;
            o << ind << ctype(in.t) << " " << v((int)i) << " = (" << ctype(in.t) << ")0;\n";
        }
        o << ind << "if (" << cond << ") {\n";
        for (size_t i = 0; i < p.ins.size(); i++) {
            const Ins &in = p.ins[i];
            if (in.uniform || in.k != Ins::LD_VEC) continue;
            o << ind << "  " << v((int)i) << " = " << ld(in) << ";\n";
        }
        o << ind << "}\n";
    }

    // per-element body: non-uniform instructions; LD_VEC reads `ld(slot)`; outputs/reductions
    // through the given callbacks.
    template <class LD, class ST, class RD>
    void emit_body(const std::string &ind, LD ld, ST st, RD rd, const std::string &accname, bool hoisted = false) {
        for (size_t i = 0; i < p.ins.size(); i++) {
            const Ins &in = p.ins[i];
            if (in.uniform) continue;
            if (in.k == Ins::LD_VEC) {
                if (!hoisted) o << ind << "const " << ctype(in.t) << " " << v((int)i) << " = " << ld(in) << ";\n";
            } else {
                o << ind << "const " << ctype(in.t) << " " << v((int)i) << " = " << expr(in, accname) << ";\n";
            }
        }
        for (const OutV &ov : p.outs) o << ind << st(ov) << "\n";
        for (size_t j = 0; j < p.reds.size(); j++) o << ind << rd(j) << "\n";
    }
};

// vector load / store helpers for 4 consecutive elements of type t at vector index `vi`
std::string vload(int t, const std::string &ptr, const std::string &vi, const std::string &dst) {
    std::ostringstream s;
    switch (t) {
        case NBG_FP32:
            s << "{ const float4 q = __ldg(((const float4*)(" << ptr << ")) + " << vi << "); " << dst << "[0]=q.x; "
              << dst << "[1]=q.y; " << dst << "[2]=q.z; " << dst << "[3]=q.w; }";
            break;
        case NBG_INT32:
            s << "{ const int4 q = __ldg(((const int4*)(" << ptr << ")) + " << vi << "); " << dst << "[0]=q.x; "
              << dst << "[1]=q.y; " << dst << "[2]=q.z; " << dst << "[3]=q.w; }";
            break;
        case NBG_FP64:
            s << "{ const double2 q0 = __ldg(((const double2*)(" << ptr << ")) + 2*" << vi << "); const double2 q1 = __ldg(((const double2*)(" << ptr
              << ")) + 2*" << vi << "+1); " << dst << "[0]=q0.x; " << dst << "[1]=q0.y; " << dst << "[2]=q1.x; " << dst
              << "[3]=q1.y; }";
            break;
        case NBG_INT64:
            s << "{ const longlong2 q0 = __ldg(((const longlong2*)(" << ptr << ")) + 2*" << vi
              << "); const longlong2 q1 = __ldg(((const longlong2*)(" << ptr << ")) + 2*" << vi << "+1); " << dst
              << "[0]=q0.x; " << dst << "[1]=q0.y; " << dst << "[2]=q1.x; " << dst << "[3]=q1.y; }";
            break;
        case NBG_BOOL:
            s << "{ const uchar4 q = ((const uchar4*)(" << ptr << "))[" << vi << "]; " << dst << "[0]=q.x; " << dst
              << "[1]=q.y; " << dst << "[2]=q.z; " << dst << "[3]=q.w; }";
            break;
    }
    return s.str();
}
std::string vstore(int t, const std::string &ptr, const std::string &vi, const std::string &src) {
    std::ostringstream s;
    switch (t) {
        case NBG_FP32:
            s << "((float4*)(" << ptr << "))[" << vi << "] = make_float4(" << src << "[0], " << src << "[1], " << src << "[2], " << src << "[3]);";
            break;
        case NBG_INT32:
            s << "((int4*)(" << ptr << "))[" << vi << "] = make_int4(" << src << "[0], " << src << "[1], " << src << "[2], " << src << "[3]);";
            break;
        case NBG_FP64:
            s << "((double2*)(" << ptr << "))[2*" << vi << "] = make_double2(" << src << "[0], " << src << "[1]); ((double2*)(" << ptr
              << "))[2*" << vi << "+1] = make_double2(" << src << "[2], " << src << "[3]);";
            break;
        case NBG_INT64:
            s << "((longlong2*)(" << ptr << "))[2*" << vi << "] = make_longlong2(" << src << "[0], " << src << "[1]); ((longlong2*)(" << ptr
              << "))[2*" << vi << "+1] = make_longlong2(" << src << "[2], " << src << "[3]);";
            break;
        case NBG_BOOL:
            s << "((uchar4*)(" << ptr << "))[" << vi << "] = make_uchar4(" << src << "[0], " << src << "[1], " << src << "[2], " << src << "[3]);";
            break;
    }
    return s.str();
}

int gen_ewise(Gen &g, const std::string &kname, bool vec) {
    const Prog &p = g.p;
    auto &o = g.o;
    // which slots are loaded, with their types
    std::vector<int> slot_type(p.n_in, -1);
    for (const Ins &in : p.ins)
        if (in.k == Ins::LD_VEC) slot_type[in.slot] = in.t;
    std::vector<int> out_type(p.n_out, -1);
    for (const OutV &ov : p.outs)
        if (!ov.scatter) out_type[ov.out] = p.ins[ov.ins].t;

    // an exact reduction (nbg_xt) raises register use: keep 6 blocks of 256 threads resident so the
    // grid-stride loads keep enough bytes in flight
    o << "extern \"C\" __global__ void __launch_bounds__(256" << (g.n_exact() ? ", 6" : "") << ") " << kname << "(const KArgs a) {\n";
    o << "  __shared__ double nbg_sh[32];\n";
    g.emit_uniform();
    g.emit_red_decl();
    o << "  const long long n = a.n;\n";
    o << "  const long long stride = (long long)gridDim.x * blockDim.x;\n";
    o << "  long long tail0 = 0;\n";
    int smem = 0;
    long long v0 = 0;   // first vector index of the register skeleton (after the TMA tiles)
    (void)v0;
    if (vec && p.tma) {
        // TMA skeleton: the CTA's tiles of TV 4-element vectors of every loaded input are staged
        // in shared memory by bulk copies, NST stages deep (one thread arms each stage's mbarrier
        // with the byte count; the copies complete on it); all threads compute from shared memory.
        // Bytes in flight per SM no longer depend on registers per thread.  Whole tiles only; the
        // rest goes through the register skeleton below.
        int sumsz = 0;
        for (int s2 = 0; s2 < p.n_in; s2++)
            if (slot_type[s2] >= 0) sumsz += (int)type_size(slot_type[s2]);
        const int TV = sumsz <= 8 ? 512 : 256, NST = 4;
        std::vector<int> off(p.n_in, -1);
        int stage_bytes = 0;
        for (int s2 = 0; s2 < p.n_in; s2++)
            if (slot_type[s2] >= 0) { off[s2] = stage_bytes; stage_bytes += TV * 4 * (int)type_size(slot_type[s2]); }
        smem = NST * stage_bytes;
        o << "  extern __shared__ __align__(128) unsigned char nbg_dyn[];\n";
        o << "  __shared__ __align__(8) u64 nbg_full[" << NST << "];\n";
        o << "  const long long ntile = (n >> 2) / " << TV << ";\n";
        o << "  if (threadIdx.x == 0) {\n";
        o << "    for (int s_ = 0; s_ < " << NST << "; s_++) nbg_mbar_init(&nbg_full[s_], 1);\n";
        o << "    nbg_fence_proxy_async();\n";
        o << "  }\n";
        o << "  __syncthreads();\n";
        // issue tile t into stage s_
        o << "  auto nbg_issue = [&](int s_, long long t_) {\n";
        o << "    nbg_mbar_expect_tx(&nbg_full[s_], " << stage_bytes << "u);\n";
        for (int s2 = 0; s2 < p.n_in; s2++)
            if (slot_type[s2] >= 0) {
                const int bytes = TV * 4 * (int)type_size(slot_type[s2]);
                o << "    nbg_bulk_g2s(nbg_dyn + s_ * " << stage_bytes << " + " << off[s2] << ", (const unsigned char*)a.in[" << s2 << "] + t_ * "
                  << bytes << "ll, " << bytes << "u, &nbg_full[s_]);\n";
            }
        o << "  };\n";
        o << "  if (threadIdx.x == 0)\n";
        o << "    for (int s_ = 0; s_ < " << NST << "; s_++) { const long long t_ = blockIdx.x + (long long)s_ * gridDim.x; if (t_ < ntile) nbg_issue(s_, t_); }\n";
        o << "  int it_ = 0;\n";
        o << "  for (long long t_ = blockIdx.x; t_ < ntile; t_ += gridDim.x, it_++) {\n";
        o << "    const int s_ = it_ % " << NST << ";\n";
        o << "    nbg_mbar_wait(&nbg_full[s_], (unsigned)((it_ / " << NST << ") & 1));\n";
        o << "    for (int u_ = threadIdx.x; u_ < " << TV << "; u_ += blockDim.x) {\n";
        o << "      const long long vi = t_ * " << TV << " + u_;\n";
        for (int s2 = 0; s2 < p.n_in; s2++)
            if (slot_type[s2] >= 0) {
                const std::string T = ctype(slot_type[s2]);
                o << "      " << T << " L" << s2 << "[4];\n";
                o << "      { const " << T << " *q_ = (const " << T << "*)(nbg_dyn + s_ * " << stage_bytes << " + " << off[s2]
                  << ") + 4 * u_; L" << s2 << "[0] = q_[0]; L" << s2 << "[1] = q_[1]; L" << s2 << "[2] = q_[2]; L" << s2 << "[3] = q_[3]; }\n";
            }
        for (int k = 0; k < p.n_out; k++)
            if (out_type[k] >= 0) o << "      " << ctype(out_type[k]) << " O" << k << "[4];\n";
        o << "      #pragma unroll\n      for (int e = 0; e < 4; e++) {\n";
        g.emit_body(
            "        ", [&](const Ins &in) { return "L" + std::to_string(in.slot) + "[e]"; },
            [&](const OutV &ov) {
                if (ov.scatter) return g.scat(ov, "(vi * 4 + e)");
                return "O" + std::to_string(ov.out) + "[e] = " + g.v(ov.ins) + ";";
            },
            [&](size_t j) { return g.red_update(p.reds[j], "r" + std::to_string(j), g.v(p.reds[j].ins)); }, "");
        o << "      }\n";
        for (int k = 0; k < p.n_out; k++)
            if (out_type[k] >= 0) o << "      " << vstore(out_type[k], "a.out[" + std::to_string(k) + "]", "vi", "O" + std::to_string(k)) << "\n";
        o << "    }\n";
        // every thread is done with stage s_: refill it (generic-proxy reads before async-proxy writes)
        o << "    __syncthreads();\n";
        o << "    if (threadIdx.x == 0) { const long long t2_ = t_ + (long long)" << NST << " * gridDim.x; if (t2_ < ntile) { nbg_fence_proxy_async(); nbg_issue(s_, t2_); } }\n";
        o << "  }\n";
        o << "  const long long vstart_ = ntile * " << TV << ";\n";
    } else {
        o << "  const long long vstart_ = 0;\n";
    }
    if (vec) {
        // 4 grid-stride iterations per trip: all 16-byte loads of the trip are issued before any
        // use, so every thread keeps 4 loads per input in flight (memory-level parallelism)
        o << "  const long long nv = n >> 2;\n  tail0 = nv << 2;\n";
        const char *eu = getenv("NBG_EWISE_UNROLL");
        const int U = (eu && (eu[0] == '1' || eu[0] == '2' || eu[0] == '4' || eu[0] == '8')) ? eu[0] - '0' : 1;
        o << "  for (long long vb_ = vstart_ + (long long)blockIdx.x * blockDim.x + threadIdx.x; vb_ < nv; vb_ += " << U << " * stride) {\n";
        for (int s = 0; s < p.n_in; s++)
            if (slot_type[s] >= 0) o << "    " << ctype(slot_type[s]) << " L" << s << "[" << U << "][4];\n";
        o << "    #pragma unroll\n    for (int u = 0; u < " << U << "; u++) {\n";
        o << "      const long long vi = vb_ + u * stride;\n";
        o << "      if (vi < nv) {\n";
        for (int s = 0; s < p.n_in; s++)
            if (slot_type[s] >= 0)
                o << "        " << vload(slot_type[s], "a.in[" + std::to_string(s) + "]", "vi", "L" + std::to_string(s) + "[u]") << "\n";
        o << "      }\n";
        o << "    }\n";
        o << "    #pragma unroll\n    for (int u = 0; u < " << U << "; u++) {\n";
        o << "      const long long vi = vb_ + u * stride;\n";
        o << "      if (vi >= nv) break;\n";
        for (const OutV &ov : p.outs)
            if (ov.scatter) o << "      " << g.scat_preload(ov, "vi") << "\n";
        for (int k = 0; k < p.n_out; k++)
            if (out_type[k] >= 0) o << "      " << ctype(out_type[k]) << " O" << k << "[4];\n";
        o << "      #pragma unroll\n      for (int e = 0; e < 4; e++) {\n";
        g.emit_body(
            "        ", [&](const Ins &in) { return "L" + std::to_string(in.slot) + "[u][e]"; },
            [&](const OutV &ov) {
                if (ov.scatter) return g.scat_pre(ov, "e", "(vi * 4 + e)");
                return "O" + std::to_string(ov.out) + "[e] = " + g.v(ov.ins) + ";";
            },
            [&](size_t j) { return g.red_update(p.reds[j], "r" + std::to_string(j), g.v(p.reds[j].ins)); }, "");
        o << "      }\n";
        for (int k = 0; k < p.n_out; k++)
            if (out_type[k] >= 0) o << "      " << vstore(out_type[k], "a.out[" + std::to_string(k) + "]", "vi", "O" + std::to_string(k)) << "\n";
        o << "    }\n";
        o << "  }\n";
    }
    o << "  for (long long i = tail0 + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {\n";
    g.emit_body(
        "    ",
        [&](const Ins &in) { return std::string("((const ") + ctype(in.t) + "*)a.in[" + std::to_string(in.slot) + "])[i]"; },
        [&](const OutV &ov) { return g.store(ov, "i"); },
        [&](size_t j) { return g.red_update(p.reds[j], "r" + std::to_string(j), g.v(p.reds[j].ins)); }, "");
    o << "  }\n";
    g.emit_red_finish();
    o << "}\n";
    return smem;
}

static int redkind(const Gen &g, const RedOut &r) { return g.redkind(r).kind; }

// SpMV skeleton v6.  The matrix plan stores every row padded to 4-entry
// groups (index -1 = padding), so one 16-byte index load never mixes two rows.  One CTA of 1024
// threads per SM; the CTA owns tasks b, b + G, ... (G = grid size) and its 32 warps pull them
// from a shared-memory counter.
//   row task  (<= 128 consecutive rows, <= 512 groups): the warp streams the task's groups, lane l
//             owning group base + l (one row) per step; the next step's indices are prefetched;
//             the 4 gathers per lane are predicated loads (hot-column cache in shared memory, else
//             L1/L2).  Row starts/ends of the step are two warp OR-reductions; a segmented warp
//             scan keyed by those starts combines lane sums into row totals (carry across steps).
//             Lane j then runs the fused epilogue for rows rb + j + 32 r (coalesced loads/stores).
//   chunk task (512 groups of a longer row): lane-strided 16-entry batches, fixed shuffle tree ->
//             chunk partial; the warp that completes the row's last chunk (atomic ticket) sums
//             the chunk partials in chunk order and runs the epilogue.
// Floating PLUS reductions of the epilogue are summed per task in fp64 (fixed tree) and the task
// partials added EXACTLY into per-warp fixed-point limbs, so the dynamic task order changes
// nothing: every result is deterministic.  Summation order inside a row is fixed by the matrix
// plan (the same for the fused and the per-op mxv).
// The task's step loop with G groups per lane (step = 32 G groups, 4 G gathers in flight per lane):
// lane l owns groups b + G l .. b + G l + G - 1.  Same row bookkeeping as the G = 2 loop (row-start
// bitmask s_sbm, one segmented warp scan per step, carry across steps), generalised over the G
// group positions of a lane: the scan value is the sum since the lane's last row start (the whole
// lane when none starts in it); rows that end inside the lane are written after the scan.
static void gen_spmv_steps_g(Gen &g, int G, const std::string &ACC, const std::string &IDENT, const char *XT) {
    auto &o = g.o;
    const std::string gs = std::to_string(G), ss = std::to_string(32 * G);
    for (int k = 0; k < G; k++)
        o << "      int4 q" << k << " = (" << gs << " * lane + " << k << " < NG) ? __ldcs(CG + G0 + " << gs << " * lane + " << k
          << ") : make_int4(-1, -1, -1, -1);\n";
    o << "      int rs_[4];\n";
    o << "      #pragma unroll\n      for (int r = 0; r < 4; r++) { const int j = lane + 32 * r; rs_[r] = (j <= R) ? (int)(GRP[tl.x + j] - G0) : NG; }\n";
    o << "      const int r128_ = (lane == 0 && 128 <= R) ? (int)(GRP[tl.x + 128] - G0) : NG;\n";
    o << "      unsigned nem_[4];\n";
    o << "      #pragma unroll\n      for (int r = 0; r < 4; r++) {\n";
    o << "        const int nx = __shfl_down_sync(0xffffffffu, rs_[r], 1);\n";
    o << "        const int nf = __shfl_sync(0xffffffffu, r < 3 ? rs_[r < 3 ? r + 1 : 3] : r128_, 0);\n";
    o << "        const int re = (lane == 31) ? nf : nx;\n";
    o << "        nem_[r] = __ballot_sync(0xffffffffu, lane + 32 * r < R && re > rs_[r]);\n";
    o << "      }\n";
    o << "      s_sbm[lane] = 0u;\n";
    o << "      __syncwarp();\n";
    o << "      #pragma unroll\n      for (int r = 0; r < 4; r++) if ((nem_[r] >> lane) & 1u) atomicOr(&s_sbm[rs_[r] >> 5], 1u << (rs_[r] & 31));\n";
    o << "      __syncwarp();\n";
    o << "      " << ACC << " carry = " << IDENT << ";\n";
    o << "      int nstarted = 0;\n";
    o << "      for (int b = 0; b < NG; b += " << ss << ") {\n";
    o << "        const long long P_ = 4 * (G0 + b + " << gs << " * lane);\n";
    for (int k = 0; k < G; k++) o << "        const int4 c" << k << " = q" << k << ";\n";
    for (int k = 0; k < G; k++)
        o << "        const " << XT << " g" << k << "x = NBG_GV(c" << k << ".x), g" << k << "y = NBG_GV(c" << k << ".y), g" << k
          << "z = NBG_GV(c" << k << ".z), g" << k << "w = NBG_GV(c" << k << ".w);\n";
    o << "        if (b + " << ss << " < NG) {\n";
    for (int k = 0; k < G; k++)
        o << "          q" << k << " = (b + " << ss << " + " << gs << " * lane + " << k << " < NG) ? __ldcs(CG + G0 + b + " << ss << " + " << gs
          << " * lane + " << k << ") : make_int4(-1, -1, -1, -1);\n";
    o << "        }\n";
    // row starts of the step: G words over positions [b, b + 32 G)
    o << "        const int lw_ = (" << gs << " * lane) >> 5, sh_ = (" << gs << " * lane) & 31;\n";
    o << "        int before = 0, total_ = 0;\n";
    o << "        #pragma unroll\n        for (int w = 0; w < " << gs << "; w++) { const int pc = __popc(s_sbm[(b >> 5) + w]); total_ += pc; if (w < lw_) before += pc; }\n";
    o << "        const unsigned Mw = s_sbm[(b >> 5) + lw_];\n";
    o << "        before += __popc(Mw & ((1u << sh_) - 1u));\n";
    o << "        const unsigned bits_ = (Mw >> sh_) & " << ((1u << G) - 1u) << "u;\n";
    const char *f4[4] = {"x", "y", "z", "w"};
    for (int k = 0; k < G; k++) {
        o << "        " << ACC << " v" << k << " = NBG_TV(c" << k << ".x, P_ + " << 4 * k << ", g" << k << "x);";
        for (int e = 1; e < 4; e++)
            o << " v" << k << " = NBG_ADD(v" << k << ", NBG_TV(c" << k << "." << f4[e] << ", P_ + " << 4 * k + e << ", g" << k << f4[e] << "));";
        o << "\n";
    }
    // scan value: sum since the lane's last row start (whole lane if none)
    o << "        " << ACC << " S = " << IDENT << ";\n";
    for (int k = 0; k < G; k++) o << "        S = ((bits_ >> " << k << ") & 1u) ? v" << k << " : NBG_ADD(S, v" << k << ");\n";
    o << "        if (lane == 0 && bits_ == 0u) S = NBG_ADD(carry, S);\n";
    o << "        const unsigned H_ = __ballot_sync(0xffffffffu, bits_ != 0u) | 1u;\n";
    o << "        const int seg_ = 31 - __clz(H_ & ((2u << lane) - 1u));\n";
    o << "        #pragma unroll\n        for (int d = 1; d < 32; d <<= 1) {\n";
    o << "          const " << ACC << " Sy = __shfl_up_sync(0xffffffffu, S, d);\n";
    o << "          if (lane - d >= seg_) S = NBG_ADD(Sy, S);\n";
    o << "        }\n";
    o << "        " << ACC << " Sp = __shfl_up_sync(0xffffffffu, S, 1);\n";
    o << "        if (lane == 0) Sp = carry;\n";
    // rows ending inside the lane: before its first start the row continues from Sp
    o << "        {\n";
    o << "          " << ACC << " run_ = Sp; int wi_ = nstarted + before - 1; bool st_ = false;\n";
    for (int k = 0; k < G; k++) {
        o << "          if ((bits_ >> " << k << ") & 1u) { if (st_ || " << (k > 0 ? "true" : "lane > 0 || nstarted > 0")
          << ") s_racc[wi_] = run_; wi_++; st_ = true; run_ = v" << k << "; }";
        o << (k + 1 < G ? " else run_ = NBG_ADD(run_, v" + std::to_string(k) + ");\n" : "\n");
    }
    o << "        }\n";
    o << "        carry = __shfl_sync(0xffffffffu, S, 31);\n";
    o << "        nstarted += total_;\n";
    o << "      }\n";
}

int gen_spmv(Gen &g, const std::string &kname, int *hot_entries) {
    const Prog &p = g.p;
    auto &o = g.o;
    const SpmvSig &sp = p.sp;
    const char *C = ctype_compute(sp.T);
    const char *XT = ctype(sp.xt);
    std::string VT = C;
    std::string ACC, IDENT, ADD;
    bool fT = is_float(sp.T);
    if (sp.add == NBG_PLUS) {
        ACC = fT ? "double" : "long long";
        IDENT = fT ? "0.0" : "0ll";
        ADD = "(A_ + B_)";
    } else if (sp.add == NBG_MIN) {
        ACC = C;
        IDENT = fT ? (sp.T == NBG_FP32 ? "__int_as_float(0x7f800000)" : "__longlong_as_double(0x7ff0000000000000ll)")
                   : (sp.T == NBG_INT32 ? "0x7fffffff" : "0x7fffffffffffffffll");
        ADD = "nbg_min(A_, B_)";
    } else {
        ACC = C;
        IDENT = fT ? (sp.T == NBG_FP32 ? "__int_as_float((int)0xff800000)" : "__longlong_as_double((long long)0xfff0000000000000ull)")
                   : (sp.T == NBG_INT32 ? "((int)0x80000000)" : "((long long)0x8000000000000000ull)");
        ADD = "nbg_max(A_, B_)";
    }
    std::string av = sp.has_vals ? std::string("((") + C + ")(((const " + ctype(sp.at) + "*)a.aval)[P_]))"
                                 : std::string("((") + C + ")(a.imm[0]))";
    std::string xv = std::string("((") + C + ")(X_))";
    std::string mul;
    switch (sp.mul) {
        case NBG_PLUS: mul = "(" + av + " + " + xv + ")"; break;
        case NBG_MINUS: mul = "(" + av + " - " + xv + ")"; break;
        case NBG_TIMES: mul = "(" + av + " * " + xv + ")"; break;
        case NBG_DIV: mul = "nbg_div(" + av + ", " + xv + ")"; break;
        case NBG_MIN: mul = "nbg_min(" + av + ", " + xv + ")"; break;
        case NBG_MAX: mul = "nbg_max(" + av + ", " + xv + ")"; break;
        case NBG_FIRST: mul = av; break;
        case NBG_SECOND: mul = xv; break;
        case NBG_ABSDIFF: mul = "nbg_abs(" + av + " - " + xv + ")"; break;
        case NBG_MAX_DIVX_C: mul = "nbg_max(nbg_div(" + av + ", ((" + std::string(C) + ")(a.imm[1]))), " + xv + ")"; break;
        default: {
            const UserOp *u = user_op(sp.mul);
            if (!u || u->arity != 2) fail(NBG_INVALID_VALUE, "codegen: semiring mul");
            mul = user_op_call(*u, C, av, xv, "a.imm[1]", "0");
        }
    }
    std::vector<int> fplus;
    for (size_t j = 0; j < p.reds.size(); j++)
        if (redkind(g, p.reds[j]) == 0) fplus.push_back((int)j);
    const int NF = (int)fplus.size();
    const int accw = (ACC == "double" || ACC == "long long") ? 8 : 4;
    // row totals of the task + row-start bitmask; an fp32 mxv keeps its fp64 row sums rounded to
    // fp32 here (the epilogue rounds them to fp32 anyway: identical values, half the bytes, which
    // leaves room for hot entries inside the shared-memory carveout step)
    const bool rt_narrow = (ACC == "double" && sp.T == NBG_FP32);
    const std::string RT = rt_narrow ? "float" : ACC;
    const int rt_bytes = rt_narrow ? 4 : 8;
    const int warp_bytes = 128 * rt_bytes + 32 * 4;
    const int xacc_bytes = 32 * NF * 12 * 8;
    const int x_bytes = (int)type_size(sp.xt);
    int nt_ = p.nt, hk_ = p.hot_kb;
    if (nt_ <= 0) spmv_variant((int)type_size(sp.xt), 0, &nt_, &hk_);
    const int NT = nt_, NW = NT / 32;
    int hot_bytes = hk_ * 1024;
    {   // keep all shared memory inside the carveout step the size aims at (132 / 164 / 196 KB):
        // crossing a step halves the L1 left beside it (measured cliffs)
        const int other = NW * warp_bytes + NW * NF * 12 * 8 + 3072;   // + static smem + the driver's 1 KB per CTA
        const int step = (hk_ >= 140 ? 196 : (hk_ >= 100 ? 164 : 132)) * 1024;
        if (hot_bytes > step - other) hot_bytes = std::max(0, step - other);
    }
    int hot_cap = hot_bytes / x_bytes;
    hot_cap = (hot_cap / 4) * 4;
    const int hot_region = (hot_cap * x_bytes + 15) / 16 * 16;
    const int dyn_bytes = hot_region + NW * warp_bytes + NW * NF * 12 * 8;
    if (hot_entries) *hot_entries = hot_cap;
    (void)accw;
    // gathered element: predicated shared/global load of the raw bits, reinterpreted as XT
    std::string gx;
    const char *ecold = getenv("NBG_SPMV_COLD");
    const std::string sfx = (ecold && std::string(ecold) == "nc") ? "nc" : "";
    switch (sp.xt) {
        case NBG_FP32: gx = "__uint_as_float(nbg_gx32" + sfx + "(s_base, X, C_, hc))"; break;
        case NBG_INT32: gx = "((int)nbg_gx32" + sfx + "(s_base, X, C_, hc))"; break;
        case NBG_FP64: gx = "__longlong_as_double((long long)nbg_gx64" + sfx + "(s_base, X, C_, hc))"; break;
        case NBG_INT64: gx = "((long long)nbg_gx64" + sfx + "(s_base, X, C_, hc))"; break;
        default: gx = "((C_) < hc ? s_hot[(C_)] : X[(C_)])"; break;
    }

    o << "#define NBG_HOT_CAP " << hot_cap << "\n#define NBG_NF " << NF << "\n";
    o << "#define NBG_ADD(A_, B_) " << ADD << "\n";
    o << "__device__ __forceinline__ " << VT << " nbg_mul(const KArgs &a, long long P_, " << XT << " X_) { return " << mul
      << "; }\n";
    // one padded position: index c (-1 = padding) at position P_ -> term of the row's sum
    o << "#define NBG_TERM(C_, P_) (((C_) >= 0) ? (" << ACC << ")nbg_mul(a, (P_), nbg_gxv(s_base, s_hot, X, (C_), hc)) : (" << ACC
      << ")(" << IDENT << "))\n";
    // split form: gather (index clamped, always safe) now, turn into a term later
    o << "#define NBG_GV(C_) nbg_gxv(s_base, s_hot, X, ((C_) > 0 ? (C_) : 0), hc)\n";
    // PLUS with SECOND (or TIMES on an iso matrix): a padding position contributes x = 0 (one select
    // on the gathered value instead of one on the accumulator type)
    const bool zero_pad = sp.add == NBG_PLUS && !sp.has_vals && (sp.mul == NBG_SECOND || sp.mul == NBG_TIMES);
    if (zero_pad)
        o << "#define NBG_TV(C_, P_, V_) ((" << ACC << ")nbg_mul(a, (P_), ((C_) >= 0) ? (V_) : (" << XT << ")0))\n";
    else
        o << "#define NBG_TV(C_, P_, V_) (((C_) >= 0) ? (" << ACC << ")nbg_mul(a, (P_), (V_)) : (" << ACC << ")(" << IDENT << "))\n";
    o << "__device__ __forceinline__ " << XT << " nbg_gxv(unsigned s_base, const " << XT << "* s_hot, const " << XT
      << "* X, int C_, int hc) { return " << gx << "; }\n";
    o << "#define NBG_NW " << NW << "\n";
    o << "extern \"C\" __global__ void __launch_bounds__(" << NT << ", 1) " << kname << "(const KArgs a) {\n";
    o << "  extern __shared__ __align__(16) unsigned char nbg_dyn[];\n";
    o << "  __shared__ double nbg_sh[32];\n";
    o << "  __shared__ int s_ctr;\n";
    o << "  " << XT << "* s_hot = (" << XT << "*)nbg_dyn;\n";
    o << "  const unsigned s_base = (unsigned)__cvta_generic_to_shared(nbg_dyn);\n";
    o << "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n";
    o << "  " << RT << "* s_racc = (" << RT << "*)(nbg_dyn + " << hot_region << " + warp * " << warp_bytes << ");   // [128] row totals\n";
    o << "  unsigned* s_sbm = (unsigned*)(nbg_dyn + " << hot_region << " + warp * " << warp_bytes << " + " << 128 * rt_bytes << ");   // [32] row starts\n";
    if (NF)
        o << "  u64* s_x = (u64*)(nbg_dyn + " << hot_region << " + NBG_NW * " << warp_bytes << ");   // [warp][NF][11]\n";
    o << "  const " << XT << "* __restrict__ X = (const " << XT << "*)a.x;\n";
    o << "  const int4* __restrict__ CG = (const int4*)a.colidx;\n";
    o << "  const long long* __restrict__ GRP = a.rowptr;\n";
    o << "  const int hc = (int)a.hc;\n";
    o << "  if (threadIdx.x == 0) s_ctr = 0;\n";
    if (NF) o << "  for (int k = threadIdx.x; k < NBG_NW * NBG_NF * 12; k += blockDim.x) s_x[k] = 0ull;\n";
    // hot-column cache: 16-byte loads, 4 in flight per thread (X is 16-byte aligned, hc % 16 == 0 or tail)
    o << "  {\n";
    o << "    const int nv_ = ((((unsigned long long)X) & 15ull) == 0ull) ? (int)((hc * sizeof(" << XT << ")) >> 4) : 0;\n";
    o << "    const uint4* src_ = (const uint4*)X; uint4* dst_ = (uint4*)nbg_dyn;\n";
    o << "    for (int k = threadIdx.x; k < nv_; k += 4 * blockDim.x) {\n";
    o << "      uint4 w_[4];\n";
    o << "      #pragma unroll\n      for (int u = 0; u < 4; u++) if (k + u * (int)blockDim.x < nv_) w_[u] = __ldg(src_ + k + u * blockDim.x);\n";
    o << "      #pragma unroll\n      for (int u = 0; u < 4; u++) if (k + u * (int)blockDim.x < nv_) dst_[k + u * blockDim.x] = w_[u];\n";
    o << "    }\n";
    o << "    for (int k = (nv_ << 4) / (int)sizeof(" << XT << ") + threadIdx.x; k < hc; k += blockDim.x) s_hot[k] = X[k];\n";
    o << "  }\n";
    const int NU = std::max(1, g.n_uniform());
    o << "  __shared__ unsigned long long s_uni[" << NU << "];\n";
    g.emit_uniform_to_smem("s_uni");
    o << "  __syncthreads();\n";
    g.emit_red_decl();
    o << "  const long long items = a.nchunks + a.ntiles;\n";
    // tasks are claimed one ahead so the next row task's header load overlaps this task
    o << "  int ln_ = 0;\n";
    o << "  if (lane == 0) ln_ = atomicAdd(&s_ctr, 1);\n";
    o << "  ln_ = __shfl_sync(0xffffffffu, ln_, 0);\n";
    o << "  long long itn_ = (long long)blockIdx.x + (long long)ln_ * gridDim.x;\n";
    o << "  int4 tn_ = (itn_ >= a.nchunks && itn_ < items) ? ((const int4*)a.tiles)[itn_ - a.nchunks] : make_int4(0, 0, 0, 0);\n";
    o << "  for (;;) {\n";
    o << "    const long long it = itn_;\n";
    o << "    if (it >= items) break;\n";
    o << "    const int4 tl = tn_;\n";
    o << "    if (lane == 0) ln_ = atomicAdd(&s_ctr, 1);\n";
    o << "    ln_ = __shfl_sync(0xffffffffu, ln_, 0);\n";
    o << "    itn_ = (long long)blockIdx.x + (long long)ln_ * gridDim.x;\n";
    o << "    if (itn_ >= a.nchunks && itn_ < items) tn_ = ((const int4*)a.tiles)[itn_ - a.nchunks];\n";
    // ---------------- one task: a row task (<= 128 rows, lane l owns rows l, l + 32, l + 64,
    // l + 96) or a chunk of one long row (R = 0: no row starts, the whole chunk is one segment)
    o << "    {\n";
    o << "      const bool is_chunk = it < a.nchunks;\n";
    o << "      int4 ch = make_int4(0, 0, 0, 0);\n";
    o << "      if (is_chunk) ch = ((const int4*)a.chunks)[it];\n";
    o << "      const int R = is_chunk ? 0 : (tl.y & 0xff), NG = is_chunk ? ch.w : (tl.y >> 8);\n";
    o << "      const long long G0 = is_chunk ? (((long long)(unsigned)ch.z << 32) | (long long)(unsigned)ch.y)\n";
    o << "                                    : (((long long)(unsigned)tl.w << 32) | (long long)(unsigned)tl.z);\n";
    // step = 64 groups: lane l owns groups b + 2l and b + 2l + 1 (8 gathers in flight per lane);
    // the next step's indices are prefetched while this step is reduced
    const bool gpipe = spmv_gather_pipeline();
    // the epilogue's per-row inputs (and scatter maps) are prefetched into L1 when the task starts,
    // so the epilogue does not wait a global round trip after the step loop (NBG_SPMV_PF=0: off)
    if (spmv_epilogue_prefetch()) {
        std::vector<int> slot_sz(p.n_in, 0);
        for (const Ins &in : p.ins)
            if (in.k == Ins::LD_VEC) slot_sz[in.slot] = (int)type_size(in.t);
        std::ostringstream pf;
        for (int s = 0; s < p.n_in; s++)
            if (slot_sz[s] > 0)
                pf << " asm volatile(\"prefetch.global.L1 [%0];\" :: \"l\"((const char*)a.in[" << s << "] + " << slot_sz[s] << " * i));";
        for (const OutV &ov : p.outs)
            if (ov.scatter && !ov.affine) pf << " asm volatile(\"prefetch.global.L1 [%0];\" :: \"l\"(a.oscat[" << ov.out << "] + i));";
        if (!pf.str().empty()) {
            o << "      if (!is_chunk) {\n";
            o << "        #pragma unroll\n        for (int r = 0; r < 4; r++) { const long long i = (long long)tl.x + lane + 32 * r; if (lane + 32 * r < R) {" << pf.str() << " } }\n";
            o << "      }\n";
        }
    }
    const int GPL = gpipe ? 2 : spmv_groups_per_lane();
    if (GPL != 2) {
        gen_spmv_steps_g(g, GPL, ACC, IDENT, XT);
    } else {
        o << "      int4 qa = (2 * lane < NG) ? __ldcs(CG + G0 + 2 * lane) : make_int4(-1, -1, -1, -1);\n";
        o << "      int4 qb = (2 * lane + 1 < NG) ? __ldcs(CG + G0 + 2 * lane + 1) : make_int4(-1, -1, -1, -1);\n";
        if (gpipe) {
            // gathers one step ahead: step b + 64's values are in flight while step b is reduced
            o << "      int4 ca = qa, cb = qb;\n";
            o << "      " << XT << " h0 = NBG_GV(ca.x), h1 = NBG_GV(ca.y), h2 = NBG_GV(ca.z), h3 = NBG_GV(ca.w);\n";
            o << "      " << XT << " h4 = NBG_GV(cb.x), h5 = NBG_GV(cb.y), h6 = NBG_GV(cb.z), h7 = NBG_GV(cb.w);\n";
            o << "      qa = (64 + 2 * lane < NG) ? __ldcs(CG + G0 + 64 + 2 * lane) : make_int4(-1, -1, -1, -1);\n";
            o << "      qb = (65 + 2 * lane < NG) ? __ldcs(CG + G0 + 65 + 2 * lane) : make_int4(-1, -1, -1, -1);\n";
        }
        o << "      int rs_[4];\n";
        o << "      #pragma unroll\n      for (int r = 0; r < 4; r++) { const int j = lane + 32 * r; rs_[r] = (j <= R) ? (int)(GRP[tl.x + j] - G0) : NG; }\n";
        o << "      const int r128_ = (lane == 0 && 128 <= R) ? (int)(GRP[tl.x + 128] - G0) : NG;\n";
        o << "      unsigned nem_[4];\n";
        o << "      #pragma unroll\n      for (int r = 0; r < 4; r++) {\n";
        o << "        const int nx = __shfl_down_sync(0xffffffffu, rs_[r], 1);\n";
        o << "        const int nf = __shfl_sync(0xffffffffu, r < 3 ? rs_[r < 3 ? r + 1 : 3] : r128_, 0);\n";
        o << "        const int re = (lane == 31) ? nf : nx;                     // end (exclusive) of row lane + 32 r\n";
        o << "        nem_[r] = __ballot_sync(0xffffffffu, lane + 32 * r < R && re > rs_[r]);\n";
        o << "      }\n";
        // the task's row starts as a bitmask over its groups (tasks hold < 1024 groups): one bit per
        // non-empty row, set once per task instead of recomputed every step
        o << "      s_sbm[lane] = 0u;\n";
        o << "      __syncwarp();\n";
        o << "      #pragma unroll\n      for (int r = 0; r < 4; r++) if ((nem_[r] >> lane) & 1u) atomicOr(&s_sbm[rs_[r] >> 5], 1u << (rs_[r] & 31));\n";
        o << "      __syncwarp();\n";
        o << "      " << ACC << " carry = " << IDENT << ";\n";
        o << "      int nstarted = 0;                                          // nonempty rows started before the step\n";
        o << "      for (int b = 0; b < NG; b += 64) {\n";
        o << "        const long long P_ = 4 * (G0 + b + 2 * lane);\n";
        if (gpipe) {
            o << "        const int4 ca_ = ca, cb_ = cb;\n";
            o << "        const " << XT << " g0 = h0, g1 = h1, g2 = h2, g3 = h3, g4 = h4, g5 = h5, g6 = h6, g7 = h7;\n";
            o << "        if (b + 64 < NG) {\n";
            o << "          ca = qa; cb = qb;\n";
            o << "          h0 = NBG_GV(ca.x); h1 = NBG_GV(ca.y); h2 = NBG_GV(ca.z); h3 = NBG_GV(ca.w);\n";
            o << "          h4 = NBG_GV(cb.x); h5 = NBG_GV(cb.y); h6 = NBG_GV(cb.z); h7 = NBG_GV(cb.w);\n";
            o << "          if (b + 128 < NG) {\n";
            o << "            qa = (b + 128 + 2 * lane < NG) ? __ldcs(CG + G0 + b + 128 + 2 * lane) : make_int4(-1, -1, -1, -1);\n";
            o << "            qb = (b + 129 + 2 * lane < NG) ? __ldcs(CG + G0 + b + 129 + 2 * lane) : make_int4(-1, -1, -1, -1);\n";
            o << "          }\n";
            o << "        }\n";
            o << "        const int4 ca0 = ca_, cb0 = cb_;\n";
            o << "#define ca ca0\n#define cb cb0\n";
        } else {
            o << "        const int4 ca = qa, cb = qb;\n";
            o << "        const " << XT << " g0 = NBG_GV(ca.x), g1 = NBG_GV(ca.y), g2 = NBG_GV(ca.z), g3 = NBG_GV(ca.w);\n";
            o << "        const " << XT << " g4 = NBG_GV(cb.x), g5 = NBG_GV(cb.y), g6 = NBG_GV(cb.z), g7 = NBG_GV(cb.w);\n";
            o << "        if (b + 64 < NG) {\n";
            o << "          qa = (b + 64 + 2 * lane < NG) ? __ldcs(CG + G0 + b + 64 + 2 * lane) : make_int4(-1, -1, -1, -1);\n";
            o << "          qb = (b + 65 + 2 * lane < NG) ? __ldcs(CG + G0 + b + 65 + 2 * lane) : make_int4(-1, -1, -1, -1);\n";
            o << "        }\n";
        }
        // row starts of this step: two 32-bit words over positions [0, 64)
        o << "        const unsigned M0 = s_sbm[b >> 5], M1 = s_sbm[(b >> 5) + 1];\n";
        o << "        const unsigned Mw = lane < 16 ? M0 : M1;\n";
        o << "        const int sh_ = (2 * lane) & 31;\n";
        o << "        const bool s0 = (Mw >> sh_) & 1u, s1 = (Mw >> (sh_ + 1)) & 1u;\n";
        o << "        const int before = (lane < 16 ? 0 : __popc(M0)) + __popc(Mw & ((1u << sh_) - 1u));   // starts before position 2 lane\n";
        o << "        " << ACC << " v0 = NBG_TV(ca.x, P_, g0);\n";
        o << "        v0 = NBG_ADD(v0, NBG_TV(ca.y, P_ + 1, g1)); v0 = NBG_ADD(v0, NBG_TV(ca.z, P_ + 2, g2)); v0 = NBG_ADD(v0, NBG_TV(ca.w, P_ + 3, g3));\n";
        o << "        " << ACC << " v1 = NBG_TV(cb.x, P_ + 4, g4);\n";
        o << "        v1 = NBG_ADD(v1, NBG_TV(cb.y, P_ + 5, g5)); v1 = NBG_ADD(v1, NBG_TV(cb.z, P_ + 6, g6)); v1 = NBG_ADD(v1, NBG_TV(cb.w, P_ + 7, g7));\n";
        // scan value: the segment open at the lane's end; lane 0 continues the carried row
        o << "        " << ACC << " S = s1 ? v1 : NBG_ADD(v0, v1);\n";
        o << "        if (lane == 0 && !s0 && !s1) S = NBG_ADD(carry, S);\n";
        // segmented inclusive scan bounded by the lane's segment start (highest head lane <= lane)
        o << "        const unsigned H_ = __ballot_sync(0xffffffffu, s0 || s1) | 1u;\n";
        o << "        const int seg_ = 31 - __clz(H_ & ((2u << lane) - 1u));\n";
        o << "        #pragma unroll\n        for (int d = 1; d < 32; d <<= 1) {\n";
        o << "          const " << ACC << " Sy = __shfl_up_sync(0xffffffffu, S, d);\n";
        o << "          if (lane - d >= seg_) S = NBG_ADD(Sy, S);\n";
        o << "        }\n";
        o << "        " << ACC << " Sp = __shfl_up_sync(0xffffffffu, S, 1);\n";
        o << "        if (lane == 0) Sp = carry;                                   // running total before position 0\n";
        o << "        if (s0 && (lane > 0 || nstarted > 0)) s_racc[nstarted + before - 1] = Sp;          // row ending at 2 lane - 1\n";
        o << "        if (s1) s_racc[nstarted + before + (s0 ? 1 : 0) - 1] = s0 ? v0 : NBG_ADD(Sp, v0);   // row ending at 2 lane\n";
        o << "        carry = __shfl_sync(0xffffffffu, S, 31);\n";
        o << "        nstarted += __popc(M0) + __popc(M1);\n";
        if (gpipe) o << "#undef ca\n#undef cb\n";
        o << "      }\n";
    }
    o << "      if (is_chunk) {\n";
    o << "        if (lane == 0) {\n";
    o << "          const " << ACC << " t = carry;\n";
    o << "          ((" << ACC << "*)a.partials)[it] = t;\n";
    // release on the ticket (no L1 invalidation for the other chunks), acquire fence for the winner
    o << "          const int4 lr = ((const int4*)a.longs)[ch.x];\n";
    o << "          int tk;\n";
    o << "          asm volatile(\"atom.add.release.gpu.s32 %0, [%1], 1;\" : \"=r\"(tk) : \"l\"(&a.counters[ch.x]) : \"memory\");\n";
    o << "          if (tk == lr.z - 1) {\n";
    o << "            asm volatile(\"fence.acq_rel.gpu;\" ::: \"memory\");\n";
    o << "            " << ACC << " acc = " << IDENT << ";\n";
    o << "            for (int j = 0; j < lr.z; j++) { const " << ACC << " pj = *(volatile const " << ACC << "*)(((const " << ACC
      << "*)a.partials) + lr.y + j); acc = NBG_ADD(acc, pj); }\n";
    o << "            a.counters[ch.x] = 0;\n";
    o << "            const long long i = lr.x;\n";
    g.emit_uniform_reload("            ", "s_uni");
    g.emit_body(
        "            ",
        [&](const Ins &in) { return std::string("((const ") + ctype(in.t) + "*)a.in[" + std::to_string(in.slot) + "])[i]"; },
        [&](const OutV &ov) { return g.store(ov, "i"); },
        [&](size_t j) { return g.red_direct(p.reds[j], g.v(p.reds[j].ins)); }, "acc");
    o << "          }\n";
    o << "        }\n";
    o << "        __syncwarp();\n";
    o << "        continue;\n";
    o << "      }\n";
    o << "      if (lane == 0 && nstarted > 0) s_racc[nstarted - 1] = carry;          // the task's last row\n";
    o << "      __syncwarp();\n";
    for (int j : fplus) o << "      r" << j << " = 0.0;\n";
    o << "      int rb_ = 0;                                               // nonempty rows before block r\n";
    o << "      for (int r = 0; r < 4; r++) {\n";
    o << "        const long long i = (long long)tl.x + lane + 32 * r;\n";
    o << "        const unsigned nm = r == 0 ? nem_[0] : (r == 1 ? nem_[1] : (r == 2 ? nem_[2] : nem_[3]));\n";
    o << "        if (lane + 32 * r < R) {\n";
    o << "          const " << ACC << " acc = ((nm >> lane) & 1u) ? (" << ACC << ")s_racc[rb_ + __popc(nm & ((1u << lane) - 1u))] : (" << ACC << ")(" << IDENT << ");\n";
    g.emit_uniform_reload("          ", "s_uni");
    g.emit_body(
        "          ",
        [&](const Ins &in) { return std::string("((const ") + ctype(in.t) + "*)a.in[" + std::to_string(in.slot) + "])[i]"; },
        [&](const OutV &ov) { return g.store(ov, "i"); },
        [&](size_t j) { return g.red_update(p.reds[j], "r" + std::to_string(j), g.v(p.reds[j].ins)); }, "acc");
    o << "        }\n";
    o << "        rb_ += __popc(nm);\n";
    o << "        if (32 * (r + 1) >= R) break;\n";
    o << "      }\n";
    for (int f = 0; f < NF; f++) {
        int j = fplus[f];
        o << "      { double t_ = nbg_warp_sum(r" << j << "); if (lane == 0) nbg_xacc_add_local(s_x + (warp * NBG_NF + " << f
          << ") * 12, t_); }\n";
    }
    o << "      __syncwarp();\n";
    o << "    }\n";
    o << "  }\n";
    o << "  __syncthreads();\n";
    for (int f = 0; f < NF; f++) {
        int j = fplus[f];
        o << "  if (threadIdx.x < 12) {\n";
        o << "    u64 v_ = 0ull; double d_ = 0.0;\n";
        o << "    for (int w = 0; w < NBG_NW; w++) { const u64 x_ = s_x[(w * NBG_NF + " << f << ") * 12 + threadIdx.x]; if (threadIdx.x == 11) d_ += __longlong_as_double((long long)x_); else v_ = threadIdx.x == 10 ? (v_ | x_) : v_ + x_; }\n";
        o << "    if (threadIdx.x == 11) { if (d_ != 0.0) atomicAdd((double*)&a.racc[" << p.reds[j].racc << "][12], d_); }\n";
        o << "    else if (threadIdx.x == 10) { if (v_) atomicAdd(&a.racc[" << p.reds[j].racc << "][10], nbg_xacc_flag_counts(v_)); }\n";
        o << "    else if (v_) atomicAdd(&a.racc[" << p.reds[j].racc << "][threadIdx.x], v_);\n";
        o << "  }\n";
    }
    for (size_t j = 0; j < p.reds.size(); j++) {
        if (std::find(fplus.begin(), fplus.end(), (int)j) != fplus.end()) continue;
        int kind = redkind(g, p.reds[j]);
        if (kind == 6) { o << g.red_finish_xt(j); continue; }
        if (kind == 0 || kind == 2 || kind == 3)
            o << "  nbg_block_finish_f(r" << j << ", " << kind << ", a.racc[" << p.reds[j].racc << "], nbg_sh);\n";
        else
            o << "  nbg_block_finish_i(r" << j << ", " << kind << ", a.racc[" << p.reds[j].racc << "], nbg_sh);\n";
    }
    o << "}\n";
    return dyn_bytes;
}

// ---------------------------------------------------------------- two-phase SpMV

struct SemiringCode {
    std::string C, XT, ACC, IDENT, ADD, mul;
};

SemiringCode semiring_code(const SpmvSig &sp) {
    SemiringCode r;
    r.C = ctype_compute(sp.T);
    r.XT = ctype(sp.xt);
    const bool fT = is_float(sp.T);
    if (sp.add == NBG_PLUS) {
        r.ACC = fT ? "double" : "long long";
        r.IDENT = fT ? "0.0" : "0ll";
        r.ADD = "(A_ + B_)";
    } else if (sp.add == NBG_MIN) {
        r.ACC = r.C;
        r.IDENT = fT ? (sp.T == NBG_FP32 ? "__int_as_float(0x7f800000)" : "__longlong_as_double(0x7ff0000000000000ll)")
                     : (sp.T == NBG_INT32 ? "0x7fffffff" : "0x7fffffffffffffffll");
        r.ADD = "nbg_min(A_, B_)";
    } else {
        r.ACC = r.C;
        r.IDENT = fT ? (sp.T == NBG_FP32 ? "__int_as_float((int)0xff800000)" : "__longlong_as_double((long long)0xfff0000000000000ull)")
                     : (sp.T == NBG_INT32 ? "((int)0x80000000)" : "((long long)0x8000000000000000ull)");
        r.ADD = "nbg_max(A_, B_)";
    }
    const std::string C = r.C;
    const std::string av = sp.has_vals ? "((" + C + ")(((const " + std::string(ctype(sp.at)) + "*)a.aval)[P_]))" : "((" + C + ")(a.imm[0]))";
    const std::string xv = "((" + C + ")(X_))";
    switch (sp.mul) {
        case NBG_PLUS: r.mul = "(" + av + " + " + xv + ")"; break;
        case NBG_MINUS: r.mul = "(" + av + " - " + xv + ")"; break;
        case NBG_TIMES: r.mul = "(" + av + " * " + xv + ")"; break;
        case NBG_DIV: r.mul = "nbg_div(" + av + ", " + xv + ")"; break;
        case NBG_MIN: r.mul = "nbg_min(" + av + ", " + xv + ")"; break;
        case NBG_MAX: r.mul = "nbg_max(" + av + ", " + xv + ")"; break;
        case NBG_FIRST: r.mul = av; break;
        case NBG_SECOND: r.mul = xv; break;
        case NBG_ABSDIFF: r.mul = "nbg_abs(" + av + " - " + xv + ")"; break;
        case NBG_MAX_DIVX_C: r.mul = "nbg_max(nbg_div(" + av + ", ((" + C + ")(a.imm[1]))), " + xv + ")"; break;
        default: {
            const UserOp *u = user_op(sp.mul);
            if (!u || u->arity != 2) fail(NBG_INVALID_VALUE, "codegen: semiring mul");
            r.mul = user_op_call(*u, C, av, xv, "a.imm[1]", "0");
        }
    }
    return r;
}

// Lane-per-row SpMV skeleton (SURVEY 8(a) K4 notes, "low skew": max row <= 4 x mean, mean <= 32
// entries, e.g. C3's Erdos-Renyi rows of 8-39 entries).  A warp takes 32 consecutive rows, lane j
// row rb + j: the row's 4-entry groups two at a time (8 gathers in flight per lane), summed in
// order (the same per-row order as the fused and the per-op mxv), then the fused epilogue straight
// from registers -- no tasks, scans or shared memory.  Grid-stride over 32-row tiles; epilogue
// reductions per thread, then the block finish of the elementwise skeleton.
int gen_spmv_lpr(Gen &g, const std::string &kname) {
    const Prog &p = g.p;
    auto &o = g.o;
    SemiringCode k = semiring_code(p.sp);
    const bool zero_pad = p.sp.add == NBG_PLUS && !p.sp.has_vals && (p.sp.mul == NBG_SECOND || p.sp.mul == NBG_TIMES);
    o << "#define NBG_ADD(A_, B_) " << k.ADD << "\n";
    o << "__device__ __forceinline__ " << k.C << " nbg_mul(const KArgs &a, long long P_, " << k.XT << " X_) { return " << k.mul << "; }\n";
    if (zero_pad)
        o << "#define NBG_TV(C_, P_, V_) ((" << k.ACC << ")nbg_mul(a, (P_), ((C_) >= 0) ? (V_) : (" << k.XT << ")0))\n";
    else
        o << "#define NBG_TV(C_, P_, V_) (((C_) >= 0) ? (" << k.ACC << ")nbg_mul(a, (P_), (V_)) : (" << k.ACC << ")(" << k.IDENT << "))\n";
    o << "#define NBG_G(C_) __ldg(X + ((C_) > 0 ? (C_) : 0))\n";
    o << "extern \"C\" __global__ void __launch_bounds__(256) " << kname << "(const KArgs a) {\n";
    o << "  __shared__ double nbg_sh[32];\n";
    o << "  const int lane = threadIdx.x & 31;\n";
    o << "  const " << k.XT << "* __restrict__ X = (const " << k.XT << "*)a.x;\n";
    o << "  const int4* __restrict__ CG = (const int4*)a.colidx;\n";
    o << "  const long long* __restrict__ GRP = a.rowptr;\n";
    g.emit_uniform();
    g.emit_red_decl();
    o << "  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;\n";
    o << "  for (long long rb = (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5) << 5; rb < a.n; rb += nw << 5) {\n";
    o << "    const long long i = rb + lane;\n";
    o << "    if (i >= a.n) continue;\n";
    o << "    const long long g1 = GRP[i + 1];\n";
    o << "    " << k.ACC << " acc = " << k.IDENT << ";\n";
    // UG groups per iteration (4 UG gathers in flight per lane); groups past the row end are
    // padding (-1) and contribute nothing
    const char *eug = getenv("NBG_LPR_UG");
    const int UG = (eug && (eug[0] == '1' || eug[0] == '2' || eug[0] == '4')) ? eug[0] - '0' : 4;
    o << "    for (long long gg = GRP[i]; gg < g1; gg += " << UG << ") {\n";
    o << "      const long long P_ = 4 * gg;\n";
    for (int u = 0; u < UG; u++)
        o << "      const int4 c" << u << " = (gg + " << u << " < g1) ? __ldcs(CG + gg + " << u << ") : make_int4(-1, -1, -1, -1);\n";
    for (int u = 0; u < UG; u++)
        o << "      const " << k.XT << " x" << u << "a = NBG_G(c" << u << ".x), x" << u << "b = NBG_G(c" << u << ".y), x" << u << "c = NBG_G(c" << u
          << ".z), x" << u << "d = NBG_G(c" << u << ".w);\n";
    for (int u = 0; u < UG; u++) {
        o << "      if (gg + " << u << " < g1) {\n";
        o << "        acc = NBG_ADD(acc, NBG_TV(c" << u << ".x, P_ + " << 4 * u << ", x" << u << "a)); acc = NBG_ADD(acc, NBG_TV(c" << u
          << ".y, P_ + " << 4 * u + 1 << ", x" << u << "b));\n";
        o << "        acc = NBG_ADD(acc, NBG_TV(c" << u << ".z, P_ + " << 4 * u + 2 << ", x" << u << "c)); acc = NBG_ADD(acc, NBG_TV(c" << u
          << ".w, P_ + " << 4 * u + 3 << ", x" << u << "d));\n";
        o << "      }\n";
    }
    o << "    }\n";
    g.emit_body(
        "    ",
        [&](const Ins &in) { return std::string("((const ") + ctype(in.t) + "*)a.in[" + std::to_string(in.slot) + "])[i]"; },
        [&](const OutV &ov) { return g.store(ov, "i"); },
        [&](size_t j) { return g.red_update(p.reds[j], "r" + std::to_string(j), g.v(p.reds[j].ins)); }, "acc");
    o << "  }\n";
    g.emit_red_finish();
    o << "}\n";
    return 0;
}

// Row-binned SpMV skeleton (DESIGN.md §7 "row-binned SpMV", plan RbPlan in graph.cu).  One
// persistent CTA per SM, hot-column cache in shared memory as in the task skeleton.  Warps claim
// tasks from one global counter (the largest first; the whole grid shares the tail):
//   hub chunk   : 512 groups of a row > 2048 entries; lane l sums groups l, l + 32, ... in order,
//                 fixed shuffle tree -> chunk partial; the last chunk (ticket) combines in order;
//   long rows   : up to 32 rows of T+1..512 groups, one after another by the whole warp (same
//                 lane-strided order + tree); the next step's indices load during this one;
//   short slices: up to 32 slices of 32 rows, lane l owns slot l of each slice and sums its row
//                 sequentially (entries in order); sell[base + 32 j + l] is the j-th group of the
//                 lane's run, so every index load is one coalesced 512-byte warp load and row ends
//                 are warp-uniform (no scans, no shuffles, no shared-memory bookkeeping);
//   empty rows  : (inline mode) ranges of 512 rows, the epilogue of the rows without entries.
// Epilogue, two modes:
//   inline (default): the fused epilogue of a row runs where its total completes -- per lane at a
//     slice end, per lane for the task's long rows at the task end, by the combining lane for a
//     hub -- so its loads and stores overlap the gathers of other warps; floating PLUS reductions
//     are summed per task in fp64 (fixed tree) and added exactly into per-warp limbs;
//   barrier: row totals to tot[row]; grid barrier; the epilogue over rows in index order
//     (coalesced, 4 rows per thread and trip).
// A row's summation order depends on its length only, so fused / per-op mxv and every row
// partition give identical row sums; every reduction is deterministic.
int gen_spmv_rb(Gen &g, const std::string &kname, int *hot_entries) {
    const Prog &p = g.p;
    auto &o = g.o;
    const SpmvSig &sp = p.sp;
    const bool IE = p.rb_inline, PIPE = p.rb_pipe && !IE;
    const bool PT = IE || PIPE;   // reductions summed per task (dynamic task order) rather than per thread
    SemiringCode k = semiring_code(sp);
    const std::string &ACC = k.ACC, &IDENT = k.IDENT;
    const char *XT = ctype(sp.xt);
    const bool rt_narrow = (ACC == "double" && sp.T == NBG_FP32);
    const std::string RT = rt_narrow ? "float" : ACC;
    const int x_bytes = (int)type_size(sp.xt);
    int nt_ = p.nt, hk_ = p.hot_kb;
    if (nt_ <= 0) spmv_variant(x_bytes, 0, &nt_, &hk_);
    const int NT = nt_, NW = NT / 32;
    // inline mode: floating PLUS reductions flushed per task into per-warp exact limbs
    std::vector<int> fplus;
    if (PT)
        for (size_t j = 0; j < p.reds.size(); j++)
            if (redkind(g, p.reds[j]) == 0) fplus.push_back((int)j);
    const int NF = (int)fplus.size();
    int hot_bytes = hk_ * 1024;
    {
        const int other = 4096 + NW * NF * 12 * 8;   // static shared memory + the driver's 1 KB per CTA, warp limbs
        const int step = (hk_ >= 140 ? 196 : (hk_ >= 100 ? 164 : 132)) * 1024;
        if (hot_bytes > step - other) hot_bytes = std::max(0, step - other);
    }
    int hot_cap = (hot_bytes / x_bytes / 4) * 4;
    const int hot_region = (hot_cap * x_bytes + 15) / 16 * 16;
    const int dyn_bytes = std::max(16, hot_region + NW * NF * 12 * 8);
    if (hot_entries) *hot_entries = hot_cap;
    std::string gx;
    // cold-gather qualifier: ld.global.cg (L2 only, default) or, NBG_SPMV_COLD=nc / el, the read-only path
    // with L1 allocation (plain / L1::evict_last); DESIGN.md section 7 has the measured sweep
    const char *ecold = getenv("NBG_SPMV_COLD");
    const std::string ec = ecold ? ecold : "";
    const std::string sfx = ec == "nc" ? "nc" : (ec == "el" ? "el" : "");
    switch (sp.xt) {
        case NBG_FP32: gx = "__uint_as_float(nbg_gx32" + sfx + "(s_base, X, C_, hc))"; break;
        case NBG_INT32: gx = "((int)nbg_gx32" + sfx + "(s_base, X, C_, hc))"; break;
        case NBG_FP64: gx = "__longlong_as_double((long long)nbg_gx64" + sfx + "(s_base, X, C_, hc))"; break;
        case NBG_INT64: gx = "((long long)nbg_gx64" + sfx + "(s_base, X, C_, hc))"; break;
        default: gx = "((C_) < hc ? s_hot[(C_)] : X[(C_)])"; break;
    }
    const bool zero_pad = sp.add == NBG_PLUS && !sp.has_vals && (sp.mul == NBG_SECOND || sp.mul == NBG_TIMES);
    o << "#define NBG_ADD(A_, B_) " << k.ADD << "\n";
    o << "__device__ __forceinline__ " << k.C << " nbg_mul(const KArgs &a, long long P_, " << XT << " X_) { return " << k.mul << "; }\n";
    o << "__device__ __forceinline__ " << XT << " nbg_gxv(unsigned s_base, const " << XT << "* s_hot, const " << XT
      << "* X, int C_, int hc) { return " << gx << "; }\n";
    o << "#define NBG_GV(C_) nbg_gxv(s_base, s_hot, X, ((C_) > 0 ? (C_) : 0), hc)\n";
    // term of a stored position B_ (1) or a padding position (0)
    if (zero_pad)
        o << "#define NBG_TV(B_, V_) ((" << ACC << ")nbg_mul(a, 0, (B_) ? (V_) : (" << XT << ")0))\n";
    else
        o << "#define NBG_TV(B_, V_) ((B_) ? (" << ACC << ")nbg_mul(a, 0, (V_)) : (" << ACC << ")(" << IDENT << "))\n";
    // the 4 gathers of a group and its presence bits (the indices die here), then its 4 terms in order
    o << "#define NBG_G4(Q_, V_) const " << XT << " V_##0 = NBG_GV(Q_.x), V_##1 = NBG_GV(Q_.y), V_##2 = NBG_GV(Q_.z), V_##3 = NBG_GV(Q_.w); "
         "const unsigned V_##m = (unsigned)(Q_.x >= 0) | ((unsigned)(Q_.y >= 0) << 1) | ((unsigned)(Q_.z >= 0) << 2) | ((unsigned)(Q_.w >= 0) << 3)\n";
    o << "#define NBG_A4(ACC_, V_) ACC_ = NBG_ADD(ACC_, NBG_TV(V_##m & 1u, V_##0)); ACC_ = NBG_ADD(ACC_, NBG_TV((V_##m >> 1) & 1u, V_##1)); "
         "ACC_ = NBG_ADD(ACC_, NBG_TV((V_##m >> 2) & 1u, V_##2)); ACC_ = NBG_ADD(ACC_, NBG_TV((V_##m >> 3) & 1u, V_##3))\n";
    o << "#define NBG_NEG make_int4(-1, -1, -1, -1)\n";
    o << "__device__ __forceinline__ " << ACC << " nbg_tree(" << ACC << " v) {   // fixed shuffle tree, lane 0 holds the total\n";
    o << "  for (int d = 16; d > 0; d >>= 1) { const " << ACC << " w = __shfl_down_sync(0xffffffffu, v, d); v = NBG_ADD(v, w); }\n";
    o << "  return v;\n}\n";
    if (NF) o << "#define NBG_NF " << NF << "\n";
    o << "extern \"C\" __global__ void __launch_bounds__(" << NT << ", 1) " << kname << "(const KArgs a) {\n";
    o << "  extern __shared__ __align__(16) unsigned char nbg_dyn[];\n";
    o << "  __shared__ double nbg_sh[32];\n";
    o << "  " << XT << "* s_hot = (" << XT << "*)nbg_dyn;\n";
    o << "  const unsigned s_base = (unsigned)__cvta_generic_to_shared(nbg_dyn);\n";
    o << "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n";
    if (NF) {
        o << "  u64* s_x = (u64*)(nbg_dyn + " << hot_region << ");   // [warp][NF][12] exact limbs\n";
        o << "  for (int k = threadIdx.x; k < " << NW * NF * 12 << "; k += blockDim.x) s_x[k] = 0ull;\n";
    }
    (void)NW;
    o << "  const " << XT << "* __restrict__ X = (const " << XT << "*)a.x;\n";
    o << "  const int4* __restrict__ CG = (const int4*)a.colidx;\n";
    o << "  const int4* __restrict__ SELL = (const int4*)a.rb_sell;\n";
    o << "  const long long* __restrict__ GRP = a.rowptr;\n";
    // barrier mode: row totals go to a plain output of the region with the row-total width when there
    // is one (the epilogue pass reads each total and overwrites it in place: one 4-byte array less in
    // L2 next to the index stream), else to the plan's tot buffer
    std::string totbuf = "a.rb_tot";
    if (!IE) {
        const char *e = PIPE ? "0" : getenv("NBG_RB_TOTOUT");   // pipelined: epilogue chunks of a group run while other
                                                                  // groups still write totals -- keep them apart from the outputs
        if (!(e && e[0] == '0'))
            for (const OutV &ov : p.outs)
                if (!ov.scatter && !ov.multi && type_size(p.ins[ov.ins].t) == (RT == "float" || RT == "int" ? 4u : 8u)) {
                    totbuf = "a.out[" + std::to_string(ov.out) + "]";
                    break;
                }
        o << "  " << RT << "* TOT = (" << RT << "*)" << totbuf << ";\n";
    }
    o << "  const int hc = (int)a.hc;\n";
    o << "  {\n";
    o << "    const int nv_ = ((((unsigned long long)X) & 15ull) == 0ull) ? (int)((hc * sizeof(" << XT << ")) >> 4) : 0;\n";
    o << "    const uint4* src_ = (const uint4*)X; uint4* dst_ = (uint4*)nbg_dyn;\n";
    o << "    for (int k = threadIdx.x; k < nv_; k += 4 * blockDim.x) {\n";
    o << "      uint4 w_[4];\n";
    o << "      #pragma unroll\n      for (int u = 0; u < 4; u++) if (k + u * (int)blockDim.x < nv_) w_[u] = __ldg(src_ + k + u * blockDim.x);\n";
    o << "      #pragma unroll\n      for (int u = 0; u < 4; u++) if (k + u * (int)blockDim.x < nv_) dst_[k + u * blockDim.x] = w_[u];\n";
    o << "    }\n";
    o << "    for (int k = (nv_ << 4) / (int)sizeof(" << XT << ") + threadIdx.x; k < hc; k += blockDim.x) s_hot[k] = X[k];\n";
    o << "  }\n";
    // uniform values (device scalars of earlier kernels, constants) read once per CTA into shared
    // memory: re-read per use, they take no registers across the step loops
    const int NU = std::max(1, g.n_uniform());
    o << "  __shared__ unsigned long long s_uni[" << NU << "];\n";
    g.emit_uniform_to_smem("s_uni");
    o << "  __syncthreads();\n";
    g.emit_red_decl();
    // the fused epilogue of row `i` with row total `acc` (inline mode), in its own scope
    auto epi = [&](const std::string &ind, const std::string &idx, const std::string &accx) {
        o << ind << "{\n";
        o << ind << "  const long long i = " << idx << ";\n";
        o << ind << "  const " << ACC << " eacc_ = " << accx << ";\n";
        g.emit_uniform_reload(ind + "  ", "s_uni");
        g.emit_body(
            ind + "  ",
            [&](const Ins &in) { return std::string("((const ") + ctype(in.t) + "*)a.in[" + std::to_string(in.slot) + "])[i]"; },
            [&](const OutV &ov) { return g.store(ov, "i"); },
            [&](size_t j) { return g.red_update(p.reds[j], "r" + std::to_string(j), g.v(p.reds[j].ins)); }, "eacc_");
        o << ind << "}\n";
    };
    // row total of a completed row: inline epilogue or tot[]
    auto done = [&](const std::string &ind, const std::string &idx, const std::string &accx) {
        if (IE) epi(ind, idx, accx);
        else o << ind << "TOT[" << idx << "] = (" << RT << ")(" << accx << ");\n";
    };
    // one trip of the vector epilogue: rows 4 vi .. 4 vi + 3, every load of the trip (inputs, totals,
    // non-empty mask word, scatter map) before any store
    std::vector<int> slot_type(p.n_in, -1);
    for (const Ins &in : p.ins)
        if (in.k == Ins::LD_VEC) slot_type[in.slot] = in.t;
    std::vector<int> out_type(p.n_out, -1);
    for (const OutV &ov : p.outs)
        if (!ov.scatter) out_type[ov.out] = p.ins[ov.ins].t;
    const int rtt = RT == "float" ? NBG_FP32 : (RT == "double" ? NBG_FP64 : (RT == "int" ? NBG_INT32 : NBG_INT64));
    auto red_of = [&](size_t j) { return g.red_update(p.reds[j], "r" + std::to_string(j), g.v(p.reds[j].ins)); };
    // NBG_RB_EPI_HINT: L2 cache-policy hints on the epilogue pass's
    // fp32 vector accesses -- "el": input loads evict_last, "els": loads and output stores
    // evict_last, "ef" / "efs": the same with evict_first.  A hint only; values are unchanged.
    // Default: "ef" when the gathered vector stays L2-resident (the matrix has the 196 KB hot-cache
    // launch shape, spmv_variant): the epilogue's inputs are read once per sweep, and evict_first keeps
    // them from displacing the gathered vector and the row totals (C4 152.3 -> 149.9 us per sweep);
    // off when it does not (C5: 3.53 ms without, 3.58 ms with).  NBG_RB_EPI_HINT=0 turns it off.
    const char *ehint = getenv("NBG_RB_EPI_HINT");
    const std::string eh = PIPE ? "" : (ehint && *ehint ? std::string(ehint) : std::string(hk_ >= 140 ? "ef" : ""));
    // "efl": evict_first loads, evict_last stores (the stored r is the next sweep's t)
    const bool hint_ld = eh == "el" || eh == "els" || eh == "ef" || eh == "efs" || eh == "efl", hint_st = eh == "els" || eh == "efs" || eh == "efl";
    auto vec_trip = [&](const std::string &ind) {
        o << ind << "{\n";
        if (hint_ld)
            o << ind << "  unsigned long long pol_; asm(\"createpolicy.fractional.L2::" << (eh[1] == 'f' ? "evict_first" : "evict_last")
              << ".b64 %0, 1.0;\" : \"=l\"(pol_));\n";
        if (eh == "efl")
            o << ind << "  unsigned long long pols_; asm(\"createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\" : \"=l\"(pols_));\n";
        for (int s2 = 0; s2 < p.n_in; s2++)
            if (slot_type[s2] >= 0) {
                o << ind << "  " << ctype(slot_type[s2]) << " L" << s2 << "[4];\n";
                if (hint_ld && slot_type[s2] == NBG_FP32) {
                    const std::string L = "L" + std::to_string(s2);
                    o << ind << "  asm volatile(\"ld.global.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;\" : \"=f\"(" << L << "[0]), \"=f\"(" << L
                      << "[1]), \"=f\"(" << L << "[2]), \"=f\"(" << L << "[3]) : \"l\"(((const float4*)(a.in[" << s2 << "])) + vi), \"l\"(pol_));\n";
                    continue;
                }
                o << ind << "  " << vload(slot_type[s2], "a.in[" + std::to_string(s2) + "]", "vi", "L" + std::to_string(s2)) << "\n";
            }
        std::string tl = vload(rtt, totbuf, "vi", "T_");
        for (size_t q = tl.find("__ldg("); q != std::string::npos; q = tl.find("__ldg(", q)) tl.replace(q, 6, "__ldcg(");
        o << ind << "  " << RT << " T_[4];\n" << ind << "  " << tl << "\n";
        o << ind << "  const unsigned mb_ = (__ldcg(a.rb_mask + ((vi << 2) >> 5)) >> ((vi << 2) & 31)) & 15u;\n";
        for (const OutV &ov : p.outs)
            if (ov.scatter && !ov.affine) o << ind << "  " << g.scat_preload(ov, "vi") << "\n";
        for (int k2 = 0; k2 < p.n_out; k2++)
            if (out_type[k2] >= 0) o << ind << "  " << ctype(out_type[k2]) << " O" << k2 << "[4];\n";
        g.emit_uniform_reload(ind + "  ", "s_uni");
        o << ind << "  #pragma unroll\n" << ind << "  for (int e = 0; e < 4; e++) {\n";
        o << ind << "    const " << ACC << " acc = ((mb_ >> e) & 1u) ? (" << ACC << ")T_[e] : (" << ACC << ")(" << IDENT << ");\n";
        g.emit_body(
            ind + "    ", [&](const Ins &in) { return "L" + std::to_string(in.slot) + "[e]"; },
            [&](const OutV &ov) {
                if (ov.scatter) return g.scat_pre(ov, "e", "(vi * 4 + e)");
                return "O" + std::to_string(ov.out) + "[e] = " + g.v(ov.ins) + ";";
            },
            red_of, "acc");
        o << ind << "  }\n";
        for (int k2 = 0; k2 < p.n_out; k2++)
            if (out_type[k2] >= 0) {
                if (hint_st && out_type[k2] == NBG_FP32) {
                    const std::string O = "O" + std::to_string(k2);
                    o << ind << "  asm volatile(\"st.global.L2::cache_hint.v4.f32 [%0], {%1,%2,%3,%4}, %5;\" :: \"l\"(((float4*)(a.out[" << k2
                      << "])) + vi), \"f\"(" << O << "[0]), \"f\"(" << O << "[1]), \"f\"(" << O << "[2]), \"f\"(" << O << "[3]), \"l\"(" << (eh == "efl" ? "pols_" : "pol_") << ") : \"memory\");\n";
                    continue;
                }
                o << ind << "  " << vstore(out_type[k2], "a.out[" + std::to_string(k2) + "]", "vi", "O" + std::to_string(k2)) << "\n";
            }
        o << ind << "}\n";
    };
    // the epilogue of row i from its total (tail rows and unaligned buffers)
    auto row_epi = [&](const std::string &ind) {
        o << ind << "const unsigned mw_ = __ldcg(a.rb_mask + (i >> 5));\n";
        o << ind << "const " << RT << " t_ = __ldcg(((const " << RT << "*)" << totbuf << ") + i);\n";
        o << ind << "const " << ACC << " acc = ((mw_ >> (i & 31)) & 1u) ? (" << ACC << ")t_ : (" << ACC << ")(" << IDENT << ");\n";
        g.emit_uniform_reload(ind, "s_uni");
        g.emit_body(
            ind,
            [&](const Ins &in) { return std::string("((const ") + ctype(in.t) + "*)a.in[" + std::to_string(in.slot) + "])[i]"; },
            [&](const OutV &ov) { return g.store(ov, "i"); }, red_of, "acc");
    };
    o << "  {\n";
    o << "  const int items = (int)a.rb_ntasks;\n";
    o << "  const int4* __restrict__ TK = (const int4*)a.rb_tasks;\n";
    // tasks from one global counter (bar[2]; reset by the grid barrier's last arriver / the last CTA
    // out), claimed one ahead
    const std::string claim = PIPE ? "(int)atomicAdd(a.rb_done + 1 + 2 * a.rb_ngrp, 1ull)" : "(int)atomicAdd(a.rb_bar + 2, 1u)";
    o << "  int itn_ = 0;\n";
    o << "  if (lane == 0) itn_ = " << claim << ";\n";
    o << "  itn_ = __shfl_sync(0xffffffffu, itn_, 0);\n";
    o << "  int4 tn_ = itn_ < items ? TK[itn_] : make_int4(0, 0, 0, 0);\n";
    if (PIPE) {
        o << "  int qlo_ = 0;          // lane 0: first row group whose epilogue chunks are not all taken\n";
        o << "  bool hd_ = false;      // lane 0: every hub / long task has completed\n";
        o << "  const int ngk_ = (int)a.rb_ngrp;\n";
    }
    o << "  for (;;) {\n";
    if (PIPE) {
        // an epilogue chunk (512 rows) of a row group whose totals are complete -- every hub / long task
        // and every slice run of the group done (acquire loads of the completion counters) -- before
        // the next row task: the DRAM-bound epilogue overlaps the gather-bound rows of later groups
        o << "    int eq_ = -1; long long ec_ = 0;\n";
        // polled only once every slice run of group qlo_ has been claimed (before that it cannot be complete)
        // while row tasks remain, only every NBG_RB_EW-th warp takes epilogue chunks (the rest keep the
        // gathers going); once the queue is empty every warp does
        int ew = 4;
        {
            const char *e = getenv("NBG_RB_EW");
            if (e && *e) ew = std::max(1, std::min(32, atoi(e)));
        }
        o << "    if (lane == 0 && qlo_ < ngk_ && itn_ >= a.rb_gcnt[1 + ngk_ + qlo_] && (itn_ >= items || (warp % " << ew << ") == 0)) {\n";
        o << "      unsigned long long d_;\n";
        // relaxed polls (an acquire load invalidates the SM's L1 each time); one acquire fence once a chunk is taken
        o << "      if (!hd_) { asm volatile(\"ld.relaxed.gpu.global.u64 %0, [%1];\" : \"=l\"(d_) : \"l\"(a.rb_done) : \"memory\"); hd_ = d_ >= (unsigned long long)a.rb_gcnt[0]; }\n";
        o << "      if (hd_)\n";
        o << "        for (int q = qlo_; q < ngk_; q++) {\n";
        o << "          asm volatile(\"ld.relaxed.gpu.global.u64 %0, [%1];\" : \"=l\"(d_) : \"l\"(a.rb_done + 1 + q) : \"memory\");\n";
        o << "          if (d_ < (unsigned long long)a.rb_gcnt[1 + q]) break;\n";
        o << "          const long long r0q_ = (long long)q * a.rb_gsize, r1q_ = min(a.n, r0q_ + a.rb_gsize);\n";
        o << "          const unsigned long long c_ = atomicAdd(a.rb_done + 1 + ngk_ + q, 1ull);\n";
        o << "          if ((long long)c_ < (r1q_ - r0q_ + 511) / 512) { eq_ = q; ec_ = (long long)c_; asm volatile(\"fence.acq_rel.gpu;\" ::: \"memory\"); break; }\n";
        o << "          if (q == qlo_) qlo_++;\n";
        o << "        }\n";
        o << "    }\n";
        o << "    eq_ = __shfl_sync(0xffffffffu, eq_, 0);\n";
        o << "    ec_ = __shfl_sync(0xffffffffu, ec_, 0);\n";
        o << "    if (eq_ >= 0) {\n";
        o << "      const long long rb0_ = (long long)eq_ * a.rb_gsize + 512 * ec_;\n";
        o << "      const long long re_ = min(min(a.n, (long long)(eq_ + 1) * a.rb_gsize), rb0_ + 512);\n";
        if (p.vec) {
            o << "      for (long long vi = (rb0_ >> 2) + lane; vi < (re_ >> 2); vi += 32)\n";
            vec_trip("      ");
            o << "      for (long long i = (re_ & ~3ll) + lane; i < re_; i += 32) {\n";
        } else {
            o << "      for (long long i = rb0_ + lane; i < re_; i += 32) {\n";
        }
        row_epi("        ");
        o << "      }\n";
        for (int f = 0; f < NF; f++) {
            const int j = fplus[f];
            o << "      { const double t_ = nbg_warp_sum(r" << j << "); if (lane == 0) nbg_xacc_add_local(s_x + (warp * NBG_NF + " << f
              << ") * 12, t_); r" << j << " = 0.0; }\n";
        }
        o << "      continue;\n";
        o << "    }\n";
    }
    o << "    const int it = itn_;\n";
    if (PIPE)
        o << "    if (it >= items) { if (__shfl_sync(0xffffffffu, qlo_, 0) >= ngk_) break; __nanosleep(200); continue; }\n";
    else
        o << "    if (it >= items) break;\n";
    o << "    const int4 tk = tn_;\n";
    o << "    if (lane == 0) itn_ = " << claim << ";\n";
    o << "    itn_ = __shfl_sync(0xffffffffu, itn_, 0);\n";
    o << "    if (itn_ < items) tn_ = TK[itn_];\n";
    o << "    const int kind = tk.x & 3, cnt = tk.x >> 2;\n";
    // ---- short slices
    o << "    if (kind == 2) {\n";
    o << "      const int s0 = tk.y;\n";
    if (PIPE)   // pipelined records: 32-bit slice offset, .w = the row group
        o << "      const long long base = (long long)(unsigned)tk.z;\n";
    else
        o << "      const long long base = ((long long)(unsigned)tk.w << 32) | (long long)(unsigned)tk.z;\n";
    o << "      const int myw = lane < cnt ? a.rb_swid[s0 + lane] : 0;\n";
    o << "      const int W = __reduce_add_sync(0xffffffffu, (unsigned)myw);\n";
    o << "      const int4* __restrict__ Q = SELL + base + lane;\n";
    o << "      int4 q0 = __ldcs(Q), q1 = (1 < W) ? __ldcs(Q + 32) : NBG_NEG;\n";
    o << "      int si = 0, send = __shfl_sync(0xffffffffu, myw, 0);\n";
    o << "      int row = a.rb_srow[32ll * s0 + lane];\n";
    o << "      " << ACC << " acc = " << IDENT << ";\n";
    o << "      for (int j = 0; j < W; j += 2) {\n";
    o << "        const int4 c0 = q0, c1 = q1;\n";
    o << "        NBG_G4(c0, u); NBG_G4(c1, v);\n";
    o << "        if (j + 2 < W) q0 = __ldcs(Q + 32 * (j + 2));\n";
    o << "        if (j + 3 < W) q1 = __ldcs(Q + 32 * (j + 3)); else q1 = NBG_NEG;\n";
    o << "        NBG_A4(acc, u);\n";
    o << "        if (j + 1 == send) {\n";
    o << "          if (row >= 0)\n";
    done("          ", "row", "acc");
    o << "          acc = " << IDENT << ";\n";
    o << "          if (++si < cnt) { send += __shfl_sync(0xffffffffu, myw, si); row = a.rb_srow[32ll * (s0 + si) + lane]; }\n";
    o << "        }\n";
    o << "        if (j + 1 < W) {\n";
    o << "          NBG_A4(acc, v);\n";
    o << "          if (j + 2 == send) {\n";
    o << "            if (row >= 0)\n";
    done("            ", "row", "acc");
    o << "            acc = " << IDENT << ";\n";
    o << "            if (++si < cnt) { send += __shfl_sync(0xffffffffu, myw, si); row = a.rb_srow[32ll * (s0 + si) + lane]; }\n";
    o << "          }\n";
    o << "        }\n";
    o << "      }\n";
    o << "    }\n";
    if (IE) {
        // ---- empty rows: 4 consecutive rows per lane and trip (vector loads when aligned)
        o << "    else if (kind == 3) {\n";
        o << "      const long long rb0_ = tk.y;\n";
        o << "      for (int j = lane; j < cnt; j += 32) {\n";
        o << "        const long long i_ = rb0_ + j;\n";
        o << "        if (!((__ldg(a.rb_mask + (i_ >> 5)) >> (i_ & 31)) & 1u))\n";
        epi("          ", "i_", "(" + ACC + ")(" + IDENT + ")");
        o << "      }\n";
        o << "    }\n";
    }
    // ---- long rows / hub chunk: lane-strided groups (lane l: l, l + 32, l + 64, ...), tree
    o << "    else {\n";
    o << "    int myrow = 0, myng = 0;\n";
    o << "    long long mygb = 0;\n";
    o << "    int nrow = 1;\n";
    if (IE) o << "    " << ACC << " mytot = " << IDENT << ";\n";
    o << "    if (kind == 0) {\n";
    o << "      const int4 ch = ((const int4*)a.chunks)[tk.y];\n";
    o << "      mygb = ((long long)(unsigned)ch.z << 32) | (long long)(unsigned)ch.y;\n";
    o << "      myng = ch.w;\n";
    o << "    } else {\n";
    o << "      nrow = cnt;\n";
    o << "      if (lane < cnt) { myrow = a.rb_lrows[tk.y + lane]; mygb = GRP[myrow]; myng = (int)(GRP[myrow + 1] - mygb); }\n";
    o << "    }\n";
    o << "    int r = 0, b = 0;\n";
    o << "    long long gb = __shfl_sync(0xffffffffu, mygb, 0);\n";
    o << "    int ng = __shfl_sync(0xffffffffu, myng, 0);\n";
    // LG groups per lane per step (steps of 32 LG groups): lane l sums groups l, l + 32, l + 64, ...
    // whatever LG is -- the order (and every bit of the result) does not depend on it
    int LG = 2;
    {
        const char *e = getenv("NBG_RB_LG");
        if (e && (e[0] == '1' || e[0] == '2' || e[0] == '3' || e[0] == '4')) LG = e[0] - '0';
    }
    const char *gv[4] = {"u", "v", "w", "z"};
    for (int k2 = 0; k2 < LG; k2++)
        o << "    int4 q" << k2 << " = (" << 32 * k2 << " + lane < ng) ? __ldcs(CG + gb + " << 32 * k2 << " + lane) : NBG_NEG;\n";
    o << "    " << ACC << " acc = " << IDENT << ";\n";
    o << "    for (;;) {\n";
    for (int k2 = 0; k2 < LG; k2++) o << "      const int4 c" << k2 << " = q" << k2 << ";\n";
    for (int k2 = 0; k2 < LG; k2++) o << "      NBG_G4(c" << k2 << ", " << gv[k2] << ");\n";
    o << "      int nb = b + " << 32 * LG << ", nr = r;\n";
    o << "      long long ngb = gb; int nng = ng;\n";
    o << "      if (nb >= ng) { nr = r + 1; nb = 0; if (nr < nrow) { ngb = __shfl_sync(0xffffffffu, mygb, nr); nng = __shfl_sync(0xffffffffu, myng, nr); } }\n";
    o << "      if (nr < nrow) {\n";
    for (int k2 = 0; k2 < LG; k2++)
        o << "        q" << k2 << " = (nb + " << 32 * k2 << " + lane < nng) ? __ldcs(CG + ngb + nb + " << 32 * k2 << " + lane) : NBG_NEG;\n";
    o << "      }\n";
    o << "      ";
    for (int k2 = 0; k2 < LG; k2++) o << "NBG_A4(acc, " << gv[k2] << "); ";
    o << "\n";
    o << "      if (nr != r) {\n";
    o << "        const " << ACC << " t = nbg_tree(acc);\n";
    if (IE) {
        o << "        { const " << ACC << " tt = __shfl_sync(0xffffffffu, t, 0); if (lane == r) mytot = tt; }\n";
    } else {
        o << "        const int orow = __shfl_sync(0xffffffffu, myrow, r);\n";
    }
    o << "        acc = " << IDENT << ";\n";
    o << "        if (lane == 0) {\n";
    if (!IE) o << "          if (kind != 0) TOT[orow] = (" << RT << ")t;\n          else {\n";
    else o << "          if (kind == 0) {\n";
    o << "            ((" << ACC << "*)a.partials)[tk.y] = t;\n";
    o << "            const int cx = ((const int4*)a.chunks)[tk.y].x;\n";
    o << "            const int4 lr = ((const int4*)a.longs)[cx];\n";
    o << "            int tk_;\n";
    o << "            asm volatile(\"atom.add.release.gpu.s32 %0, [%1], 1;\" : \"=r\"(tk_) : \"l\"(&a.counters[cx]) : \"memory\");\n";
    o << "            if (tk_ == lr.z - 1) {\n";
    o << "              asm volatile(\"fence.acq_rel.gpu;\" ::: \"memory\");\n";
    o << "              " << ACC << " s_ = " << IDENT << ";\n";
    o << "              for (int q = 0; q < lr.z; q++) { const " << ACC << " pq = *(volatile const " << ACC << "*)(((const " << ACC
      << "*)a.partials) + lr.y + q); s_ = NBG_ADD(s_, pq); }\n";
    o << "              a.counters[cx] = 0;\n";
    done("              ", "lr.x", "s_");
    o << "            }\n";
    o << "          }\n";
    o << "        }\n";
    o << "        if (nr >= nrow) break;\n";
    o << "      }\n";
    o << "      r = nr; b = nb; gb = ngb; ng = nng;\n";
    o << "    }\n";
    if (IE) {
        o << "    if (kind == 1 && lane < nrow)\n";
        epi("      ", "myrow", "mytot");
    }
    o << "    }\n";
    if (PIPE) {   // a slice / long / hub task is complete: its totals are visible before the count
        // release by lane 0 after the warp barrier (which orders the other lanes' total stores before it):
        // no full fence and no L1 invalidation per task
        o << "    __syncwarp();\n";
        o << "    if (lane == 0) asm volatile(\"red.release.gpu.global.add.u64 [%0], 1;\" :: \"l\"(a.rb_done + (kind == 2 ? 1 + tk.w : 0)) : \"memory\");\n";
    }
    if (NF && IE) {   // the task's floating PLUS partials: fixed tree, exact add into the warp's limbs
        for (int f = 0; f < NF; f++) {
            const int j = fplus[f];
            o << "    { const double t_ = nbg_warp_sum(r" << j << "); if (lane == 0) nbg_xacc_add_local(s_x + (warp * NBG_NF + " << f
              << ") * 12, t_); r" << j << " = 0.0; }\n";
        }
    }
    o << "  }\n";
    o << "  }\n";
    if (PT) {
        o << "  __syncthreads();\n";
        // inline: the last CTA out resets the task counter for the next launch (every CTA is done with it);
        // pipelined: monotonic counters, nothing to reset
        if (IE)
            o << "  if (threadIdx.x == 0) { __threadfence(); if (atomicAdd(a.rb_bar, 1u) == gridDim.x - 1) { atomicExch(a.rb_bar, 0u); atomicExch(a.rb_bar + 2, 0u); } }\n";
        else   // pipelined: the last CTA out zeroes every counter for the next launch
            o << "  if (threadIdx.x == 0) { __threadfence(); if (atomicAdd(a.rb_done + 2 + 2 * a.rb_ngrp, 1ull) == gridDim.x - 1) { for (long long k_ = 0; k_ < 3 + 2 * a.rb_ngrp; k_++) atomicExch(a.rb_done + k_, 0ull); } }\n";
        for (int f = 0; f < NF; f++) {
            const int j = fplus[f];
            o << "  if (threadIdx.x < 12) {\n";
            o << "    u64 v_ = 0ull; double d_ = 0.0;\n";
            o << "    for (int w = 0; w < " << NW << "; w++) { const u64 x_ = s_x[(w * NBG_NF + " << f << ") * 12 + threadIdx.x]; if (threadIdx.x == 11) d_ += __longlong_as_double((long long)x_); else v_ = threadIdx.x == 10 ? (v_ | x_) : v_ + x_; }\n";
            o << "    if (threadIdx.x == 11) { if (d_ != 0.0) atomicAdd((double*)&a.racc[" << p.reds[j].racc << "][12], d_); }\n";
            o << "    else if (threadIdx.x == 10) { if (v_) atomicAdd(&a.racc[" << p.reds[j].racc << "][10], nbg_xacc_flag_counts(v_)); }\n";
            o << "    else if (v_) atomicAdd(&a.racc[" << p.reds[j].racc << "][threadIdx.x], v_);\n";
            o << "  }\n";
        }
        for (size_t j = 0; j < p.reds.size(); j++) {
            if (std::find(fplus.begin(), fplus.end(), (int)j) != fplus.end()) continue;
            const int kind = redkind(g, p.reds[j]);
            if (kind == 6) { o << g.red_finish_xt(j); continue; }
            if (kind == 0 || kind == 2 || kind == 3)
                o << "  nbg_block_finish_f(r" << j << ", " << kind << ", a.racc[" << p.reds[j].racc << "], nbg_sh);\n";
            else
                o << "  nbg_block_finish_i(r" << j << ", " << kind << ", a.racc[" << p.reds[j].racc << "], nbg_sh);\n";
        }
        o << "}\n";
        return dyn_bytes;
    }
    // ---------------- grid barrier (all CTAs are resident: one per SM, grid <= SMs)
    o << "  nbg_grid_sync(a.rb_bar, a.rb_bar + 2);\n";
    // ---------------- phase B: the epilogue over rows in index order.  Vector form (all buffers
    // 16-byte aligned): 4 consecutive rows per thread and trip (vec_trip); then the tail.  (Two or four
    // trips per iteration measured slower: 167.0 / 178.8 vs 165.0 us at C4.)
    o << "  const long long stride_ = (long long)gridDim.x * blockDim.x;\n";
    o << "  long long tail0_ = 0;\n";
    if (p.vec) {
        o << "  const long long nv_ = a.n >> 2;\n  tail0_ = nv_ << 2;\n";
        o << "  for (long long vi = (long long)blockIdx.x * blockDim.x + threadIdx.x; vi < nv_; vi += stride_)\n";
        vec_trip("  ");
    }
    o << "  for (long long i = tail0_ + (long long)blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += stride_) {\n";
    row_epi("    ");
    o << "  }\n";
    g.emit_red_finish();
    o << "}\n";
    return dyn_bytes;
}

// Phase 1: per-pair partial sums with the column block in shared memory.  The CTA walks its task
// range block by block (loads the block's slice of x, then its warps claim the block's tasks); a
// task is the single-pass row task on pairs instead of rows (same 64-group steps, lane-local split
// + one segmented scan), gathering only from shared memory; pair totals go to part[pslot[pair]].
// Chunks of a long pair: the chunk total to partials[], the last chunk (ticket) combines in order.
std::string gen_tp1(const SpmvSig &sp, const std::string &kname, int xsize, long long S, int *dyn_smem) {
    SemiringCode k = semiring_code(sp);
    const int NT = spmv_threads(xsize), NW = NT / 32;
    const long long slice = (S * xsize + 15) / 16 * 16;
    const int dyn = (int)slice + NW * 128 * 8;
    if (dyn_smem) *dyn_smem = dyn;
    std::ostringstream o;
    o << "#define NBG_ADD(A_, B_) " << k.ADD << "\n";
    o << "__device__ __forceinline__ " << k.C << " nbg_mul(const KArgs &a, long long P_, " << k.XT << " X_) { return " << k.mul << "; }\n";
    o << "#define NBG_TV(C_, P_, V_) (((C_) >= 0) ? (" << k.ACC << ")nbg_mul(a, (P_), (V_)) : (" << k.ACC << ")(" << k.IDENT << "))\n";
    o << "#define NBG_GS(C_) xs[(C_) > 0 ? (C_) : 0]\n";
    o << "extern \"C\" __global__ void __launch_bounds__(" << NT << ", 1) " << kname << "(const KArgs a) {\n";
    o << "  extern __shared__ __align__(16) unsigned char nbg_dyn[];\n";
    o << "  __shared__ int s_ctr;\n";
    o << "  " << k.XT << "* xs = (" << k.XT << "*)nbg_dyn;\n";
    o << "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n";
    o << "  " << k.ACC << "* s_racc = (" << k.ACC << "*)(nbg_dyn + " << slice << " + warp * 1024);\n";
    o << "  const int4* __restrict__ CG = (const int4*)a.colidx;\n";
    o << "  const long long* __restrict__ GRP = a.rowptr;\n";
    o << "  const " << k.XT << "* __restrict__ X = (const " << k.XT << "*)a.x;\n";
    o << "  " << k.ACC << "* __restrict__ PART = (" << k.ACC << "*)a.part;\n";
    o << "  const int q1 = a.cta[blockIdx.x + 1];\n";
    o << "  int q = a.cta[blockIdx.x];\n";
    o << "  while (q < q1) {\n";
    o << "    const int blk = a.tblk[q];\n";
    o << "    int lo = q, hi = q1;\n";
    o << "    while (lo < hi) { const int mid = (lo + hi) >> 1; if (a.tblk[mid] <= blk) lo = mid + 1; else hi = mid; }\n";
    o << "    const int qe = lo;\n";
    o << "    __syncthreads();\n";
    o << "    if (threadIdx.x == 0) s_ctr = q;\n";
    // the block's slice of x (16-byte loads when aligned)
    o << "    {\n";
    o << "      const long long c0 = (long long)blk * a.S;\n";
    o << "      const int cn = (int)((a.ncols_g - c0) < a.S ? (a.ncols_g - c0) : a.S);\n";
    o << "      const " << k.XT << "* src = X + c0;\n";
    o << "      const bool al = ((((unsigned long long)src) & 15ull) == 0ull);\n";
    o << "      const int nv = al ? (int)((cn * (int)sizeof(" << k.XT << ")) >> 4) : 0;\n";
    o << "      for (int v = threadIdx.x; v < nv; v += 4 * blockDim.x) {\n";
    o << "        uint4 w_[4];\n";
    o << "        #pragma unroll\n        for (int u = 0; u < 4; u++) if (v + u * (int)blockDim.x < nv) w_[u] = __ldg((const uint4*)src + v + u * blockDim.x);\n";
    o << "        #pragma unroll\n        for (int u = 0; u < 4; u++) if (v + u * (int)blockDim.x < nv) ((uint4*)xs)[v + u * blockDim.x] = w_[u];\n";
    o << "      }\n";
    o << "      for (int j = (nv << 4) / (int)sizeof(" << k.XT << ") + threadIdx.x; j < cn; j += blockDim.x) xs[j] = src[j];\n";
    o << "    }\n";
    o << "    __syncthreads();\n";
    o << "    for (;;) {\n";
    o << "      int t_ = 0;\n";
    o << "      if (lane == 0) t_ = atomicAdd(&s_ctr, 1);\n";
    o << "      t_ = __shfl_sync(0xffffffffu, t_, 0);\n";
    o << "      if (t_ >= qe) break;\n";
    o << "      const int4 tl = ((const int4*)a.tiles)[t_];\n";
    o << "      const bool is_chunk = (tl.y & 0xff) == 255;\n";
    o << "      const int R = is_chunk ? 0 : (tl.y & 0xff), NG = tl.y >> 8;\n";
    o << "      const long long G0 = ((long long)(unsigned)tl.w << 32) | (long long)(unsigned)tl.z;\n";
    o << "      int4 qa = (2 * lane < NG) ? __ldcs(CG + G0 + 2 * lane) : make_int4(-1, -1, -1, -1);\n";
    o << "      int4 qb = (2 * lane + 1 < NG) ? __ldcs(CG + G0 + 2 * lane + 1) : make_int4(-1, -1, -1, -1);\n";
    o << "      int rs_[4];\n";
    o << "      #pragma unroll\n      for (int r = 0; r < 4; r++) { const int j = lane + 32 * r; rs_[r] = (j <= R) ? (int)(GRP[tl.x + j] - G0) : NG; }\n";
    o << "      const int r128_ = (lane == 0 && 128 <= R) ? (int)(GRP[tl.x + 128] - G0) : NG;\n";
    o << "      unsigned nem_[4];\n";
    o << "      #pragma unroll\n      for (int r = 0; r < 4; r++) {\n";
    o << "        const int nx = __shfl_down_sync(0xffffffffu, rs_[r], 1);\n";
    o << "        const int nf = __shfl_sync(0xffffffffu, r < 3 ? rs_[r < 3 ? r + 1 : 3] : r128_, 0);\n";
    o << "        const int re = (lane == 31) ? nf : nx;\n";
    o << "        nem_[r] = __ballot_sync(0xffffffffu, lane + 32 * r < R && re > rs_[r]);\n";
    o << "      }\n";
    o << "      " << k.ACC << " carry = " << k.IDENT << ";\n";
    o << "      int nstarted = 0;\n";
    o << "      for (int b = 0; b < NG; b += 64) {\n";
    o << "        const long long P_ = 4 * (G0 + b + 2 * lane);\n";
    o << "        const int4 ca = qa, cb = qb;\n";
    o << "        if (b + 64 < NG) {\n";
    o << "          qa = (b + 64 + 2 * lane < NG) ? __ldcs(CG + G0 + b + 64 + 2 * lane) : make_int4(-1, -1, -1, -1);\n";
    o << "          qb = (b + 65 + 2 * lane < NG) ? __ldcs(CG + G0 + b + 65 + 2 * lane) : make_int4(-1, -1, -1, -1);\n";
    o << "        }\n";
    o << "        const " << k.XT << " g0 = NBG_GS(ca.x), g1 = NBG_GS(ca.y), g2 = NBG_GS(ca.z), g3 = NBG_GS(ca.w);\n";
    o << "        const " << k.XT << " g4 = NBG_GS(cb.x), g5 = NBG_GS(cb.y), g6 = NBG_GS(cb.z), g7 = NBG_GS(cb.w);\n";
    o << "        unsigned m0_ = 0u, m1_ = 0u;\n";
    o << "        #pragma unroll\n        for (int r = 0; r < 4; r++) {\n";
    o << "          const int os_ = rs_[r] - b;\n";
    o << "          if (((nem_[r] >> lane) & 1u) && os_ >= 0 && os_ < 64) { if (os_ < 32) m0_ |= 1u << os_; else m1_ |= 1u << (os_ - 32); }\n";
    o << "        }\n";
    o << "        const unsigned M0 = __reduce_or_sync(0xffffffffu, m0_), M1 = __reduce_or_sync(0xffffffffu, m1_);\n";
    o << "        const unsigned Mw = lane < 16 ? M0 : M1;\n";
    o << "        const int sh_ = (2 * lane) & 31;\n";
    o << "        const bool s0 = (Mw >> sh_) & 1u, s1 = (Mw >> (sh_ + 1)) & 1u;\n";
    o << "        const int before = (lane < 16 ? 0 : __popc(M0)) + __popc(Mw & ((1u << sh_) - 1u));\n";
    o << "        " << k.ACC << " v0 = NBG_TV(ca.x, P_, g0);\n";
    o << "        v0 = NBG_ADD(v0, NBG_TV(ca.y, P_ + 1, g1)); v0 = NBG_ADD(v0, NBG_TV(ca.z, P_ + 2, g2)); v0 = NBG_ADD(v0, NBG_TV(ca.w, P_ + 3, g3));\n";
    o << "        " << k.ACC << " v1 = NBG_TV(cb.x, P_ + 4, g4);\n";
    o << "        v1 = NBG_ADD(v1, NBG_TV(cb.y, P_ + 5, g5)); v1 = NBG_ADD(v1, NBG_TV(cb.z, P_ + 6, g6)); v1 = NBG_ADD(v1, NBG_TV(cb.w, P_ + 7, g7));\n";
    o << "        " << k.ACC << " Sv = s1 ? v1 : NBG_ADD(v0, v1);\n";
    o << "        if (lane == 0 && !s0 && !s1) Sv = NBG_ADD(carry, Sv);\n";
    o << "        bool F = s0 || s1 || lane == 0;\n";
    o << "        #pragma unroll\n        for (int d = 1; d < 32; d <<= 1) {\n";
    o << "          const " << k.ACC << " Sy = __shfl_up_sync(0xffffffffu, Sv, d);\n";
    o << "          const bool Fy = __shfl_up_sync(0xffffffffu, F, d);\n";
    o << "          if (lane >= d && !F) { Sv = NBG_ADD(Sy, Sv); F = Fy; }\n";
    o << "        }\n";
    o << "        " << k.ACC << " Sp = __shfl_up_sync(0xffffffffu, Sv, 1);\n";
    o << "        if (lane == 0) Sp = carry;\n";
    o << "        if (s0 && (lane > 0 || nstarted > 0)) s_racc[nstarted + before - 1] = Sp;\n";
    o << "        if (s1) s_racc[nstarted + before + (s0 ? 1 : 0) - 1] = s0 ? v0 : NBG_ADD(Sp, v0);\n";
    o << "        carry = __shfl_sync(0xffffffffu, Sv, 31);\n";
    o << "        nstarted += __popc(M0) + __popc(M1);\n";
    o << "      }\n";
    o << "      if (is_chunk) {\n";
    o << "        if (lane == 0) {\n";
    o << "          const int ci = a.chunks[t_];                              // global chunk index\n";
    o << "          ((" << k.ACC << "*)a.partials)[ci] = carry;\n";
    o << "          const int4 lr = ((const int4*)a.longs)[tl.x];\n";
    o << "          int tk;\n";
    o << "          asm volatile(\"atom.add.release.gpu.s32 %0, [%1], 1;\" : \"=r\"(tk) : \"l\"(&a.counters[tl.x]) : \"memory\");\n";
    o << "          if (tk == lr.z - 1) {\n";
    o << "            asm volatile(\"fence.acq_rel.gpu;\" ::: \"memory\");\n";
    o << "            " << k.ACC << " acc = " << k.IDENT << ";\n";
    o << "            for (int j = 0; j < lr.z; j++) { const " << k.ACC << " pj = *(volatile const " << k.ACC << "*)(((const " << k.ACC
      << "*)a.partials) + lr.y + j); acc = NBG_ADD(acc, pj); }\n";
    o << "            a.counters[tl.x] = 0;\n";
    o << "            PART[a.pslot[lr.x]] = acc;\n";
    o << "          }\n";
    o << "        }\n";
    o << "        __syncwarp();\n";
    o << "        continue;\n";
    o << "      }\n";
    o << "      if (lane == 0 && nstarted > 0) s_racc[nstarted - 1] = carry;\n";
    o << "      __syncwarp();\n";
    // pairs are never empty: pair j of the task -> rank j
    o << "      #pragma unroll\n      for (int r = 0; r < 4; r++) {\n";
    o << "        const int j = lane + 32 * r;\n";
    o << "        if (j < R) PART[a.pslot[tl.x + j]] = s_racc[j];\n";
    o << "      }\n";
    o << "      __syncwarp();\n";
    o << "    }\n";
    o << "    q = qe;\n";
    o << "  }\n";
    o << "}\n";
    return o.str();
}

// Phase 2: row i = its pair partials (slots rowslot[i] .. rowslot[i+1], block order) combined in
// order, then the fused epilogue.  Warp tiles of 128 rows (lane l: rows l, l + 32, l + 64, l + 96),
// claimed from a shared-memory counter; reductions as in the single-pass skeleton.
int gen_tp2(Gen &g, const std::string &kname) {
    const Prog &p = g.p;
    auto &o = g.o;
    SemiringCode k = semiring_code(p.sp);
    std::vector<int> fplus;
    for (size_t j = 0; j < p.reds.size(); j++)
        if (redkind(g, p.reds[j]) == 0) fplus.push_back((int)j);
    const int NF = (int)fplus.size();
    const int NT = 256, NW = NT / 32;
    o << "#define NBG_ADD(A_, B_) " << k.ADD << "\n#define NBG_NF " << NF << "\n#define NBG_NW " << NW << "\n";
    o << "extern \"C\" __global__ void __launch_bounds__(" << NT << ") " << kname << "(const KArgs a) {\n";
    o << "  __shared__ double nbg_sh[32];\n";
    o << "  __shared__ int s_ctr;\n";
    if (NF) o << "  __shared__ u64 s_x[NBG_NW * NBG_NF * 12];\n";
    const int NU = std::max(1, g.n_uniform());
    o << "  __shared__ unsigned long long s_uni[" << NU << "];\n";
    o << "  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;\n";
    o << "  const " << k.ACC << "* __restrict__ PART = (const " << k.ACC << "*)a.part;\n";
    o << "  const long long* __restrict__ RS = a.rowslot;\n";
    o << "  if (threadIdx.x == 0) s_ctr = 0;\n";
    if (NF) o << "  for (int k = threadIdx.x; k < NBG_NW * NBG_NF * 12; k += blockDim.x) s_x[k] = 0ull;\n";
    g.emit_uniform_to_smem("s_uni");
    o << "  __syncthreads();\n";
    g.emit_red_decl();
    o << "  const long long ntl = (a.n + 127) / 128;\n";
    o << "  for (;;) {\n";
    o << "    int l_ = 0;\n";
    o << "    if (lane == 0) l_ = atomicAdd(&s_ctr, 1);\n";
    o << "    l_ = __shfl_sync(0xffffffffu, l_, 0);\n";
    o << "    const long long tt = (long long)blockIdx.x + (long long)l_ * gridDim.x;\n";
    o << "    if (tt >= ntl) break;\n";
    o << "    long long s0_[4], s1_[4];\n";
    o << "    #pragma unroll\n    for (int r = 0; r < 4; r++) {\n";
    o << "      const long long i = 128 * tt + lane + 32 * r;\n";
    o << "      s0_[r] = (i < a.n) ? RS[i] : 0; s1_[r] = (i < a.n) ? RS[i + 1] : 0;\n";
    o << "    }\n";
    for (int j : fplus) o << "    r" << j << " = 0.0;\n";
    o << "    #pragma unroll\n    for (int r = 0; r < 4; r++) {\n";
    o << "      const long long i = 128 * tt + lane + 32 * r;\n";
    o << "      if (i < a.n) {\n";
    o << "        " << k.ACC << " acc = " << k.IDENT << ";\n";
    o << "        for (long long s = s0_[r]; s < s1_[r]; s++) acc = NBG_ADD(acc, PART[s]);\n";
    g.emit_uniform_reload("        ", "s_uni");
    g.emit_body(
        "        ",
        [&](const Ins &in) { return std::string("((const ") + ctype(in.t) + "*)a.in[" + std::to_string(in.slot) + "])[i]"; },
        [&](const OutV &ov) { return g.store(ov, "i"); },
        [&](size_t j) { return g.red_update(p.reds[j], "r" + std::to_string(j), g.v(p.reds[j].ins)); }, "acc");
    o << "      }\n";
    o << "    }\n";
    for (int f = 0; f < NF; f++) {
        int j = fplus[f];
        o << "    { double t_ = nbg_warp_sum(r" << j << "); if (lane == 0) nbg_xacc_add_local(s_x + (warp * NBG_NF + " << f << ") * 12, t_); }\n";
    }
    o << "  }\n";
    o << "  __syncthreads();\n";
    for (int f = 0; f < NF; f++) {
        int j = fplus[f];
        o << "  if (threadIdx.x < 12) {\n";
        o << "    u64 v_ = 0ull; double d_ = 0.0;\n";
        o << "    for (int w = 0; w < NBG_NW; w++) { const u64 x_ = s_x[(w * NBG_NF + " << f << ") * 12 + threadIdx.x]; if (threadIdx.x == 11) d_ += __longlong_as_double((long long)x_); else v_ = threadIdx.x == 10 ? (v_ | x_) : v_ + x_; }\n";
        o << "    if (threadIdx.x == 11) { if (d_ != 0.0) atomicAdd((double*)&a.racc[" << p.reds[j].racc << "][12], d_); }\n";
        o << "    else if (threadIdx.x == 10) { if (v_) atomicAdd(&a.racc[" << p.reds[j].racc << "][10], nbg_xacc_flag_counts(v_)); }\n";
        o << "    else if (v_) atomicAdd(&a.racc[" << p.reds[j].racc << "][threadIdx.x], v_);\n";
        o << "  }\n";
    }
    for (size_t j = 0; j < p.reds.size(); j++) {
        if (std::find(fplus.begin(), fplus.end(), (int)j) != fplus.end()) continue;
        int kind = redkind(g, p.reds[j]);
        if (kind == 6) { o << g.red_finish_xt(j); continue; }
        if (kind == 0 || kind == 2 || kind == 3)
            o << "  nbg_block_finish_f(r" << j << ", " << kind << ", a.racc[" << p.reds[j].racc << "], nbg_sh);\n";
        else
            o << "  nbg_block_finish_i(r" << j << ", " << kind << ", a.racc[" << p.reds[j].racc << "], nbg_sh);\n";
    }
    o << "}\n";
    return 0;
}

}  // namespace

extern const char *NBG_PRELUDE_SRC;

// ---------------------------------------------------------------- structured regions (NEXT-3)
//
// A region over sparse / bitset / full leaves: every instruction carries a
// presence bit next to its value -- leaves: full = present, bitset = bit test, sparse = binary
// search of its sorted indices; apply / bind2nd keep the operand's presence, ewise_mult ANDs
// (intersection), ewise_add ORs (union; the value is op(u, v) where both are present, else the
// present operand converted to the output type).  Two loops (chosen by the
// estimator in structured.cpp):
//   dense : one thread per element, one warp per 32 consecutive elements; the output presence is
//           one __ballot_sync word per warp (the output bitset, coalesced), values are dense
//           (absent = 0) and the present count goes to a.part
//   index : one thread per entry of a sorted driver index list (a sparse operand's indices, or the
//           union of several); per entry a presence flag (a.out[1], bytes) and a value, compacted
//           afterwards in index order
// Reductions count present elements only.
std::string SProg::signature() const {
    std::ostringstream s;
    s << "X" << (index_mode ? "i" : "d") << (vec_out ? "v" : "r") << "|" << p.signature() << "|";
    for (uint8_t m : pmode) s << (int)m;
    s << "|";
    for (uint8_t l : leaf) s << (int)l;
    return s.str();
}

std::string codegen_structured(const SProg &sp, const std::string &kname) {
    const Prog &p = sp.p;
    Gen g(p);
    auto &o = g.o;
    o << NBG_PRELUDE_SRC << "\n// ---- structured region: " << sp.signature() << "\n";
    o << "extern \"C\" __global__ void __launch_bounds__(256) " << kname << "(const KArgs a) {\n";
    o << "  __shared__ double nbg_sh[32];\n";
    o << "  const int lane = threadIdx.x & 31;\n";
    g.emit_uniform();
    for (size_t k = 0; k < p.ins.size(); k++)
        if (p.ins[k].uniform) o << "  const bool p" << k << " = true;\n";
    g.emit_red_decl();
    const int NI = p.n_in;
    auto body = [&](const std::string &ind) {
        for (size_t k = 0; k < p.ins.size(); k++) {
            const Ins &in = p.ins[k];
            if (in.uniform) continue;
            const std::string T = ctype(in.t), vk = g.v((int)k), pk = "p" + std::to_string(k);
            if (in.k == Ins::LD_VEC) {
                const std::string vals = "((const " + T + "*)a.in[" + std::to_string(in.slot) + "])";
                const int lk = sp.leaf[in.slot];
                if (lk == 0) {
                    o << ind << "const bool " << pk << " = true;\n";
                    o << ind << "const " << T << " " << vk << " = " << vals << "[ic];\n";
                } else if (lk == 3) {   // an empty operand: never present
                    o << ind << "const bool " << pk << " = false;\n";
                    o << ind << "const " << T << " " << vk << " = (" << T << ")0;\n";
                } else if (lk == 1) {
                    o << ind << "const bool " << pk << " = ((((const unsigned*)a.in[" << NI + in.slot << "])[ic >> 5]) >> (ic & 31)) & 1u;\n";
                    o << ind << "const " << T << " " << vk << " = " << vals << "[ic];\n";
                } else {
                    o << ind << "long long lo" << k << " = 0;\n";
                    o << ind << "{ const int* ix_ = (const int*)a.in[" << NI + in.slot << "]; long long hi_ = (long long)a.imm[" << in.imm0
                      << "]; while (lo" << k << " < hi_) { const long long m_ = (lo" << k << " + hi_) >> 1; if ((long long)ix_[m_] < ic) lo" << k
                      << " = m_ + 1; else hi_ = m_; } }\n";
                    o << ind << "const bool " << pk << " = lo" << k << " < (long long)a.imm[" << in.imm0 << "] && (long long)((const int*)a.in["
                      << NI + in.slot << "])[lo" << k << "] == ic;\n";
                    o << ind << "const " << T << " " << vk << " = " << pk << " ? " << vals << "[lo" << k << "] : (" << T << ")0;\n";
                }
                continue;
            }
            const std::string pa = "p" + std::to_string(in.a), pb = in.b >= 0 ? "p" + std::to_string(in.b) : "true";
            const int pm = sp.pmode[k];
            if (pm == 2) {
                o << ind << "const " << T << " t" << k << " = " << g.expr(in, "") << ";\n";
                o << ind << "const " << T << " " << vk << " = (" << pa << " && " << pb << ") ? t" << k << " : (" << pa << " ? "
                  << g.cvt(in.t, g.v(in.a)) << " : " << g.cvt(in.t, g.v(in.b)) << ");\n";
                o << ind << "const bool " << pk << " = " << pa << " || " << pb << ";\n";
            } else {
                o << ind << "const " << T << " " << vk << " = " << g.expr(in, "") << ";\n";
                o << ind << "const bool " << pk << " = " << (pm == 1 ? pa + " && " + pb : pa) << ";\n";
            }
        }
    };
    const int root = sp.vec_out ? p.outs[0].ins : p.reds[0].ins;
    const std::string RT = ctype(p.ins[root].t);
    if (!sp.index_mode) {
        o << "  const long long nwords = (a.n + 31) >> 5;\n";
        o << "  unsigned long long cnt_ = 0ull;\n";
        o << "  for (long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nwords; w += ((long long)gridDim.x * blockDim.x) >> 5) {\n";
        o << "    const long long i = (w << 5) + lane;\n";
        o << "    const bool inb = i < a.n;\n";
        o << "    const long long ic = inb ? i : 0;\n";
        body("    ");
        o << "    const bool P_ = inb && p" << root << ";\n";
        if (sp.vec_out) {
            o << "    const unsigned m_ = __ballot_sync(0xffffffffu, P_);\n";
            o << "    if (lane == 0) { ((unsigned*)a.out[1])[w] = m_; cnt_ += (unsigned long long)__popc(m_); }\n";
            o << "    if (inb) ((" << RT << "*)a.out[0])[i] = P_ ? " << g.v(root) << " : (" << RT << ")0;\n";
        } else {
            o << "    if (P_) { " << g.red_update(p.reds[0], "r0", g.v(root)) << " }\n";
        }
        o << "  }\n";
        if (sp.vec_out) o << "  if (lane == 0 && cnt_) atomicAdd((unsigned long long*)a.part, cnt_);\n";
    } else {
        o << "  const int* __restrict__ D_ = (const int*)a.rowptr;\n";
        o << "  for (long long k_ = (long long)blockIdx.x * blockDim.x + threadIdx.x; k_ < a.nnz; k_ += (long long)gridDim.x * blockDim.x) {\n";
        o << "    const long long ic = (long long)D_[k_];\n";
        body("    ");
        if (sp.vec_out) {
            o << "    ((unsigned char*)a.out[1])[k_] = p" << root << " ? 1 : 0;\n";
            o << "    ((" << RT << "*)a.out[0])[k_] = p" << root << " ? " << g.v(root) << " : (" << RT << ")0;\n";
        } else {
            o << "    if (p" << root << ") { " << g.red_update(p.reds[0], "r0", g.v(root)) << " }\n";
        }
        o << "  }\n";
    }
    g.emit_red_finish();
    o << "}\n";
    return g.o.str();
}

// mxv with a structured x (SPEC.md:206 reading: dense output, identity where no stored entry of
// the row meets a present x entry): one warp per row of the CSR, lane-strided entries, presence by
// bit test, fixed xor-shuffle tree -> deterministic.
std::string codegen_smxv(const SpmvSig &sp, const std::string &kname) {
    SemiringCode k = semiring_code(sp);
    std::ostringstream o;
    o << NBG_PRELUDE_SRC << "\n// ---- structured mxv\n";
    o << "#define NBG_ADD(A_, B_) " << k.ADD << "\n";
    o << "__device__ __forceinline__ " << k.C << " nbg_mul(const KArgs &a, long long P_, " << k.XT << " X_) { return " << k.mul << "; }\n";
    o << "extern \"C\" __global__ void __launch_bounds__(256) " << kname << "(const KArgs a) {\n";
    o << "  const int lane = threadIdx.x & 31;\n";
    o << "  const long long* __restrict__ RP = a.rowptr;\n";
    o << "  const int* __restrict__ CI = a.colidx;\n";
    o << "  const " << k.XT << "* __restrict__ X = (const " << k.XT << "*)a.x;\n";
    o << "  const unsigned* __restrict__ XB = (const unsigned*)a.in[0];\n";
    o << "  for (long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < a.n; i += ((long long)gridDim.x * blockDim.x) >> 5) {\n";
    o << "    " << k.ACC << " acc = " << k.IDENT << ";\n";
    o << "    const long long s1 = RP[i + 1];\n";
    o << "    for (long long P_ = RP[i] + lane; P_ < s1; P_ += 32) {\n";
    o << "      const int j = CI[P_];\n";
    o << "      if ((XB[j >> 5] >> (j & 31)) & 1u) acc = NBG_ADD(acc, (" << k.ACC << ")nbg_mul(a, P_, X[j]));\n";
    o << "    }\n";
    o << "    #pragma unroll\n    for (int d = 16; d >= 1; d >>= 1) { const " << k.ACC << " y_ = __shfl_xor_sync(0xffffffffu, acc, d); acc = NBG_ADD(acc, y_); }\n";
    o << "    if (lane == 0) ((" << ctype(sp.T) << "*)a.out[0])[i] = (" << ctype(sp.T) << ")acc;\n";
    o << "  }\n";
    o << "}\n";
    return o.str();
}


bool spmv_epilogue_prefetch() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("NBG_SPMV_PF");
        v = (e && *e) ? (e[0] == '1') : 1;
    }
    return v == 1;
}

bool spmv_gather_pipeline() {
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("NBG_SPMV_GPIPE");
        v = (e && *e) ? (e[0] == '1') : 0;
    }
    return v == 1;
}

int spmv_lpr_mode() {   // read at every region launch (the signature records the skeleton)
    const char *e = getenv("NBG_SPMV_LPR");
    return (e && *e) ? (e[0] == '1' ? 1 : 0) : -1;
}

int spmv_groups_per_lane() {   // NBG_SPMV_GPL: groups per lane per step of the task skeleton (2 or 4)
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("NBG_SPMV_GPL");
        v = (e && *e) ? atoi(e) : 2;
        if (v != 1 && v != 2 && v != 4) v = 2;
    }
    return v;
}

int spmv_threads(int xsize) {
    // measured (DESIGN.md §7 sweep): 1024 threads for 4-byte gathered elements; 8-byte ones spill
    // at the 64-register cap of 1024 threads, so 768
    static int v = -1;
    if (v < 0) {
        const char *e = getenv("NBG_SPMV_THREADS");
        v = (e && *e) ? atoi(e) : 0;
        if (v != 0 && v != 32 && v != 64 && v != 128 && v != 256 && v != 512 && v != 640 && v != 768 && v != 1024) v = 0;
    }
    return v ? v : (xsize <= 4 ? 1024 : 768);
}

bool spmv_threads_overridden() {
    const char *e = getenv("NBG_SPMV_THREADS");
    if (!(e && *e)) return false;
    const int v = atoi(e);
    return v == 32 || v == 64 || v == 128 || v == 256 || v == 512 || v == 640 || v == 768 || v == 1024;
}

// Launch shape of the task skeleton (DESIGN.md §7 "L2-only cold gathers"): 1024 threads for 4-byte
// gathered elements (768 for 8-byte ones: spills); the hot cache fills the 196 KB carveout step when
// the gathered vector stays L2-resident (C4: 16.8 MB) and only the 132 KB step when it does not
// (C5: 108 MB), because then the L1 left beside it is worth more than hot entries: C5 3.88 ms per
// sweep at 99 KB vs 4.55 ms at 96 KB in the 164 KB step and 5.79 ms at 144 KB.
// NBG_SPMV_THREADS / NBG_SPMV_HOT_KB override both.
void spmv_variant(int xsize, long long gathered_bytes, int *nt, int *hot_kb) {
    const bool resident = gathered_bytes <= (48ll << 20);
    static int et = -1, eh = -2;
    if (et < 0) {
        const char *e = getenv("NBG_SPMV_THREADS");
        et = (e && *e) ? atoi(e) : 0;
        if (et != 0 && et != 32 && et != 64 && et != 128 && et != 256 && et != 512 && et != 640 && et != 768 && et != 1024) et = 0;
        const char *h = getenv("NBG_SPMV_HOT_KB");
        eh = (h && *h) ? std::max(0, std::min(200, atoi(h))) : -1;
    }
    *nt = et ? et : (xsize <= 4 ? 1024 : 768);
    // targets clamped to their carveout step by gen_spmv: 192 -> fills the 196 KB step, 99 -> the 132 KB step
    *hot_kb = eh >= 0 ? eh : (resident ? 192 : 99);
}

std::string codegen_tp1(const SpmvSig &sp, const std::string &kname, int xsize, long long S, int *dyn_smem) {
    return std::string(NBG_PRELUDE_SRC) + "\n// ---- two-phase spmv, phase 1\n" + gen_tp1(sp, kname, xsize, S, dyn_smem);
}

std::string codegen(const Prog &p, const std::string &kname, int *dyn_smem, int *hot_entries) {
    Gen g(p);
    g.o << NBG_PRELUDE_SRC << "\n// ---- generated region: " << p.signature() << "\n";
    int smem = 0;
    if (p.spmv && p.tp)
        smem = gen_tp2(g, kname);
    else if (p.spmv && p.lpr)
        smem = gen_spmv_lpr(g, kname);
    else if (p.spmv && p.rb)
        smem = gen_spmv_rb(g, kname, hot_entries);
    else if (p.spmv)
        smem = gen_spmv(g, kname, hot_entries);
    else
        smem = gen_ewise(g, kname, p.vec);
    if (dyn_smem) *dyn_smem = smem;
    return g.o.str();
}

}  // namespace nbg
