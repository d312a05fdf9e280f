// selftest.cpp -- GPU-free checks of the code generator: builds representative region programs
// (the config-2 elementwise chain, the fused PageRank sweep with its speculative side outputs,
// plain mxv for every monoid x type) and compiles them with NVRTC for sm_100a.  Exported as
// nbg_debug_jit_selftest (not part of nbg.h) so the CPU test-suite can run it without a device.
#include <nvrtc.h>

#include <cstdio>

#include "nbg_internal.hpp"

using namespace nbg;

static bool compile_only(const std::string &src, const std::string &kname, std::string &log) {
    const char *dump = getenv("NBG_JIT_DUMP");
    if (dump && *dump) {
        FILE *f = fopen((std::string(dump) + "/" + kname + ".cu").c_str(), "w");
        if (f) { fputs(src.c_str(), f); fclose(f); }
    }
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, src.c_str(), (kname + ".cu").c_str(), 0, nullptr, nullptr) != NVRTC_SUCCESS) {
        log += "create failed\n";
        return false;
    }
    const char *opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "-std=c++17", "-default-device", "--device-int128"};
    nvrtcResult r = nvrtcCompileProgram(prog, 5, opts);
    if (r != NVRTC_SUCCESS) {
        size_t ls = 0;
        nvrtcGetProgramLogSize(prog, &ls);
        std::string l(ls, '\0');
        nvrtcGetProgramLog(prog, &l[0]);
        log += kname + ": " + l.substr(0, 3000) + "\n";
    }
    nvrtcDestroyProgram(&prog);
    return r == NVRTC_SUCCESS;
}

static Ins I(Ins::K k, int t, int code = 0, int a = -1, int b = -1, int slot = -1, bool uni = false) {
    Ins in{};
    in.k = k;
    in.t = t;
    in.code = code;
    in.a = a;
    in.b = b;
    in.slot = slot;
    in.uniform = uni;
    return in;
}

extern "C" int nbg_debug_jit_selftest(char *out, size_t len) {
    std::string log;
    int fails = 0;
    try {
        // (1) config-2 chain: z = x*(y+1); c1 = 0.5z; c2 = c1+x; c3 = c2*y; c4 = |c3-0.25|; c5 = max(c4,z); s = sum c5
        for (int T : {NBG_FP32, NBG_FP64}) {
            for (bool vec : {true, false}) {
                Prog p;
                p.vec = vec;
                p.ins.push_back(I(Ins::LD_VEC, T, 0, -1, -1, 0));            // 0 x
                p.ins.push_back(I(Ins::LD_VEC, T, 0, -1, -1, 1));            // 1 y
                Ins a = I(Ins::UN, T, NBG_ADD_C, 1); a.imm0 = 2; p.ins.push_back(a);   // 2
                p.ins.push_back(I(Ins::BIN, T, NBG_TIMES, 0, 2));            // 3 z
                Ins h = I(Ins::UN, T, NBG_MUL_C, 3); h.imm0 = 3; p.ins.push_back(h);   // 4
                p.ins.push_back(I(Ins::BIN, T, NBG_PLUS, 4, 0));             // 5
                p.ins.push_back(I(Ins::BIN, T, NBG_TIMES, 5, 1));            // 6
                Ins q = I(Ins::UN, T, NBG_ABS_SUB_C, 6); q.imm0 = 4; p.ins.push_back(q);  // 7
                p.ins.push_back(I(Ins::BIN, T, NBG_MAX, 7, 3));              // 8
                p.ins.push_back(I(Ins::CVT, NBG_FP64, 0, 8));                // 9
                p.reds.push_back(RedOut{9, NBG_PLUS, 0, (uint8_t)SFmt::XACC});
                p.outs.push_back(OutV{3, 0});
                p.n_in = 2; p.n_out = 1; p.n_imm = 5; p.n_red = 1;
                std::string nm = std::string("selftest_chain_") + (T == NBG_FP32 ? "f32" : "f64") + (vec ? "_v" : "_s");
                if (!compile_only(codegen(p, nm), nm, log)) fails++;
            }
        }
        // (2) fused PageRank sweep + side outputs (y_next, ds_next), fp32 / fp64
        for (int T : {NBG_FP32, NBG_FP64}) {
            Prog p;
            p.spmv = true;
            p.sp.add = NBG_PLUS; p.sp.mul = NBG_SECOND; p.sp.T = T; p.sp.xt = T; p.sp.at = NBG_FP32;
            p.ins.push_back(I(Ins::MXV_ACC, T));                                  // 0 m
            p.ins.push_back(I(Ins::LD_SDEV, NBG_FP64, 0, -1, -1, 0, true));       // 1 ds
            p.ins.back().fmt = (uint8_t)SFmt::XACC;
            Ins ax = I(Ins::UN, NBG_FP64, NBG_AXPB, 1, -1, -1, true); ax.imm0 = 2; ax.imm1 = 3; p.ins.push_back(ax);  // 2 c
            p.ins.push_back(I(Ins::BIN, T, NBG_PLUS, 0, 2));                       // 3 r
            p.ins.push_back(I(Ins::LD_VEC, T, 0, -1, -1, 0));                      // 4 t
            p.ins.push_back(I(Ins::BIN, T, NBG_ABSDIFF, 4, 3));                    // 5 e
            p.ins.push_back(I(Ins::CVT, NBG_FP64, 0, 5));                          // 6
            p.ins.push_back(I(Ins::LD_VEC, T, 0, -1, -1, 1));                      // 7 dinv
            p.ins.push_back(I(Ins::BIN, T, NBG_TIMES, 3, 7));                      // 8 y_next
            p.ins.push_back(I(Ins::UN, T, NBG_ISZERO, 7));                         // 9 mask
            p.ins.push_back(I(Ins::BIN, T, NBG_TIMES, 3, 9));                      // 10
            p.ins.push_back(I(Ins::CVT, NBG_FP64, 0, 10));                         // 11
            p.outs.push_back(OutV{3, 0});
            p.outs.push_back(OutV{8, 1});
            p.reds.push_back(RedOut{6, NBG_PLUS, 0, (uint8_t)SFmt::XACC});
            p.reds.push_back(RedOut{11, NBG_PLUS, 1, (uint8_t)SFmt::XACC});
            p.n_in = 2; p.n_out = 2; p.n_imm = 4; p.n_sin = 1; p.n_red = 2;
            std::string nm = std::string("selftest_pr_") + (T == NBG_FP32 ? "f32" : "f64");
            if (!compile_only(codegen(p, nm), nm, log)) fails++;
            p.lpr = true;
            p.outs[1].scatter = true;        // y_next written in the gather layout (side output)
            if (!compile_only(codegen(p, nm + "_lpr"), nm + "_lpr", log)) fails++;
            p.lpr = false;
            p.rb = true;                     // row-binned skeleton (the C4 default), both epilogue modes
            if (!compile_only(codegen(p, nm + "_rb"), nm + "_rb", log)) fails++;
            p.rb_inline = true;
            if (!compile_only(codegen(p, nm + "_rbi"), nm + "_rbi", log)) fails++;
            p.rb_inline = false;
            p.rb_pipe = true;                // pipelined epilogue chunks
            if (!compile_only(codegen(p, nm + "_rbp"), nm + "_rbp", log)) fails++;
            p.outs[1].affine = true;         // y_next into this rank's slice of the exchange buffer
            if (!compile_only(codegen(p, nm + "_rba"), nm + "_rba", log)) fails++;
            p.outs[1].multi = true;          // ... and into every peer's (NVLink peer stores)
            if (!compile_only(codegen(p, nm + "_rbam"), nm + "_rbam", log)) fails++;
            p.rb = false;                    // the task skeleton with the same outputs
            if (!compile_only(codegen(p, nm + "_am"), nm + "_am", log)) fails++;
        }
        // (3) plain mxv for every monoid x type x mul, iso and valued matrices
        int k = 0;
        for (int add : {NBG_PLUS, NBG_MIN, NBG_MAX})
            for (int T : {NBG_BOOL, NBG_INT32, NBG_INT64, NBG_FP32, NBG_FP64})
                for (int mul : {NBG_TIMES, NBG_SECOND, NBG_MAX_DIVX_C})
                    for (bool vals : {false, true}) {
                        if (mul == NBG_MAX_DIVX_C && vals) continue;
                        Prog p;
                        p.spmv = true;
                        p.sp.add = add; p.sp.mul = mul; p.sp.T = T; p.sp.xt = NBG_FP32; p.sp.at = NBG_INT32; p.sp.has_vals = vals;
                        p.ins.push_back(I(Ins::MXV_ACC, T));
                        p.outs.push_back(OutV{0, 0});
                        p.n_out = 1; p.n_imm = 2;
                        std::string nm = "selftest_mxv_" + std::to_string(k++);
                        if (!compile_only(codegen(p, nm), nm, log)) fails++;
                    }
        // (3b) the lane-per-row skeleton for the same semirings (low-skew matrices)
        for (int add : {NBG_PLUS, NBG_MIN, NBG_MAX})
            for (int T : {NBG_INT32, NBG_FP32, NBG_FP64}) {
                Prog p;
                p.spmv = true;
                p.lpr = true;
                p.sp.add = add; p.sp.mul = NBG_TIMES; p.sp.T = T; p.sp.xt = T; p.sp.at = NBG_FP32; p.sp.has_vals = add != NBG_PLUS;
                p.ins.push_back(I(Ins::MXV_ACC, T));
                p.outs.push_back(OutV{0, 0});
                p.n_out = 1; p.n_imm = 2;
                std::string nm = "selftest_mxvl_" + std::to_string(k++);
                if (!compile_only(codegen(p, nm), nm, log)) fails++;
            }
        // (3c) the row-binned skeleton for every monoid x type (iso matrices)
        for (int add : {NBG_PLUS, NBG_MIN, NBG_MAX})
            for (int T : {NBG_BOOL, NBG_INT32, NBG_INT64, NBG_FP32, NBG_FP64})
                for (int mul : {NBG_TIMES, NBG_SECOND}) {
                    Prog p;
                    p.spmv = true;
                    p.rb = true;
                    p.rb_inline = (k % 3) == 1;
                    p.rb_pipe = (k % 3) == 2;
                    p.sp.add = add; p.sp.mul = mul; p.sp.T = T; p.sp.xt = T == NBG_BOOL ? NBG_FP32 : T; p.sp.at = NBG_INT32;
                    p.ins.push_back(I(Ins::MXV_ACC, T));
                    p.outs.push_back(OutV{0, 0});
                    p.n_out = 1; p.n_imm = 2;
                    std::string nm = "selftest_mxvr_" + std::to_string(k++);
                    if (!compile_only(codegen(p, nm), nm, log)) fails++;
                }
        // (4) reductions of every kind
        for (int T : {NBG_INT32, NBG_INT64, NBG_FP32, NBG_FP64})
            for (int mono : {NBG_PLUS, NBG_MIN, NBG_MAX}) {
                Prog p;
                p.ins.push_back(I(Ins::LD_VEC, T, 0, -1, -1, 0));
                uint8_t fmt;
                if (mono == NBG_PLUS) fmt = (uint8_t)(is_float(T) ? SFmt::XACC : SFmt::I64);
                else if (mono == NBG_MAX) fmt = (uint8_t)(is_float(T) ? SFmt::FMAX : SFmt::IMAX);
                else fmt = (uint8_t)(is_float(T) ? SFmt::FMIN : SFmt::IMIN);
                p.reds.push_back(RedOut{0, mono, 0, fmt});
                p.n_in = 1; p.n_red = 1; p.n_imm = 2;
                std::string nm = "selftest_red_" + std::to_string(k++);
                if (!compile_only(codegen(p, nm), nm, log)) fails++;
            }
        // (5) every unop / binop in every type (bool outputs included)
        for (int T : {NBG_BOOL, NBG_INT32, NBG_INT64, NBG_FP32, NBG_FP64}) {
            Prog p;
            p.ins.push_back(I(Ins::LD_VEC, NBG_INT32, 0, -1, -1, 0));
            p.ins.push_back(I(Ins::LD_VEC, NBG_FP64, 0, -1, -1, 1));
            int nimm = 2;
            for (int code = NBG_IDENTITY; code <= NBG_ISZERO; code++) {
                Ins u = I(Ins::UN, T, code, 1);
                u.imm0 = nimm; u.imm1 = nimm + 1;
                nimm += 2;
                p.ins.push_back(u);
                p.outs.push_back(OutV{(int)p.ins.size() - 1, (int)p.outs.size()});
                if (p.outs.size() == 8) break;
            }
            p.n_in = 2; p.n_out = (int)p.outs.size(); p.n_imm = nimm;
            std::string nm = "selftest_un_" + std::to_string(k++);
            if (!compile_only(codegen(p, nm), nm, log)) fails++;
            Prog q;
            q.ins.push_back(I(Ins::LD_VEC, NBG_INT32, 0, -1, -1, 0));
            q.ins.push_back(I(Ins::LD_VEC, NBG_FP64, 0, -1, -1, 1));
            for (int code = NBG_PLUS; code <= NBG_MAX_DIVX_C; code++) {
                Ins b = I(Ins::BIN, T, code, 0, 1);
                b.imm0 = 2;
                q.ins.push_back(b);
                q.reds.push_back(RedOut{(int)q.ins.size() - 1, NBG_MAX, (int)q.reds.size(),
                                        (uint8_t)(is_float(T) ? SFmt::FMAX : SFmt::IMAX)});
                if (q.reds.size() == 8) break;
            }
            q.n_in = 2; q.n_red = (int)q.reds.size(); q.n_imm = 3;
            std::string nm2 = "selftest_bin_" + std::to_string(k++);
            if (!compile_only(codegen(q, nm2), nm2, log)) fails++;
        }
        // (6) structured regions (NEXT-3): z = (x .* s) (+) apply(b) over full / bitset / sparse leaves,
        // dense and index loops, vector and reduce roots; structured mxv for every monoid
        for (int T : {NBG_INT32, NBG_FP32, NBG_FP64})
            for (int im : {0, 1})
                for (int vec : {0, 1}) {
                    SProg sp;
                    sp.index_mode = im;
                    sp.vec_out = vec;
                    Prog &p = sp.p;
                    p.ins.push_back(I(Ins::LD_VEC, T, 0, -1, -1, 0));                      // 0 x (full)
                    p.ins.push_back(I(Ins::LD_VEC, T, 0, -1, -1, 1));                      // 1 s (sparse / bitset)
                    p.ins.push_back(I(Ins::LD_VEC, NBG_FP64, 0, -1, -1, 2));               // 2 b (bitset)
                    p.ins.push_back(I(Ins::BIN, T, NBG_TIMES, 0, 1));                      // 3 x .* s
                    Ins u = I(Ins::UN, T, NBG_ADD_C, 2); u.imm0 = 1; p.ins.push_back(u);   // 4 b + c
                    p.ins.push_back(I(Ins::BIN, T, NBG_MAX, 3, 4));                        // 5 union
                    p.ins[1].imm0 = 0;
                    sp.pmode = {3, 3, 3, 1, 0, 2};
                    sp.leaf = {0, (uint8_t)(im ? 2 : 1), 1};
                    if (vec) { p.outs.push_back(OutV{5, 0}); p.n_out = 1; }
                    else {
                        p.reds.push_back(RedOut{5, NBG_PLUS, 0, (uint8_t)(is_float(T) ? SFmt::XACC : SFmt::I64)});
                        p.n_red = 1;
                    }
                    p.n_in = 3; p.n_imm = 2;
                    std::string nm = "selftest_sreg_" + std::to_string(k++);
                    if (!compile_only(codegen_structured(sp, nm), nm, log)) fails++;
                }
        for (int add : {NBG_PLUS, NBG_MIN, NBG_MAX})
            for (int T : {NBG_INT32, NBG_FP32, NBG_FP64}) {
                SpmvSig sg;
                sg.add = add; sg.mul = NBG_TIMES; sg.T = T; sg.xt = T; sg.at = NBG_FP32; sg.has_vals = true;
                std::string nm = "selftest_smxv_" + std::to_string(k++);
                if (!compile_only(codegen_smxv(sg, nm), nm, log)) fails++;
            }
    } catch (const Error &e) {
        log += "exception: " + e.msg;
        fails++;
    }
    if (out && len) snprintf(out, len, "%s", log.c_str());
    return fails;
}

// host twin of the exact accumulator: sum of n doubles through the fixed-point limbs, decoded
// with round-to-nearest-even (CPU-testable against math.fsum).
extern "C" double nbg_debug_xacc_sum(const double *v, long long n) {
    unsigned long long limbs[SLOT_U64] = {0};
    for (long long i = 0; i < n; i++) host_xacc_add(limbs, v[i]);
    return xacc_to_double(limbs);
}
