import re
p='paper_2509_14211_b200/csrc/codegen.cpp'; s=open(p).read()
s=s.replace("int gen_spmv(Gen &g, const std::string &kname) {","int gen_spmv(Gen &g, const std::string &kname, int *hot_entries) {")
s=s.replace("    const int dyn_bytes = hot_cap * x_bytes + ci_bytes + xacc_bytes;\n","    const int dyn_bytes = hot_cap * x_bytes + ci_bytes + xacc_bytes;\n    if (hot_entries) *hot_entries = hot_cap;\n")
s=s.replace("std::string codegen(const Prog &p, const std::string &kname, int *dyn_smem) {","std::string codegen(const Prog &p, const std::string &kname, int *dyn_smem, int *hot_entries) {")
s=s.replace("        smem = gen_spmv(g, kname);","        smem = gen_spmv(g, kname, hot_entries);")
open(p,'w').write(s)
p='paper_2509_14211_b200/csrc/nbg_internal.hpp'; s=open(p).read()
s=s.replace("std::string codegen(const Prog &p, const std::string &kname, int *dyn_smem = nullptr);","std::string codegen(const Prog &p, const std::string &kname, int *dyn_smem = nullptr, int *hot_entries = nullptr);")
s=s.replace("    int smem = 0;            // dynamic shared memory per CTA\n","    int smem = 0;            // dynamic shared memory per CTA\n    int hot = 0;             // spmv: capacity of the hot-column cache (entries)\n")
open(p,'w').write(s)
p='paper_2509_14211_b200/csrc/planner.cpp'; s=open(p).read()
s=s.replace("""        int smem = 0;
        std::string src = codegen(p, nm, &smem);
        kern = jit_compile(c, src, nm, p.spmv, smem);""","""        int smem = 0, hot = 0;
        std::string src = codegen(p, nm, &smem, &hot);
        kern = jit_compile(c, src, nm, p.spmv, smem);
        kern->hot = hot;""")
a=s.index("// hot-cache capacity (entries) of a generated SpMV kernel")
b=s.index("struct HintOut {")
s=s[:a]+s[b:]
s=s.replace("""        const long long cap = (long long)(kern->smem - 0) > 0 ? hot_capacity(*kern, p) : 0;
        if (args.hc > cap) args.hc = cap;""","""        if (args.hc > kern->hot) args.hc = kern->hot;""")
open(p,'w').write(s)
