p='paper_2509_14211_b200/csrc/codegen.cpp'; s=open(p).read()
start=s.index("// SpMV skeleton v2")
end=s.index("}  // namespace\n\nextern const char *NBG_PRELUDE_SRC;")
new=open('scratch/gen_spmv_v3.txt').read()
s=s[:start]+new+s[end:]
open(p,'w').write(s)

p='paper_2509_14211_b200/csrc/planner.cpp'; s=open(p).read()
s=s.replace("""        items = (A.plan->ntiles + A.plan->nchunks + 3) / 4;   // 4 independent groups per CTA""","""        items = (A.plan->ntiles + A.plan->nchunks + 31) / 32;   // one task per warp, 32 warps per CTA""")
a=s.index("// hot-cache capacity (entries) of a generated SpMV kernel")
b=s.index("struct HintOut {")
s=s[:a]+"""// hot-cache capacity (entries) of a generated SpMV kernel: its whole dynamic shared memory
static long long hot_capacity(const Kernel &k, const Prog &p) {
    return (long long)k.smem / (long long)type_size(p.sp.xt);
}

"""+s[b:]
open(p,'w').write(s)

p='paper_2509_14211_b200/csrc/graph.cu'; s=open(p).read()
s=s.replace("constexpr int SP_CHUNK = 2048;   // nonzeros per chunk of a long row","constexpr int SP_CHUNK = 1024;   // nonzeros per chunk of a long row (one warp)\nconstexpr int SP_TASK_ROWS = 32;  // rows per warp task (one per lane)\nconstexpr int SP_TASK_NNZ = 2048; // nonzero budget of a warp task")
old=s[s.index("    // tile boundaries = merge-path cuts U {L, L+1 : L long}"):s.index("    std::vector<int> chunks, longs;")]
new="""    // warp tasks: runs of <= 32 consecutive non-long rows with <= SP_TASK_NNZ nonzeros (greedy,
    // on the host from the row pointers; once per matrix)
    std::vector<long long> rph((size_t)n + 1);
    NBG_CUDA(cudaMemcpyAsync(rph.data(), A.rowptr->d, (size_t)(n + 1) * 8, cudaMemcpyDeviceToHost, c.stream));
    NBG_CUDA(cudaStreamSynchronize(c.stream));
    std::vector<int> tiles;
    tiles.reserve((size_t)(n / 16 + 16));
    for (long long i = 0; i < n;) {
        long long len = rph[i + 1] - rph[i];
        if (len > SP_LONG) { i++; continue; }
        long long st = i, nz = 0;
        while (i < n && i - st < SP_TASK_ROWS) {
            long long l2 = rph[i + 1] - rph[i];
            if (l2 > SP_LONG) break;
            if (i > st && nz + l2 > SP_TASK_NNZ) break;
            nz += l2;
            i++;
        }
        tiles.push_back((int)st);
        tiles.push_back((int)i);
    }
    (void)s;
"""
s=s.replace(old,new)
open(p,'w').write(s)
