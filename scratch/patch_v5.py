p='paper_2509_14211_b200/csrc/codegen.cpp'; s=open(p).read()
start=s.index("// SpMV skeleton v4")
end=s.index("}  // namespace\n\nextern const char *NBG_PRELUDE_SRC;")
new=open('scratch/gen_spmv_v5.txt').read()
new=new.replace('''    o << "      s_racc[lane] = " << IDENT << ";\\n";''','''    o << "      s_racc[lane] = " << IDENT << ";\\n";
    o << "      __syncwarp();\\n";''')
new=new.replace('''    o << "        if (lane < 4) s_fl[lane] = 0u;\\n";''','''    o << "        if (lane < 4) s_fl[lane] = 0u;\\n";
    o << "        __syncwarp();\\n";''')
s=s[:start]+new+s[end:]
open(p,'w').write(s)
p='paper_2509_14211_b200/csrc/graph.cu'; s=open(p).read()
s=s.replace("constexpr int SP_LONG = 512;     // rows with more nonzeros are processed as chunks","constexpr int SP_LONG = 2048;    // rows with more nonzeros are processed as chunks")
s=s.replace("constexpr int SP_CHUNK = 512;    // nonzeros per chunk of a long row (one warp)","constexpr int SP_CHUNK = 2048;   // nonzeros per chunk of a long row (one warp)")
s=s.replace("constexpr int SP_TASK_NNZ = 512;  // nonzero budget of a warp task (= its staging buffer)","constexpr int SP_TASK_NNZ = 2048; // nonzero budget of a warp task")
open(p,'w').write(s)
p='paper_2509_14211_b200/csrc/capi.cpp'; s=open(p).read()
s=s.replace("""    if (space == NBG_DEVICE && own == NBG_BORROW) return borrow_buf(c, const_cast<void *>(p), bytes);""","""    // borrowed device memory is used in place when 16-byte aligned (vector loads); else copied
    if (space == NBG_DEVICE && own == NBG_BORROW && ((uintptr_t)p % 16) == 0) return borrow_buf(c, const_cast<void *>(p), bytes);""")
open(p,'w').write(s)
