// jit.cpp -- NVRTC compilation of generated regions and their launch.
//
// (1) signature, (2) cache lookup, (3) on a miss generate + compile + insert,
// (4) execute.  Steps 1/2/4 live in planner.cpp; this file is step 3 and the launch of step 4.
// Kernels are compiled for sm_100a only (--gpu-architecture=sm_100a), with --fmad=false so that
// no multiply-add contraction changes a rounding point.  The compiled cubin is loaded with the
// CUDA 12 library API (cudaLibraryLoadData / cudaLibraryGetKernel), so no driver-API link is
// needed.  A persistent cubin cache keyed by a hash of the source (the paper's future-work
// "persistent cache") is used when NBG_JIT_CACHE names a directory.
#include <cuda.h>
#include <nvrtc.h>
#include <algorithm>
#include <sys/stat.h>
#include <unistd.h>

#include <cstdio>
#include <fstream>
#include <sstream>

#include "nbg_internal.hpp"

namespace nbg {

static std::string cache_dir() {
    const char *e = getenv("NBG_JIT_CACHE");
    if (!e || !*e) return "";
    return e;
}

static bool read_file(const std::string &path, std::string &out) {
    std::ifstream f(path, std::ios::binary);
    if (!f) return false;
    std::ostringstream ss;
    ss << f.rdbuf();
    out = ss.str();
    return !out.empty();
}

static void write_file(const std::string &path, const std::string &data) {
    std::string tmp = path + ".tmp" + std::to_string(getpid());
    {
        std::ofstream f(tmp, std::ios::binary);
        if (!f) return;
        f.write(data.data(), (std::streamsize)data.size());
    }
    rename(tmp.c_str(), path.c_str());
}

static std::string nvrtc_compile(Ctx &c, const std::string &src, const std::string &kname) {
    std::string dir = cache_dir();
    char hbuf[40];
    snprintf(hbuf, sizeof hbuf, "%016llx", (unsigned long long)hash_str(src + "|sm_100a|v1"));
    std::string cpath = dir.empty() ? "" : dir + "/" + kname + "_" + hbuf + ".cubin";
    std::string cubin;
    if (!cpath.empty() && read_file(cpath, cubin)) {
        c.stats.jit_disk_hits++;
        return cubin;
    }

    double t0 = now_ns();
    nvrtcProgram prog;
    if (nvrtcCreateProgram(&prog, src.c_str(), (kname + ".cu").c_str(), 0, nullptr, nullptr) != NVRTC_SUCCESS)
        fail(NBG_PANIC, "nvrtcCreateProgram failed");
    const char *opts[] = {"--gpu-architecture=sm_100a", "--fmad=false", "--prec-div=true", "--prec-sqrt=true",
                          "--ftz=false", "-std=c++17", "--generate-line-info", "-default-device", "--device-int128"};
    nvrtcResult r = nvrtcCompileProgram(prog, (int)(sizeof opts / sizeof opts[0]), opts);
    if (r != NVRTC_SUCCESS) {
        size_t ls = 0;
        nvrtcGetProgramLogSize(prog, &ls);
        std::string log(ls, '\0');
        nvrtcGetProgramLog(prog, &log[0]);
        nvrtcDestroyProgram(&prog);
        const char *dump = getenv("NBG_JIT_DUMP");
        if (dump && *dump) write_file(std::string(dump) + "/" + kname + "_failed.cu", src);
        fail(NBG_PANIC, std::string("NVRTC compile failed: ") + nvrtcGetErrorString(r) + "\n" + log.substr(0, 4000));
    }
    size_t cs = 0;
    nvrtcGetCUBINSize(prog, &cs);
    cubin.resize(cs);
    nvrtcGetCUBIN(prog, &cubin[0]);
    nvrtcDestroyProgram(&prog);
    c.stats.jit_compiles++;
    c.stats.jit_ms += (now_ns() - t0) * 1e-6;
    if (!cpath.empty()) {
        mkdir(dir.c_str(), 0755);
        write_file(cpath, cubin);
    }
    return cubin;
}

KernelP jit_compile(Ctx &c, const std::string &src, const std::string &kname, bool spmv, int dyn_smem, int block) {
    const char *dump = getenv("NBG_JIT_DUMP");
    if (dump && *dump) write_file(std::string(dump) + "/" + kname + ".cu", src);
    std::string cubin = nvrtc_compile(c, src, kname);
    auto k = std::make_shared<Kernel>();
    k->name = kname;
    NBG_CUDA(cudaLibraryLoadData(&k->lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0));
    NBG_CUDA(cudaLibraryGetKernel(&k->k, k->lib, kname.c_str()));
    k->block = block > 0 ? block : (spmv ? spmv_threads(4) : 256);
    k->smem = dyn_smem;
    if (dyn_smem > 48 * 1024)
        NBG_CUDA(cudaFuncSetAttribute((const void *)k->k, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem));
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, (const void *)k->k, k->block, dyn_smem);
    if (e != cudaSuccess || per_sm <= 0) {
        cudaGetLastError();
        per_sm = spmv ? 1 : 8;
    }
    k->grid_cap = c.num_sms * per_sm;
    return k;
}

// Raise the device's persisting-L2 set-aside to `want` bytes (once per context; the previous limit
// is saved and restored at finalize, ~Ctx).  Acts on c.device, restoring the caller's current
// device.  Returns the granted set-aside (0 if the device refuses).
static size_t l2_setaside(Ctx &c, size_t want) {
    if (c.l2_limit_set) return c.l2_limit_granted;
    c.l2_limit_set = true;   // one attempt per context
    int prev_dev = -1, mx = 0;
    if (cudaGetDevice(&prev_dev) != cudaSuccess) { cudaGetLastError(); return 0; }
    if (prev_dev != c.device && cudaSetDevice(c.device) != cudaSuccess) { cudaGetLastError(); return 0; }
    size_t prev = 0, got = 0;
    bool ok = cudaDeviceGetAttribute(&mx, cudaDevAttrMaxPersistingL2CacheSize, c.device) == cudaSuccess && mx > 0 &&
              cudaDeviceGetLimit(&prev, cudaLimitPersistingL2CacheSize) == cudaSuccess;
    if (ok) {
        c.l2_limit_prev = prev;
        ok = cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, std::min<size_t>(want, (size_t)mx)) == cudaSuccess &&
             cudaDeviceGetLimit(&got, cudaLimitPersistingL2CacheSize) == cudaSuccess;
    }
    if (!ok) { cudaGetLastError(); got = 0; c.l2_limit_set = false; c.l2_limit_prev = 0; }
    c.l2_limit_granted = got;
    if (prev_dev != c.device) cudaSetDevice(prev_dev);
    return got;
}

void launch(Ctx &c, const Kernel &k, const KArgs &args, long long work_items, const char *cls, long long l2_window) {
    long long g = work_items;
    if (g > k.grid_cap) g = k.grid_cap;
    if (g < 1) g = 1;
    void *params[] = {(void *)&args};
    // SpMV over a gathered vector that does not stay L2-resident (> 48 MB, C5: 108 MB): a persisting
    // L2 window over its head -- the hottest columns in the degree-sorted gather layout -- keeps
    // them in L2 against the streamed indices.  C5 sweep: no window 3.86-3.93 ms,
    // 48 / 56 / 64 MB 3.80-3.81 ms, 72 / 80 MB 4.10 ms (past the persisting capacity).
    // NBG_L2_PERSIST_MB overrides the 56 MB default (0: off); resident vectors get no window.
    static long long persist = -1;
    if (persist < 0) {
        const char *e = getenv("NBG_L2_PERSIST_MB");
        persist = (e && *e) ? std::max(0ll, atoll(e)) << 20 : (56ll << 20);
    }
    size_t granted = 0;
    if (persist > 0 && args.x && l2_window > (48ll << 20)) granted = l2_setaside(c, (size_t)persist);
    const size_t win = granted ? (size_t)std::min<long long>(persist, l2_window) : 0;
    if (!win && c.l2_win_base) {
        // lines marked persisting stay set aside until demoted: touch the region once with a
        // Normal window, in stream order after the SpMV that marked them (never while it runs)
        cudaLaunchAttribute dm[1];
        dm[0].id = cudaLaunchAttributeAccessPolicyWindow;
        dm[0].val.accessPolicyWindow.base_ptr = const_cast<void *>(c.l2_win_base);
        dm[0].val.accessPolicyWindow.num_bytes = c.l2_win_bytes;
        dm[0].val.accessPolicyWindow.hitRatio = 1.0f;
        dm[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyNormal;
        dm[0].val.accessPolicyWindow.missProp = cudaAccessPropertyNormal;
        gpu_l2_touch(c, c.l2_win_base, c.l2_win_bytes, dm);
        c.l2_win_base = nullptr;
        c.l2_win_bytes = 0;
    }
    cudaEvent_t ev0 = nullptr;
    timing_begin(c, cls, &ev0);
    if (win) {
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeAccessPolicyWindow;
        at[0].val.accessPolicyWindow.base_ptr = const_cast<void *>(args.x);
        at[0].val.accessPolicyWindow.num_bytes = win;
        // hit ratio so that the persisting lines fit the granted set-aside (no thrashing inside it)
        at[0].val.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)granted / (double)win);
        at[0].val.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
        at[0].val.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3((unsigned)g);
        cfg.blockDim = dim3((unsigned)k.block);
        cfg.dynamicSmemBytes = (size_t)k.smem;
        cfg.stream = c.stream;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        NBG_CUDA(cudaLaunchKernelExC(&cfg, (const void *)k.k, params));
        c.l2_win_base = args.x;
        c.l2_win_bytes = win;
    } else {
        // the driver's cuLaunchKernel takes the library kernel handle directly (CUkernel in place of
        // CUfunction), skipping the runtime's per-launch handle translation: ~0.5 us of host time per
        // launch, which small graphs (C1) pay every sweep.  Resolved once through the runtime, no link
        // against libcuda.
        using LaunchFn = CUresult (*)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned, CUstream,
                                      void **, void **);
        using GetFn = CUresult (*)(CUfunction *, CUkernel);
        auto entry = [](const char *sym) -> void * {
            void *f = nullptr;
            cudaDriverEntryPointQueryResult q;
            if (cudaGetDriverEntryPoint(sym, &f, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess) f = nullptr;
            return f;
        };
        static LaunchFn drv = (LaunchFn)entry("cuLaunchKernel");
        static GetFn getfn = (GetFn)entry("cuKernelGetFunction");
        Kernel &km = const_cast<Kernel &>(k);
        if (!km.fn && getfn) {   // the kernel's function in the current context, once per kernel
            CUfunction f = nullptr;
            if (getfn(&f, (CUkernel)(void *)k.k) == CUDA_SUCCESS) km.fn = (void *)f;
        }
        if (drv) {
            plan_prof_t0();
            const CUresult r = drv(km.fn ? (CUfunction)km.fn : (CUfunction)(void *)k.k, (unsigned)g, 1, 1, (unsigned)k.block, 1, 1,
                                   (unsigned)k.smem, (CUstream)c.stream, params, nullptr);
            plan_prof_t1(8);
            if (r != CUDA_SUCCESS) fail(NBG_PANIC, "cuLaunchKernel failed (" + std::to_string((int)r) + ") for " + k.name);
        } else {
            NBG_CUDA(cudaLaunchKernel((const void *)k.k, dim3((unsigned)g), dim3((unsigned)k.block), params, (size_t)k.smem,
                                      c.stream));
        }
    }
    timing_end(c, cls, ev0);
    c.stats.kernels_launched++;
    if (guard_enabled()) guard_check(c, k.name.c_str());
    static int dbg_sync = -1;
    if (dbg_sync < 0) dbg_sync = (getenv("NBG_SYNC_DEBUG") && *getenv("NBG_SYNC_DEBUG")) ? 1 : 0;
    if (dbg_sync) {
        cudaError_t e = cudaStreamSynchronize(c.stream);
        if (e != cudaSuccess) fail(NBG_PANIC, "kernel " + k.name + " failed: " + cudaGetErrorString(e));
    }
}

}  // namespace nbg
