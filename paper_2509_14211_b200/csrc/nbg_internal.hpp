// nbg_internal.hpp -- internal data structures of the nonblocking GraphBLAS runtime.
//
// Layer map:
//   capi.cpp      C ABI: validation + DAG recording ("return once validated")
//   planner.cpp   wait(): region collection, signature, plan cache, memo, speculation, launch
//                 (PAPER.md:301-306 the four wait steps)
//   codegen.cpp   region IR -> CUDA C++ source (multi-stage programming)
//   jit.cpp       NVRTC -> cubin -> cudaLibrary, cached by signature
//   graph.cu      generators, CSR(AT) build, SpMV tile plan (static sm_100a kernels)
//   pagerank.cpp  Fig. 6 written on the C ABI
//   dist.cpp      NCCL (dlopen'ed) allgather-v + exact scalar allreduce
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <functional>
#include <memory>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/nbg.h"

namespace nbg {

// ---------------------------------------------------------------- errors

struct Error {
    nbg_status st;
    std::string msg;
};

[[noreturn]] void fail(nbg_status st, const std::string &msg);
[[noreturn]] void cuda_fail(cudaError_t e, const char *what, const char *file, int line);

#define NBG_CUDA(x)                                                     \
    do {                                                                \
        cudaError_t e_ = (x);                                           \
        if (e_ != cudaSuccess) ::nbg::cuda_fail(e_, #x, __FILE__, __LINE__); \
    } while (0)

inline size_t type_size(int t) {
    switch (t) {
        case NBG_BOOL: return 1;
        case NBG_INT32: return 4;
        case NBG_INT64: return 8;
        case NBG_FP32: return 4;
        case NBG_FP64: return 8;
    }
    return 0;
}
inline bool is_float(int t) { return t == NBG_FP32 || t == NBG_FP64; }
inline bool valid_type(int t) { return t >= NBG_BOOL && t <= NBG_FP64; }

struct Ctx;

// ---------------------------------------------------------------- device buffers

// A device allocation.  Owned buffers are released with cudaFreeAsync on the context stream
// (stream-ordered, so kernels already queued that read it stay valid).
struct Buf {
    Ctx *ctx = nullptr;
    uint64_t id = 0;           // never reused: memo keys and hints refer to buffers by id
    void *d = nullptr;
    size_t bytes = 0;
    bool owned = true;
    uint64_t prod_sig = 0;     // signature hash of the region that wrote it (0 = none)
    int prod_out = -1;         // output index within that region
    uint64_t prod_seq = 0;     // launch sequence number of that region
    ~Buf();
};
using BufP = std::shared_ptr<Buf>;

// ---------------------------------------------------------------- device scalar slots
// Every reduction result lives in a 128-byte slot of a zero-initialised slab; each slot has a
// pinned host mirror for asynchronous read-back.
//   u64[0..9]  signed 32-bit-piece limbs of the exact fixed-point accumulator (LSB = 2^-160)
//   u64[10]    flags: bit0 NaN, bit1 +inf, bit2 -inf, bit3 out of exact range
//   u64[11]    int64 sum (integer PLUS) or order-preserving key (MIN/MAX; 0 = no value)
constexpr int SLOT_U64 = 16;
constexpr int SLAB_SLOTS = 4096;

struct Slab {
    Ctx *ctx = nullptr;
    unsigned long long *d = nullptr;   // device, SLAB_SLOTS * SLOT_U64
    unsigned long long *h = nullptr;   // pinned host mirror
    int used = 0;
    ~Slab();
};
using SlabP = std::shared_ptr<Slab>;

enum class SFmt : uint8_t { HOST = 0, XACC = 1, I64 = 2, FMAX = 3, FMIN = 4, IMAX = 5, IMIN = 6 };

// an event recorded on the context's stream right after the launch (or collective) that produced
// one or more scalar slots: a deferred readback orders its copy after it (one record per launch)
struct ProdEv {
    Ctx *ctx = nullptr;
    cudaEvent_t e = nullptr;
    ~ProdEv();
};
using ProdEvP = std::shared_ptr<ProdEv>;

struct Slot {
    SlabP slab;
    int idx = 0;
    uint64_t id = 0;
    cudaEvent_t ev = nullptr;          // recorded after the D2H copy of the mirror
    bool rb_issued = false;
    ProdEvP pev;                       // producer position of a slot the host may read (mark_readable)
    ProdEvP cev;                       // completion of a bulk readback that covered this slot
    unsigned long long *dptr() const { return slab->d + (size_t)idx * SLOT_U64; }
    unsigned long long *hptr() const { return slab->h + (size_t)idx * SLOT_U64; }
    ~Slot();
};
using SlotP = std::shared_ptr<Slot>;

// decode helpers (host side; device side lives in jit/prelude.cuh)
double xacc_to_double(const unsigned long long *limbs);
double slot_value(const unsigned long long *s, SFmt fmt);

// ---------------------------------------------------------------- matrices

struct TpPlan;

struct RbPlan;
struct SpmvPlan {
    // Rows are stored in 4-entry groups (padded with index -1) so a 16-byte index load never mixes
    // two rows.  Tiles: runs of <= 32 consecutive rows with <= 512 groups (one warp task, lane j ->
    // row j).  Long rows (> 512 groups) are cut into chunks of 512 groups processed by separate
    // warps; the warp that finishes a long row's last chunk (atomic ticket) combines the chunk
    // partials in chunk order and runs the epilogue.  DESIGN.md "K4 SpMV".
    int64_t ntiles = 0, nchunks = 0, nlong = 0, ngroups = 0;
    int64_t max_row_groups = 0;   // longest row, in 4-entry groups
    bool low_skew = false;        // max row <= 4 x mean and mean <= 32 entries: lane-per-row SpMV
    BufP grp;        // int64[n + 1]  first group of each row
    BufP cg;         // int32[4 * ngroups]  column index per padded position (gather layout), -1 = pad
    BufP vals_g;     // values per padded position (valued matrices only)
    BufP tiles;      // int4  {row_begin, rows | ngroups << 8, first_group_lo, first_group_hi}
    BufP chunks;     // int4  {long_idx, first_group_lo, first_group_hi, ngroups}
    BufP longs;      // int4  {row, first_chunk, nchunks, 0}
    BufP counters;   // int[nlong], zero between launches
    BufP partials;   // double[nchunks]
    // Gather layout: columns renumbered by descending column count,
    // empty columns dropped.  The gathered vector is stored in that order so the hot entries are
    // dense and the first ones fit a shared-memory cache; rows keep their entry order.
    bool relabel = false;
    int64_t ncols_g = 0;     // number of non-empty columns
    BufP perm;               // int32[ncols] old -> new id, -1 for an empty column
    BufP iperm;              // int32[ncols_g] new -> old id
    BufP colidx_g;           // int32[nnz] gather-layout column indices (relabelled matrices; two-phase build)
    std::unique_ptr<TpPlan> tp[2];   // two-phase plans for 4- and 8-byte gathered elements (lazy)
    std::unique_ptr<RbPlan> rb;   // row-binned plan (lazy, DESIGN.md §7 "row-binned SpMV")
    bool filled = false;          // stage 2 (column indices) done
};

// Row-binned SpMV plan (DESIGN.md §7 "row-binned SpMV"), built once per matrix on top of the
// group-padded plan.  Rows are binned by length in 4-entry groups g:
//   short (1 <= g <= T): sorted by g descending (ties by row id), cut into 32-row slices; a slice
//        is stored column-major (group k of its lane-l row at soff + 32 k + l, -1 padded to the
//        slice width), so one warp sums 32 rows lane-per-row with coalesced 512-byte index loads;
//   long  (T < g <= 512): g descending, one warp per row over the group-padded CSR;
//   hub   (g > 512): the group-padded plan's chunks (one warp each, combined in chunk order).
// Every row total goes to tot[row]; after a grid barrier the same kernel runs the fused epilogue
// over the rows in index order.  A row's summation order depends on its length only.
struct RbPlan {
    int T = 32;                  // short-row bound in groups (C4: T 8 / 16 / 32 / 64 / 128 -> 209 / 171 / 168 / 171 / 194 us)
    int64_t nshort = 0, nslices = 0, nlong = 0, ntasks = 0, ntasks_main = 0, sell_groups = 0;
    BufP sell;      // int4[sell_groups]  short slices, column-major, -1 padded
    BufP srow;      // int32[32 * nslices]  destination row of each slice slot (-1: none)
    BufP swid;      // int32[nslices]  slice width in groups
    BufP lrows;     // int32[nlong]  long rows, g descending
    BufP tasks;     // int4[ntasks]  {kind | count << 2, first, base_lo, base_hi}: 0 hub chunk, 1 long rows, 2 short slices,
                    //   3 empty-row range (inline-epilogue mode), interleaved
    BufP tasks_main;   // int4[ntasks_main]  the same without kind 3 (barrier mode)
    BufP tasks_pipe;   // int4[ntasks_pipe]  pipelined mode: hub + long tasks, then slice runs by row group (.w = group)
    int64_t ntasks_pipe = 0;
    int ngrp = 1;      // row groups: rows [q gsize, (q + 1) gsize)
    int64_t gsize = 0;
    bool pipe_ok = false;
    BufP gcnt;      // int[2 ngrp + 1]  tasks per counter: [0] hub + long, [1 + q] slice runs of group q; [1 + ngrp + q] end of group q's runs
    BufP done;      // u64[2 ngrp + 3]  pipelined counters (zero between launches; see rb_task_list)
    bool filled = false;                      // slices filled (sell / srow); before: pend_* hold the fill's inputs
    BufP pend_sorted, pend_fc, pend_so;
    std::vector<int> h_head;                  // host copies for the lazily built lists: hub + long task records,
    std::vector<std::vector<int>> h_sruns;    // and the slice runs per row group (pipelined form, .w = group)
    BufP mask;      // u32[(n + 31) / 32]  bit i: row i is non-empty
    BufP tot;       // 8 bytes per row: row totals (the kernel's row-total type)
    BufP bar;       // u32[2]  grid barrier {arrivals, generation}
};

// Two-phase column-blocked SpMV plan, one per gathered element size.
// Phase 1: the gather layout's columns are cut into blocks of S columns (S * element size = 128 KB,
// one block in shared memory at a time); the entries of row i in block b form a "pair" (b, i).
// Pairs are stored block-major in the same 4-entry group layout as the single-pass plan, with
// block-local column indices, and processed by warp tasks (<= 128 pairs, one block per task);
// each pair's partial sum goes to part[slot], where slots are ordered (row, block).
// Phase 2: row i's value = its slots rowslot[i] .. rowslot[i+1] combined in block order.
struct TpPlan {
    int xsize = 4;               // gathered element size this plan is for
    int64_t S = 0;               // columns per block
    int64_t nblocks = 0, npairs = 0, ngroups = 0, ntasks = 0, nchunks = 0, nlong = 0;
    BufP grp;        // int64[npairs + 1]  first group of each pair
    BufP cg;         // int32[4 * ngroups]  block-local column index per padded position, -1 = pad
    BufP tasks;      // int4 {pair_begin, npairs | ngroups << 8, first_group_lo, first_group_hi}
    BufP tblk;       // int32[ntasks]  column block of each task (tasks are block-major)
    BufP cta;        // int32[ncta + 1]  task range of each CTA
    int ncta = 0;
    BufP chunks;     // int32[ntasks]  global chunk index of a chunk task, -1 for a pair task
    BufP longs;      // int4 {pair, first_chunk, nchunks, 0}
    BufP counters;   // int[nlong]
    BufP partials;   // double[nchunks]
    BufP slot;       // int32[npairs]  (row, block)-ordered slot of each pair
    BufP rowslot;    // int64[n + 1]   first slot of each row
    BufP part;       // double[npairs] per-pair partial sums (phase 1 -> phase 2)
};

struct Mat {
    Ctx *ctx = nullptr;
    uint64_t id = 0;
    int64_t nrows = 0, ncols = 0, nnz = 0;
    int type = NBG_FP32;     // value type (iso or vals)
    double iso = 1.0;
    BufP rowptr, colidx, vals;   // vals null => iso
    std::unique_ptr<SpmvPlan> plan;
    int64_t max_row = -1;
    bool prelabeled = false;     // columns already in a gather layout (multi-GPU row blocks): no relabel
};
using MatP = std::shared_ptr<Mat>;

// ---------------------------------------------------------------- DAG nodes

enum class Op : uint8_t { LEAF = 0, APPLY, BIND2ND, EMULT, EADD, MXV, REDUCE, SAPPLY };
// vector representations (PAPER.md:185 SparseVector / BitSetVector / FullVector).  EMPTY and ISO
// are folded at record time; SPARSE and BITSET carry a structure.
enum class VKind : uint8_t { EMPTY = 0, ISO = 1, FULL = 2, SPARSE = 3, BITSET = 4 };

struct Node;
using NodeP = std::shared_ptr<Node>;

struct Node {
    Op op = Op::LEAF;
    bool scalar = false;
    int type = NBG_FP32;
    int64_t n = 0;               // vector length (vectors)
    int code = 0;                // unop / binop code, or monoid for REDUCE
    double c0 = 0.0, c1 = 0.0;   // operator constants
    int add = 0, mul = 0;        // MXV semiring
    NodeP a, b;                  // operands (b: second vector, or bound scalar)
    MatP A;                      // MXV matrix
    uint64_t uid = 0;
    int user_refs = 0;           // live user handles (liveness rule)

    // materialised state
    bool mat = false;
    VKind kind = VKind::FULL;    // kind is known at record time (EMPTY/ISO folded eagerly)
    BufP buf;                    // FULL: n values; SPARSE: nvals values; BITSET: n values
    BufP idx;                    // SPARSE: int32[nvals] strictly ascending indices
    BufP bits;                   // BITSET: uint32[(n + 31) / 32], bit i = entry i present
    int64_t nvals = 0;           // SPARSE / BITSET: number of present entries
    double iso = 0.0;            // ISO vector value (already rounded to type)
    // scalar state
    SFmt sfmt = SFmt::HOST;
    double hval = 0.0;           // HOST scalar value (already rounded to type)
    SlotP slot;                  // device scalar
    BufP full_cache;             // ISO vector expanded to a buffer (used as an mxv input)
};

// ---------------------------------------------------------------- region IR (codegen input)

struct Ins {
    enum K : uint8_t { LD_VEC = 0, LD_ISO, LD_SHOST, LD_SDEV, MXV_ACC, UN, BIN, CVT } k;
    int t = NBG_FP32;       // output type
    int code = 0;
    int a = -1, b = -1;     // operand instruction indices
    int imm0 = -1, imm1 = -1;
    int slot = -1;          // LD_VEC input index / LD_ISO, LD_SHOST imm index / LD_SDEV sin index
    uint8_t fmt = 0;        // LD_SDEV format
    bool uniform = false;   // value independent of the element index
};

// scatter: out[oscat[i]] (skip < 0); multi: the scattered value stored into every a.peer[q] buffer
// (the multi-GPU exchange fused into the producing kernel, dist.cpp peer mode)
struct OutV { int ins; int out; bool scatter = false; bool multi = false; bool affine = false; };   // affine: out[ooff + i], i < olim (no map)
struct RedOut { int ins; int monoid; int racc; uint8_t fmt; };

struct SpmvSig {
    int add = NBG_PLUS, mul = NBG_SECOND;
    int T = NBG_FP32;       // type of the mxv node (mul evaluated in T)
    int xt = NBG_FP32;      // x buffer type
    int at = NBG_FP32;      // matrix value type
    bool has_vals = false;
};

struct Prog {
    std::vector<Ins> ins;
    std::vector<OutV> outs;
    std::vector<RedOut> reds;
    bool spmv = false;
    bool tp = false;        // spmv through the two-phase plan: this program is phase 2 (combine + epilogue)
    bool lpr = false;       // spmv, lane-per-row skeleton (low-skew matrices)
    bool rb = false;        // spmv, row-binned skeleton (RbPlan)
    bool rb_inline = false; // row-binned: epilogue at each row's completion (no barrier)
    bool rb_pipe = false;   // row-binned: epilogue chunks of a row group once its totals are complete (no barrier)
                            // neither: totals + grid barrier + epilogue pass
    int nt = 0, hot_kb = 0; // spmv (task skeleton): threads per CTA and hot-cache KB, chosen per matrix
    bool vec = true;        // 16-byte vector loads/stores (all buffers aligned)
    bool tma = false;       // ewise: inputs staged through shared memory by TMA bulk copies (large n)
    SpmvSig sp;
    int n_in = 0, n_out = 0, n_imm = 0, n_sin = 0, n_red = 0;
    std::string signature() const;
    uint64_t sig_hash() const;   // hash of the signature's token stream (no string)
};

// Kernel arguments (one struct passed by value; mirrored in jit/prelude.cuh).
constexpr int MAX_IN = 16, MAX_OUT = 8, MAX_IMM = 32, MAX_SIN = 8, MAX_RED = 8;
constexpr int MAX_PEER = 8;   // ranks a multi-store output writes to (one NVSwitch node)
struct KArgs {
    long long n;
    const void *in[MAX_IN];
    void *out[MAX_OUT];
    double imm[MAX_IMM];
    const unsigned long long *sin[MAX_SIN];
    unsigned long long *racc[MAX_RED];
    // spmv
    const long long *rowptr;
    const int *colidx;
    const void *aval;
    const void *x;
    const int *tiles;        // int2 pairs
    const int *chunks;       // int4
    const int *longs;        // int4
    int *counters;
    double *partials;
    long long ntiles, nchunks;
    long long row_offset;    // global index of local row 0 (distributed); 0 otherwise
    const int *oscat[MAX_OUT];   // per output: scatter map (gather layout) or null
    long long hc;                // spmv: entries of the gathered vector cached in shared memory
    long long nnz;               // spmv: number of stored entries (bounds of vector index loads)
    // two-phase spmv (TpPlan)
    const int *tblk;             // phase 1: column block of each task
    const int *cta;              // phase 1: task range of each CTA
    const int *pslot;            // phase 1: (row, block) slot of each pair
    const long long *rowslot;    // phase 2: first slot of each row
    void *part;                  // per-slot partial sums (accumulator type)
    long long S;                 // phase 1: columns per block
    long long ncols_g;           // phase 1: columns of the gather layout
    void *peer[MAX_PEER];        // multi-store output: the exchange buffers of all ranks
    int npeer;
    // row-binned spmv (RbPlan)
    const int *rb_tasks;         // int4 task records
    const int *rb_sell;          // int4 short-slice groups
    const int *rb_srow;
    const int *rb_swid;
    const int *rb_lrows;
    const unsigned *rb_mask;
    void *rb_tot;
    unsigned *rb_bar;
    long long rb_ntasks;
    long long ooff[MAX_OUT], olim[MAX_OUT];   // affine outputs: out[ooff + i] for i < olim
    // row-binned, pipelined mode: counters (gpu_rb_plan), tasks per completion counter, row groups
    unsigned long long *rb_done;
    const int *rb_gcnt;
    long long rb_ngrp, rb_gsize;
};

struct Kernel {
    ~Kernel();
    cudaLibrary_t lib = nullptr;
    cudaKernel_t k = nullptr;
    void *fn = nullptr;      // CUfunction of k in the context's device (driver launch), resolved once
    int block = 256;
    int smem = 0;            // dynamic shared memory per CTA
    int hot = 0;             // spmv: capacity of the hot-column cache (entries)
    int grid_cap = 0;        // persistent grid size (SMs * resident CTAs)
    std::string name;
};
using KernelP = std::shared_ptr<Kernel>;

struct Hint {           // speculative loop-carried side output (planner rule 3)
    NodeP tmpl;         // pending template expression
    Node *placeholder;  // leaf inside tmpl standing for the region output
    NodeP ph_keep;
    // the template's other vector leaves, held weakly: placeholder -> original leaf
    std::vector<std::pair<NodeP, std::weak_ptr<Node>>> fixed;
    std::string key;    // dedupe key (expression with the loop-carried leaf as "P")
    std::weak_ptr<Mat> consumer;   // mxv whose gather input this expression was (layout of the output)
};

struct TimingClass {
    double ms = 0.0;
    int64_t launches = 0;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> pending;
};

// ---------------------------------------------------------------- context

struct LoopGroup;   // dist.cpp: in-process transport (P contexts in P host threads on one GPU, tests)
struct Dist {
    int rank = 0, nranks = 1;
    void *comm = nullptr;   // ncclComm_t
    std::shared_ptr<LoopGroup> loop;   // set instead of comm by nbg_dist_init_loopback
    int xmode = 0;          // NBG_DIST_EXCHANGE_{COLLECTIVE,PEER} (nbg_dist_set_exchange)
    // peer mode: per (ncols_g, element size) a ping-pong pair of exchange buffers on every rank
    // and the peers' addresses (IPC-mapped under NCCL, plain pointers under loopback)
    struct PeerSet {
        size_t bytes = 0;
        void *own[2] = {nullptr, nullptr};
        std::vector<void *> peer[2];     // indexed by rank (own included)
        std::vector<void *> opened;      // IPC mappings to close
        int parity = 0;
    };
    std::map<std::pair<int64_t, size_t>, PeerSet> peersets;
    ~Dist();
};

// memo key: 128-bit hash of an expression's structural token stream (planner.cpp memo_key)
struct MKey {
    uint64_t a = 0, b = 0;
    bool operator==(const MKey &o) const { return a == o.a && b == o.b; }
};
struct MKeyHash {
    size_t operator()(const MKey &k) const { return (size_t)(k.a ^ (k.b * 0x9E3779B97F4A7C15ull)); }
};

struct Ctx {
    int mode = NBG_NONBLOCKING;
    int device = 0;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    int num_sms = 148;
    uint64_t next_id = 1;
    uint64_t launch_seq = 0;
    std::string last_error;
    nbg_status latched = NBG_SUCCESS;
    nbg_stats stats{};

    // scalar slabs
    SlabP cur_slab;
    std::vector<cudaEvent_t> event_pool;
    std::vector<cudaEvent_t> timing_pool;   // recycled timing events (nbg_set_timing)
    std::map<void *, size_t> guard_live;   // NBG_GUARD=1: live pool buffers (red zone after each)
    std::string guard_msg;                  // a red-zone violation found at free
    std::deque<std::weak_ptr<Slot>> deferred;   // readable slots not yet copied, in production order
    cudaStream_t rb_stream = nullptr;      // scalar readbacks (issue_readback), ordered after the producer
    cudaEvent_t rb_dep = nullptr;
    // persisting-L2 window over the head of a large gathered vector (launch(), NBG_L2_PERSIST_MB)
    bool l2_limit_set = false;             // this context raised the device's persisting set-aside
    size_t l2_limit_prev = 0;              // ... from this value (restored at finalize)
    size_t l2_limit_granted = 0;           // set-aside the device granted
    const void *l2_win_base = nullptr;     // region whose lines were last marked persisting
    size_t l2_win_bytes = 0;               // (demoted in stream order before the next other kernel)

    // freed device buffers kept for reuse by size (all work is ordered on `stream`, so a buffer
    // whose last handle died can back a later allocation without a cudaFreeAsync/MallocAsync pair)
    std::unordered_map<size_t, std::vector<void *>> buf_pool;
    size_t pooled_bytes = 0;
    bool closing = false;
    // plan cache: signature -> kernel ("GraphBLAS method signatures as keys")
    std::unordered_map<std::string, KernelP> plans;
    // memo: structural key over materialised leaves -> result (derived views)
    struct MemoEntry {
        std::vector<std::weak_ptr<Buf>> deps;
        NodeP result;            // a materialised node
        uint64_t stamp = 0;      // last use (LRU bound)
    };
    uint64_t memo_clock = 0;
    std::unordered_map<MKey, MemoEntry, MKeyHash> memo;
    // learned hints: producer signature hash + output index -> templates
    std::map<std::pair<uint64_t, int>, std::vector<Hint>> hints;

    // output targets of the current materialize call (multi-GPU: a block written straight into
    // the exchange buffer through a scatter map); see dist.cpp nbg_vector_allgather_reduce
    // peers: multi-store; alim >= 0: the map is affine (row i -> aoff + i for i < alim, else skipped) and
    // the kernels store without it
    struct OutTarget { BufP buf; const int *map = nullptr; std::vector<void *> peers; int64_t aoff = 0, alim = -1; };
    std::unordered_map<const Node *, OutTarget> out_targets;
    // nodes user handles point to (weak): nbg_wait_all materialises the live pending ones
    std::vector<std::weak_ptr<Node>> user_nodes;
    size_t user_nodes_live = 0;

    // timing
    bool timing = false;
    std::map<std::string, TimingClass> tclass;

    // distributed
    std::unique_ptr<Dist> dist;
    // row -> position maps of this rank's block in the exchange buffer, per (first row, rows)
    std::shared_ptr<std::map<std::pair<int64_t, int64_t>, BufP>> dist_maps;

    uint64_t new_id() { return next_id++; }
    ~Ctx();
};

// ---------------------------------------------------------------- helpers shared by the runtime

BufP alloc_buf(Ctx &c, size_t bytes);
BufP borrow_buf(Ctx &c, void *d, size_t bytes);
SlotP alloc_slot(Ctx &c);
cudaEvent_t get_event(Ctx &c);
void put_event(Ctx &c, cudaEvent_t e);
void issue_readback(Ctx &c, Slot &s);
// record (once per producing launch: pass the same ProdEvP) the stream position after which slot s
// is final; the D2H copy itself is issued only when the host reads it (issue_readback)
ProdEvP record_prod_event(Ctx &c);
void mark_readable(Ctx &c, const SlotP &s, const ProdEvP &pe);

void timing_begin(Ctx &c, const char *cls, cudaEvent_t *ev0);
void timing_end(Ctx &c, const char *cls, cudaEvent_t ev0);
void timing_collect(Ctx &c);

// user-defined operators (userops.cpp)
struct UserOp { int arity = 1; std::string name, expr; };
const UserOp *user_op(int code);   // null unless `code` is a registered user operator
int user_op_define(int arity, const std::string &name, const std::string &expr, std::string *err);
std::string user_op_call(const UserOp &op, const std::string &C, const std::string &x, const std::string &y,
                         const std::string &k0, const std::string &k1);

// planner entry points
void materialize(Ctx &c, const std::vector<NodeP> &roots);
double scalar_read(Ctx &c, const NodeP &s);
void ensure_full(Ctx &c, const NodeP &v);   // ISO leaf -> FULL buffer

// structured (sparse / bitset) vectors: structured.cpp, sparse.cu
bool structured_kind(VKind k);                       // SPARSE or BITSET
bool needs_structured(const NodeP &r);               // root whose region reads a sparse/bitset leaf
void materialize_structured(Ctx &c, const NodeP &r); // one structured region (vector or reduce root)
double estimated_fill(const Node *x);                // naive metadata estimator
// structured region program: Prog + presence algebra
struct SProg {
    Prog p;
    std::vector<uint8_t> pmode;   // per instruction: 0 inherit a, 1 AND (ewise_mult), 2 OR (ewise_add), 3 leaf
    std::vector<uint8_t> leaf;    // per input slot: 0 full, 1 bitset (bits in in[n_in + slot]), 2 sparse (binary search)
    bool index_mode = false;      // iterate a sorted index list (a.rowptr as int*, a.nnz entries) instead of [0, n)
    bool vec_out = true;          // root is a vector (else a reduction)
    std::string signature() const;
};
std::string codegen_structured(const SProg &sp, const std::string &kname);
std::string codegen_smxv(const SpmvSig &sp, const std::string &kname);
// device helpers (sparse.cu)
int gpu_check_sparse(Ctx &c, int64_t n, int64_t nv, const int32_t *idx);   // 0 ok, 1 not ascending, 2 out of range
void gpu_sparse_to_bitset(Ctx &c, int64_t n, int64_t nv, const int32_t *idx, const void *vals, int type, uint32_t *bits,
                          void *dense);
int64_t gpu_bitset_to_sparse(Ctx &c, int64_t n, const uint32_t *bits, const void *dense, int type, BufP *idx, BufP *vals);
int64_t gpu_select_flagged(Ctx &c, int64_t m, const int32_t *idx, const void *vals, const uint8_t *flags, int type, BufP *oidx,
                           BufP *ovals);
int64_t gpu_union_indices(Ctx &c, const std::vector<std::pair<const int32_t *, int64_t>> &lists, BufP *out);
void gpu_bitset_full(Ctx &c, int64_t n, uint32_t *bits);   // all n bits set, tail bits clear

// codegen / jit
bool spmv_gather_pipeline();   // SpMV gathers one step ahead (NBG_SPMV_GPIPE=1)
bool spmv_epilogue_prefetch();  // SpMV prefetches the epilogue's row inputs at task start (NBG_SPMV_PF, default on)
int spmv_threads(int xsize);
bool spmv_threads_overridden();   // NBG_SPMV_THREADS set to a valid CTA size
int spmv_groups_per_lane();   // SpMV task skeleton: groups per lane per step (NBG_SPMV_GPL, default 2)
void spmv_variant(int xsize, long long gathered_bytes, int *nt, int *hot_kb);   // per-matrix SpMV launch shape   // threads per SpMV CTA for a gathered element size (NBG_SPMV_THREADS overrides)
int spmv_rb_mode();    // NBG_SPMV_RB: -1 auto (skewed matrices), 0 never, 1 always
char spmv_rb_epi_mode(); // NBG_RB_MODE: b (default) totals + grid barrier + epilogue pass, p pipelined epilogue chunks, i epilogue at each row's completion
int spmv_lpr_mode();   // NBG_SPMV_LPR: -1 auto (by skew), 0 never, 1 always   // threads per SpMV CTA (NBG_SPMV_THREADS, default 1024)
std::string codegen_tp1(const SpmvSig &sp, const std::string &kname, int xsize, long long S, int *dyn_smem);
std::string codegen(const Prog &p, const std::string &kname, int *dyn_smem = nullptr, int *hot_entries = nullptr);
KernelP jit_compile(Ctx &c, const std::string &src, const std::string &kname, bool spmv, int dyn_smem = 0, int block = 0);
// Launch k on the context stream.  l2_window > 0: an SpMV over a gathered vector args.x of that many
// bytes; large ones get a persisting L2 access-policy window over their head.
void launch(Ctx &c, const Kernel &k, const KArgs &args, long long work_items, const char *cls, long long l2_window = 0);
void gpu_l2_touch(Ctx &c, const void *base, size_t bytes, const cudaLaunchAttribute *attr);   // graph.cu

// graph (graph.cu)
void gpu_graph_edges(Ctx &c, const nbg_graphgen &g, int32_t *d_src, int32_t *d_dst);
MatP gpu_build_csr(Ctx &c, int64_t n, int64_t m, const int32_t *d_src, const int32_t *d_dst, BufP *deg_out);
// stage 0: the whole plan; 1: the structure (row pointers only); 2: the fill of a stage-1 plan
// (column indices) -- nbg_matrix_from_csr overlaps stage 1 with the column-index upload
void gpu_build_spmv_plan(Ctx &c, Mat &A, int stage = 0);
// per-rank multi-GPU graph setup (graph.cu)
struct DistGraph {
    MatP blk;                    // rows pi in [cuts[rank], cuts[rank+1]) x ncols_g columns (pi ids)
    BufP deg_blk;                // int32 out-degrees of the block's vertices (pi order)
    BufP order;                  // int32[n]: pi^-1 (vertex of each pi position)
    std::vector<int64_t> cuts;   // P + 1 row cuts in pi-space
    int64_t n = 0, ncols_g = 0;
};
DistGraph gpu_dist_graph(Ctx &c, const nbg_graphgen &g, int rank, int P, long long bytes_per_row,
                         const std::function<void(int *, long long)> &allreduce_int_sum);
TpPlan *gpu_tp_plan(Ctx &c, Mat &A, int xsize, int ncta);   // null if not applicable
RbPlan *gpu_rb_plan(Ctx &c, Mat &A, bool fill = true);      // null if not applicable (valued matrices); fill = false:
                                                             // everything but the slice fill (needs the plan's fill)
void gpu_rb_fill(Ctx &c, Mat &A);                            // the slice fill of a gpu_rb_plan(.., false) plan
const int *rb_task_list(Ctx &c, RbPlan &R, char mode, long long n, int64_t *ntasks);   // task list of an epilogue mode (lazy)
void gpu_fill_iso(Ctx &c, void *d, int type, int64_t n, double v);
void gpu_permute(Ctx &c, const void *x, void *xg, int type, const int *iperm, int64_t ng);
int gpu_validate_csr(Ctx &c, long long n, long long ncols, long long nnz, const long long *rp, const int *ci);
void gpu_rebase_rowptr(Ctx &c, long long n, const long long *rp, long long base, long long *out);
void host_xacc_add(unsigned long long *limbs, double d);
void gpu_offset_map(Ctx &c, int64_t nb, int64_t c0, int64_t limit, int *map);   // map[i] = c0+i < limit ? c0+i : -1
void gpu_sum_i32(Ctx &c, int64_t n, int nsrc, const int *const *srcs, int *dst);      // dst = sum of nsrc arrays (host ptr list)
void gpu_sum_slots(Ctx &c, int nsrc, const unsigned long long *const *slots, unsigned long long *dst);  // exact slot sum

// host arithmetic (used for eager iso folding and host-side scalar ops)
double host_unop(int code, int t, double x, double c0, double c1);
double host_binop(int code, int t, double x, double y, double c0);
double host_round(int t, double v);
double monoid_identity(int monoid, int type);   // identity of PLUS / MIN / MAX in type
uint64_t hash_str(const std::string &s);
bool guard_enabled();                   // NBG_GUARD=1 (runtime.cpp)
void guard_check(Ctx &c, const char *where);
int gpu_guard_scan(Ctx &c, const unsigned char *const *zones, int nzones, size_t bytes);   // graph.cu: first bad zone or -1
void plan_prof_t0();          // NBG_PLAN_PROFILE probes (planner.cpp)
void plan_prof_t1(int phase);

double now_ns();

}  // namespace nbg

// opaque handle structs of the C ABI
struct nbg_ctx_s : nbg::Ctx {};
struct nbg_matrix_s { nbg_ctx *ctx; nbg::MatP m; };
struct nbg_vector_s { nbg_ctx *ctx; nbg::NodeP node; };
struct nbg_scalar_s { nbg_ctx *ctx; nbg::NodeP node; };
