/*
 * nbg.h -- C ABI of the B200-native nonblocking GraphBLAS hot path (arxiv 2509.14211).
 *
 * The calls follow the paper's statement of the problem: GraphBLAS operations in program order
 * define a DAG (Sec. 2); in NONBLOCKING mode an operation returns once its
 * arguments are validated and the DAG is materialised at `wait` as fused GPU
 * passes; in BLOCKING mode every operation is complete on return
 * (PAPER.md:48, 255).  Results of both modes are equal up to floating-point rounding order
 * (PAPER.md:52); this library keeps the blocking mode's rounding points in its fused kernels,
 * so ranks agree bit for bit.
 *
 * Conventions (apply to every function):
 *  - Return value: nbg_status.  NBG_SUCCESS = 0.  Validation errors (null handle, dimension or
 *    domain mismatch, bad enum) are returned AT CALL TIME in both modes (PAPER.md:49,
 *    SPEC.md:237).  Execution errors (a CUDA/NVRTC/NCCL failure, out of memory on the device)
 *    are returned by the call that materialises the object (a wait, an export, a scalar read,
 *    or any op in blocking mode) and latched on the context: nbg_last_error() returns the text.
 *  - Handles (nbg_matrix, nbg_vector, nbg_scalar) are opaque and immutable: an operation never
 *    modifies its inputs, it returns a NEW handle through its first out-parameter
 *    (PAPER.md:113).  The caller owns every returned handle and releases it with
 *    the matching nbg_*_free().  Freeing a handle that pending operations still reference is
 *    safe: the library keeps the definition alive internally.
 *  - Liveness: in nonblocking mode a pending node is materialised at wait iff it is requested
 *    or the user still holds a handle to it; otherwise it is fused and elided.
 *  - Memory spaces: NBG_HOST pointers are ordinary host memory (pinned or pageable);
 *    NBG_DEVICE pointers are device memory of the context's GPU.  NBG_COPY copies the data;
 *    NBG_BORROW keeps the device pointer (it must outlive the object and stay unmodified).
 *  - Streams: every kernel and every host<->device copy of a context is issued on the context's
 *    CUDA stream (config.stream, or a library-owned stream when NULL), except the device->host
 *    readback of a reduction's value, which runs on an internal side stream ordered after the
 *    producing kernel by an event (so the next kernels on the context stream do not wait behind
 *    the copy).  Exports synchronise the context stream; nbg_scalar_get waits only for the
 *    readback of that scalar; nbg_sync waits for both streams (all outstanding work).
 *  - Index types: row pointers are int64, column indices int32 ("32 bit indices");
 *    dimensions must be < 2^31 (NBG_INVALID_VALUE otherwise).
 *  - A context is single-threaded: calls on one context must not run concurrently.
 */
#ifndef NBG_H
#define NBG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---------------------------------------------------------------- status, types, modes */

typedef enum {
    NBG_SUCCESS = 0,
    NBG_NULL_POINTER = 1,          /* a required pointer/handle argument is NULL */
    NBG_INVALID_VALUE = 2,         /* bad enum, negative/oversized dimension, bad parameter */
    NBG_DIMENSION_MISMATCH = 3,    /* operand lengths / matrix shape disagree */
    NBG_DOMAIN_MISMATCH = 4,       /* operator not defined for the requested type */
    NBG_INDEX_OUT_OF_BOUNDS = 5,   /* an index in user data is out of range */
    NBG_INVALID_OBJECT = 6,        /* handle from another context, or an empty vector exported */
    NBG_OUT_OF_MEMORY = 7,
    NBG_NOT_IMPLEMENTED = 8,       /* valid request outside this subset (e.g. sparse vectors) */
    NBG_PANIC = 9                  /* CUDA / NVRTC / NCCL failure; see nbg_last_error */
} nbg_status;

typedef enum { NBG_BOOL = 0, NBG_INT32 = 1, NBG_INT64 = 2, NBG_FP32 = 3, NBG_FP64 = 4 } nbg_type;

typedef enum { NBG_BLOCKING = 0, NBG_NONBLOCKING = 1 } nbg_mode;

typedef enum { NBG_HOST = 0, NBG_DEVICE = 1 } nbg_space;
typedef enum { NBG_COPY = 0, NBG_BORROW = 1 } nbg_ownership;

typedef struct nbg_ctx_s nbg_ctx;
typedef struct nbg_matrix_s *nbg_matrix;
typedef struct nbg_vector_s *nbg_vector;
typedef struct nbg_scalar_s *nbg_scalar;

/* nbg_config.flags bits.
 * NBG_FLAG_DETERMINISTIC (SURVEY 8(b) `deterministic=1`): request run-to-run bit-reproducible
 *   results.  This library has no nondeterministic fast path, so the flag changes nothing and
 *   results are always deterministic: floating PLUS reductions are accumulated per thread / task
 *   in a fixed order and combined across blocks EXACTLY (order-independent fixed-point limbs;
 *   across ranks by an integer allreduce), SpMV row sums have an order fixed by the matrix plan,
 *   and integer MIN/MAX/PLUS are associative.  (The one exception is documented at nbg_reduce:
 *   partials of magnitude >= 2^128 or < 2^-160 are added in arrival order.)  Other bits:
 *   NBG_INVALID_VALUE. */
enum { NBG_FLAG_DETERMINISTIC = 1 };

typedef struct {
    int mode;        /* nbg_mode; fixed for the context's lifetime */
    int device;      /* CUDA device ordinal */
    void *stream;    /* cudaStream_t to issue work on (borrowed), or NULL for a library stream */
    int flags;       /* 0 or NBG_FLAG_DETERMINISTIC (see above); checked before any CUDA call */
} nbg_config;

/* ---------------------------------------------------------------- operators
 * Operators are plain descriptors (no function pointers): the operation is inlined into the
 * generated kernel per signature, as PAPER.md:227 specialises "the concrete operations".
 * Every operator is evaluated in the OUTPUT type T of the operation that uses it: its inputs
 * and constants are first converted to T (round to nearest for floating T, truncation toward
 * zero for integer T; bool T computes in int64 and stores x != 0).  One IEEE round-to-nearest
 * rounding per arithmetic step, no FMA contraction.                                          */

typedef enum {
    NBG_IDENTITY = 0,      /* x                                       */
    NBG_AINV = 1,          /* -x                                      */
    NBG_ABS = 2,           /* |x|                                     */
    NBG_MINV = 3,          /* 1/x   (integer: 0 when x == 0)          */
    NBG_ADD_C = 4,         /* x + c0        (Fig. 2: x -> x + 1)       */
    NBG_MUL_C = 5,         /* x * c0                                  */
    NBG_AXPB = 6,          /* (c0 * x) + c1, two roundings            */
    NBG_ABS_SUB_C = 7,     /* |x - c0|                                */
    NBG_RECIP_SCALED = 8,  /* x != 0 ? c0 / x : 0                     */
    NBG_ISZERO = 9         /* x == 0 ? 1 : 0                          */
} nbg_unop_code;

typedef struct { int code; double c0; double c1; } nbg_unop;

typedef enum {
    NBG_PLUS = 0, NBG_MINUS = 1, NBG_TIMES = 2, NBG_DIV = 3, /* integer DIV: x/0 := 0 */
    NBG_MIN = 4, NBG_MAX = 5,        /* IEEE minNum/maxNum (a NaN operand yields the other) */
    NBG_FIRST = 6, NBG_SECOND = 7,   /* (x, y) -> x ; (x, y) -> y  (Fig. 6 mul "(_, x) -> x") */
    NBG_ABSDIFF = 8,                 /* |x - y|       (Fig. 6)                      */
    NBG_MAX_DIVX_C = 9               /* max(x / c0, y) (Fig. 6, c0 = damping)       */
} nbg_binop_code;

typedef struct { int code; double c0; } nbg_binop;

/* User-defined operators (the paper splices the user's function into the
 * generated loop, Fig. 2, specialising on "the concrete operations").
 * `expr` is a CUDA C++ expression over the operand `x` (binary: `x` and `y`) and the descriptor's
 * constants `c0`, `c1` (binary: `c0`); the prelude's helpers nbg_abs / nbg_min / nbg_max / nbg_div
 * and CUDA math functions may be used.  Like the built-in operators it is evaluated in the
 * operation's compute type (inputs and constants converted first; bool outputs store x != 0),
 * IEEE round to nearest, no FMA contraction.  The expression is compiled by NVRTC (no GPU needed)
 * for float, double, int and long long at definition time: NBG_INVALID_VALUE if it does not compile
 * or contains ';' / unbalanced brackets (the log goes to stderr).  *code (>= NBG_USER_OP_BASE) is
 * valid for the whole process in nbg_unop / nbg_binop descriptors of every context: apply, bind2nd,
 * ewise_mult, ewise_add, and as the multiply of a semiring (nbg_mxv); not in nbg_scalar_apply
 * (scalar ops are host-evaluated: NBG_NOT_IMPLEMENTED).  Operations over iso operands are not
 * folded on the host for user operators (they run in the generated kernel).  The expression text
 * is part of every generated kernel's source, hence of the persistent cubin cache key
 * (NBG_JIT_CACHE). */
enum { NBG_USER_OP_BASE = 1000 };
nbg_status nbg_unop_define(const char *name, const char *expr, int *code);
nbg_status nbg_binop_define(const char *name, const char *expr, int *code);

/* Monoids (add of a semiring, reduce): NBG_PLUS (identity 0), NBG_MIN (+inf / INT_MAX),
 * NBG_MAX (-inf / INT_MIN).  Floating PLUS folds accumulate in fp64. */
typedef struct {
    int add;        /* monoid: NBG_PLUS | NBG_MIN | NBG_MAX               (Fig. 3 `add`, `identity`) */
    int mul;        /* any nbg_binop_code (Fig. 3 `mul`; x = A(i,j), y = u(j)) */
    double mul_c0;  /* constant of `mul` when it takes one */
} nbg_semiring;

/* ---------------------------------------------------------------- context */

/* Create a context on cfg->device.  Errors: NBG_NULL_POINTER, NBG_INVALID_VALUE (mode),
 * NBG_PANIC (no CUDA device / driver error). */
nbg_status nbg_init(nbg_ctx **ctx, const nbg_config *cfg);

/* Destroy the context and every object still owned by it (outstanding handles become invalid). */
nbg_status nbg_finalize(nbg_ctx *ctx);

/* Copy the last latched error message (NUL-terminated, truncated to len) into buf. */
nbg_status nbg_last_error(nbg_ctx *ctx, char *buf, size_t len);

/* Block until all work of the context has finished (its stream and the scalar-readback side
 * stream); returns a latched execution error if one occurred.  With NBG_GUARD=1 in the
 * environment it also checks the red zones of all live buffers (see nbg_guard_selftest). */
nbg_status nbg_sync(nbg_ctx *ctx);

/* Guard mode (test instrument; compute-sanitizer is unavailable on the GPU pool): with NBG_GUARD=1
 * every pool buffer carries a 256-byte red zone after its end, checked on the device after every
 * generated-kernel launch, at the end of every wait and when the buffer is freed; an overwritten
 * zone fails the call with NBG_PANIC ("guard: ...").  This entry point writes one byte past the end
 * of a fresh 1000-byte buffer and runs the check: NBG_PANIC when guard mode is on and detects it,
 * NBG_NOT_IMPLEMENTED when NBG_GUARD is not set. */
nbg_status nbg_guard_selftest(nbg_ctx *ctx);

/* Planner / executor counters (SPEC.md:338-341 cache counters; PAPER.md:301-306 wait steps). */
typedef struct {
    uint64_t waits;                 /* regions materialised                                   */
    uint64_t plans_built;           /* plan-cache misses (signature seen for the first time)  */
    uint64_t plan_hits;             /* plan-cache hits (step 3 skipped)          */
    uint64_t jit_compiles;          /* NVRTC compilations                       */
    uint64_t kernels_launched;      /* kernels this library launched                          */
    uint64_t vectors_materialized;  /* vector buffers written by kernels                      */
    uint64_t intermediates_elided;  /* pending nodes computed in registers, never stored      */
    uint64_t memo_hits;             /* pending nodes bound to an already computed result      */
    uint64_t side_outputs;          /* speculative loop-carried outputs emitted               */
    uint64_t bytes_materialized;    /* bytes of vector buffers written by kernels             */
    uint64_t host_plan_ns;          /* host time spent planning (signature..launch)           */
    double jit_ms;                  /* host time spent in NVRTC                               */
    uint64_t structured_regions;    /* regions over sparse / bitset vectors (NEXT-3)          */
    uint64_t structured_index_loops;/* ... of those, run over a sparse index list (estimator)  */
    uint64_t jit_disk_hits;         /* kernels loaded from the persistent cubin cache (NBG_JIT_CACHE) */
} nbg_stats;

nbg_status nbg_get_stats(nbg_ctx *ctx, nbg_stats *out);
nbg_status nbg_reset_stats(nbg_ctx *ctx);

/* Per-kernel-class device timing with CUDA events recorded on the context stream around every
 * launch of that class (used by bench.py for the roofline).  Classes: "spmv" (any kernel with
 * an mxv, fused or not), "ewise" (elementwise/reduce regions), "graph" (generation/CSR build).
 * nbg_get_timing synchronises and returns the summed device milliseconds and launch count
 * since the last nbg_set_timing(ctx, 1). */
nbg_status nbg_set_timing(nbg_ctx *ctx, int enable);
nbg_status nbg_get_timing(nbg_ctx *ctx, const char *kernel_class, double *total_ms, int64_t *launches);

/* ---------------------------------------------------------------- matrices (CSR)
 * A matrix is CSR with int64 row pointers and int32 column indices, columns strictly
 * ascending within a row.  vals == NULL makes it iso-valued (every stored
 * entry equals `iso`, PAPER.md:227 iso facet); otherwise vals has nnz entries of `type`. */
nbg_status nbg_matrix_from_csr(nbg_ctx *ctx, nbg_matrix *A, int64_t nrows, int64_t ncols, int64_t nnz,
                               const int64_t *rowptr, const int32_t *colidx, const void *vals,
                               int type, double iso, int space, int ownership);

/* Build AT (edge u->v stored at AT[v,u], PAPER.md:266 `AT`) and the INT32 out-degree vector
 * (`out_degree`) from an edge list of m edges (src[e] -> dst[e], ids in [0,n)).
 * Self-loops are dropped and duplicate edges removed (BASELINE configs).  Runs on the GPU
 * (radix sort by (dst, src), unique, histograms).  deg may be NULL.
 * Errors: NBG_INDEX_OUT_OF_BOUNDS if an id is outside [0, n). */
nbg_status nbg_matrix_from_edges(nbg_ctx *ctx, nbg_matrix *AT, nbg_vector *deg, int64_t n, int64_t m,
                                 const int32_t *src, const int32_t *dst, int space);

/* Matrix Market ingestion (the paper's experiment reads GAP-web.mtx).
 * `path` names a coordinate-format file ("%%MatrixMarket matrix coordinate <field> <symmetry>",
 * field pattern | real | integer, symmetry general | symmetric; '%' comment lines; a size line
 * "M N NNZ"; NNZ lines "i j [value]" with 1-based indices).  Entry (i, j) is the edge i -> j
 * (row = source, GAP/LAGraph convention); a symmetric file contributes both directions; values are
 * ignored (the PageRank matrix is a pattern).  The graph has n = max(M, N)
 * vertices and goes through nbg_matrix_from_edges (self-loops dropped, duplicates removed).
 * Errors: NBG_INVALID_VALUE for an unreadable file or a malformed / unsupported header or line
 * (array format, complex or hermitian fields), NBG_INDEX_OUT_OF_BOUNDS for an index outside
 * [1, M] x [1, N]. */
nbg_status nbg_matrix_from_mtx(nbg_ctx *ctx, nbg_matrix *AT, nbg_vector *deg, const char *path);

/* Synthetic graphs (input recipe of DESIGN.md; BASELINE configs 1,3,4,5).
 * kind NBG_GRAPH_RMAT: n = 2^scale, m = edge_factor * n, (a,b,c,d) = (0.57,0.19,0.19,0.05),
 *   edge e level l draws u = SplitMix64(seed, e*64 + l) >> 11 (reading Q9).
 * kind NBG_GRAPH_ER: n = 2^scale, m = edge_factor * n, src/dst = top scale bits of
 *   SplitMix64(seed, 2e) / SplitMix64(seed, 2e+1) (reading Q11). */
typedef enum { NBG_GRAPH_RMAT = 0, NBG_GRAPH_ER = 1 } nbg_graph_kind;
typedef struct { int kind; int scale; int edge_factor; uint64_t seed; } nbg_graphgen;

/* Write the m generated edges into src/dst (int32[m] each, in `space`). */
nbg_status nbg_graph_edges(nbg_ctx *ctx, const nbg_graphgen *g, int32_t *src, int32_t *dst, int space);

/* Generate on the device and build AT + out-degree (= nbg_graph_edges + nbg_matrix_from_edges
 * without a host round trip). */
nbg_status nbg_matrix_from_generator(nbg_ctx *ctx, nbg_matrix *AT, nbg_vector *deg, const nbg_graphgen *g);

nbg_status nbg_matrix_nrows(nbg_ctx *ctx, nbg_matrix A, int64_t *out);
nbg_status nbg_matrix_ncols(nbg_ctx *ctx, nbg_matrix A, int64_t *out);
nbg_status nbg_matrix_nnz(nbg_ctx *ctx, nbg_matrix A, int64_t *out);

/* Copy the structure out (rowptr: nrows+1 int64, colidx: nnz int32) into `space`.  Synchronises. */
nbg_status nbg_matrix_export_csr(nbg_ctx *ctx, nbg_matrix A, int64_t *rowptr, int32_t *colidx, int space);
nbg_status nbg_matrix_free(nbg_ctx *ctx, nbg_matrix A);

/* ---------------------------------------------------------------- vectors
 * Representations in this subset: FULL (dense values), ISO full (one value, "iso
 * value only once"), EMPTY (no stored entries).  Sparse/bitset vectors are
 * outside the hot path and return NBG_NOT_IMPLEMENTED. */

/* Empty vector of length n (Fig. 6 line 276 `GrBVector{Float32}(n)`). */
nbg_status nbg_vector_new(nbg_ctx *ctx, nbg_vector *v, int type, int64_t n);

/* Iso full vector, every entry = (type)value (Fig. 6 line 277 `GrBVector(n, 1/n)`). */
nbg_status nbg_vector_new_const(nbg_ctx *ctx, nbg_vector *v, int type, int64_t n, double value);

/* Full vector from n dense values of `type` in `space` (NBG_BORROW: device pointer kept). */
nbg_status nbg_vector_from_dense(nbg_ctx *ctx, nbg_vector *v, int type, int64_t n, const void *data,
                                 int space, int ownership);

/* Materialise v (forces wait) and copy its n values (of v's type) to out in `space`.
 * Errors: NBG_INVALID_OBJECT if v is empty, sparse or bitset (not every entry present; use
 * nbg_vector_export_sparse).  Synchronises. */
nbg_status nbg_vector_export_dense(nbg_ctx *ctx, nbg_vector v, void *out, int space);

nbg_status nbg_vector_size(nbg_ctx *ctx, nbg_vector v, int64_t *n);
nbg_status nbg_vector_type(nbg_ctx *ctx, nbg_vector v, int *type);
/* Number of stored (present) entries.  Full / iso / empty vectors and operations over them know
 * it at record time (n or 0); a vector over sparse or bitset operands is materialised first. */
nbg_status nbg_vector_nvals(nbg_ctx *ctx, nbg_vector v, int64_t *nvals);
/* 1 if v is currently materialised (FULL buffer, ISO or EMPTY), 0 if it is a pending node. */
nbg_status nbg_vector_is_materialized(nbg_ctx *ctx, nbg_vector v, int *out);
/* Materialise v and return the device address of its dense values (FULL vectors; an ISO vector
 * is expanded once).  The pointer stays valid while v (or a handle to the same node) lives;
 * the caller must not write through it (handles are immutable).  Used for zero-copy interop
 * (e.g. torch) and to build row-block views for the multi-GPU driver. */
nbg_status nbg_vector_device_ptr(nbg_ctx *ctx, nbg_vector v, void **ptr);
nbg_status nbg_vector_free(nbg_ctx *ctx, nbg_vector v);

/* ---------------------------------------------------------------- sparse and bitset vectors
 * (PAPER.md:185 SparseVector / BitSetVector / FullVector, PAPER.md:234-246
 * estimated fill ratios; GraphBLAS structure semantics: apply / bind2nd keep the operand's
 * structure, ewise_mult = intersection, ewise_add = union with the present operand's value where
 * only one is present, reduce = monoid over the present entries (identity if none), mxv = dense
 * output (SPEC.md:206 reading) summing the stored entries whose x entry is present.)
 * Representations: */
enum { NBG_FORMAT_FULL = 0, NBG_FORMAT_ISO = 1, NBG_FORMAT_SPARSE = 2, NBG_FORMAT_BITSET = 3, NBG_FORMAT_EMPTY = 4 };

/* Sparse vector of length n with nvals entries: indices (int32, strictly ascending, in [0, n))
 * and values (nvals of `type`), both in `space`; copied.  Errors: NBG_INVALID_VALUE (bad sizes or
 * indices not strictly ascending), NBG_INDEX_OUT_OF_BOUNDS (index outside [0, n)), NBG_NULL_POINTER. */
nbg_status nbg_vector_from_sparse(nbg_ctx *ctx, nbg_vector *v, int type, int64_t n, int64_t nvals,
                                  const int32_t *indices, const void *values, int space);

/* Materialise v (forces wait) and export its present entries in ascending index order.  Call with
 * indices == values == NULL to read *nvals only; otherwise both arrays must hold *nvals entries
 * (the count from the first call) in `space`.  Works for every representation (a full vector
 * exports all n entries, an empty one none).  Synchronises. */
nbg_status nbg_vector_export_sparse(nbg_ctx *ctx, nbg_vector v, int64_t *nvals, int32_t *indices, void *values,
                                    int space);

/* Materialise v and return its representation (NBG_FORMAT_*): chosen by the library from the
 * estimated fill of the result (sparse below 1/8, bitset above, full when every
 * entry is present). */
nbg_status nbg_vector_format(nbg_ctx *ctx, nbg_vector v, int *format);

/* The naive metadata estimate of v's fill ratio (present entries / n) without materialising it
 * (PAPER.md:236-240): materialised = nvals / n; apply, bind2nd = operand; ewise_mult = product;
 * ewise_add = f_u + f_v - f_u f_v; mxv = 1.  Used only to choose loops and representations. */
nbg_status nbg_vector_estimated_fill(nbg_ctx *ctx, nbg_vector v, double *fill);

/* ---------------------------------------------------------------- scalars */

/* Materialised scalar (Fig. 6 line 275 `GrBScalar(1.0f0)`). */
nbg_status nbg_scalar_new(nbg_ctx *ctx, nbg_scalar *s, int type, double value);
/* Force materialisation and read the value as double (Fig. 6 `rdiff()`).
 * Synchronises only on the event of the kernel that produced s. */
nbg_status nbg_scalar_get(nbg_ctx *ctx, nbg_scalar s, double *value);
nbg_status nbg_scalar_free(nbg_ctx *ctx, nbg_scalar s);

/* ---------------------------------------------------------------- operations
 * Each returns a new handle of output type `type` and the operand length; operands must be
 * of equal length (NBG_DIMENSION_MISMATCH).  Full/iso operands: ewise_mult and ewise_add both
 * apply op everywhere; with an EMPTY operand ewise_mult is empty (intersection)
 * and ewise_add yields the other operand converted to `type` (union). */
nbg_status nbg_apply(nbg_ctx *ctx, nbg_vector *w, int type, nbg_unop op, nbg_vector u);           /* Fig. 4 VectorApply */
nbg_status nbg_apply_bind2nd(nbg_ctx *ctx, nbg_vector *w, int type, nbg_binop op, nbg_vector u,
                             nbg_scalar s);                                                       /* w = op(u, s) */
nbg_status nbg_ewise_mult(nbg_ctx *ctx, nbg_vector *w, int type, nbg_binop op, nbg_vector u, nbg_vector v);  /* Fig. 1 */
nbg_status nbg_ewise_add(nbg_ctx *ctx, nbg_vector *w, int type, nbg_binop op, nbg_vector u, nbg_vector v);   /* Fig. 6 l.288 */
nbg_status nbg_convert(nbg_ctx *ctx, nbg_vector *w, int type, nbg_vector u);                      /* Fig. 6 `conv` */

/* w(i) = add-fold over stored A(i,j) of mul(A(i,j), u(j)), identity for an empty row (dense
 * output); A.ncols must equal len(u) (Fig. 3, Fig. 6). */
nbg_status nbg_mxv(nbg_ctx *ctx, nbg_vector *w, int type, nbg_semiring sr, nbg_matrix A, nbg_vector u);

/* s = add-fold of u's stored values (identity if empty) (Fig. 6).  Floating PLUS:
 *   - fp64 terms (a reduction of an fp64 vector, or over fp64 values of a fused region): every
 *     term is added EXACTLY (per-thread 128-bit fixed-point accumulators flushed into the block's
 *     limbs, limbs combined across blocks by integer atomics), so s is the exact sum of the terms
 *     rounded once to fp64 -- independent of grouping, block count and rank count (P9);
 *   - fp32 terms (and the per-row / per-task partials of a fused SpMV epilogue) are accumulated in
 *     fp64 in a fixed order per thread / task, and those fp64 partials are combined exactly.
 * Terms outside the exact window [2^-160, 2^128) are summed in fp64 on the side (slot word 12),
 * in arrival order -- the one non-deterministic case (see NBG_FLAG_DETERMINISTIC); NaN / +inf /
 * -inf terms are counted and decide the result (NaN, or inf of one sign). */
nbg_status nbg_reduce(nbg_ctx *ctx, nbg_scalar *s, int type, int monoid, nbg_vector u);

/* s_out = op(s_in) evaluated in `type` (a scalar node of the DAG, e.g. the dangling constant). */
nbg_status nbg_scalar_apply(nbg_ctx *ctx, nbg_scalar *s_out, int type, nbg_unop op, nbg_scalar s_in);

/* ---------------------------------------------------------------- wait
 * Materialise v (and every live pending node it depends on) -- the `wait` of PAPER.md:66,136
 * and Fig. 6: signature -> plan cache -> (NVRTC compile on a miss) -> launch
 * (PAPER.md:301-306).  Idempotent.  Returns after LAUNCHING (device work may be in flight);
 * exports and nbg_scalar_get synchronise. */
nbg_status nbg_vector_wait(nbg_ctx *ctx, nbg_vector v);
nbg_status nbg_scalar_wait(nbg_ctx *ctx, nbg_scalar s);

/* Materialise every pending vector and reduction the caller still holds a handle to, in one
 * planning pass (the GraphBLAS `GrB_wait()` without an object): nodes that no handle
 * reaches stay elided.  Pending scalar_apply nodes are evaluated where they are read (host
 * arithmetic on a materialised scalar), as with nbg_scalar_wait.  Idempotent; returns after
 * launching; execution errors as for nbg_vector_wait. */
nbg_status nbg_wait_all(nbg_ctx *ctx);

/* ---------------------------------------------------------------- PageRank (Fig. 6)
 * Written purely on the operations above.  AT: n x n pattern CSR (edge
 * u->v at AT[v,u]); deg: out-degrees (any numeric type).  dangling NBG_PR_UNIFORM adds the
 * dangling mass alpha*ds/n to every rank (Google matrix, ranks sum to 1; BASELINE config 4);
 * NBG_PR_DROP is Fig. 6 literally (no redistribution).  tol < 0 runs exactly itermax sweeps.
 * On return *r is the rank vector (caller frees), *sweeps the number of SpMV sweeps
 * (Fig. 6's iter = sweeps + 1), delta_hist (may be NULL, >= itermax doubles) the L1 deltas. */
typedef enum { NBG_PR_UNIFORM = 0, NBG_PR_DROP = 1 } nbg_pr_dangling;
typedef struct { double alpha; double tol; int itermax; int dangling; int type; } nbg_pr_params;

nbg_status nbg_pagerank(nbg_ctx *ctx, nbg_matrix AT, nbg_vector deg, const nbg_pr_params *p,
                        nbg_vector *r, int *sweeps, double *delta_hist);

/* ---------------------------------------------------------------- multi-GPU (1-D row partition)
 * One process per GPU; torch.distributed only broadcasts the 128-byte NCCL unique id.
 * nbg_partition_rows is host-only (no GPU): cut points cuts[0..nparts] (cuts[0]=0,
 * cuts[nparts]=n) of a contiguous row partition balanced by per-row bytes
 * 4*len(i) + 8 + bytes_per_row. */
nbg_status nbg_partition_rows(const int64_t *rowptr, int64_t n, int nparts, int64_t bytes_per_row,
                              int64_t *cuts);
nbg_status nbg_dist_unique_id(void *id128);
nbg_status nbg_dist_init(nbg_ctx *ctx, int rank, int nranks, const void *id128);

/* Rows [lo, hi) of A as a new matrix with all of A's columns (row pointers rebased to 0).
 * Used to hand each rank its block of the 1-D row partition. */
nbg_status nbg_matrix_row_block(nbg_ctx *ctx, nbg_matrix *B, nbg_matrix A, int64_t lo, int64_t hi);

/* Collective operations (require nbg_dist_init; they are fusion barriers: the input is
 * materialised, then the collective is enqueued on the context stream).
 * allgather: every rank passes its block u_blk (length cuts[rank+1]-cuts[rank]); w is the
 *   full vector of length cuts[nranks] on every rank (allgather-v as grouped ncclBroadcast).
 * allreduce: s_out = the sum (PLUS reductions, combined EXACTLY on the fixed-point limbs, so
 *   the result is independent of the rank order) or min/max of s over all ranks. */
nbg_status nbg_vector_allgather(nbg_ctx *ctx, nbg_vector *w, nbg_vector u_blk, const int64_t *cuts);
nbg_status nbg_scalar_allreduce(nbg_ctx *ctx, nbg_scalar *s_out, nbg_scalar s);

/* ---- round-2 data plane
 * Exact-accumulator slot format (the value of every floating PLUS reduction): 16 uint64 words;
 * words 0-9 are limbs of signed 32-bit pieces (LSB weight 2^-160), word 10 counts non-finite terms
 * (NaN: bits 0-20, +inf: 21-41, -inf: 42-62), word 12 is the fp64 sum of terms outside the exact
 * window [2^-160, 2^128).  Slots of several ranks combine by an integer sum of words 0-10 and an
 * fp64 sum of word 12 (what nbg_vector_allgather_reduce does over NCCL); the value is the exact sum
 * of all terms rounded once to fp64 (window terms), so it does not depend on the rank order. */

/* Host only (no GPU): encode n terms into a zeroed slot / decode a slot to its value. */
nbg_status nbg_xacc_encode(const double *terms, int64_t n, uint64_t *slot16);
nbg_status nbg_xacc_decode(const uint64_t *slot16, double *value);

/* Materialise the floating PLUS reduction s and copy its raw 16-word slot to host memory
 * (synchronises).  NBG_INVALID_OBJECT if s is not a device exact-accumulator scalar. */
nbg_status nbg_scalar_export_slot(nbg_ctx *ctx, nbg_scalar s, uint64_t *slot16);

/* Test transport: make the contexts ctxs[0..nranks) ranks 0..nranks-1 of one group whose
 * collectives run inside this process (the ranks must be driven by nranks host threads, one per
 * context, calling the same sequence of collective operations).  A collective synchronises the
 * caller's stream, meets the other ranks at a host barrier and reads their buffers with the
 * caller's own copies / sum kernels (all contexts on one device), so every N > 1 code path runs
 * on one GPU without any kernel waiting on another rank.  NCCL-based runs use nbg_dist_init. */
nbg_status nbg_dist_init_loopback(nbg_ctx **ctxs, int nranks);

/* Host only: the exchange schedule of the 1-D row partition in the gather layout.  Rank q owns
 * rows [cuts[q], cuts[q+1]) of the relabelled AT; its scaled ranks occupy positions
 * offsets[q] .. offsets[q]+counts[q] of the gathered vector (length ncols_g), i.e. the slice of its
 * rows clipped at ncols_g (rows >= ncols_g are dangling vertices: never gathered). */
nbg_status nbg_dist_exchange_plan(const int64_t *cuts, int nranks, int64_t ncols_g, int64_t *offsets, int64_t *counts);

/* Per-rank graph setup without building the whole graph on any rank (needs nbg_dist_init for
 * nranks > 1; a context without it is rank 0 of 1).  Every rank regenerates the m edges of `g`
 * (counter-based, nbg_graph_edges), deduplicates those whose destination lies in its share of the
 * original ids to obtain exact out/in-degree contributions, sums them over the ranks (NCCL), and
 * derives the same symmetric relabel pi on every rank: vertices by descending out-degree, ties by
 * id, dangling vertices last (the single-GPU gather layout).  Rows are cut in pi-space balanced by
 * bytes (4*len + 8 + bytes_per_row per row, as nbg_partition_rows).  Out: AT_blk = rows
 * pi in [cuts[rank], cuts[rank+1]) with pi column ids (ncols = ncols_g = number of non-dangling
 * vertices; every row keeps its original ascending-source entry order, so row sums are the
 * single-GPU ones); deg_blk = INT32 out-degrees of those rows' vertices; cuts (nranks + 1 entries);
 * ncols_g.  Errors: NBG_INVALID_VALUE (generator parameters), NBG_NOT_IMPLEMENTED (> 64 ranks). */
nbg_status nbg_dist_graph_from_generator(nbg_ctx *ctx, const nbg_graphgen *g, int64_t bytes_per_row, nbg_matrix *AT_blk,
                                         nbg_vector *deg_blk, int64_t *cuts, int64_t *ncols_g);

/* The per-sweep exchange in one call: u_blk (this rank's block, length cuts[rank+1]-cuts[rank]) is
 * materialised -- together with the pending reductions s_in[0..nscal) and every pending node the
 * caller holds, in ONE fused kernel -- with its values written straight into positions
 * cuts[rank] + i (< ncols_g) of a new full vector w of length ncols_g; then ONE NCCL group
 * broadcasts every rank's slice in place (peer mode: the kernel already stored it on every rank,
 * see nbg_dist_set_exchange) and sums the scalars' exact slots (s_out[i] = global sum
 * of s_in[i], float PLUS reductions).  u_blk itself stays pending (its values live only inside w).
 * With one rank no collective runs.  Errors: NBG_DIMENSION_MISMATCH (u_blk length),
 * NBG_NOT_IMPLEMENTED (sparse/bitset u_blk, non-PLUS scalars across ranks), NBG_INVALID_VALUE. */
nbg_status nbg_vector_allgather_reduce(nbg_ctx *ctx, nbg_vector *w, nbg_vector u_blk, const int64_t *cuts, int64_t ncols_g,
                                       int nscal, const nbg_scalar *s_in, nbg_scalar *s_out);

/* Exchange mode of nbg_vector_allgather_reduce (per context; every rank of a group must set the
 * same mode before its first exchange):
 *   NBG_DIST_EXCHANGE_COLLECTIVE (default): the producing kernel writes this rank's slice of w,
 *     then one NCCL group broadcasts the slices (loopback: device copies) and sums the slots.
 *   NBG_DIST_EXCHANGE_PEER: the exchange is fused into the producing kernel -- every element it
 *     computes is stored straight into ALL ranks' w buffers (peer stores over NVLink/NVSwitch:
 *     buffers mapped with CUDA IPC handles exchanged once per (ncols_g, type) through NCCL;
 *     loopback: plain pointers), so the data movement overlaps the SpMV row by row and only the
 *     scalar sums (plus, with no scalars, a one-word barrier) remain as a collective.  w lives in
 *     one of two exchange buffers per rank used alternately: it is valid until the exchange after
 *     next of the same (ncols_g, type) overwrites it (nbg_pagerank_dist frees each gathered vector
 *     before that).  At most 8 ranks.
 * Errors: NBG_INVALID_VALUE (unknown mode, > 8 ranks for PEER, no nbg_dist_init / loopback). */
enum { NBG_DIST_EXCHANGE_COLLECTIVE = 0, NBG_DIST_EXCHANGE_PEER = 1 };
nbg_status nbg_dist_set_exchange(nbg_ctx *ctx, int mode);

/* Distributed PageRank on the output of nbg_dist_graph_from_generator: one fused kernel and one
 * exchange per sweep (nbg_vector_allgather_reduce, in the context's exchange mode).  r_blk
 * receives this rank's ranks in pi order (rows [cuts[rank], cuts[rank+1])); sweeps / delta_hist as
 * nbg_pagerank.  Every row sum keeps the row's original entry order, the delta and dangling mass
 * are exact sums over all ranks (identical on every rank); ranks agree with the single-GPU
 * nbg_pagerank of the same graph (permuted by pi) up to the fp64 grouping of long rows' partial
 * sums, which follows each block's SpMV task layout. */
nbg_status nbg_pagerank_dist(nbg_ctx *ctx, nbg_matrix AT_blk, nbg_vector deg_blk, const int64_t *cuts, int64_t ncols_g,
                             const nbg_pr_params *p, nbg_vector *r_blk, int *sweeps, double *delta_hist);

#ifdef __cplusplus
}
#endif
#endif /* NBG_H */
