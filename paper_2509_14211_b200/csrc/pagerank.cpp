// pagerank.cpp -- PAPER.md Fig. 6 (`pagerank_gap`, lines 266-294) written ONLY on the public C ABI,
// which shows the ABI suffices for the paper's algorithm.
//
// Per sweep (t = previous ranks; all handles are immutable, so `t = r` aliases):
//   mask  = apply(iszero, dinv)                       dangling vertices (dinv == 0 iff deg == 0)
//   ds    = reduce(+, ewise_mult(*, t, mask))         dangling mass of t      [UNIFORM only]
//   c     = (alpha/n) * ds + (1-alpha)/n               scalar node (Q1, Q3)     [DROP: c = (1-alpha)/n]
//   y     = ewise_mult(*, t, dinv)                    Fig. 6 l.286 `t / d` (reading Q2)
//   m     = mxv(+, second, AT, y)                     Fig. 6 l.287
//   r     = apply_bind2nd(+, m, c)                    Fig. 6 l.288 `ewise_add(+, rt, r)` + dangling
//   e     = ewise_add(|x-y|, t, r); delta = reduce(+, e)   Fig. 6 l.290-291
//   wait(delta)   -- r is live (the driver holds it), so ONE fused kernel materialises r and delta
//                    (Fig. 6 waits on r first; waiting on delta instead lets the planner fuse the
//                    residual into the same pass -- the placement SPEC.md:474 leaves open).
// Convergence (Fig. 6 l.284): sweep k+1 is recorded and launched BEFORE delta_k is read, so the
// device never idles on the host's read-back; if delta_k <= tol the speculative sweep is dropped
// (immutable handles keep r_k intact).  When the deltas' geometric decay predicts that sweep k is
// the last (within a margin set by how steady the decay ratio is), sweep k+1 is launched only
// after delta_k is read (no discarded sweep at the end).
// tol < 0 runs exactly itermax sweeps with no host sync.
#include <algorithm>
#include <cmath>
#include <vector>

#include "nbg_internal.hpp"

#define TRY(x)                                   \
    do {                                         \
        nbg_status s_ = (x);                     \
        if (s_ != NBG_SUCCESS) return s_;        \
    } while (0)

namespace {

struct PR {
    nbg_ctx *ctx;
    nbg_matrix AT;
    nbg_vector dinv;
    int T;
    bool uniform;
    double a_n, tele;

    // one sweep over t; returns the new ranks and the delta scalar (both launched)
    nbg_status sweep(nbg_vector t, nbg_vector *r_new, nbg_scalar *delta) {
        nbg_scalar c = nullptr;
        if (uniform) {
            nbg_vector mask, tm;
            nbg_scalar ds;
            TRY(nbg_apply(ctx, &mask, T, nbg_unop{NBG_ISZERO, 0, 0}, dinv));
            TRY(nbg_ewise_mult(ctx, &tm, T, nbg_binop{NBG_TIMES, 0}, t, mask));
            nbg_vector_free(ctx, mask);
            TRY(nbg_reduce(ctx, &ds, NBG_FP64, NBG_PLUS, tm));
            nbg_vector_free(ctx, tm);
            TRY(nbg_scalar_apply(ctx, &c, NBG_FP64, nbg_unop{NBG_AXPB, a_n, tele}, ds));
            nbg_scalar_free(ctx, ds);
        } else {
            TRY(nbg_scalar_new(ctx, &c, NBG_FP64, tele));
        }
        nbg_vector y, m, e;
        TRY(nbg_ewise_mult(ctx, &y, T, nbg_binop{NBG_TIMES, 0}, t, dinv));
        TRY(nbg_mxv(ctx, &m, T, nbg_semiring{NBG_PLUS, NBG_SECOND, 0.0}, AT, y));
        nbg_vector_free(ctx, y);
        TRY(nbg_apply_bind2nd(ctx, r_new, T, nbg_binop{NBG_PLUS, 0}, m, c));
        nbg_vector_free(ctx, m);
        nbg_scalar_free(ctx, c);
        TRY(nbg_ewise_add(ctx, &e, T, nbg_binop{NBG_ABSDIFF, 0}, t, *r_new));
        TRY(nbg_reduce(ctx, delta, NBG_FP64, NBG_PLUS, e));
        nbg_vector_free(ctx, e);
        TRY(nbg_scalar_wait(ctx, *delta));
        return NBG_SUCCESS;
    }
};

}  // namespace

extern "C" nbg_status nbg_pagerank(nbg_ctx *ctx, nbg_matrix AT, nbg_vector deg, const nbg_pr_params *p, nbg_vector *r_out,
                                   int *sweeps_out, double *delta_hist) {
    if (!ctx || !AT || !deg || !p || !r_out) return NBG_NULL_POINTER;
    if (!(p->alpha > 0.0 && p->alpha < 1.0) || p->itermax < 0) return NBG_INVALID_VALUE;
    if (p->type != NBG_FP32 && p->type != NBG_FP64) return NBG_DOMAIN_MISMATCH;
    if (p->dangling != NBG_PR_UNIFORM && p->dangling != NBG_PR_DROP) return NBG_INVALID_VALUE;
    int64_t n = 0, nc = 0, nd = 0;
    TRY(nbg_matrix_nrows(ctx, AT, &n));
    TRY(nbg_matrix_ncols(ctx, AT, &nc));
    TRY(nbg_vector_size(ctx, deg, &nd));
    if (n != nc || nd != n) return NBG_DIMENSION_MISMATCH;
    if (n == 0) return NBG_INVALID_VALUE;

    PR pr;
    pr.ctx = ctx;
    pr.AT = AT;
    pr.T = p->type;
    pr.uniform = p->dangling == NBG_PR_UNIFORM;
    pr.a_n = p->alpha / (double)n;
    pr.tele = (1.0 - p->alpha) / (double)n;

    // Fig. 6 l.278-281: d, then wait(d).  Reading Q2: dinv = (T)(alpha / deg) in double, 0 if deg == 0.
    nbg_vector d64;
    TRY(nbg_apply(ctx, &d64, NBG_FP64, nbg_unop{NBG_RECIP_SCALED, p->alpha, 0.0}, deg));
    TRY(nbg_convert(ctx, &pr.dinv, pr.T, d64));
    nbg_vector_free(ctx, d64);
    TRY(nbg_vector_wait(ctx, pr.dinv));

    nbg_vector t;   // Fig. 6 l.277: r = GrBVector(n, 1/n)
    TRY(nbg_vector_new_const(ctx, &t, pr.T, n, 1.0 / (double)n));
    if (p->itermax == 0) {
        *r_out = t;
        if (sweeps_out) *sweeps_out = 0;
        nbg_vector_free(ctx, pr.dinv);
        return NBG_SUCCESS;
    }
    const bool conv = p->tol >= 0.0;
    nbg_vector rk;
    nbg_scalar dk;
    TRY(pr.sweep(t, &rk, &dk));
    std::vector<nbg_scalar> deltas;   // fixed-count mode: read after the loop
    int k = 1;
    double dm1 = -1.0, dm2 = -1.0, dm3 = -1.0;   // delta_{k-1}, delta_{k-2}, delta_{k-3} (convergence mode)
    for (;;) {
        nbg_vector rnext = nullptr;
        nbg_scalar dnext = nullptr;
        const bool more = k < p->itermax;
        // speculate (launch sweep k+1 before delta_k is read) unless the geometric decay of the
        // deltas predicts that sweep k is the last one: then the host waits for delta_k instead
        // of paying a whole discarded sweep (results are identical either way).  Prediction
        // delta_k ~ delta_{k-1} q with q = delta_{k-1} / delta_{k-2}; the margin grows with the
        // disagreement of the last two ratios (a waited sweep costs the device ~ one host round
        // trip, a discarded one a whole sweep, so waiting pays once P(delta_k <= tol) > ~0.2)
        bool last_likely = false;
        if (conv && dm1 > 0.0 && dm2 > 0.0) {
            const double q1 = dm1 / dm2;
            const double spread = dm3 > 0.0 ? std::fabs(q1 - dm2 / dm3) / q1 : 1.0;
            last_likely = dm1 * q1 <= p->tol * (1.0 + std::min(1.0, 3.0 * spread));
        }
        const bool spec = more && !last_likely;
        if (spec) TRY(pr.sweep(rk, &rnext, &dnext));   // launched before delta_k is read
        bool stop = !more;
        if (conv) {
            double v = 0.0;
            TRY(nbg_scalar_get(ctx, dk, &v));
            if (delta_hist) delta_hist[k - 1] = v;
            nbg_scalar_free(ctx, dk);
            dk = nullptr;
            if (!(v > p->tol)) stop = true;
            dm3 = dm2;
            dm2 = dm1;
            dm1 = v;
            if (!stop && more && !spec) TRY(pr.sweep(rk, &rnext, &dnext));   // mispredicted: launch now
        } else {
            deltas.push_back(dk);
            dk = nullptr;
        }
        if (stop) {
            if (rnext) nbg_vector_free(ctx, rnext);
            if (dnext) nbg_scalar_free(ctx, dnext);
            break;
        }
        nbg_vector_free(ctx, t);
        t = rk;
        rk = rnext;
        dk = dnext;
        k++;
    }
    for (size_t j = 0; j < deltas.size(); j++) {
        double v = 0.0;
        TRY(nbg_scalar_get(ctx, deltas[j], &v));
        if (delta_hist) delta_hist[j] = v;
        nbg_scalar_free(ctx, deltas[j]);
    }
    if (dk) nbg_scalar_free(ctx, dk);
    nbg_vector_free(ctx, t);
    nbg_vector_free(ctx, pr.dinv);
    *r_out = rk;
    if (sweeps_out) *sweeps_out = k;
    return NBG_SUCCESS;
}

// ---------------------------------------------------------------- distributed
// Every rank holds its row block of the symmetrically relabelled AT (nbg_dist_graph_from_generator:
// rows and columns in the gather layout pi, so rank r's scaled ranks are the contiguous slice
// [cuts[r], cuts[r+1]) of the next gathered vector).  One sweep = ONE fused kernel (mxv + teleport /
// dangling epilogue + the delta and next dangling-mass reductions + the scaled ranks written straight
// into this rank's slice of the exchange buffer) and ONE NCCL group (the P slices broadcast in place,
// the two scalars' exact limbs summed): nbg_vector_allgather_reduce.  Row sums keep each row's
// original entry order, so the ranks are bit-identical for every P.
extern "C" nbg_status nbg_pagerank_dist(nbg_ctx *ctx, nbg_matrix AT_blk, nbg_vector deg_blk, const int64_t *cuts,
                                        int64_t ncols_g, const nbg_pr_params *p, nbg_vector *r_out, int *sweeps_out,
                                        double *delta_hist) {
    if (!ctx || !AT_blk || !deg_blk || !cuts || !p || !r_out) return NBG_NULL_POINTER;
    if (!(p->alpha > 0.0 && p->alpha < 1.0) || p->itermax < 1) return NBG_INVALID_VALUE;
    if (p->dangling != NBG_PR_UNIFORM && p->dangling != NBG_PR_DROP) return NBG_INVALID_VALUE;
    if (p->type != NBG_FP32 && p->type != NBG_FP64) return NBG_DOMAIN_MISMATCH;
    const int rank = ctx->dist ? ctx->dist->rank : 0, P = ctx->dist ? ctx->dist->nranks : 1;
    const int64_t n = cuts[P], nb = cuts[rank + 1] - cuts[rank];
    int64_t rows = 0, cols = 0, nd = 0;
    TRY(nbg_matrix_nrows(ctx, AT_blk, &rows));
    TRY(nbg_matrix_ncols(ctx, AT_blk, &cols));
    TRY(nbg_vector_size(ctx, deg_blk, &nd));
    if (rows != nb || cols != ncols_g || nd != nb || ncols_g > n) return NBG_DIMENSION_MISMATCH;
    const int T = p->type;
    const bool uniform = p->dangling == NBG_PR_UNIFORM;
    const double a_n = p->alpha / (double)n, tele = (1.0 - p->alpha) / (double)n;

    // Fig. 6 l.278-281 `d` (reading Q2: dinv = (T)(alpha / deg), 0 for dangling vertices)
    nbg_vector d64, dinv_blk;
    TRY(nbg_apply(ctx, &d64, NBG_FP64, nbg_unop{NBG_RECIP_SCALED, p->alpha, 0.0}, deg_blk));
    TRY(nbg_convert(ctx, &dinv_blk, T, d64));
    nbg_vector_free(ctx, d64);
    TRY(nbg_vector_wait(ctx, dinv_blk));

    // exchange of y = t * dinv (+ the local partials of the given scalars) -> full x on every rank
    auto exchange = [&](nbg_vector t, int ns, nbg_scalar *loc, nbg_vector *x, nbg_scalar *glob) -> nbg_status {
        nbg_vector u;
        TRY(nbg_ewise_mult(ctx, &u, T, nbg_binop{NBG_TIMES, 0}, t, dinv_blk));
        nbg_status st = nbg_vector_allgather_reduce(ctx, x, u, cuts, ncols_g, ns, loc, glob);
        nbg_vector_free(ctx, u);
        for (int i = 0; i < ns; i++) nbg_scalar_free(ctx, loc[i]);
        return st;
    };
    // the dangling mask is recorded afresh per sweep and released at once (as in nbg_pagerank): not
    // user-live at the wait, it is elided and fused as iszero(dinv[i]) on the dinv the epilogue loads
    // anyway -- a held mask would be materialised and read as a third n-vector every sweep
    auto dangling_mass = [&](nbg_vector r, nbg_scalar *s) -> nbg_status {
        nbg_vector mask, tm;
        TRY(nbg_apply(ctx, &mask, T, nbg_unop{NBG_ISZERO, 0, 0}, dinv_blk));
        nbg_status st = nbg_ewise_mult(ctx, &tm, T, nbg_binop{NBG_TIMES, 0}, r, mask);
        nbg_vector_free(ctx, mask);
        if (st != NBG_SUCCESS) return st;
        st = nbg_reduce(ctx, s, NBG_FP64, NBG_PLUS, tm);
        nbg_vector_free(ctx, tm);
        return st;
    };
    // one sweep: t, x (gathered y), ds (global dangling mass of t) -> r, x', delta, ds'
    auto sweep = [&](nbg_vector t, nbg_vector x, nbg_scalar ds, nbg_vector *r_new, nbg_vector *x_next, nbg_scalar *delta,
                     nbg_scalar *ds_next) -> nbg_status {
        nbg_scalar c;
        if (uniform) TRY(nbg_scalar_apply(ctx, &c, NBG_FP64, nbg_unop{NBG_AXPB, a_n, tele}, ds));
        else TRY(nbg_scalar_new(ctx, &c, NBG_FP64, tele));
        nbg_vector m, e;
        TRY(nbg_mxv(ctx, &m, T, nbg_semiring{NBG_PLUS, NBG_SECOND, 0.0}, AT_blk, x));
        TRY(nbg_apply_bind2nd(ctx, r_new, T, nbg_binop{NBG_PLUS, 0}, m, c));
        nbg_vector_free(ctx, m);
        nbg_scalar_free(ctx, c);
        nbg_scalar loc[2];
        TRY(nbg_ewise_add(ctx, &e, T, nbg_binop{NBG_ABSDIFF, 0}, t, *r_new));
        TRY(nbg_reduce(ctx, &loc[0], NBG_FP64, NBG_PLUS, e));
        nbg_vector_free(ctx, e);
        if (uniform) TRY(dangling_mass(*r_new, &loc[1]));
        nbg_scalar glob[2] = {nullptr, nullptr};
        TRY(exchange(*r_new, uniform ? 2 : 1, loc, x_next, glob));
        *delta = glob[0];
        *ds_next = glob[1];
        return NBG_SUCCESS;
    };

    nbg_vector t, x;
    nbg_scalar ds = nullptr;
    TRY(nbg_vector_new_const(ctx, &t, T, nb, 1.0 / (double)n));      // Fig. 6 l.277
    {
        nbg_scalar loc[1];
        if (uniform) TRY(dangling_mass(t, &loc[0]));
        TRY(exchange(t, uniform ? 1 : 0, loc, &x, &ds));
    }
    const bool conv = p->tol >= 0.0;
    nbg_vector rk, xk;
    nbg_scalar dk, dsk;
    TRY(sweep(t, x, ds, &rk, &xk, &dk, &dsk));
    nbg_vector_free(ctx, x);
    if (ds) nbg_scalar_free(ctx, ds);
    std::vector<nbg_scalar> deltas;
    int k = 1;
    double dm1 = -1.0, dm2 = -1.0, dm3 = -1.0;   // delta_{k-1}, delta_{k-2}, delta_{k-3} (convergence mode)
    for (;;) {
        nbg_vector rnext = nullptr, xnext = nullptr;
        nbg_scalar dnext = nullptr, dsnext = nullptr;
        const bool more = k < p->itermax;
        // the same convergence prediction as nbg_pagerank (every rank sees the same exact deltas, so
        // every rank takes the same decision): wait for delta_k instead of speculating when the
        // geometric decay predicts that sweep k is the last one
        bool last_likely = false;
        if (conv && dm1 > 0.0 && dm2 > 0.0) {
            const double q1 = dm1 / dm2;
            const double spread = dm3 > 0.0 ? std::fabs(q1 - dm2 / dm3) / q1 : 1.0;
            last_likely = dm1 * q1 <= p->tol * (1.0 + std::min(1.0, 3.0 * spread));
        }
        const bool spec = more && !last_likely;
        if (spec) TRY(sweep(rk, xk, dsk, &rnext, &xnext, &dnext, &dsnext));   // launched before delta_k is read
        bool stop = !more;
        if (conv) {
            double v = 0.0;
            TRY(nbg_scalar_get(ctx, dk, &v));
            if (delta_hist) delta_hist[k - 1] = v;
            nbg_scalar_free(ctx, dk);
            dk = nullptr;
            if (!(v > p->tol)) stop = true;   // identical on every rank: the sum is exact
            dm3 = dm2;
            dm2 = dm1;
            dm1 = v;
            if (!stop && more && !spec) TRY(sweep(rk, xk, dsk, &rnext, &xnext, &dnext, &dsnext));   // mispredicted: launch now
        } else {
            deltas.push_back(dk);
            dk = nullptr;
        }
        nbg_vector_free(ctx, xk);
        if (dsk) nbg_scalar_free(ctx, dsk);
        if (stop) {
            if (rnext) nbg_vector_free(ctx, rnext);
            if (xnext) nbg_vector_free(ctx, xnext);
            if (dnext) nbg_scalar_free(ctx, dnext);
            if (dsnext) nbg_scalar_free(ctx, dsnext);
            break;
        }
        nbg_vector_free(ctx, t);
        t = rk;
        rk = rnext;
        xk = xnext;
        dk = dnext;
        dsk = dsnext;
        k++;
    }
    for (size_t j = 0; j < deltas.size(); j++) {
        double v = 0.0;
        TRY(nbg_scalar_get(ctx, deltas[j], &v));
        if (delta_hist) delta_hist[j] = v;
        nbg_scalar_free(ctx, deltas[j]);
    }
    nbg_vector_free(ctx, t);
    nbg_vector_free(ctx, dinv_blk);
    *r_out = rk;
    if (sweeps_out) *sweeps_out = k;
    return NBG_SUCCESS;
}
