// structured.cpp -- sparse and bitset vectors at wait.
//
// materialised vectors are SparseVector, BitSetVector or FullVector.  A region whose
// elementwise DAG reads a sparse or bitset leaf is materialised here (the full/iso regions keep
// the planner's fused kernels): ONE generated kernel evaluates every op of the region with a
// presence bit per value (codegen_structured), on a loop chosen by the naive metadata estimators
// of PAPER.md:234-246:
//   * estimated fill of a node (fraction of present entries): materialised = nvals / n, apply /
//     bind2nd = operand, ewise_mult = product, ewise_add = f_u + f_v - f_u f_v, mxv = 1;
//   * "element-wise multiplications: which of the two input containers drives the loop" -- the
//     driver of an intersection is the operand cover with the fewest estimated entries;
//   * "element-wise additions: an outer loop over the full dimension when the result is expected
//     to be (almost) dense, else over the indices of the inputs" -- a union is driven by the merged
//     index lists of its sparse operands;
//   * "the representation of the result (sparse, bitset or full)" -- full when presence is
//     structurally complete (or every entry turned out present), sparse below the fill threshold,
//     bitset above it.
// The estimators only select the loop and the representation; values never depend on them.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <sstream>
#include <unordered_map>
#include <unordered_set>

#include "nbg_internal.hpp"

namespace nbg {

static constexpr double SPARSE_FILL = 1.0 / 16.0;  // estimated fill at or below: sparse representation, else bitset
static constexpr double INDEX_FILL = 1.0 / 16.0;    // driver entries / n at or below: loop over the driver's indices (measured crossover, bench.py --workload sparse)

bool structured_kind(VKind k) { return k == VKind::SPARSE || k == VKind::BITSET; }

static bool reaches_structured(const Node *x, std::unordered_set<const Node *> &seen) {
    if (!seen.insert(x).second) return false;
    // an EMPTY leaf here is a pending structured result that materialised with no entries
    if (x->mat) return !x->scalar && (structured_kind(x->kind) || x->kind == VKind::EMPTY);
    switch (x->op) {
        case Op::APPLY:
        case Op::BIND2ND: return reaches_structured(x->a.get(), seen);
        case Op::EMULT:
        case Op::EADD: return reaches_structured(x->a.get(), seen) || reaches_structured(x->b.get(), seen);
        default: return false;   // MXV / REDUCE / SAPPLY are barriers (their results are full or scalars)
    }
}

bool needs_structured(const NodeP &r) {
    if (r->mat) return false;
    std::unordered_set<const Node *> seen;
    if (r->op == Op::REDUCE) return reaches_structured(r->a.get(), seen);
    if (r->op == Op::MXV) {
        const Node *u = r->a.get();
        return u->mat && !u->scalar && (structured_kind(u->kind) || u->kind == VKind::EMPTY);
    }
    if (r->scalar) return false;
    return reaches_structured(r.get(), seen);
}

static double fill_rec(const Node *x, std::unordered_map<const Node *, double> &memo) {
    auto it = memo.find(x);
    if (it != memo.end()) return it->second;
    double f = 1.0;
    if (x->scalar) f = 1.0;
    else if (x->mat) {
        switch (x->kind) {
            case VKind::EMPTY: f = 0.0; break;
            case VKind::SPARSE:
            case VKind::BITSET: f = x->n ? (double)x->nvals / (double)x->n : 0.0; break;
            default: f = 1.0;
        }
    } else {
        switch (x->op) {
            case Op::APPLY:
            case Op::BIND2ND: f = fill_rec(x->a.get(), memo); break;
            case Op::EMULT: f = fill_rec(x->a.get(), memo) * fill_rec(x->b.get(), memo); break;
            case Op::EADD: {
                const double fa = fill_rec(x->a.get(), memo), fb = fill_rec(x->b.get(), memo);
                f = fa + fb - fa * fb;
                break;
            }
            default: f = 1.0;   // mxv output is dense (SPEC.md:206 reading)
        }
    }
    memo[x] = f;
    return f;
}

double estimated_fill(const Node *x) {
    std::unordered_map<const Node *, double> memo;
    return fill_rec(x, memo);
}

namespace {

// presence that holds for every index without looking at data
bool static_full(const Node *x) {
    if (x->scalar) return true;
    if (x->mat) return x->kind == VKind::FULL || x->kind == VKind::ISO;
    switch (x->op) {
        case Op::APPLY:
        case Op::BIND2ND: return static_full(x->a.get());
        case Op::EMULT: return static_full(x->a.get()) && static_full(x->b.get());
        case Op::EADD: return static_full(x->a.get()) || static_full(x->b.get());
        default: return true;
    }
}

// a set of sparse leaves whose index union contains every present index of x (false: none exists)
bool cover(const Node *x, std::vector<const Node *> &out) {
    if (x->mat) {
        if (!x->scalar && x->kind == VKind::SPARSE) { out.push_back(x); return true; }
        return !x->scalar && x->kind == VKind::EMPTY;   // no entries: covered by nothing
    }
    switch (x->op) {
        case Op::APPLY:
        case Op::BIND2ND: return cover(x->a.get(), out);
        case Op::EMULT: {
            std::vector<const Node *> ca, cb;
            const bool ha = cover(x->a.get(), ca), hb = cover(x->b.get(), cb);
            if (!ha && !hb) return false;
            auto sz = [](const std::vector<const Node *> &v) { int64_t s = 0; for (auto *l : v) s += l->nvals; return s; };
            const std::vector<const Node *> &pick = (ha && (!hb || sz(ca) <= sz(cb))) ? ca : cb;
            out.insert(out.end(), pick.begin(), pick.end());
            return true;
        }
        case Op::EADD: {
            std::vector<const Node *> ca, cb;
            if (!cover(x->a.get(), ca) || !cover(x->b.get(), cb)) return false;
            out.insert(out.end(), ca.begin(), ca.end());
            for (auto *l : cb)
                if (std::find(out.begin(), out.end(), l) == out.end()) out.push_back(l);
            return true;
        }
        default: return false;
    }
}

struct SBuilder {
    Ctx &c;
    SProg sp;
    bool index_mode;
    std::vector<double> imm;
    std::vector<SlotP> sin;
    std::vector<NodeP> in_nodes;
    std::vector<BufP> keep;                 // temporaries alive until the launch is queued
    std::vector<const void *> in_vals, in_aux;
    std::unordered_map<const Node *, int> ins_of;
    std::vector<NodeP> visited;

    SBuilder(Ctx &cc, bool im) : c(cc), index_mode(im) {}

    int add(const Ins &in, uint8_t pm) {
        sp.p.ins.push_back(in);
        sp.pmode.push_back(pm);
        return (int)sp.p.ins.size() - 1;
    }
    int imm_slot(double v) {
        imm.push_back(v);
        return (int)imm.size() - 1;
    }

    int emit(const NodeP &x) {
        auto it = ins_of.find(x.get());
        if (it != ins_of.end()) return it->second;
        int r;
        Ins in{};
        in.t = x->type;
        if (x->mat) {
            if (x->scalar) {
                in.uniform = true;
                if (x->sfmt == SFmt::HOST) {
                    in.k = Ins::LD_SHOST;
                    in.slot = imm_slot(x->hval);
                } else {
                    in.k = Ins::LD_SDEV;
                    in.slot = (int)sin.size();
                    sin.push_back(x->slot);
                    in.fmt = (uint8_t)x->sfmt;
                }
                r = add(in, 3);
            } else if (x->kind == VKind::ISO) {
                in.k = Ins::LD_ISO;
                in.uniform = true;
                in.slot = imm_slot(x->iso);
                r = add(in, 3);
            } else {
                in.k = Ins::LD_VEC;
                in.slot = (int)in_nodes.size();
                in_nodes.push_back(x);
                uint8_t lk = 0;
                const void *aux = nullptr;
                const void *vals = x->buf ? x->buf->d : nullptr;
                if (x->kind == VKind::EMPTY) {
                    lk = 3;                  // never present
                    vals = nullptr;
                } else if (x->kind == VKind::BITSET) {
                    lk = 1;
                    aux = x->bits->d;
                } else if (x->kind == VKind::SPARSE) {
                    if (index_mode) {
                        lk = 2;
                        aux = x->idx->d;
                        in.imm0 = imm_slot((double)x->nvals);
                    } else {   // dense loop: the sparse operand is scattered into a bitset first
                        lk = 1;
                        BufP bits = alloc_buf(c, (size_t)((x->n + 31) / 32) * 4);
                        BufP dense = alloc_buf(c, (size_t)x->n * type_size(x->type));
                        gpu_sparse_to_bitset(c, x->n, x->nvals, (const int32_t *)x->idx->d, x->buf->d, x->type, (uint32_t *)bits->d,
                                             dense->d);
                        keep.push_back(bits);
                        keep.push_back(dense);
                        aux = bits->d;
                        vals = dense->d;
                    }
                } else if (x->kind != VKind::FULL) {
                    fail(NBG_PANIC, "structured region: unexpected leaf");
                }
                sp.leaf.push_back(lk);
                in_vals.push_back(vals);
                in_aux.push_back(aux);
                r = add(in, 3);
            }
        } else {
            switch (x->op) {
                case Op::APPLY:
                case Op::SAPPLY: {
                    const int a = emit(x->a);
                    in.k = Ins::UN;
                    in.code = x->code;
                    in.a = a;
                    if (x->code == NBG_ADD_C || x->code == NBG_MUL_C || x->code == NBG_AXPB || x->code == NBG_ABS_SUB_C ||
                        x->code == NBG_RECIP_SCALED || x->code >= NBG_USER_OP_BASE)
                        in.imm0 = imm_slot(x->c0);
                    if (x->code == NBG_AXPB || x->code >= NBG_USER_OP_BASE) in.imm1 = imm_slot(x->c1);
                    in.uniform = sp.p.ins[a].uniform;
                    r = add(in, 0);
                    break;
                }
                case Op::BIND2ND:
                case Op::EMULT:
                case Op::EADD: {
                    const int a = emit(x->a), b = emit(x->b);
                    in.k = Ins::BIN;
                    in.code = x->code;
                    in.a = a;
                    in.b = b;
                    if (x->code == NBG_MAX_DIVX_C || x->code >= NBG_USER_OP_BASE) in.imm0 = imm_slot(x->c0);
                    in.uniform = sp.p.ins[a].uniform && sp.p.ins[b].uniform;
                    r = add(in, x->op == Op::EMULT ? 1 : (x->op == Op::EADD ? 2 : 0));
                    break;
                }
                default: fail(NBG_PANIC, "structured region: unexpected node (prerequisite not materialised)");
            }
            visited.push_back(x);
        }
        ins_of[x.get()] = r;
        return r;
    }
};

// pending barriers under x (mxv results and scalars feeding bind2nd) materialised before the region
void collect_prereq(const NodeP &x, std::vector<NodeP> &out, std::unordered_set<const Node *> &seen) {
    if (x->mat || !seen.insert(x.get()).second) return;
    switch (x->op) {
        case Op::APPLY: collect_prereq(x->a, out, seen); break;
        case Op::SAPPLY: {
            NodeP r = x->a;
            while (r && !r->mat && r->op == Op::SAPPLY) r = r->a;
            if (r && !r->mat) out.push_back(r);
            break;
        }
        case Op::BIND2ND:
            collect_prereq(x->a, out, seen);
            if (!x->b->mat) collect_prereq(x->b, out, seen);
            break;
        case Op::EMULT:
        case Op::EADD:
            collect_prereq(x->a, out, seen);
            collect_prereq(x->b, out, seen);
            break;
        default: out.push_back(x);   // MXV, REDUCE
    }
}

void drop(Node &x) {
    x.a.reset();
    x.b.reset();
    x.A.reset();
}

// structured mxv: x scattered into (bitset, dense values); one warp per CSR row
void materialize_smxv(Ctx &c, const NodeP &r) {
    const NodeP u = r->a;
    Mat &A = *r->A;
    BufP bits, dense;
    if (u->kind == VKind::BITSET) {
        bits = u->bits;
        dense = u->buf;
    } else if (u->kind == VKind::EMPTY) {   // no x entry present: every row is the identity
        bits = alloc_buf(c, (size_t)std::max<int64_t>((u->n + 31) / 32, 1) * 4);
        dense = alloc_buf(c, (size_t)std::max<int64_t>(u->n, 1) * type_size(u->type));
        NBG_CUDA(cudaMemsetAsync(bits->d, 0, bits->bytes, c.stream));
        NBG_CUDA(cudaMemsetAsync(dense->d, 0, dense->bytes, c.stream));
    } else {
        bits = alloc_buf(c, (size_t)((u->n + 31) / 32) * 4);
        dense = alloc_buf(c, (size_t)u->n * type_size(u->type));
        gpu_sparse_to_bitset(c, u->n, u->nvals, (const int32_t *)u->idx->d, u->buf->d, u->type, (uint32_t *)bits->d, dense->d);
    }
    SpmvSig sig;
    sig.add = r->add;
    sig.mul = r->mul;
    sig.T = r->type;
    sig.xt = u->type;
    sig.at = A.type;
    sig.has_vals = (bool)A.vals;
    std::ostringstream key;
    key << "XM|" << sig.add << "," << sig.mul << "," << sig.T << "," << sig.xt << "," << sig.at << "," << sig.has_vals;
    KernelP k;
    auto it = c.plans.find(key.str());
    if (it == c.plans.end()) {
        char nm[48];
        snprintf(nm, sizeof nm, "nbg_smxv_%016llx", (unsigned long long)hash_str(key.str()));
        k = jit_compile(c, codegen_smxv(sig, nm), nm, false);
        c.plans[key.str()] = k;
        c.stats.plans_built++;
    } else {
        k = it->second;
        c.stats.plan_hits++;
    }
    KArgs a;
    memset(&a, 0, sizeof a);
    a.n = A.nrows;
    a.rowptr = (const long long *)A.rowptr->d;
    a.colidx = (const int *)A.colidx->d;
    a.aval = A.vals ? A.vals->d : nullptr;
    a.x = dense->d;
    a.in[0] = bits->d;
    a.imm[0] = A.iso;
    a.imm[1] = r->c0;
    BufP out = alloc_buf(c, (size_t)A.nrows * type_size(r->type));
    a.out[0] = out->d;
    if (A.nrows > 0) launch(c, *k, a, (A.nrows + 7) / 8, "spmv");
    r->mat = true;
    r->kind = VKind::FULL;
    r->buf = out;
    drop(*r);
    c.stats.vectors_materialized++;
    c.stats.bytes_materialized += out->bytes;
    c.stats.structured_regions++;
    c.stats.waits++;
}

}  // namespace

void materialize_structured(Ctx &c, const NodeP &r) {
    if (r->mat) return;
    if (r->op == Op::MXV) {
        materialize_smxv(c, r);
        return;
    }
    const bool vec_out = !r->scalar;
    const NodeP R = vec_out ? r : r->a;           // the vector expression (reduce operand)
    {
        std::vector<NodeP> pre;
        std::unordered_set<const Node *> seen;
        if (!R->mat) collect_prereq(R, pre, seen);
        if (!pre.empty()) materialize(c, pre);
        if (r->mat) return;
    }
    const int64_t n = R->n;
    const bool sfull = static_full(R.get());
    const double f_est = estimated_fill(R.get());
    std::vector<const Node *> cov;
    const bool has_cover = !sfull && cover(R.get(), cov);
    int64_t cov_n = 0;
    for (const Node *l : cov) cov_n += l->nvals;
    bool index_mode = has_cover && n > 0 && (double)cov_n <= INDEX_FILL * (double)n;
    // NBG_STRUCT_LOOP=index|dense overrides the estimator's choice (benchmarking the choice itself)
    const char *force = getenv("NBG_STRUCT_LOOP");
    if (force && has_cover && !strcmp(force, "index")) index_mode = true;
    if (force && !strcmp(force, "dense")) index_mode = false;
    const bool want_sparse = f_est <= SPARSE_FILL;

    SBuilder B(c, index_mode);
    B.sp.index_mode = index_mode;
    B.sp.vec_out = vec_out;
    int root = B.emit(R);
    Prog &p = B.sp.p;
    if (vec_out) {
        p.outs.push_back(OutV{root, 0});
    } else {
        if (p.ins[root].t != r->type) {
            Ins cv{};
            cv.k = Ins::CVT;
            cv.t = r->type;
            cv.a = root;
            cv.uniform = p.ins[root].uniform;
            root = B.add(cv, 0);
        }
        const bool f = is_float(r->type);
        uint8_t fmt;
        if (r->code == NBG_PLUS) fmt = (uint8_t)(f ? SFmt::XACC : SFmt::I64);
        else if (r->code == NBG_MAX) fmt = (uint8_t)(f ? SFmt::FMAX : SFmt::IMAX);
        else fmt = (uint8_t)(f ? SFmt::FMIN : SFmt::IMIN);
        p.reds.push_back(RedOut{root, r->code, 0, fmt});
    }
    p.n_in = (int)B.in_nodes.size();
    p.n_out = vec_out ? 1 : 0;
    p.n_imm = (int)B.imm.size();
    p.n_sin = (int)B.sin.size();
    p.n_red = vec_out ? 0 : 1;
    if (2 * p.n_in > MAX_IN || p.n_imm > MAX_IMM || p.n_sin > MAX_SIN)
        fail(NBG_NOT_IMPLEMENTED, "structured region exceeds kernel argument limits");

    // driver index list (index loop)
    BufP drv;
    int64_t m = 0;
    if (index_mode) {
        if (cov.size() == 1) {
            drv = cov[0]->idx;
            m = cov[0]->nvals;
        } else {
            std::vector<std::pair<const int32_t *, int64_t>> lists;
            for (const Node *l : cov) lists.push_back({(const int32_t *)l->idx->d, l->nvals});
            m = gpu_union_indices(c, lists, &drv);
        }
    }

    const std::string sig = B.sp.signature();
    KernelP k;
    auto it = c.plans.find(sig);
    if (it == c.plans.end()) {
        char nm[48];
        snprintf(nm, sizeof nm, "nbg_sreg_%016llx", (unsigned long long)hash_str(sig));
        k = jit_compile(c, codegen_structured(B.sp, nm), nm, false);
        c.plans[sig] = k;
        c.stats.plans_built++;
    } else {
        k = it->second;
        c.stats.plan_hits++;
    }

    KArgs a;
    memset(&a, 0, sizeof a);
    a.n = n;
    for (int s = 0; s < p.n_in; s++) {
        a.in[s] = B.in_vals[s];
        a.in[p.n_in + s] = B.in_aux[s];
    }
    for (int s = 0; s < p.n_imm; s++) a.imm[s] = B.imm[s];
    for (int s = 0; s < p.n_sin; s++) a.sin[s] = B.sin[s]->dptr();
    const int T = vec_out ? R->type : r->type;
    const size_t w = type_size(vec_out ? p.ins[p.outs[0].ins].t : T);
    BufP ovals, oaux, cnt;
    SlotP slot;
    if (vec_out) {
        const int64_t len = index_mode ? m : n;
        ovals = alloc_buf(c, (size_t)std::max<int64_t>(len, 1) * w);
        oaux = alloc_buf(c, index_mode ? (size_t)std::max<int64_t>(m, 1) : (size_t)std::max<int64_t>((n + 31) / 32, 1) * 4);
        a.out[0] = ovals->d;
        a.out[1] = oaux->d;
        if (!index_mode) {
            cnt = alloc_buf(c, 8);
            NBG_CUDA(cudaMemsetAsync(cnt->d, 0, 8, c.stream));
            a.part = cnt->d;
        }
    } else {
        slot = alloc_slot(c);
        a.racc[0] = slot->dptr();
    }
    if (index_mode) {
        a.rowptr = (const long long *)(drv ? drv->d : nullptr);
        a.nnz = m;
        if (m > 0) launch(c, *k, a, (m + 255) / 256, "ewise");
        else if (!vec_out) {          // no entry can be present: the monoid identity
            r->mat = true;
            r->sfmt = SFmt::HOST;
            r->hval = monoid_identity(r->code, r->type);
            r->hval = host_round(r->type, r->hval);
            drop(*r);
            c.stats.structured_regions++;
            c.stats.structured_index_loops++;
            c.stats.waits++;
            return;
        }
    } else if (n > 0) {
        launch(c, *k, a, (n + 255) / 256, "ewise");
    }
    c.stats.structured_regions++;
    if (index_mode) c.stats.structured_index_loops++;

    if (vec_out) {
        const int OT = p.ins[p.outs[0].ins].t;
        if (index_mode) {
            BufP oi, ov;
            const int64_t nv = gpu_select_flagged(c, m, (const int32_t *)(drv ? drv->d : nullptr), ovals->d, (const uint8_t *)oaux->d, OT,
                                                  &oi, &ov);
            r->nvals = nv;
            if (nv == 0) {
                r->kind = VKind::EMPTY;
            } else if (nv == n) {   // every entry present: dense values in index order
                r->kind = VKind::FULL;
                r->buf = ov;
            } else if (want_sparse) {
                r->kind = VKind::SPARSE;
                r->idx = oi;
                r->buf = ov;
            } else {
                r->kind = VKind::BITSET;
                r->bits = alloc_buf(c, (size_t)((n + 31) / 32) * 4);
                r->buf = alloc_buf(c, (size_t)n * type_size(OT));
                gpu_sparse_to_bitset(c, n, nv, (const int32_t *)oi->d, ov->d, OT, (uint32_t *)r->bits->d, r->buf->d);
            }
        } else {
            int64_t nv = 0;
            NBG_CUDA(cudaMemcpyAsync(&nv, cnt->d, 8, cudaMemcpyDeviceToHost, c.stream));
            NBG_CUDA(cudaStreamSynchronize(c.stream));
            if (nv == n) {
                r->kind = VKind::FULL;
                r->buf = ovals;
            } else if (nv == 0) {
                r->kind = VKind::EMPTY;
            } else if (want_sparse) {
                BufP oi, ov;
                gpu_bitset_to_sparse(c, n, (const uint32_t *)oaux->d, ovals->d, OT, &oi, &ov);
                r->kind = VKind::SPARSE;
                r->idx = oi;
                r->buf = ov;
            } else {
                r->kind = VKind::BITSET;
                r->bits = oaux;
                r->buf = ovals;
            }
            r->nvals = nv;
        }
        if (r->kind == VKind::FULL) r->nvals = n;
        r->mat = true;
        c.stats.vectors_materialized++;
        if (r->buf) c.stats.bytes_materialized += r->buf->bytes;
    } else {
        r->mat = true;
        r->slot = slot;
        r->sfmt = (SFmt)p.reds[0].fmt;
        if (r->user_refs > 0) mark_readable(c, slot, record_prod_event(c));
    }
    c.stats.intermediates_elided += B.visited.size() > 0 ? B.visited.size() - (vec_out ? 1 : 0) : 0;
    drop(*r);
    c.stats.waits++;
}

}  // namespace nbg
