// planner.cpp -- materialisation at wait.
//
// wait(roots):
//   1. Region: walk the pending DAG from the roots down to materialised leaves.  Every pending
//      elementwise node (apply / ewise_mult / ewise_add / apply_bind2nd / convert) joins the
//      region; at most ONE mxv joins it and then the whole region runs in that mxv's epilogue
//      (per output row).  Fusion barriers: an mxv's vector input must be
//      materialised (it is gathered), a reduction feeding a scalar operand must be materialised
//      (every block needs its value), a second mxv is materialised separately.  Those become
//      prerequisites, materialised first (recursively, jointly when independent).
//   2. Memo: before computing a prerequisite, look it up by its structural key over the
//      identities of its materialised leaves (immutable buffers) -- a derived view computed
//      earlier is bound instead of recomputed.
//   3. Speculation (loop-carried elision): when a prerequisite depends on exactly one buffer that
//      an earlier region wrote, remember "region S's output o tends to be consumed through
//      expression E"; the next time a region with signature S runs, E(output o) is emitted as an
//      extra output of that same kernel and memoised.  For PageRank this turns y = t/d and the
//      dangling sum of t into side outputs of the previous sweep.
//   4. Signature of the region program -> plan cache -> (NVRTC on a miss) -> bind -> launch.
//   Liveness ("elide unneeded objects"): besides the requested roots, only pending
//   nodes a user still holds a handle to are stored; every other intermediate lives in registers.
#include <algorithm>
#include <charconv>
#include <cstring>
#include <cstdio>
#include <functional>
#include <sstream>
#include <unordered_set>

#include "nbg_internal.hpp"

namespace nbg {

// host-side phase profile of the planner (NBG_PLAN_PROFILE=1: printed at exit)
struct PlanProf {
    double t[10] = {0};
    long long n[10] = {0};
    bool on = false;
    PlanProf() { const char *e = getenv("NBG_PLAN_PROFILE"); on = e && e[0] == '1'; }
    ~PlanProf() {
        if (!on) return;
        const char *nm[10] = {"purge+bind", "region", "hints", "keys", "run:sig+plan", "run:args+launch", "memo_insert", "total",
                              "  launch call", "  readable mark"};
        for (int i = 0; i < 10; i++)
            if (n[i]) fprintf(stderr, "[nbg plan] %-16s %10.2f us/call  (%lld calls)\n", nm[i], t[i] / 1e3 / n[i], n[i]);
    }
};
PlanProf g_prof;
static thread_local double g_pp_t0 = 0.0;
void plan_prof_t0() {
    if (g_prof.on) g_pp_t0 = now_ns();
}
void plan_prof_t1(int k) {
    if (!g_prof.on) return;
    const double d = now_ns() - g_pp_t0;
    if (d < 500e3) { g_prof.t[k] += d; g_prof.n[k]++; }
}
struct PTimer {
    int k;
    double t0;
    explicit PTimer(int kk) : k(kk), t0(g_prof.on ? now_ns() : 0.0) {}
    ~PTimer() {
        if (!g_prof.on) return;
        const double d = now_ns() - t0;
        if (d < 500e3) { g_prof.t[k] += d; g_prof.n[k]++; }   // steady state only (no JIT compiles)
    }
};

static std::string dbits(double v) {
    uint64_t b;
    memcpy(&b, &v, 8);
    char s[24];
    snprintf(s, sizeof s, "%llx", (unsigned long long)b);
    return s;
}

// flat containers for the few-node sets of one wait (a region has tens of nodes): linear search
// over a vector beats hashing and node allocation at this size (host time per wait)
template <class K, class V>
struct SmallMap {
    std::vector<std::pair<K, V>> v;
    using iterator = typename std::vector<std::pair<K, V>>::iterator;
    iterator begin() { return v.begin(); }
    iterator end() { return v.end(); }
    iterator find(const K &k) {
        for (auto it = v.begin(); it != v.end(); ++it)
            if (it->first == k) return it;
        return v.end();
    }
    size_t count(const K &k) { return find(k) != v.end() ? 1 : 0; }
    V &operator[](const K &k) {
        auto it = find(k);
        if (it != v.end()) return it->second;
        v.emplace_back(k, V{});
        return v.back().second;
    }
};
template <class K>
struct SmallSet {
    std::vector<K> v;
    size_t count(const K &k) const {
        for (const K &x : v)
            if (x == k) return 1;
        return 0;
    }
    std::pair<size_t, bool> insert(const K &k) {
        if (count(k)) return {0, false};
        v.push_back(k);
        return {v.size() - 1, true};
    }
};

// ---------------------------------------------------------------- structural keys

// The key is a token stream over the expression (ops, types, sizes, operator codes and constants,
// leaf identities); it is emitted into a sink: a string (hint templates, debug output) or a
// 128-bit hash (the memo key, computed at every wait without building the string; two
// independent 64-bit streams, so a collision needs both to collide).
struct KStr {
    std::string s;
    void put(long long v) {
        char buf[24];
        auto r = std::to_chars(buf, buf + sizeof buf, v);
        s.append(buf, r.ptr);
    }
    void bits(double v) {
        uint64_t b;
        memcpy(&b, &v, 8);
        char buf[24];
        auto r = std::to_chars(buf, buf + sizeof buf, (unsigned long long)b, 16);
        s.append(buf, r.ptr);
    }
    void ch(char c) { s.push_back(c); }
};
struct KHash {
    uint64_t a = 1469598103934665603ull, b = 0x9E3779B97F4A7C15ull;
    void put(long long v) {
        const uint64_t u = (uint64_t)v;
        a = (a ^ u) * 1099511628211ull;
        b = (b ^ (u + 0x632BE59BD9B4E019ull)) * 0xFF51AFD7ED558CCDull;
        b ^= b >> 29;
    }
    void bits(double v) {
        uint64_t u;
        memcpy(&u, &v, 8);
        put((long long)u);
    }
    void ch(char c) { put((long long)(unsigned char)c | (1ll << 40)); }
    MKey key() const { return MKey{a, b}; }
};
template <class S>
static void key_rec(const Node *x, S &s, const Node *ph) {
    if (x == ph) { s.ch('P'); return; }
    if (x->mat) {
        if (x->scalar) {
            if (x->sfmt == SFmt::HOST) { s.ch('h'); s.put(x->type); s.ch(':'); s.bits(x->hval); }
            else { s.ch('d'); s.put(x->type); s.ch(':'); s.put((long long)x->slot->id); }
        } else if (x->kind == VKind::FULL) { s.ch('F'); s.put((long long)x->buf->id); }
        else if (x->kind == VKind::ISO) { s.ch('I'); s.put(x->type); s.ch(':'); s.bits(x->iso); }
        else if (x->kind == VKind::SPARSE) { s.ch('S'); s.put((long long)x->buf->id); }
        else if (x->kind == VKind::BITSET) { s.ch('B'); s.put((long long)x->buf->id); }
        else s.ch('E');
        return;
    }
    s.ch('(');
    s.put((int)x->op); s.ch(',');
    s.put(x->type); s.ch(',');
    s.put(x->n); s.ch(',');
    s.put(x->code); s.ch(',');
    s.bits(x->c0); s.ch(',');
    s.bits(x->c1); s.ch(',');
    s.put(x->add); s.ch(',');
    s.put(x->mul); s.ch(',');
    if (x->A) s.put((long long)x->A->id); else s.ch('-');
    s.ch(';');
    if (x->a) key_rec(x->a.get(), s, ph);
    s.ch(';');
    if (x->b) key_rec(x->b.get(), s, ph);
    s.ch(')');
}

static std::string node_key(const Node *x, const Node *ph = nullptr) {
    KStr s;
    key_rec(x, s, ph);
    return s.s;
}

// memo key of x; `pending`: as if x were still pending (x materialised, its inputs still
// attached) -- the lookup key the next wait builds for the same expression; `perm`: the view of x
// in matrix perm's gather layout
static MKey memo_key(const Node *x, bool pending = false, const Mat *perm = nullptr) {
    KHash h;
    if (perm) { h.ch('!'); h.put((long long)perm->id); h.ch('('); }
    Node *m = const_cast<Node *>(x);
    const bool flip = pending && x->mat;
    if (flip) m->mat = false;
    key_rec(x, h, nullptr);
    if (flip) m->mat = true;
    if (perm) h.ch(')');
    return h.key();
}

static void leaf_bufs(const Node *x, std::vector<std::weak_ptr<Buf>> &deps, SmallSet<const Node *> &seen) {
    if (!seen.insert(x).second) return;
    if (x->mat) {
        if (!x->scalar && (x->kind == VKind::FULL || structured_kind(x->kind)) && x->buf) deps.push_back(x->buf);
        return;
    }
    if (x->a) leaf_bufs(x->a.get(), deps, seen);
    if (x->b) leaf_bufs(x->b.get(), deps, seen);
}

static void memo_purge(Ctx &c) {
    for (auto it = c.memo.begin(); it != c.memo.end();) {
        bool dead = false;
        for (auto &w : it->second.deps)
            if (w.expired()) { dead = true; break; }
        if (dead) it = c.memo.erase(it);
        else ++it;
    }
}

static void drop_inputs(Node &x) {
    x.a.reset();
    x.b.reset();
    x.A.reset();
}

static void copy_result(Node &dst, const Node &src) {
    dst.mat = true;
    dst.kind = src.kind;
    dst.buf = src.buf;
    dst.idx = src.idx;
    dst.bits = src.bits;
    dst.nvals = src.nvals;
    dst.iso = src.iso;
    dst.sfmt = src.sfmt;
    dst.hval = src.hval;
    dst.slot = src.slot;
    drop_inputs(dst);
}

static bool dbg() {
    static int v = -1;
    if (v < 0) v = getenv("NBG_DEBUG") && *getenv("NBG_DEBUG") ? 1 : 0;
    return v == 1;
}

static bool memo_bind(Ctx &c, const NodeP &x) {
    if (x->mat) return true;
    if (dbg()) fprintf(stderr, "[nbg] memo lookup %s (%zu entries)\n", node_key(x.get()).c_str(), c.memo.size());
    auto it = c.memo.find(memo_key(x.get()));
    if (it == c.memo.end()) return false;
    for (auto &w : it->second.deps)
        if (w.expired()) return false;
    copy_result(*x, *it->second.result);
    it->second.stamp = ++c.memo_clock;
    c.stats.memo_hits++;
    return true;
}

// Results are immutable and keyed by the identities of immutable leaves, so a memo entry stays
// valid while its leaves live; the table is bounded (LRU) so it cannot pin unbounded memory.
static const size_t MEMO_CAP = 64;
static void memo_insert(Ctx &c, const MKey &k, const NodeP &result) {
    std::vector<std::weak_ptr<Buf>> deps;
    SmallSet<const Node *> seen;
    // leaves of the expression: walk the (still attached) inputs of the result node
    seen.insert(result.get());
    if (result->a) leaf_bufs(result->a.get(), deps, seen);
    if (result->b) leaf_bufs(result->b.get(), deps, seen);
    if (c.memo.size() >= MEMO_CAP) {
        auto victim = c.memo.begin();
        for (auto it = c.memo.begin(); it != c.memo.end(); ++it)
            if (it->second.stamp < victim->second.stamp) victim = it;
        c.memo.erase(victim);
    }
    c.memo.insert_or_assign(k, Ctx::MemoEntry{std::move(deps), result, ++c.memo_clock});
}

// ---------------------------------------------------------------- cloning (hint templates)

// clone the pending part of x; `subst` maps leaves to replacements (pre-seeded in `seen`)
static NodeP clone_subst(Ctx &c, const NodeP &x, SmallMap<const Node *, NodeP> &seen) {
    auto it = seen.find(x.get());
    if (it != seen.end()) return it->second;
    if (x->mat) return x;
    auto y = std::make_shared<Node>(*x);
    y->uid = c.new_id();
    y->user_refs = 0;
    if (x->a) y->a = clone_subst(c, x->a, seen);
    if (x->b) y->b = clone_subst(c, x->b, seen);
    seen[x.get()] = y;
    return y;
}

static NodeP make_placeholder(Ctx &c, const Node *like) {
    auto ph = std::make_shared<Node>();
    ph->op = Op::LEAF;
    ph->mat = true;
    ph->kind = VKind::FULL;
    ph->type = like->type;
    ph->n = like->n;
    ph->uid = c.new_id();
    return ph;
}

static void full_leaves(const NodeP &x, std::vector<NodeP> &out, std::unordered_set<const Node *> &seen) {
    if (!seen.insert(x.get()).second) return;
    if (x->mat) {
        if (!x->scalar && x->kind == VKind::FULL) out.push_back(x);
        return;
    }
    if (x->a) full_leaves(x->a, out, seen);
    if (x->b) full_leaves(x->b, out, seen);
}

// a template can be instantiated inside another region only if it needs no prerequisite
static bool fusable_template(const Node *x, bool root) {
    if (x->mat) return true;
    if (x->op == Op::MXV) return false;
    if (x->op == Op::REDUCE && !root) return false;
    if (x->a && !fusable_template(x->a.get(), false)) return false;
    if (x->b && !fusable_template(x->b.get(), false)) return false;
    return true;
}

static void find_produced_leaves(const Node *x, std::vector<const Node *> &out, std::unordered_set<const Node *> &seen) {
    if (!seen.insert(x).second) return;
    if (x->mat) {
        if (!x->scalar && x->kind == VKind::FULL && x->buf && x->buf->prod_sig) out.push_back(x);
        return;
    }
    if (x->a) find_produced_leaves(x->a.get(), out, seen);
    if (x->b) find_produced_leaves(x->b.get(), out, seen);
}

static void learn_hint(Ctx &c, const NodeP &p, const MatP &consumer) {
    if (!fusable_template(p.get(), true)) return;
    std::vector<const Node *> prod;
    std::unordered_set<const Node *> seen;
    find_produced_leaves(p.get(), prod, seen);
    if (prod.empty()) return;
    // the loop-carried operand is the most recently produced buffer (e.g. the previous sweep's
    // ranks); older products (dinv) are loop invariants and stay leaves of the template
    const Node *L = prod[0];
    for (const Node *q : prod)
        if (q->buf->prod_seq > L->buf->prod_seq) L = q;
    for (const Node *q : prod)
        if (q != L && q->buf->prod_seq == L->buf->prod_seq) return;   // ambiguous
    auto key = std::make_pair(L->buf->prod_sig, L->buf->prod_out);
    const std::string k = node_key(p.get(), L);
    auto &vec = c.hints[key];
    // drop hints whose loop-invariant leaves died (e.g. a previous run's dinv)
    vec.erase(std::remove_if(vec.begin(), vec.end(),
                             [](const Hint &h) {
                                 for (auto &f : h.fixed)
                                     if (f.second.expired()) return true;
                                 return false;
                             }),
              vec.end());
    for (auto &h : vec)
        if (h.key == k) return;
    if (vec.size() >= 4) return;
    Hint h;
    h.key = k;
    h.consumer = consumer;
    SmallMap<const Node *, NodeP> cs;
    h.ph_keep = make_placeholder(c, L);
    h.placeholder = h.ph_keep.get();
    cs[L] = h.ph_keep;
    std::vector<NodeP> leaves;
    std::unordered_set<const Node *> sl;
    full_leaves(p, leaves, sl);
    for (const NodeP &q : leaves) {
        if (q.get() == L) continue;
        NodeP px = make_placeholder(c, q.get());
        cs[q.get()] = px;
        h.fixed.push_back({px, std::weak_ptr<Node>(q)});
    }
    h.tmpl = clone_subst(c, p, cs);
    if (dbg()) fprintf(stderr, "[nbg] learn hint sig=%llx out=%d tmpl=%s\n", (unsigned long long)key.first, key.second, k.c_str());
    vec.push_back(std::move(h));
}

// instantiate a hint over the region output R (nullptr if a loop-invariant leaf died)
static NodeP instantiate(Ctx &c, const Hint &h, const NodeP &R) {
    SmallMap<const Node *, NodeP> cs;
    cs[h.placeholder] = R;
    for (auto &f : h.fixed) {
        NodeP q = f.second.lock();
        if (!q) return nullptr;
        cs[f.first.get()] = q;
    }
    return clone_subst(c, h.tmpl, cs);
}

static NodeP memo_get(Ctx &c, const MKey &k) {
    auto it = c.memo.find(k);
    if (it == c.memo.end()) return nullptr;
    for (auto &w : it->second.deps)
        if (w.expired()) return nullptr;
    it->second.stamp = ++c.memo_clock;
    c.stats.memo_hits++;
    return it->second.result;
}

static MKey perm_key(const Mat &A, const Node *u) { return memo_key(u, false, &A); }

// x in the matrix's gather layout: xg[k] = x[iperm[k]] (a static permute kernel), memoised
static NodeP permuted_view(Ctx &c, Mat &A, const NodeP &u, const MKey &pk) {
    auto g = std::make_shared<Node>();
    g->op = Op::LEAF;
    g->type = u->type;
    g->n = A.plan->ncols_g;
    g->uid = c.new_id();
    g->kind = VKind::FULL;
    g->buf = alloc_buf(c, (size_t)A.plan->ncols_g * type_size(u->type));
    if (u->kind == VKind::ISO) gpu_fill_iso(c, g->buf->d, u->type, A.plan->ncols_g, u->iso);
    else gpu_permute(c, u->buf->d, g->buf->d, u->type, (const int *)A.plan->iperm->d, A.plan->ncols_g);
    g->a = u;            // the memo entry depends on u's leaves
    g->mat = true;
    if (c.mode == NBG_NONBLOCKING) memo_insert(c, pk, g);
    g->a.reset();
    return g;
}

// ---------------------------------------------------------------- region builder

struct Builder {
    Ctx &c;
    Prog prog;
    SmallMap<const Node *, int> ins_of;
    SmallMap<const Node *, int> in_slot_of;
    std::vector<NodeP> in_nodes;
    std::vector<double> imm;
    std::vector<SlotP> sin;
    SmallMap<const Slot *, int> sin_of;
    std::vector<NodeP> prereq;
    SmallSet<const Node *> prereq_set;
    NodeP mxv;
    BufP mxv_x;                        // the gathered vector (in the matrix's gather layout)
    SmallMap<const Node *, MatP> need_mx;   // prerequisite -> the mxv that gathers it
    std::vector<NodeP> visited;        // pending nodes of the region
    std::vector<NodeP> out_nodes;      // vector outputs, index = out slot
    std::vector<NodeP> red_nodes;      // reductions, index = racc slot
    SmallSet<const Node *> is_out;

    explicit Builder(Ctx &cc) : c(cc) {
        imm.push_back(0.0);   // imm[0]: iso value of the matrix (spmv)
        imm.push_back(0.0);   // imm[1]: constant of the semiring mul (spmv)
    }

    int add(const Ins &in) {
        prog.ins.push_back(in);
        return (int)prog.ins.size() - 1;
    }
    int imm_slot(double v) {
        imm.push_back(v);
        return (int)imm.size() - 1;
    }
    void need(const NodeP &x) {
        if (prereq_set.insert(x.get()).second) prereq.push_back(x);
    }

    static bool unop_has_c0(int code) {
        return code == NBG_ADD_C || code == NBG_MUL_C || code == NBG_AXPB || code == NBG_ABS_SUB_C || code == NBG_RECIP_SCALED ||
               code >= NBG_USER_OP_BASE;
    }

    int emit(const NodeP &x) {
        auto it = ins_of.find(x.get());
        if (it != ins_of.end()) return it->second;
        int r = -1;
        if (x->mat) {
            Ins in{};
            in.t = x->type;
            if (x->scalar) {
                in.uniform = true;
                if (x->sfmt == SFmt::HOST) {
                    in.k = Ins::LD_SHOST;
                    in.slot = imm_slot(x->hval);
                } else {
                    in.k = Ins::LD_SDEV;
                    auto s = sin_of.find(x->slot.get());
                    int si;
                    if (s == sin_of.end()) {
                        si = (int)sin.size();
                        sin.push_back(x->slot);
                        sin_of[x->slot.get()] = si;
                    } else si = s->second;
                    in.slot = si;
                    in.fmt = (uint8_t)x->sfmt;
                }
            } else if (x->kind == VKind::ISO) {
                in.k = Ins::LD_ISO;
                in.uniform = true;
                in.slot = imm_slot(x->iso);
            } else if (x->kind == VKind::FULL) {
                in.k = Ins::LD_VEC;
                auto s = in_slot_of.find(x.get());
                int si;
                if (s == in_slot_of.end()) {
                    si = (int)in_nodes.size();
                    in_nodes.push_back(x);
                    in_slot_of[x.get()] = si;
                } else si = s->second;
                in.slot = si;
            } else if (structured_kind(x->kind)) {
                fail(NBG_PANIC, "planner: structured vector inside a dense region");
            } else {
                fail(NBG_PANIC, "planner: empty vector inside a region");
            }
            r = add(in);
        } else {
            switch (x->op) {
                case Op::APPLY:
                case Op::SAPPLY: {
                    int a = emit(x->a);
                    if (a < 0) return -1;
                    Ins in{};
                    in.k = Ins::UN;
                    in.t = x->type;
                    in.code = x->code;
                    in.a = a;
                    if (unop_has_c0(x->code)) in.imm0 = imm_slot(x->c0);
                    if (x->code == NBG_AXPB || x->code >= NBG_USER_OP_BASE) in.imm1 = imm_slot(x->c1);
                    in.uniform = prog.ins[a].uniform;
                    r = add(in);
                    break;
                }
                case Op::BIND2ND:
                case Op::EMULT:
                case Op::EADD: {
                    int a = emit(x->a);
                    int b = emit(x->b);
                    if (a < 0 || b < 0) return -1;
                    Ins in{};
                    in.k = Ins::BIN;
                    in.t = x->type;
                    in.code = x->code;
                    in.a = a;
                    in.b = b;
                    if (x->code == NBG_MAX_DIVX_C || x->code >= NBG_USER_OP_BASE) in.imm0 = imm_slot(x->c0);
                    in.uniform = prog.ins[a].uniform && prog.ins[b].uniform;
                    r = add(in);
                    break;
                }
                case Op::MXV: {
                    if (mxv && mxv.get() != x.get()) { need(x); return -1; }
                    const NodeP &u = x->a;
                    // a sparse / bitset x: the mxv runs on its own (structured.cpp), then feeds this region
                    if (u->mat && !u->scalar && structured_kind(u->kind)) { need(x); return -1; }
                    Mat &A = *x->A;
                    if (!A.plan) gpu_build_spmv_plan(c, A);
                    if (A.plan->relabel) {
                        // gather input in the relabelled layout: a memoised permuted view of u
                        const MKey pk = perm_key(A, u.get());
                        NodeP gx = memo_get(c, pk);
                        if (!gx) {
                            if (!u->mat) { need(u); need_mx[u.get()] = x->A; return -1; }
                            gx = permuted_view(c, A, u, pk);
                        }
                        mxv_x = gx->buf;
                    } else {
                        if (!u->mat) { need(u); need_mx[u.get()] = x->A; return -1; }
                        if (u->kind == VKind::ISO) ensure_full(c, u);
                        mxv_x = u->kind == VKind::ISO ? u->full_cache : u->buf;
                    }
                    mxv = x;
                    Ins in{};
                    in.k = Ins::MXV_ACC;
                    in.t = x->type;
                    r = add(in);
                    break;
                }
                case Op::REDUCE:
                    need(x);
                    return -1;
                default:
                    fail(NBG_PANIC, "planner: unexpected node");
            }
            visited.push_back(x);
        }
        ins_of[x.get()] = r;
        return r;
    }

    // returns false if prerequisites are missing; scatter_perm: store out[perm[i]] (gather layout)
    std::vector<MatP> out_scatter;     // per output: matrix whose gather layout it is written in
    bool add_vector_output(const NodeP &x, const MatP &scatter = nullptr) {
        if (is_out.count(x.get())) return true;
        int i = emit(x);
        if (i < 0) return false;
        OutV ov{i, (int)out_nodes.size()};
        // scattered store out[map[i]]: into a consumer's gather layout, or into a caller's target
        // (multi-GPU exchange buffer, Ctx::out_targets; map < 0 skips the row)
        auto tg = c.out_targets.find(x.get());
        ov.scatter = (bool)scatter || tg != c.out_targets.end();
        ov.multi = tg != c.out_targets.end() && !tg->second.peers.empty();
        ov.affine = tg != c.out_targets.end() && tg->second.alim >= 0;
        prog.outs.push_back(ov);
        out_nodes.push_back(x);
        out_scatter.push_back(scatter);
        is_out.insert(x.get());
        return true;
    }

    bool add_reduction(const NodeP &x) {
        if (is_out.count(x.get())) return true;
        int i = emit(x->a);
        if (i < 0) return false;
        if (prog.ins[i].t != x->type) {
            Ins cv{};
            cv.k = Ins::CVT;
            cv.t = x->type;
            cv.a = i;
            cv.uniform = prog.ins[i].uniform;
            i = add(cv);
        }
        uint8_t fmt;
        bool f = is_float(x->type);
        if (x->code == NBG_PLUS) fmt = (uint8_t)(f ? SFmt::XACC : SFmt::I64);
        else if (x->code == NBG_MAX) fmt = (uint8_t)(f ? SFmt::FMAX : SFmt::IMAX);
        else fmt = (uint8_t)(f ? SFmt::FMIN : SFmt::IMIN);
        prog.reds.push_back(RedOut{i, x->code, (int)red_nodes.size(), fmt});
        red_nodes.push_back(x);
        is_out.insert(x.get());
        return true;
    }
};

// ---------------------------------------------------------------- ISO -> FULL

void ensure_full(Ctx &c, const NodeP &v) {
    if (v->kind != VKind::ISO || v->full_cache) return;
    size_t bytes = (size_t)v->n * type_size(v->type);
    v->full_cache = alloc_buf(c, bytes);
    if (v->n) gpu_fill_iso(c, v->full_cache->d, v->type, v->n, v->iso);
}

// ---------------------------------------------------------------- launch of one region

struct HintOut {
    NodeP node;       // instantiated template root (pending until launch)
    MatP scatter;     // written in this matrix's gather layout (memo key PERM<A>(...))
};

static void run_region(Ctx &c, Builder &B, std::vector<HintOut> &hint_outs, int64_t n) {
    Prog &p = B.prog;
    p.spmv = (bool)B.mxv;
    p.n_in = (int)B.in_nodes.size();
    p.n_out = (int)B.out_nodes.size();
    p.n_imm = (int)B.imm.size();
    p.n_sin = (int)B.sin.size();
    p.n_red = (int)B.red_nodes.size();
    if (p.n_in > MAX_IN || p.n_out > MAX_OUT || p.n_imm > MAX_IMM || p.n_sin > MAX_SIN || p.n_red > MAX_RED)
        fail(NBG_NOT_IMPLEMENTED, "planner: region exceeds kernel argument limits");

    KArgs args;
    memset(&args, 0, sizeof args);
    args.n = n;
    for (int k = 0; k < p.n_in; k++) args.in[k] = B.in_nodes[k]->buf->d;
    // outputs
    std::vector<BufP> obufs;
    for (int k = 0; k < p.n_out; k++) {
        const NodeP &x = B.out_nodes[k];
        const MatP &sc = B.out_scatter[k];
        auto tg = c.out_targets.find(x.get());
        BufP b;
        if (tg != c.out_targets.end()) {
            // caller-provided destination (multi-GPU exchange buffer): out[map[i]], map < 0 skips
            b = tg->second.buf;
            args.oscat[k] = tg->second.alim >= 0 ? nullptr : tg->second.map;
            args.ooff[k] = tg->second.aoff;
            args.olim[k] = tg->second.alim;
            if (!tg->second.peers.empty()) {
                if (args.npeer || tg->second.peers.size() > (size_t)MAX_PEER) fail(NBG_NOT_IMPLEMENTED, "planner: peer outputs");
                args.npeer = (int)tg->second.peers.size();
                for (int q = 0; q < args.npeer; q++) args.peer[q] = tg->second.peers[q];
            }
        } else {
            int64_t len = sc ? sc->plan->ncols_g : n;
            b = alloc_buf(c, (size_t)len * type_size(x->type));
            if (sc) args.oscat[k] = (const int *)sc->plan->perm->d;
        }
        obufs.push_back(b);
        args.out[k] = b->d;
        c.stats.vectors_materialized++;
        c.stats.bytes_materialized += b->bytes;
    }
    std::vector<SlotP> rslots;
    for (int k = 0; k < p.n_red; k++) {
        SlotP s = alloc_slot(c);
        rslots.push_back(s);
        args.racc[k] = s->dptr();
    }
    for (int k = 0; k < p.n_sin; k++) args.sin[k] = B.sin[k]->dptr();

    // alignment decides the vectorised ewise skeleton
    bool vec = true;
    for (int k = 0; k < p.n_in; k++) vec = vec && (((uintptr_t)args.in[k]) % 16 == 0);
    for (int k = 0; k < p.n_out; k++) vec = vec && (((uintptr_t)args.out[k]) % 16 == 0);
    for (int k = 0; k < p.n_out; k++) vec = vec && (((uintptr_t)args.oscat[k]) % 16 == 0);   // scatter maps: int4 loads
    p.vec = p.spmv ? true : vec;
    // TMA-staged elementwise skeleton (codegen gen_ewise), opt-in: NBG_EWISE_TMA=1.  Measured on
    // C2: fp32 29.8 us vs 29.1 with the register skeleton, fp64 56.1 vs 56.4 -- the
    // register skeleton already keeps enough bytes in flight at this size, so it stays the default
    p.tma = false;
    if (!p.spmv && p.vec) {
        const char *e = getenv("NBG_EWISE_TMA");   // read per region (tests switch it in-process)
        const int et = (e && *e) ? (e[0] == '1' ? 1 : 0) : -1;
        int nslots = 0, sumsz = 0;
        std::vector<bool> seen_slot(p.n_in, false);
        for (const Ins &in : p.ins)
            if (in.k == Ins::LD_VEC && in.slot >= 0 && in.slot < p.n_in && !seen_slot[in.slot]) {
                seen_slot[in.slot] = true;
                nslots++;
                sumsz += (int)type_size(in.t);
            }
        const bool fits = nslots >= 1 && nslots <= 4 && sumsz <= 32;
        p.tma = fits && et == 1;
    }

    long long items = 0;
    long long xwin = 0;   // bytes of the gathered vector (persisting L2 window of large ones)
    if (p.spmv) {
        Node &mx = *B.mxv;
        Mat &A = *mx.A;
        if (!A.plan) gpu_build_spmv_plan(c, A);
        const NodeP &u = mx.a;
        p.sp.add = mx.add;
        p.sp.mul = mx.mul;
        p.sp.T = mx.type;
        p.sp.xt = u->type;
        p.sp.at = A.type;
        p.sp.has_vals = (bool)A.vals;
        B.imm[0] = A.iso;
        B.imm[1] = mx.c0;
        args.rowptr = (const long long *)A.plan->grp->d;      // group-padded layout (graph.cu plan)
        args.colidx = (const int *)A.plan->cg->d;
        args.aval = A.vals ? A.plan->vals_g->d : nullptr;
        args.x = B.mxv_x->d;
        args.tiles = (const int *)(A.plan->tiles ? A.plan->tiles->d : nullptr);
        args.chunks = (const int *)(A.plan->chunks ? A.plan->chunks->d : nullptr);
        args.longs = (const int *)(A.plan->longs ? A.plan->longs->d : nullptr);
        args.counters = (int *)(A.plan->counters ? A.plan->counters->d : nullptr);
        args.partials = (double *)(A.plan->partials ? A.plan->partials->d : nullptr);
        args.ntiles = A.plan->ntiles;
        args.nchunks = A.plan->nchunks;
        spmv_variant((int)type_size(u->type), (A.plan->relabel ? A.plan->ncols_g : A.ncols) * (long long)type_size(u->type), &p.nt,
                     &p.hot_kb);
        const long long nw = p.nt / 32;
        items = (A.plan->ntiles + A.plan->nchunks + nw - 1) / nw;   // one task per warp
        args.nnz = 4 * A.plan->ngroups;
        args.hc = A.plan->relabel ? A.plan->ncols_g : A.ncols;   // clamped to the kernel's cache below
        xwin = (A.plan->relabel ? A.plan->ncols_g : A.ncols) * (long long)type_size(u->type);
        // two-phase column-blocked plan (large relabelled matrices, 4/8-byte gathered elements)
        TpPlan *T = (!A.vals && n > 0) ? gpu_tp_plan(c, A, (int)type_size(u->type), c.num_sms) : nullptr;
        // lane-per-row skeleton for low-skew matrices (SURVEY 8(a) K4 notes), NBG_SPMV_LPR overrides
        const int lm = spmv_lpr_mode();
        if (!T && (lm == 1 || (lm == -1 && A.plan->low_skew))) {
            p.lpr = true;
            p.nt = p.hot_kb = 0;
            items = (n + 255) / 256;
        }
        // row-binned skeleton (DESIGN.md §7 "row-binned SpMV") for large skewed matrices without
        // values (C4 165 vs 178 us, C5 3.73 vs 3.90 ms per sweep; small ones keep the task skeleton:
        // C1 21.9 vs 14.9 us).  The choice does not depend on the gather layout, so relabelled and
        // plain layouts keep identical sums.  NBG_SPMV_RB overrides (1: any matrix without values, 0: never)
        p.rb = false;
        const int rbm = spmv_rb_mode();
        if (!T && !p.lpr && !A.vals && (rbm == 1 || (rbm == -1 && !A.plan->low_skew && A.nnz >= (1ll << 19)))) {
            RbPlan *R = gpu_rb_plan(c, A);
            if (R) {
                p.rb = true;
                p.vec = vec;   // the epilogue uses 16-byte vector loads when every buffer allows them
                char md = spmv_rb_epi_mode();
                if (md == 'p' && !R->pipe_ok) md = 'b';
                p.rb_inline = md == 'i';
                p.rb_pipe = md == 'p';
                int64_t nt = 0;
                args.rb_tasks = rb_task_list(c, *R, md, n, &nt);
                args.rb_ntasks = nt;
                args.rb_done = R->done ? (unsigned long long *)R->done->d : nullptr;
                args.rb_gcnt = R->gcnt ? (const int *)R->gcnt->d : nullptr;
                args.rb_ngrp = R->ngrp;
                args.rb_gsize = R->gsize;
                args.rb_sell = (const int *)R->sell->d;
                args.rb_srow = (const int *)R->srow->d;
                args.rb_swid = (const int *)R->swid->d;
                args.rb_lrows = (const int *)R->lrows->d;
                args.rb_mask = (const unsigned *)R->mask->d;
                args.rb_tot = R->tot->d;
                args.rb_bar = (unsigned *)R->bar->d;

                items = 1ll << 40;   // persistent: one CTA per SM (clamped to the kernel's grid_cap)
            }
        }
        if (T) {
            p.tp = true;
            p.nt = p.hot_kb = 0;
            args.rowslot = (const long long *)T->rowslot->d;
            args.part = T->part->d;
            items = (n + 127) / 128 / 8 + 1;      // phase 2: 128-row tiles, 8 warps per CTA
        }
        // task skeleton on a matrix whose warp tasks would not fill the SMs at the default CTA size
        // (C1: 48 tasks in 2 CTAs of 768 threads): 256-thread CTAs spread them over more SMs and
        // shorten each CTA's block-level finish (C1 sweep kernel 14.8 -> 12.7 us, 0.43 -> 0.49
        // GTEPS/iter; 32 / 64 / 128 threads measured no better).  The task order and every row's
        // summation order are those of the task plan, independent of the CTA size.
        if (!p.tp && !p.lpr && !p.rb && !spmv_threads_overridden() && p.nt > 256 &&
            A.plan->ntiles + A.plan->nchunks < (long long)c.num_sms * (p.nt / 32)) {
            p.nt = 256;
            items = (A.plan->ntiles + A.plan->nchunks + 7) / 8;
        }
    } else {
        items = (n + 1023) / 1024;
    }
    for (int k = 0; k < p.n_imm; k++) args.imm[k] = B.imm[k];

    if (p.tp) {
        // ---- phase 1: per-(row, column block) partial sums; its kernel depends on the semiring only
        Mat &A = *B.mxv->A;
        TpPlan *T = gpu_tp_plan(c, A, (int)type_size(p.sp.xt), c.num_sms);
        std::ostringstream k1;
        k1 << "TP1|" << p.sp.add << "," << p.sp.mul << "," << p.sp.T << "," << p.sp.xt << "," << p.sp.at << "|" << T->S << "|"
           << spmv_threads((int)type_size(p.sp.xt));
        KernelP kp1;
        auto it1 = c.plans.find(k1.str());
        if (it1 == c.plans.end()) {
            char nm[48];
            snprintf(nm, sizeof nm, "nbg_tp1_%016llx", (unsigned long long)hash_str(k1.str()));
            int smem = 0;
            std::string src = codegen_tp1(p.sp, nm, (int)type_size(p.sp.xt), T->S, &smem);
            kp1 = jit_compile(c, src, nm, true, smem, spmv_threads((int)type_size(p.sp.xt)));
            c.plans[k1.str()] = kp1;
            c.stats.plans_built++;
        } else {
            kp1 = it1->second;
            c.stats.plan_hits++;
        }
        KArgs a1 = args;
        a1.rowptr = (const long long *)T->grp->d;
        a1.colidx = (const int *)T->cg->d;
        a1.tiles = (const int *)T->tasks->d;
        a1.chunks = (const int *)T->chunks->d;
        a1.longs = (const int *)(T->longs ? T->longs->d : nullptr);
        a1.counters = (int *)(T->counters ? T->counters->d : nullptr);
        a1.partials = (double *)(T->partials ? T->partials->d : nullptr);
        a1.tblk = (const int *)T->tblk->d;
        a1.cta = (const int *)T->cta->d;
        a1.pslot = (const int *)T->slot->d;
        a1.part = T->part->d;
        a1.S = T->S;
        a1.ncols_g = A.plan->ncols_g;
        a1.nnz = 4 * T->ngroups;
        if (T->ntasks > 0) launch(c, *kp1, a1, T->ncta, "spmv", xwin);
    }

    double tsig0 = now_ns();
    std::string sig = p.signature();
    KernelP kern;
    auto it = c.plans.find(sig);
    if (it == c.plans.end()) {
        char nm[48];
        snprintf(nm, sizeof nm, "nbg_%s_%016llx", p.tp ? "tp2" : (p.spmv ? (p.lpr ? "spmvl" : (p.rb ? "spmvr" : "spmv")) : "ewise"), (unsigned long long)hash_str(sig));
        int smem = 0, hot = 0;
        std::string src = codegen(p, nm, &smem, &hot);
        kern = jit_compile(c, src, nm, p.spmv && !p.tp && !p.lpr, smem, (p.spmv && !p.tp && !p.lpr) ? p.nt : 0);
        kern->hot = hot;
        c.plans[sig] = kern;
        c.stats.plans_built++;
    } else {
        kern = it->second;
        c.stats.plan_hits++;
        if (g_prof.on) { g_prof.t[4] += now_ns() - tsig0; g_prof.n[4]++; }
    }
    if (p.spmv && !p.tp) {
        if (args.hc > kern->hot) args.hc = kern->hot;
    }

    {
        PTimer pt(5);
        if (dbg()) {
            fprintf(stderr, "[nbg] launch %s n=%lld items=%lld", kern->name.c_str(), (long long)n, items);
            for (int k = 0; k < p.n_in; k++) fprintf(stderr, " in%d=%p", k, args.in[k]);
            for (int k = 0; k < p.n_out; k++) fprintf(stderr, " out%d=%p", k, args.out[k]);
            for (int k = 0; k < p.n_sin; k++) fprintf(stderr, " sin%d=%p", k, (const void *)args.sin[k]);
            for (int k = 0; k < p.n_red; k++) fprintf(stderr, " racc%d=%p", k, (void *)args.racc[k]);
            fprintf(stderr, "\n");
        }
        if (items > 0 && n > 0) launch(c, *kern, args, items, p.tp ? "spmv_p2" : (p.spmv ? "spmv" : "ewise"), p.spmv && !p.tp ? xwin : 0);
    }

    // provenance of the written buffers (for hints): base signature + output index
    // (set by the caller through B.prog before hints were appended)
    for (int k = 0; k < p.n_out; k++) {
        Node &x = *B.out_nodes[k];
        if (c.out_targets.count(&x)) continue;   // written into a target only: the node stays pending
        x.buf = obufs[k];
        x.kind = VKind::FULL;
        x.mat = true;
    }
    PTimer pt_rm(9);
    ProdEvP pe;
    for (int k = 0; k < p.n_red; k++) {
        Node &x = *B.red_nodes[k];
        x.slot = rslots[k];
        x.sfmt = (SFmt)p.reds[k].fmt;
        x.mat = true;
        if (x.user_refs > 0) {   // so a later get() only waits on this kernel (one event per launch)
            if (!pe) pe = record_prod_event(c);
            mark_readable(c, x.slot, pe);
        }
    }
    (void)hint_outs;
}

// ---------------------------------------------------------------- materialise

static int64_t root_len(const NodeP &r) {
    if (r->scalar) return r->a ? r->a->n : 0;
    if (r->op == Op::MXV) return r->A->nrows;
    return r->n;
}

// `len`: the index-space length of the group (root_len at grouping time; a root materialised by a
// prerequisite pass in the meantime has dropped its inputs, so its root_len is no longer valid)
static void materialize_group(Ctx &c, const std::vector<NodeP> &roots, int64_t len) {
    const bool nb = c.mode == NBG_NONBLOCKING;
    for (int guard = 0; guard < 256; guard++) {
        Builder B(c);
        bool ok = true;
        {
            PTimer pt(1);
            for (const NodeP &r : roots) {
                if (r->mat) continue;
                if (r->scalar) ok = B.add_reduction(r) && ok;
                else ok = B.add_vector_output(r) && ok;
            }
        }
        if (!B.prereq.empty()) {
            std::vector<NodeP> todo;
            for (const NodeP &p : B.prereq) {
                if (p->mat) continue;
                if (nb && memo_bind(c, p)) continue;
                if (nb) {
                    auto cm = B.need_mx.find(p.get());
                    learn_hint(c, p, cm == B.need_mx.end() ? nullptr : cm->second);
                }
                todo.push_back(p);
            }
            if (!todo.empty()) materialize(c, todo);
            continue;
        }
        if (!ok) fail(NBG_PANIC, "planner: region incomplete without prerequisites");
        bool any = false;
        for (const NodeP &r : roots) any = any || !r->mat;
        if (!any) return;

        // liveness: pending nodes a user still holds are stored as well (nonblocking only)
        if (nb) {
            std::vector<NodeP> vis = B.visited;
            for (const NodeP &x : vis)
                if (!x->scalar && x->user_refs > 0 && !B.is_out.count(x.get())) B.add_vector_output(x);
        }
        const int nbase = (int)B.out_nodes.size();
        const uint64_t base_hash = B.prog.sig_hash();

        // speculative side outputs learned for this signature
        std::vector<HintOut> hint_outs;
        if (nb) {
            PTimer pt_h(2);
            for (int o = 0; o < nbase; o++) {
                auto h = c.hints.find({base_hash, o});
                if (h == c.hints.end()) continue;
                for (const Hint &hint : h->second) {
                    NodeP inst = instantiate(c, hint, B.out_nodes[o]);
                    if (!inst) continue;
                    MatP cons = hint.consumer.lock();
                    MatP scat;
                    if (cons && !inst->scalar) {
                        if (!cons->plan) gpu_build_spmv_plan(c, *cons);
                        if (cons->plan->relabel) {
                            if (cons->ncols != inst->n) continue;
                            scat = cons;
                        }
                    }
                    bool added = inst->scalar ? B.add_reduction(inst) : B.add_vector_output(inst, scat);
                    if (!added || !B.prereq.empty()) fail(NBG_PANIC, "planner: hint needs a prerequisite");
                    hint_outs.push_back(HintOut{inst, scat});
                    c.stats.side_outputs++;
                }
            }
        }

        int64_t n = B.mxv ? B.mxv->A->nrows : len;
        size_t nvis = B.visited.size();
        // structural keys of the base outputs (before they become leaves)
        std::vector<MKey> base_keys;
        {
            PTimer pt(3);
            if (nb) {
                for (int k = 0; k < nbase; k++) base_keys.push_back(memo_key(B.out_nodes[k].get()));
            }
        }
        run_region(c, B, hint_outs, n);
        const uint64_t seq = ++c.launch_seq;
        for (int k = 0; k < nbase; k++) {
            if (!B.out_nodes[k]->buf) continue;   // written into a caller's target only (stays pending)
            B.out_nodes[k]->buf->prod_sig = base_hash;
            B.out_nodes[k]->buf->prod_out = k;
            B.out_nodes[k]->buf->prod_seq = seq;
        }
        if (nb) {
            PTimer pt_m(6);
            // memoise every result (common subexpressions across waits, e.g. dinv across runs)
            for (int k = 0; k < nbase; k++)
                if (!c.out_targets.count(B.out_nodes[k].get())) memo_insert(c, base_keys[k], B.out_nodes[k]);
            // side outputs are keyed with R already materialised (the next sweep's lookup key)
            for (HintOut &h : hint_outs) {
                const MKey k = memo_key(h.node.get(), true, h.scatter.get());
                if (dbg()) fprintf(stderr, "[nbg] memo insert %s%s\n", h.scatter ? "(gather layout) " : "", node_key(h.node.get()).c_str());
                memo_insert(c, k, h.node);
            }
        }
        // elided intermediates = visited pending nodes that were not stored
        size_t stored = 0;
        for (const NodeP &x : B.visited)
            if (B.is_out.count(x.get())) stored++;
        c.stats.intermediates_elided += (nvis >= stored) ? (nvis - std::min(stored, nvis)) : 0;
        for (const NodeP &x : B.out_nodes)
            if (!c.out_targets.count(x.get())) drop_inputs(*x);
        for (const NodeP &x : B.red_nodes) drop_inputs(*x);
        c.stats.waits++;
        return;
    }
    fail(NBG_PANIC, "planner did not converge");
}

void materialize(Ctx &c, const std::vector<NodeP> &roots_in) {
    double t0 = now_ns();
    PTimer pt_all(7);
    {
        PTimer pt_pb(0);
        if (c.mode == NBG_NONBLOCKING) memo_purge(c);   // dead entries release their result buffers
    }
    std::vector<NodeP> roots;
    SmallSet<const Node *> seen;
    for (const NodeP &r0 : roots_in) {
        NodeP r = r0;
        if (r->mat) continue;
        if (r->scalar && r->op == Op::SAPPLY) {   // scalar ops are evaluated where they are used
            while (r && !r->mat && r->op == Op::SAPPLY) r = r->a;
            if (!r || r->mat) continue;
        }
        if (seen.insert(r.get()).second) roots.push_back(r);
    }
    if (roots.empty()) return;
    if (c.mode == NBG_NONBLOCKING) {
        PTimer pt_b(0);
        std::vector<NodeP> left;
        for (const NodeP &r : roots)
            if (!memo_bind(c, r)) left.push_back(r);
        roots.swap(left);
    }
    // regions reading sparse / bitset vectors run through the structured executor, one each
    {
        std::vector<NodeP> left;
        for (const NodeP &r : roots) {
            if (needs_structured(r)) materialize_structured(c, r);
            else left.push_back(r);
        }
        roots.swap(left);
    }
    // group by index-space length (one kernel per group)
    std::map<int64_t, std::vector<NodeP>> groups;
    for (const NodeP &r : roots) groups[root_len(r)].push_back(r);
    for (auto &g : groups) materialize_group(c, g.second, g.first);
    c.stats.host_plan_ns += (uint64_t)(now_ns() - t0);
    if (guard_enabled()) guard_check(c, "materialize (static kernels included)");
}

double scalar_read(Ctx &c, const NodeP &s) {
    if (!s->mat) {
        if (s->op == Op::SAPPLY) {
            double v = scalar_read(c, s->a);
            return host_round(s->type, host_unop(s->code, s->type, v, s->c0, s->c1));
        }
        materialize(c, {s});
    }
    if (s->sfmt == SFmt::HOST) return s->hval;
    Slot &sl = *s->slot;
    issue_readback(c, sl);
    NBG_CUDA(cudaEventSynchronize(sl.cev ? sl.cev->e : sl.ev));
    return host_round(s->type, slot_value(sl.hptr(), s->sfmt));
}

}  // namespace nbg
