import sys; sys.path.insert(0, '.')
import numpy as np, importlib.util
from paper_2509_14211_b200 import nbg
from oracle import sparse as S
spec = importlib.util.spec_from_file_location("f", "tests/test_gpu_fuzz.py"); f = importlib.util.module_from_spec(spec); spec.loader.exec_module(f)
seed = 10
rng = np.random.default_rng(1000 + seed)
n = 3001
T = np.float64
leaves = [S.full((rng.integers(-8, 9, n) / 4.0).astype(T)), S.full((rng.integers(-8, 9, n) / 4.0).astype(T)), S.full((rng.integers(-8, 9, n) / 4.0).astype(T))]
prog = f._program(rng, 14)
exp = f._oracle(prog, leaves, T)
order = [int(a) for a in sys.argv[1].split(",")] if len(sys.argv) > 1 else [15]
c = nbg.nbg_init(nbg.NONBLOCKING, 0)
h = []; sc = {}
for k, ins in enumerate(prog):
    if ins[0] == "leaf": h.append(nbg.nbg_vector_from_dense(c, nbg.FP64, leaves[ins[1]].vals))
    elif ins[0] == "un": h.append(nbg.nbg_apply(c, nbg.FP64, ins[1], h[ins[2]], ins[3], ins[4]))
    elif ins[0] == "bin":
        fn = nbg.nbg_ewise_add if ins[1] == "add" else nbg.nbg_ewise_mult
        h.append(fn(c, nbg.FP64, ins[2], h[ins[3]], h[ins[4]]))
    else:
        s = nbg.nbg_reduce(c, nbg.FP64, "PLUS", h[ins[3]]); sc[k] = s
        h.append(nbg.nbg_apply_bind2nd(c, nbg.FP64, ins[1], h[ins[2]], s))
for k in order:
    i, x = nbg.nbg_vector_export_sparse(c, h[k])
    bad = np.nonzero(np.abs(x - exp[k].vals) > 1e-9 * np.maximum(1, np.abs(exp[k].vals)))[0]
    print("node", k, prog[k], "bad", bad.shape[0], "first", bad[:3], x[bad[:3]] if bad.size else "", exp[k].vals[bad[:3]] if bad.size else "")
for k, s in sc.items():
    print("scalar for node", k, nbg.nbg_scalar_get(c, s), "oracle", S.reduce("PLUS", exp[prog[k][3]], np.float64))
