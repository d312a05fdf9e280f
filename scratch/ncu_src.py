"""Top stall lines of an ncu report's SASS source page: python scratch/ncu_src.py rep kernel_regex [N]"""
import csv, subprocess, sys, io
rep, k = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k", "regex:" + k, "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
si, ai, ii = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
body = []
for r in rows[2:]:
    if len(r) != len(h) or r[0] == "Address":
        if body: break
        continue
    body.append(r)
num = lambda s: float(s) if s.replace('.', '', 1).isdigit() else 0.0
tot = sum(num(r[ai]) for r in body)
print("lines", len(body), "total samples", tot)
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
agg = {c: sum(num(r[h.index(c)]) for r in body) for c in cols}
print("  ".join(f"{c[6:]}={100*v/tot:.0f}%" for c, v in sorted(agg.items(), key=lambda x: -x[1]) if v > tot / 100))
top = sorted(range(len(body)), key=lambda i: -num(body[i][ai]))[:N]
for i in sorted(top):
    r = body[i]
    st = sorted(((c[6:], num(r[h.index(c)])) for c in cols), key=lambda x: -x[1])[:2]
    print(f"{i:5d} {100*num(r[ai])/tot:5.1f}% ex={r[ii]:>9} {st[0][0]}:{st[0][1]:.0f} {st[1][0]}:{st[1][1]:.0f}  {r[si].strip()[:80]}")
