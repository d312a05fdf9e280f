"""Summaries under profiles/ from a round's ncu captures (run here, no GPU):
   python scratch/ncu_summ.py <full.ncu-rep> <launches.csv> <round-tag> <workload>"""
import csv, io, json, subprocess, sys, collections, os
rep, launches, tag, workload = sys.argv[1:5]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, v = rows[0], rows[1], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum",
        "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "launch__block_size", "launch__grid_size", "sm__warps_active.avg.pct_of_peak_sustained_active"]
full = {}
for k in keys:
    if k in h:
        i = h.index(k)
        full[k] = {"value": v[i], "unit": units[i]}
def num(k):
    s = full[k]["value"].replace(",", "")
    u = full[k]["unit"]
    x = float(s)
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}.get(u, 1)
traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
# launch list: share of each kernel
lr = list(csv.reader(open(launches)))
hi = next(i for i, r in enumerate(lr) if "Kernel Name" in r)
H = lr[hi]
ki, vi = H.index("Kernel Name"), H.index("Metric Value")
agg = collections.OrderedDict()
for r in lr[hi + 1:]:
    name = r[ki]
    base = name.split("(")[0][:60]
    if base.startswith("nbg_spmv"): base = "nbg_spmv_*"
    if base.startswith("nbg_ewise"): base = "nbg_ewise_*"
    a = agg.setdefault(base, [0, 0.0])
    a[0] += 1; a[1] += float(r[vi].replace(",", ""))
tot = sum(a[1] for a in agg.values())
summary = {"round": tag, "workload": workload, "source": [os.path.basename(rep), os.path.basename(launches)],
           "top_kernel": {"name": "nbg_spmv_* (fused PageRank sweep)", "metrics": full,
                          "dram_bytes_per_launch": traffic},
           "launch_list_ns": {k: {"launches": a[0], "total_ns": a[1], "share": round(a[1] / tot, 4)} for k, a in agg.items()},
           "note": "launch list: ncu gpu__time_duration.sum per launch, cold-cache and serialised (shares, not absolutes); "
                   "includes graph generation / CSR build / plan build launches of the bench process"}
print(json.dumps(summary, indent=1))
p = os.path.join("profiles", "ncu_summary.json")
d = json.load(open(p)) if os.path.exists(p) else {}
d[workload] = {"dram_bytes_per_launch": traffic, "round": tag, "detail": f"profiles/{tag}_ncu_summary.json"}
json.dump(d, open(p, "w"), indent=1)
json.dump(summary, open(os.path.join("profiles", f"{tag}_ncu_summary.json"), "w"), indent=1)
