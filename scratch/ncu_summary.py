# summarise an ncu --set full report (one kernel) and an ncu launch list into a JSON dict
import csv, io, json, subprocess, sys

rep, launches, out = sys.argv[1], sys.argv[2], sys.argv[3]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2]
get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio"]
summ = {k: get[k][0] + (" " + get[k][1] if get[k][1] else "") for k in want if k in get}
# launch list: device time per kernel name over the captured launches
lrows = [r for r in csv.reader(open(launches)) if len(r) > 10]
lh = lrows[0]
ki, vi = lh.index("Kernel Name"), lh.index("Metric Value")
tot, by = 0.0, {}
for r in lrows[1:]:
    try:
        v = float(r[vi].replace(",", ""))
    except ValueError:
        continue
    name = r[ki].split("(")[0]
    key = "nbg_spmv" if name.startswith("nbg_spmv") else ("nbg_ewise" if name.startswith("nbg_ewise") else name[:40])
    by[key] = by.get(key, 0.0) + v
    tot += v
summ["launch_list_share"] = {k: round(v / tot, 4) for k, v in sorted(by.items(), key=lambda kv: -kv[1])[:8]}
summ["launch_list_launches"] = len(lrows) - 1
json.dump(summ, open(out, "w"), indent=1)
print(json.dumps(summ, indent=1))
