# fold `ncu --set full` captures of sweep kernels into profiles/ncu_summary.json (traffic + L2
# sectors per launch, read by bench.py) and write one detail JSON per workload
import csv, io, json, subprocess, sys
ROOT = __file__.rsplit("/scratch/", 1)[0]
WANT = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors.sum", "lts__t_sector_hit_rate.pct", "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "sm__cycles_active.avg", "gpc__cycles_elapsed.max"]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "sector": 1, "": 1}


def num(v, u):
    return float(v.replace(",", "")) * SCALE.get(u, 1)


summ_path = f"{ROOT}/profiles/ncu_summary.json"
summ = json.load(open(summ_path))
for arg in sys.argv[1:]:          # workload=report.ncu-rep[:note]
    w, rest = arg.split("=", 1)
    rep, _, note = rest.partition(":")
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    get = {h: (v, u) for h, u, v in zip(hdr, units, vals)}
    det = {k: get[k][0] + (" " + get[k][1] if get[k][1] else "") for k in WANT if k in get}
    json.dump(det, open(f"{ROOT}/profiles/r2_ncu_summary_{w}.json", "w"), indent=1)
    dram = num(*get["dram__bytes_read.sum"]) + num(*get["dram__bytes_write.sum"])
    summ[w] = {"dram_bytes_per_launch": dram, "lts_sectors_per_launch": num(*get["lts__t_sectors.sum"]),
               "round": "r2", "detail": f"profiles/r2_ncu_summary_{w}.json", "note": note}
    print(w, det.get("gpu__time_duration.sum"), "dram", dram, "lts", get["lts__t_sectors.sum"])
json.dump(summ, open(summ_path, "w"), indent=1)
