#!/bin/bash
# round-2 fourth-session bundle: C5 cold-gather qualifier sweep, C1 lane-per-row knob, then the C4
# bench line / reference arm / launch list / ncu --set full at HEAD
set -u
O=gpurun_out/r2f; mkdir -p $O
for q in cg nc el; do
  NBG_SPMV_COLD=$q python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5_$q.json 2> $O/c5_$q.err
done
NBG_SPMV_LPR=1 python bench.py --workload c1 --no-cpu-baseline --no-e2e > $O/c1_lpr.json 2> $O/c1_lpr.err
python bench.py --workload c1 --no-cpu-baseline --no-e2e > $O/c1_def.json 2> $O/c1_def.err
python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:nbg_spmv -s 20 -c 1 -o $O/spmv_c4 \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c4.log 2>&1
for f in $O/c5_*.json $O/c1_*.json $O/bench_c4.json; do python - $f <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); r=d['roofline']
    print(sys.argv[1], d['value'], d['ms_per_step'], r.get('avg_launch_us'), r.get('frac'), d['clocks']['sm_mhz'], d.get('e2e',{}).get('value'))
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done > $O/summary.txt
echo MEASURE_DONE >> $O/summary.txt
