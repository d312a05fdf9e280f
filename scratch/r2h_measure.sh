#!/bin/bash
# round-2 fourth-session final bundle after the evict_first epilogue loads: GPU suite, C5 / C1 / C4 bench lines, reference arm, launch list, ncu --set full
set -u
mkdir -p gpurun_out/r2h; timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/r2h/gpu_suite.txt 2>&1
O=gpurun_out/r2h; mkdir -p $O
python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/c5_def.json 2> $O/c5_def.err
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
    print(sys.argv[1], d['value'], d['ms_per_step'], r.get('avg_launch_us'), r.get('frac'), d['clocks']['sm_mhz'], (d.get('e2e') or {}).get('value'))
except Exception as e: print(sys.argv[1], 'ERR', e)
PY
done > $O/summary.txt
echo MEASURE_DONE >> $O/summary.txt
