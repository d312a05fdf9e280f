#!/bin/bash
# round-2 third-session C4 / C5 bundle after the fused dangling mask: bench lines with clock records,
# the C4 launch list (the ncu --set full capture of the same kernel: gpurun_out/spmv_c4_m.ncu-rep)
set -u
O=gpurun_out/r2e; mkdir -p $O
python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('SMOKE_OK')" > $O/smoke.log 2>&1
echo MEASURE_DONE > $O/done
