#!/bin/bash
# round-2 (third session, final) measurement bundle, run under gpurun from the repo root: bench lines of
# every config with clock records, the C4 launch list, ncu --set full of the C4 and C5 sweep kernels
set -u
O=gpurun_out/r2d; mkdir -p $O
python bench.py > $O/bench_c4.json 2> $O/bench_c4.err
python bench.py --workload c1 --no-cpu-baseline > $O/bench_c1.json 2> $O/bench_c1.err
python bench.py --workload c3 --no-cpu-baseline > $O/bench_c3.json 2> $O/bench_c3.err
python bench.py --workload c2 --dtype fp32 > $O/bench_c2_fp32.json 2> $O/bench_c2_fp32.err
python bench.py --workload c2 --dtype fp64 > $O/bench_c2_fp64.json 2> $O/bench_c2_fp64.err
python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/bench_c5.json 2> $O/bench_c5.err
python bench.py --workload sparse > $O/bench_sparse.json 2> $O/bench_sparse.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_ref.json 2> $O/bench_ref.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:nbg_spmv -s 20 -c 1 -o $O/spmv_c4 \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c4.log 2>&1
python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/plain_c5.log 2>&1 && \
ncu --set full --clock-control none -k regex:nbg_spmv -s 25 -c 1 -o $O/spmv_c5 \
    python bench.py --workload c5 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c5.log 2>&1
timeout 1300 python -m pytest tests -m gpu -q > $O/gpu_suite.txt 2>&1
echo MEASURE_DONE > $O/done
