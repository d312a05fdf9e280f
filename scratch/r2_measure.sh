#!/bin/bash
# round-2 measurement bundle (run under gpurun from the repo root): bench lines of every config
# with clock records, then the C4 launch list and one ncu --set full capture of the fused sweep
set -u
mkdir -p gpurun_out/r2f
python bench.py > gpurun_out/r2f/bench_c4.json 2> gpurun_out/r2f/bench_c4.err
python bench.py --workload c1 --no-cpu-baseline > gpurun_out/r2f/bench_c1.json 2> gpurun_out/r2f/bench_c1.err
python bench.py --workload c3 --no-cpu-baseline > gpurun_out/r2f/bench_c3.json 2> gpurun_out/r2f/bench_c3.err
python bench.py --workload c2 --dtype fp32 > gpurun_out/r2f/bench_c2_fp32.json 2> gpurun_out/r2f/bench_c2_fp32.err
python bench.py --workload c2 --dtype fp64 > gpurun_out/r2f/bench_c2_fp64.json 2> gpurun_out/r2f/bench_c2_fp64.err
python bench.py --workload c5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2f/bench_c5.json 2> gpurun_out/r2f/bench_c5.err
python bench.py --workload sparse > gpurun_out/r2f/bench_sparse.json 2> gpurun_out/r2f/bench_sparse.err
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2f/bench_ref.json 2> gpurun_out/r2f/bench_ref.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2f/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2f/launches_c4.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r2f/ncu_launch.log 2>&1
echo MEASURE_DONE
