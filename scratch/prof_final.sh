#!/bin/bash
# round-end profile bundle: bench line, ncu launch list of the bench command, ncu --set full of one C4 sweep (steady state)
python bench.py > gpurun_out/bench_r1z.json 2> gpurun_out/bench_r1z.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1z.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_z.log 2>&1
python scratch/prof_c4.py > gpurun_out/prof_c4.log 2>&1 && \
ncu --set full --cache-control none --clock-control none --import-source on -k regex:nbg_spmv -s 30 -c 1 -o gpurun_out/spmv_r1z python scratch/prof_c4.py > gpurun_out/ncu_full_z.log 2>&1
