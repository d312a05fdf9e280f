#!/bin/bash
# C1 launch-shape sweep: threads per CTA of the task skeleton (NBG_SPMV_THREADS), bench lines only
mkdir -p gpurun_out
for t in 768 256 128 64 32; do
  NBG_SPMV_THREADS=$t python bench.py --workload c1 --no-cpu-baseline --no-e2e > gpurun_out/c1_t$t.json 2>gpurun_out/c1_t$t.err
done
for t in 128 64; do
  NBG_SPMV_THREADS=$t timeout 600 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/c1_par_t$t.log 2>&1
done
