#!/bin/bash
for kb in ${HOTS:-64 96 128 160 192}; do for t in ${THREADS:-768}; do
  NBG_SPMV_HOT_KB=$kb NBG_SPMV_THREADS=$t timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hot $kb KB threads $t', d['value'], d['roofline']['avg_launch_us'])"
done; done
