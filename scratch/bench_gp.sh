#!/bin/bash
for gp in 0 1; do for t in ${THREADS:-768 640 512}; do
  NBG_SPMV_GPIPE=$gp NBG_SPMV_THREADS=$t timeout 120 python bench.py --no-cpu-baseline --no-e2e --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('gpipe $gp threads $t', d['value'], d['roofline']['avg_launch_us'])"
done; done
