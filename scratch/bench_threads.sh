#!/bin/bash
# SpMV block-size / groups-per-lane sweep on C4 (one bench line each)
for eg in ${EGS:-2 4}; do for t in ${THREADS:-1024 768 512}; do
  NBG_SPMV_EG=$eg NBG_SPMV_THREADS=$t timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('eg $eg threads $t', d['value'], d['roofline']['avg_launch_us'])"
done; done
