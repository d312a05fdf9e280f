#!/bin/bash
for mb in 4 6 8; do for dt in fp32 fp64; do
  NBG_EWISE_MINBLOCKS=$mb timeout 120 python bench.py --workload c2 --dtype $dt 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('minblocks $mb $dt', d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['avg_launch_us'])"
done; done
