for rep in 1 2; do for u in 1 4; do for t in fp32 fp64; do
NBG_EWISE_UNROLL=$u timeout 200 python bench.py --workload c2 --dtype $t --steps 20 --warmup 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('unroll $u $t', d['value'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['avg_launch_us'], d['blocking']['kernel_speedup_fused_vs_blocking'])"
done; done; done
