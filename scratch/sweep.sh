run() { env "$@" timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$*', d['value'], d['roofline']['avg_launch_us'])"; }
run NBG_SPMV_GENERIC=0
run NBG_SPMV_GENERIC=1
run NBG_SPMV_GENERIC=1 NBG_SPMV_THREADS=1024
run NBG_SPMV_GENERIC=1 NBG_SPMV_HOT_KB=96
