run() { env "$@" timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > /tmp/o.json; python -c "import json; d=json.load(open('/tmp/o.json')); print('$*', d['value'], d['roofline']['avg_launch_us'])"; }
run NBG_SPMV_IDXLD=cs
run NBG_SPMV_IDXLD=na
run NBG_SPMV_IDXLD=cg
run NBG_SPMV_IDXLD=na NBG_SPMV_HOT_KB=152
run NBG_SPMV_IDXLD=cs
