run() { env "$@" timeout 600 python bench.py --workload $W --steps $S --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > /tmp/o.json; python -c "import json; d=json.load(open('/tmp/o.json')); print('$W $*', d['value'], d['roofline']['avg_launch_us'])"; }
W=c5 S=1 run NBG_SPMV_HOT_KB=96
W=c5 S=1 run NBG_SPMV_HOT_KB=99
W=c5 S=1 run NBG_SPMV_HOT_KB=88
W=c5 S=1 run NBG_SPMV_HOT_KB=80
