run() { env "$@" timeout 600 python bench.py --workload $W --steps $S --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > /tmp/o.json; python -c "import json; d=json.load(open('/tmp/o.json')); print('$W $*', d['value'], d['roofline']['avg_launch_us'])"; }
W=c4 S=5 run NBG_X=default
W=c4 S=5 run NBG_SPMV_TASKG=256 NBG_SPMV_LONGG=256 NBG_SPMV_CHUNKG=256
W=c4 S=5 run NBG_SPMV_CHUNKG=1024
W=c4 S=5 run NBG_SPMV_CHUNKG=256
W=c4 S=5 run NBG_SPMV_TASKG=384 NBG_SPMV_LONGG=384
W=c4 S=5 run NBG_SPMV_LONGG=256
