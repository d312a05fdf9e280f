run() { env "$@" timeout 600 python bench.py --workload $W --steps $S --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > /tmp/o.json; python -c "import json; d=json.load(open('/tmp/o.json')); print('$W $*', d['value'], d['roofline']['avg_launch_us'])"; }
W=c4 S=5 run NBG_SPMV_WARM=0
W=c4 S=5 run NBG_SPMV_WARM=4096
W=c4 S=5 run NBG_SPMV_WARM=16384
W=c4 S=5 run NBG_SPMV_WARM=65536
W=c5 S=1 run NBG_SPMV_WARM=16384
