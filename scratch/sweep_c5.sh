run() { env "$@" timeout 600 python bench.py --workload $W --steps $S --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > /tmp/o.json; python -c "import json; d=json.load(open('/tmp/o.json')); print('$W $*', d['value'], d['roofline']['avg_launch_us'])"; }
W=c5 S=1 run NBG_Z=0
W=c5 S=1 run NBG_SPMV_THREADS=1024 NBG_SPMV_HOT_KB=64
W=c5 S=1 run NBG_SPMV_THREADS=1024 NBG_SPMV_HOT_KB=32
W=c5 S=1 run NBG_SPMV_THREADS=1024 NBG_SPMV_HOT_KB=48
W=c5 S=1 run NBG_SPMV_THREADS=1024 NBG_SPMV_HOT_KB=80
W=c5 S=1 run NBG_SPMV_THREADS=768 NBG_SPMV_HOT_KB=64
