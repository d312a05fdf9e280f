python -m paper_2509_14211_b200.build > /dev/null 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "mxv or pagerank or config or fullsize or sweep" 2>&1 | tail -1
run() { env "$@" timeout 600 python bench.py --workload $W --steps $S --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > /tmp/o.json; python -c "import json; d=json.load(open('/tmp/o.json')); print('$W $*', d['value'], d['roofline']['avg_launch_us'])"; }
W=c4 S=20 run NBG_SPMV_V8=1
W=c4 S=20 run NBG_SPMV_V8=0
W=c4 S=20 run NBG_SPMV_V8=1
W=c4 S=20 run NBG_SPMV_V8=0
W=c5 S=1 run NBG_SPMV_V8=1
W=c5 S=1 run NBG_SPMV_V8=0
