python -m paper_2509_14211_b200.build > /dev/null 2>&1
run() { env "$@" timeout 600 python bench.py --workload c4 --steps 30 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > /tmp/o.json; python -c "import json; d=json.load(open('/tmp/o.json')); print('c4 $*', d['value'], d['roofline']['avg_launch_us'])"; }
run NBG_SPMV_HOT_KB=192
run NBG_SPMV_HOT_KB=176
run NBG_SPMV_HOT_KB=160
run NBG_SPMV_THREADS=768
run NBG_SPMV_PF=0
run NBG_RELABEL=0
run NBG_SPMV_HOT_KB=192
