python -m paper_2509_14211_b200.build > /dev/null 2>&1
run() { env "$@" timeout 600 python bench.py --workload $W --steps $S --warmup 3 --no-cpu-baseline --no-e2e 2>/tmp/e.txt > /tmp/o.json; python -c "import json; d=json.load(open('/tmp/o.json')); print('$W $*', d['value'], d['roofline']['avg_launch_us'])" || tail -3 /tmp/e.txt; }
for mb in 0 48 56 64 72 80 64 0; do W=c5 S=2 run NBG_L2_PERSIST_MB=$mb; done
