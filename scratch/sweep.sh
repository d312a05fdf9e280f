run() { env "$@" timeout 600 python bench.py --workload $W --steps $S --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > /tmp/o.json; python -c "import json; d=json.load(open('/tmp/o.json')); print('$W $*', d['value'], d['roofline']['avg_launch_us'])"; }
W=c3 S=3 run NBG_LPR_UG=2
W=c3 S=3 run NBG_LPR_UG=4
W=c3 S=3 run NBG_LPR_UG=1
W=c3 S=3 run NBG_LPR_UG=4
