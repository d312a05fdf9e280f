python -m paper_2509_14211_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "timing or config1 or steady or bench" 2>&1 | tail -1
for W in c1 c4; do NBG_PLAN_PROFILE=1 timeout 300 python bench.py --workload $W --steps 20 --warmup 3 --no-cpu-baseline --no-e2e 2>/tmp/e.txt > /tmp/o.json; grep "args+launch\|total" /tmp/e.txt; python -c "import json; d=json.load(open('/tmp/o.json')); print('$W', d['value'], d['ms_per_step'], d['roofline']['avg_launch_us'], d['host_plan_us_per_wait'])"; done
