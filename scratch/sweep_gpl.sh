set -e
python -m paper_2509_14211_b200.build > /dev/null 2>&1
NBG_SPMV_GPL=4 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x -k "mxv or pagerank or config or lane or fullsize" 2>&1 | tail -2
NBG_SPMV_GPL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "mxv or config" 2>&1 | tail -2
for cfg in 2:1024 4:1024 4:768 4:512 1:1024 2:1024; do G=${cfg%%:*}; T=${cfg##*:};
  NBG_SPMV_GPL=$G NBG_SPMV_THREADS=$T timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > /tmp/o.json || true
  python -c "import json; d=json.load(open('/tmp/o.json')); print('G $G T $T', d['value'], d['roofline']['avg_launch_us'])" || true
done
