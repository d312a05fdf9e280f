python -m paper_2509_14211_b200.build > /dev/null 2>&1
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x 2>&1 | tail -1
for W in c5 c4; do S=2; [ $W = c4 ] && S=20; timeout 600 python bench.py --workload $W --steps $S --warmup 3 --no-cpu-baseline > gpurun_out/bench_l2_$W.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_l2_$W.json')); print('$W', d['value'], d['ms_per_step'], d['roofline']['avg_launch_us'], d['roofline']['frac'])"; done
