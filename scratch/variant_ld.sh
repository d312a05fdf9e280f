# builds and benches gather-load qualifier variants of the prelude (restores the original at the end)
set -e
cp paper_2509_14211_b200/csrc/jit/prelude.cuh /tmp/prelude.keep
for q in "ld.global.nc.b32" "ld.global.nc.L1::no_allocate.b32" "ld.global.cg.b32" "ld.global.nc.L1::evict_last.b32"; do
  sed "s/ld.global.nc.b32 %0, \[%4\]/$q %0, [%4]/" /tmp/prelude.keep > paper_2509_14211_b200/csrc/jit/prelude.cuh
  python -m paper_2509_14211_b200.build > /dev/null 2>&1
  timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print('$q', d['value'], d['roofline']['avg_launch_us'])"
done
cp /tmp/prelude.keep paper_2509_14211_b200/csrc/jit/prelude.cuh
python -m paper_2509_14211_b200.build > /dev/null 2>&1
