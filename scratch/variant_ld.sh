# gather-load qualifier variants of the prelude's cold gather (restores the original at the end)
set -e
cp paper_2509_14211_b200/csrc/jit/prelude.cuh /tmp/prelude.keep
for q in "ld.global.cg.b32" "ld.global.ca.b32" "ld.global.cg.L2::64B.b32" "ld.global.cg.L2::128B.b32" "ld.global.nc.L2::128B.b32"; do
  sed "s/@!p ld.global.cg.b32 %0, \[%4\]/@!p $q %0, [%4]/" /tmp/prelude.keep > paper_2509_14211_b200/csrc/jit/prelude.cuh
  python -m paper_2509_14211_b200.build > /dev/null 2>&1
  timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > /tmp/o.json || true
  python -c "import json; d=json.load(open('/tmp/o.json')); print('$q', d['value'], d['roofline']['avg_launch_us'])" || echo "$q failed"
done
cp /tmp/prelude.keep paper_2509_14211_b200/csrc/jit/prelude.cuh
python -m paper_2509_14211_b200.build > /dev/null 2>&1
