set -e
cp paper_2509_14211_b200/csrc/jit/prelude.cuh /tmp/prelude.keep
sed "s/ld.global.nc.b32 %0, \[%4\]/ld.global.cg.b32 %0, [%4]/; s/ld.global.nc.b64 %0, \[%4\]/ld.global.cg.b64 %0, [%4]/" /tmp/prelude.keep > paper_2509_14211_b200/csrc/jit/prelude.cuh
python -m paper_2509_14211_b200.build > /dev/null 2>&1
for cfg in 1024:144 1024:152 1024:160 1024:168 768:160 1024:144; do thr=${cfg%%:*}; hk=${cfg##*:};
  NBG_SPMV_THREADS=$thr NBG_SPMV_HOT_KB=$hk timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null > /tmp/o.json
  python -c "import json; d=json.load(open('/tmp/o.json')); print('cg $thr hot $hk', d['value'], d['roofline']['avg_launch_us'])"
done
cp /tmp/prelude.keep paper_2509_14211_b200/csrc/jit/prelude.cuh
python -m paper_2509_14211_b200.build > /dev/null 2>&1
