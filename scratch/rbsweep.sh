# usage: bash scratch/rbsweep.sh TAG "ENV1" "ENV2" ... -- C4 bench (20 steps) per env setting; one line each
set -u
T=$1; shift; O=gpurun_out/$T; mkdir -p $O
for e in "$@"; do
  f=$O/$(echo "$e" | tr ' =' '_-').json
  env NBG_SPMV_RB=1 $e timeout 600 python bench.py --workload ${WL:-c4} --steps ${STEPS:-20} --no-cpu-baseline --no-e2e > $f 2> $f.err
  python -c "
import json,sys
d=json.load(open('$f')); r=d['roofline']
print('$e', d['value'], r['avg_launch_us'], r['frac'], d['clocks']['sm_mhz'])" >> $O/summary.txt 2>&1
done
echo DONE >> $O/summary.txt
