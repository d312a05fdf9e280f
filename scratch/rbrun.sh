# usage: bash scratch/rbrun.sh TAG [tests] [ncu]  -- rb tests, C4 bench rb vs single-pass, optional ncu of the rb sweep
set -u
T=$1; O=gpurun_out/$T; mkdir -p $O
if [ "${2:-}" = "tests" ]; then
  timeout 900 python -m pytest tests/test_gpu_rowbinned.py -x -q > $O/t_rb.log 2>&1; echo "rb tests rc=$?" >> $O/t_rb.log
fi
NBG_SPMV_RB=1 timeout 300 python bench.py --steps 20 --no-cpu-baseline --no-e2e > $O/c4_rb.json 2> $O/c4_rb.err
if [ "${3:-}" = "ncu" ]; then
  NBG_SPMV_RB=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:nbg_spmvr -s 20 -c 1 -o $O/rb_c4 \
     python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu.log 2>&1
fi
echo DONE
