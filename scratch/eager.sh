mkdir -p gpurun_out/eager
NBG_PLAN_BUILD_PROFILE=1 timeout 300 python scratch/e2e_rb.py > gpurun_out/eager/e2e.log 2>&1
timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/eager/c4.json 2> gpurun_out/eager/c4.err
NBG_EAGER_PLAN=0 timeout 600 python bench.py --steps 20 --no-cpu-baseline > gpurun_out/eager/c4_lazy.json 2> gpurun_out/eager/c4_lazy.err
timeout 2700 python -m pytest tests -m gpu -q -x > gpurun_out/eager/suite.log 2>&1; echo "rc=$?" >> gpurun_out/eager/suite.log
