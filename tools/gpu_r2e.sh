#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_entropy.py tests/test_gpu_fused_entropy.py tests/test_gpu_ranks.py tests/test_gpu_dp.py -x -q -p no:cacheprovider > gpurun_out/e_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/e_pytest.log
timeout 300 python tools/plan_prof.py --reps 5 > gpurun_out/e_plan_set.log 2>&1
timeout 300 python tools/plan_prof.py --reps 5 --full-idx > gpurun_out/e_plan_full.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/e_plan_ncu.csv python tools/plan_prof.py --reps 1 > gpurun_out/e_plan_ncu.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/e_bench20.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/e_bench100.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --entropy off > gpurun_out/e_bench100_off.log 2>&1
exit 0
