#!/bin/bash
# round 2, call B (1 GPU): set-mode plan resolve -- parity, plan timing (old vs new), bench, ncu launch list
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_entropy.py tests/test_gpu_fused_entropy.py \
  tests/test_gpu_ranks.py tests/test_gpu_engine.py -x -q -p no:cacheprovider > gpurun_out/b_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/b_pytest.log
timeout 300 python tools/plan_prof.py --reps 5 > gpurun_out/b_plan_set.log 2>&1
EDGC_PLAN_NOSET=1 timeout 300 python tools/plan_prof.py --reps 5 > gpurun_out/b_plan_old.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b_bench20.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/b_bench100.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/b_plan_ncu.csv python tools/plan_prof.py --reps 1 > gpurun_out/b_plan_ncu.log 2>&1
exit 0
