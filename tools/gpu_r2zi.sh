#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_recon.py -x -q -p no:cacheprovider > gpurun_out/zj_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/zj_pytest.log
timeout 1200 python bench.py --model 12.1B --rank 256 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/zj_12b.log 2>&1
timeout 1200 python bench.py --model 12.1B --rank 256 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline --entropy off > gpurun_out/zj_12b_off.log 2>&1
timeout 600 python bench.py --rank 128 --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/zj_r128.log 2>&1
exit 0
timeout 300 python tools/plan_prof.py --reps 3 --ahead > gpurun_out/zj_plan.log 2>&1
