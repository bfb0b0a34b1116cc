#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_fused_entropy.py tests/test_gpu_ranks.py -x -q -p no:cacheprovider > gpurun_out/zk_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/zk_pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/zk_13.csv python tools/plan_prof.py --reps 1 --ahead > /dev/null 2>&1
EDGC_LIB_PATH=alt_libs/set14.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/zk_14.csv python tools/plan_prof.py --reps 1 --ahead > /dev/null 2>&1
for i in 1 2; do
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/zk_b13_$i.log 2>&1
EDGC_LIB_PATH=alt_libs/set14.so timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/zk_b14_$i.log 2>&1
done
exit 0
