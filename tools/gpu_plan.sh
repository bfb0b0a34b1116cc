#!/bin/bash
# sample-plan iteration on one GPU: parity tests, plan build timing, ncu launch list + full capture
#   bash tools/gpu_plan.sh TAG
T=${1:-x}
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_fused_entropy.py tests/test_gpu_ranks.py -x -q -p no:cacheprovider > gpurun_out/${T}_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/${T}_pytest.log
timeout 120 python tools/plan_prof.py --reps 5 > gpurun_out/${T}_plan.log 2>&1
timeout 120 python tools/plan_prof.py --reps 5 --ahead >> gpurun_out/${T}_plan.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/${T}_plan_ncu.csv python tools/plan_prof.py --reps 1 --ahead > gpurun_out/${T}_plan_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/${T}_plan_ncu_lat.csv python tools/plan_prof.py --reps 1 > /dev/null 2>&1
#timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_set_resolve|k_set_tail|k_walk" -c 3 \
#  -o gpurun_out/${T}_plan_full -f python tools/plan_prof.py --reps 1 --ahead > gpurun_out/${T}_ncu.log 2>&1
exit 0
