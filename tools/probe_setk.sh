#!/bin/bash
# set-mode plan kernels: words per warp in k_set_tail, segments in flight in k_set_resolve
mkdir -p gpurun_out; rm -f gpurun_out/setk_*.csv gpurun_out/setk.txt
for v in base tw8 tw2 rb8 rb2; do
  if [ $v = base ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=alt_libs/$v.so; fi
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_set_" --csv --log-file gpurun_out/setk_$v.csv python tools/plan_prof.py --reps 1 --ahead > /dev/null 2>&1
  echo "$v $(timeout 120 python tools/plan_prof.py --reps 5 --ahead 2>/dev/null | tail -1)" >> gpurun_out/setk.txt
done
timeout 300 python -m pytest tests/test_gpu_sampling.py -x -q -p no:cacheprovider > gpurun_out/setk_pytest.log 2>&1
exit 0
