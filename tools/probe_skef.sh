#!/bin/bash
# EF fused into the P_raw partials (default for 4 < r <= 16) vs separate k_ef (EDGC_SKINNY_EF_OFF=1)
mkdir -p gpurun_out; rm -f gpurun_out/skef.txt
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_compress.py tests/test_gpu_debug_rank.py tests/test_gpu_dp.py -x -q -p no:cacheprovider > gpurun_out/skef_pytest.log 2>&1
rc=$?
echo "pytest exit $rc" >> gpurun_out/skef_pytest.log
[ $rc = 0 ] || exit 0
for r in 6 8 16; do
  for v in fused sep; do
    if [ $v = sep ]; then export EDGC_SKINNY_EF_OFF=1; else unset EDGC_SKINNY_EF_OFF; fi
    echo "$v $r $(timeout 240 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{')" >> gpurun_out/skef.txt
  done
done
unset EDGC_SKINNY_EF_OFF
for r in 8 16; do
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/skef_r$r.csv python bench.py --rank $r --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --entropy off > /dev/null 2>&1
done
exit 0
