#!/bin/bash
# TcEF prefetch depth A/B (default: 3 slices, 1 operand stage; pfd2 = the earlier 2 / 2; pfd4)
mkdir -p gpurun_out
rm -f gpurun_out/tcef.txt
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_compress.py tests/test_gpu_debug_rank.py -x -q -p no:cacheprovider > gpurun_out/tcef_pytest.log 2>&1
rc=$?
echo "pytest exit $rc" >> gpurun_out/tcef_pytest.log
[ $rc = 0 ] || exit 0
for v in base pfd2 pfd4; do
  if [ $v = base ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=alt_libs/$v.so; fi
  for r in 32 128; do
    echo "$v $r $(timeout 240 python bench.py --steps 12 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{')" >> gpurun_out/tcef.txt
  done
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:TcEF --csv --log-file gpurun_out/tcef_$v.csv python bench.py --rank 64 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --entropy off > /dev/null 2>&1
done
exit 0
