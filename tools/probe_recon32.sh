#!/bin/bash
# W r = 17..32 reconstruction tile rows (256 default; 128; 64): the N = 8, r = 4 case
mkdir -p gpurun_out; rm -f gpurun_out/r32.txt
for v in base; do
  if [ $v = base ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=alt_libs/$v.so; fi
  echo "$v $(timeout 300 python tools/recon_probe.py --rank 4 --worlds 8 2>&1 | tail -1) $(timeout 300 python tools/recon_probe.py --rank 8 --worlds 4 2>&1 | tail -1)" >> gpurun_out/r32.txt
done
timeout 300 python -m pytest tests/test_gpu_recon.py tests/test_gpu_engine.py tests/test_gpu_dp.py -x -q -p no:cacheprovider > gpurun_out/r32_pytest.log 2>&1
exit 0
