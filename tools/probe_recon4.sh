#!/bin/bash
# W r <= 4 reconstruction tile rows (64 default, 128, 256): the headline's reconstruction, twice
mkdir -p gpurun_out; rm -f gpurun_out/r4.txt
for rep in 1 2; do
for v in base r4r128 r4r256; do
  if [ $v = base ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=alt_libs/$v.so; fi
  echo "$v $(timeout 300 python tools/recon_probe.py --rank 4 --worlds 1 --iters 20 2>&1 | tail -1)" >> gpurun_out/r4.txt
done
done
timeout 300 python -m pytest tests/test_gpu_recon.py tests/test_gpu_engine.py -x -q -p no:cacheprovider > gpurun_out/r4_pytest.log 2>&1
exit 0
