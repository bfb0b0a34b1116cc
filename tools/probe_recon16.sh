#!/bin/bash
# W r = 9..32 reconstruction tile rows (256 default; 128; 512 for W r <= 16)
mkdir -p gpurun_out; rm -f gpurun_out/r16.txt
for v in base t16_128 t16_512 t32_128; do
  if [ $v = base ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=alt_libs/$v.so; fi
  echo "$v $(timeout 300 python tools/recon_probe.py --rank 4 --worlds 4,8 2>&1 | tail -1) $(timeout 300 python tools/recon_probe.py --rank 16 --worlds 1 2>&1 | tail -1)" >> gpurun_out/r16.txt
done
unset EDGC_LIB_PATH
timeout 300 python -m pytest tests/test_gpu_recon.py -x -q -p no:cacheprovider > gpurun_out/r16_pytest.log 2>&1
exit 0
