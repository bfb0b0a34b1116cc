#!/bin/bash
# W r = 8 reconstruction tile rows (64 default, 128, 256)
mkdir -p gpurun_out; rm -f gpurun_out/r8.txt
for v in base r8r128 r8r256; do
  if [ $v = base ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=alt_libs/$v.so; fi
  echo "$v $(timeout 300 python tools/recon_probe.py --rank 4 --worlds 2 2>&1 | tail -1) $(timeout 300 python tools/recon_probe.py --rank 8 --worlds 1 2>&1 | tail -1)" >> gpurun_out/r8.txt
done
exit 0
