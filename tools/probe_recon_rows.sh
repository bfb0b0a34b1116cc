#!/bin/bash
# reconstruction tile heights: W r <= 8 at 512 rows; W r <= 32 at 1024 rows
mkdir -p gpurun_out; rm -f gpurun_out/rr.txt
for v in base r8_512 r16_1024; do
  if [ $v = base ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=alt_libs/$v.so; fi
  echo "$v $(timeout 300 python tools/recon_probe.py --rank 4 --worlds 2,4,8 2>&1 | tail -1) $(timeout 300 python tools/recon_probe.py --rank 8 --worlds 1 2>&1 | tail -1) $(timeout 300 python tools/recon_probe.py --rank 16 --worlds 1 2>&1 | tail -1)" >> gpurun_out/rr.txt
done
exit 0
