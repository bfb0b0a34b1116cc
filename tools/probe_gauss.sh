#!/bin/bash
# Gaussian pass variants: float4 loads in flight per thread (4 default, 2, 8), 592 blocks x 8
mkdir -p gpurun_out; rm -f gpurun_out/ga.txt
for rep in 1 2; do
for v in base gu8; do
  if [ $v = base ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=alt_libs/$v.so; fi
  echo "$v $(timeout 300 python tools/gauss_probe.py 2>&1 | tail -1)" >> gpurun_out/ga.txt
done
done
exit 0
