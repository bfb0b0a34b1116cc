#!/bin/bash
# pass-1 (k_pass1t) wait-policy / stage variants: pass1_ab timing alone, twice each
mkdir -p gpurun_out; rm -f gpurun_out/p1v.txt
for rep in 1 2; do
  for v in base ps32 ps256 cs64 wh200 ts4; do
    if [ $v = base ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=alt_libs/$v.so; fi
    echo "$v $(timeout 240 python tools/pass1_ab.py --iters 20 2>/dev/null | tail -1)" >> gpurun_out/p1v.txt
  done
done
exit 0
