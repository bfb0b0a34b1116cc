#!/bin/bash
# GPT2-12.1B at r = 256 (config 5), 12 steps: current build vs the pfd2 TcEF variant
mkdir -p gpurun_out; rm -f gpurun_out/p12.txt
for v in base pfd2; do
  if [ $v = base ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=alt_libs/$v.so; fi
  echo "$v $(timeout 900 python bench.py --model 12.1B --rank 256 --steps 12 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{')" >> gpurun_out/p12.txt
done
exit 0
