#!/bin/bash
# fused EF + P_raw: rows per CTA (128 default, 64, 256)
mkdir -p gpurun_out; rm -f gpurun_out/skr.txt
for v in base sk64 sk256; do
  if [ $v = base ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=alt_libs/$v.so; fi
  for r in 8 16; do
    echo "$v $r $(timeout 240 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{')" >> gpurun_out/skr.txt
  done
done
exit 0
