#!/bin/bash
# 16-rank fused EF + P_raw: FFMA vs FFMA2, 4 vs 3 CTAs per SM (ranks 12 / 16)
mkdir -p gpurun_out/s16; O=gpurun_out/s16; rm -f $O/ab.txt
for rep in 1 2; do
for lib in default alt_libs/s16a.so alt_libs/s16b.so; do
  if [ $lib = default ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=$PWD/$lib; fi
  for r in 12 16; do
    echo "$lib $r $(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{')" >> $O/ab.txt
  done
done
done
exit 0
