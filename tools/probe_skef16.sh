#!/bin/bash
# 16-rank fused EF + P_raw: FFMA2 in the EF blocks only (s16e) / the product tiles only (s16g) vs FFMA
mkdir -p gpurun_out/s16b; O=gpurun_out/s16b; rm -f $O/ab.txt
for rep in 1 2; do
for lib in default alt_libs/s16e.so alt_libs/s16g.so; do
  if [ $lib = default ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=$PWD/$lib; fi
  for r in 12 16; do
    echo "$lib $r $(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{')" >> $O/ab.txt
  done
done
done
exit 0
