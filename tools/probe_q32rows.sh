#!/bin/bash
# rank-32 Q partials: 64 / 128 / 256 rows (columns of w) per CTA
mkdir -p gpurun_out/q32r; O=gpurun_out/q32r; rm -f $O/ab.txt
for rep in 1 2; do
for lib in default alt_libs/q32r64.so alt_libs/q32r256.so; do
  if [ $lib = default ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=$PWD/$lib; fi
  for r in 24 32; do
    echo "$lib $r $(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{')" >> $O/ab.txt
  done
done
done
exit 0
