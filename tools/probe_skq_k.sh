#!/bin/bash
# skinny Q partials: K rows per tile (fp64 partial per block) A/B at ranks 8 / 16 / 32
mkdir -p gpurun_out/skqk; O=gpurun_out/skqk; rm -f $O/ab.txt
for lib in default alt_libs/q512.so alt_libs/q1024.so alt_libs/q2048.so; do
  if [ $lib = default ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=$PWD/$lib; fi
  for r in 8 16 32; do
  echo "$lib $r $(timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{')" >> $O/ab.txt
  done
done
exit 0
