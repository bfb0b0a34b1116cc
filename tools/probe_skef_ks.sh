#!/bin/bash
# k_skinny_ef K-split A/B: rank-16 bench lines per library variant (EDGC_LIB_PATH), ranks 6 / 8 on the default
mkdir -p gpurun_out/skks2; O=gpurun_out/skks2; rm -f $O/ab.txt
for lib in default alt_libs/r16_128ks2.so alt_libs/r16_64ks2.so alt_libs/r16_64ks1.so; do
  if [ $lib = default ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=$PWD/$lib; fi
  echo "$lib 16 $(timeout 240 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --rank 16 2>/dev/null | grep '^{')" >> $O/ab.txt
done
unset EDGC_LIB_PATH
for r in 6 8; do
  echo "default $r $(timeout 240 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{')" >> $O/ab.txt
done
exit 0
