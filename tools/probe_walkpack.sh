#!/bin/bash
# ahead-mode walk packing (plans per CTA: 16 default, 8, 4): headline bench, twice each
mkdir -p gpurun_out; rm -f gpurun_out/wp.txt
for rep in 1 2; do
  for v in base wp8 wp4; do
    if [ $v = base ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=alt_libs/$v.so; fi
    echo "$v $(timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{')" >> gpurun_out/wp.txt
  done
done
exit 0
