#!/bin/bash
# Q partial (k_skinny<1>) rows per CTA: 256 default, 128, 512
mkdir -p gpurun_out; rm -f gpurun_out/skq_*.csv gpurun_out/skq.txt
for v in base q128 q512; do
  if [ $v = base ]; then unset EDGC_LIB_PATH; else export EDGC_LIB_PATH=alt_libs/$v.so; fi
  for r in 8 16; do
    timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_skinny<1" --csv --log-file gpurun_out/skq_${v}_r$r.csv python bench.py --rank $r --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --entropy off > /dev/null 2>&1
    echo "$v $r $(timeout 240 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{')" >> gpurun_out/skq.txt
  done
done
exit 0
