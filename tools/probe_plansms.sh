#!/bin/bash
# plan kernels (sort / resolve / tail) as persistent grids on a subset of SMs vs short CTAs
mkdir -p gpurun_out; rm -f gpurun_out/ps.txt
for rep in 1 2; do
  for v in short p16 p32 p64; do
    unset EDGC_PLAN_PERSISTENT EDGC_PLAN_SMS
    if [ $v != short ]; then export EDGC_PLAN_PERSISTENT=1 EDGC_PLAN_SMS=${v#p}; fi
    echo "$v $(timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{')" >> gpurun_out/ps.txt
  done
done
exit 0
