#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/t_bench100_$i.log 2>&1
done
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/t_bench20.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --entropy off > gpurun_out/t_bench100_off.log 2>&1
EDGC_PLAN_NOSET=1 timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/t_bench100_noset.log 2>&1
exit 0
