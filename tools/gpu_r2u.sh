#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/v_bench100.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-fuse-entropy > gpurun_out/v_bench100_nofuse.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-hi-prio > gpurun_out/v_bench100_noprio.log 2>&1
exit 0
