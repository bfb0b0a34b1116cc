#!/bin/bash
# ncu --set full of the closing build's CUDA-core wide-path kernels: r = 8 fused EF + P_raw and
# Q partials, r = 32 Q partials, and the FFMA2 reconstruction at W r = 32 (r = 32, W = 1)
mkdir -p gpurun_out/nf
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_skinny" --launch-skip 4 -c 2 \
  -o gpurun_out/nf/r8 -f python bench.py --rank 8 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --entropy off > gpurun_out/nf/r8.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_skinny|k_recon4" --launch-skip 6 -c 3 \
  -o gpurun_out/nf/r32 -f python bench.py --rank 32 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --entropy off > gpurun_out/nf/r32.log 2>&1
exit 0
