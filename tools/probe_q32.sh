#!/bin/bash
# ncu --set full of the rank-32 Q partials (k_skinny<1,128,32>) and the W r = 32 reconstruction
mkdir -p gpurun_out/q32
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_skinny<1|k_recon4" --launch-skip 4 -c 2 \
  -o gpurun_out/q32/q32 -f python bench.py --rank 32 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --entropy off > gpurun_out/q32/ncu.log 2>&1
exit 0
