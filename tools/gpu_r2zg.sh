#!/bin/bash
mkdir -p gpurun_out
for i in 1 2; do
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/zg_fused_$i.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e --no-fuse-entropy > gpurun_out/zg_nofuse_$i.log 2>&1
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_pass1|k_pass2|k_recon" -c 6 \
  -o gpurun_out/zg_r8 -f python bench.py --rank 8 --layers 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --entropy off > gpurun_out/zg_r8.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/zg_r8_launch.csv python bench.py --rank 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --entropy off > /dev/null 2>&1
exit 0
