#!/bin/bash
# A/B: ranks 5..8 on the narrow register passes vs the skinny GEMM path (EDGC_NARROW_MAX=4)
mkdir -p gpurun_out; rm -f gpurun_out/pn.txt
for r in 6 8; do
  for env in 8 4; do
    EDGC_NARROW_MAX=$env timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{' | sed "s/^/$env /" >> gpurun_out/pn.txt
  done
done
EDGC_NARROW_MAX=4 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/pn_r8.csv python bench.py --rank 8 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --entropy off > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/pn_r8_narrow.csv python bench.py --rank 8 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --entropy off > /dev/null 2>&1
EDGC_NARROW_MAX=4 timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_compress.py tests/test_gpu_debug_rank.py -x -q -p no:cacheprovider > gpurun_out/pn_pytest.log 2>&1
exit 0
