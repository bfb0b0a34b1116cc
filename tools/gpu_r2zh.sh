#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_compress.py tests/test_gpu_engine.py tests/test_gpu_dp.py -x -q -p no:cacheprovider > gpurun_out/zh_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/zh_pytest.log
for r in 8 6; do timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --rank $r > gpurun_out/zh_bench_r$r.log 2>&1; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  --csv --log-file gpurun_out/zh_r8_launch.csv python bench.py --rank 8 --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --entropy off > /dev/null 2>&1
exit 0
