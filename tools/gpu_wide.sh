#!/bin/bash
# wide-rank path: parity tests, rank-sweep bench lines, launch list at r = 16 and 32
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_compress.py tests/test_gpu_debug_rank.py tests/test_gpu_dp.py tests/test_gpu_ranks.py -x -q -p no:cacheprovider > gpurun_out/wide_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/wide_pytest.log
rm -f gpurun_out/wide_sweep.jsonl
for r in 6 8 16 32 64 128; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{' >> gpurun_out/wide_sweep.jsonl
done
for r in 8 16; do
  timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file gpurun_out/wide_r$r.csv python bench.py --rank $r --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --entropy off > /dev/null 2>&1
done
exit 0
