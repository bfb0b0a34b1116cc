mkdir -p gpurun_out
for env in 16 32; do
  EDGC_TC_MIN_RANK=$env timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --rank 32 2>/dev/null | grep '^{' | sed "s/^/$env /" >> gpurun_out/p32.txt
done
EDGC_TC_MIN_RANK=32 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/p32_r32.csv python bench.py --rank 32 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --entropy off > /dev/null 2>&1
EDGC_TC_MIN_RANK=32 timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_compress.py tests/test_gpu_debug_rank.py -x -q -p no:cacheprovider > gpurun_out/p32_pytest.log 2>&1
exit 0
