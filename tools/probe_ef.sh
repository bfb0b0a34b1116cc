#!/bin/bash
# EF update A/B: k_ef vs k_gemm<2> (EDGC_EF_GEMM=1) at r = 8, 16, 32 (r = 32 with EDGC_TC_EF_MIN_RANK=32)
mkdir -p gpurun_out
for r in 8 16 32; do
  for v in ef gemm; do
    if [ $v = gemm ]; then export EDGC_EF_GEMM=1; else unset EDGC_EF_GEMM; fi
    EDGC_TC_EF_MIN_RANK=32 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/pe_${v}_r$r.csv python bench.py --rank $r --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --entropy off > /dev/null 2>&1
  done
done
unset EDGC_EF_GEMM
timeout 600 python -m pytest tests/test_gpu_engine.py tests/test_gpu_debug_rank.py -x -q -p no:cacheprovider > gpurun_out/pe_pytest.log 2>&1
exit 0
