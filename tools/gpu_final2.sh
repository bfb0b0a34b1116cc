#!/bin/bash
# round 2 closing validation on 1 GPU: full GPU suite, smoke, driver-like bench lines (ours + reference arm), launch list
mkdir -p gpurun_out/f4
O=gpurun_out/f4
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1
timeout 900 python bench.py --steps 100 --warmup 5 --no-e2e --no-cpu-baseline > $O/bench_100.log 2>&1
timeout 900 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --entropy off > $O/bench_off.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file $O/launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/launches.log 2>&1
exit 0
