#!/bin/bash
# after the k_skinny_ef K-split: full GPU suite, rank sweep 4 < r <= 16, default bench line
mkdir -p gpurun_out/skf; O=gpurun_out/skf; rm -f $O/ranks.jsonl
timeout 1200 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
for r in 6 8 12 16; do
  timeout 240 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{' >> $O/ranks.jsonl
done
timeout 300 python bench.py --no-e2e --no-cpu-baseline > $O/bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_skinny" -c 6 --csv --log-file $O/r8.csv python bench.py --rank 8 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --entropy off > /dev/null 2>&1
exit 0
