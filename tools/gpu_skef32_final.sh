#!/bin/bash
# rank <= 32 fused path on by default: full GPU suite, rank sweep, default bench line
mkdir -p gpurun_out/s32f; O=gpurun_out/s32f; rm -f $O/ranks.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
for r in 20 24 32; do
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{' >> $O/ranks.jsonl
done
timeout 300 python bench.py --no-e2e --no-cpu-baseline > $O/bench.log 2>&1
exit 0
