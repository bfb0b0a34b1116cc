#!/bin/bash
# FFMA2 build: full GPU suite, rank sweep 6..32, reconstruction probe, default bench line
mkdir -p gpurun_out/ff; O=gpurun_out/ff; rm -f $O/ranks.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1
for r in 6 8 12 16 20 24 32; do
  timeout 300 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{' >> $O/ranks.jsonl
done
timeout 300 python tools/recon_probe.py --rank 4 > $O/recon_r4.json 2>/dev/null
timeout 300 python tools/recon_probe.py --rank 32 --worlds 1 > $O/recon_r32.json 2>/dev/null
timeout 300 python bench.py --no-e2e --no-cpu-baseline > $O/bench.log 2>&1
exit 0
