#!/bin/bash
# sanitizers, the CUDA-graph test, the config-2 sampling and rank sweeps
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_engine.py -x -q -p no:cacheprovider -k "graph or accumulate or alias" > gpurun_out/y_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/y_pytest.log
timeout 300 python tools/sanitize_cases.py > gpurun_out/y_plain.log 2>&1; echo "exit $?" >> gpurun_out/y_plain.log
for tool in memcheck synccheck racecheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python tools/sanitize_cases.py > gpurun_out/y_san_$tool.log 2>&1
  echo "exit $?" >> gpurun_out/y_san_$tool.log
done
rm -f gpurun_out/y_sweep.jsonl
for a in 1 0.1; do for b in 0.05 0.25 0.5 1.0; do
  timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-e2e --alpha $a --beta $b 2>/dev/null | grep '^{' >> gpurun_out/y_sweep.jsonl
done; done
for r in 8 16 32 64 128; do
  timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-e2e --rank $r 2>/dev/null | grep '^{' >> gpurun_out/y_sweep.jsonl
done
exit 0
