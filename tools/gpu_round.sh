set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -25 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench_n1.json 2> gpurun_out/bench_n1.err
for r in 4 8 16 32 64 128 256; do timeout 300 python tools/pass1_ab.py --rank $r --iters 3; done > gpurun_out/rank_sweep.jsonl 2> gpurun_out/rank_sweep.err
timeout 900 python bench.py --model 12.1B --rank 256 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_12b.json 2> gpurun_out/bench_12b.err
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/bench_n1.json gpurun_out/rank_sweep.jsonl gpurun_out/bench_12b.json
