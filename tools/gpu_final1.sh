set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/final_bench_n1.json 2> gpurun_out/final_bench_n1.err
tail -c 600 gpurun_out/final_bench_n1.json
for r in 32 128 256; do timeout 300 python tools/pass1_ab.py --rank $r --iters 3; done > gpurun_out/final_sweep.jsonl
cat gpurun_out/final_sweep.jsonl
timeout 900 python bench.py --model 12.1B --rank 256 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final_12b.json 2>gpurun_out/final_12b.err
tail -c 400 gpurun_out/final_12b.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/final_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/final_ncu_bench.log 2>&1
