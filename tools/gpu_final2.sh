set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/f2_bench_n1.json 2> gpurun_out/f2_bench_n1.err
tail -c 300 gpurun_out/f2_bench_n1.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/f2_ref_n1.json 2> gpurun_out/f2_ref_n1.err
tail -c 300 gpurun_out/f2_ref_n1.json
for r in 4 8 16 32 64 128 256; do timeout 300 python tools/pass1_ab.py --rank $r --iters 3; done > gpurun_out/f2_sweep.jsonl
timeout 900 python bench.py --model 12.1B --rank 256 --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/f2_12b.json 2>gpurun_out/f2_12b.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/f2_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/f2_ncu_bench.log 2>&1
