set -x
timeout 900 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_fused_entropy.py tests/test_gpu_entropy.py tests/test_gpu_ranks.py -x -q 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_draws" --csv --log-file gpurun_out/launch_draws.csv python tools/plan_prof.py --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launch_draws.csv 3
timeout 300 python bench.py --steps 60 --warmup 5 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3), d['phases_ms']['step_ms'], d['clocks'])"
