set -x
timeout 900 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_fused_entropy.py tests/test_gpu_entropy.py -x -q 2>&1 | tail -3
timeout 300 python tools/plan_prof.py --reps 4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_plan.csv python tools/plan_prof.py --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launch_plan.csv 8
timeout 300 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline
