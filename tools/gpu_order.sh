set -x
timeout 900 python -m pytest tests/test_gpu_sampling.py tests/test_gpu_fused_entropy.py tests/test_gpu_ranks.py -x -q 2>&1 | tail -2
timeout 300 python tools/plan_prof.py --reps 4
for i in 1 2; do timeout 300 python bench.py --steps 60 --warmup 5 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3), d['phases_ms']['step_ms'])"; done
