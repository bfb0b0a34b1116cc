set -x
EDGC_WALK_CLUSTER=8 timeout 600 python -m pytest tests/test_gpu_sampling.py -x -q 2>&1 | tail -2
for wc in 1 8 4 1 8; do
EDGC_WALK_CLUSTER=$wc timeout 300 python bench.py --steps 60 --warmup 5 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('wc=$wc', round(d['value'],1), round(d['ms_per_step'],3), d['phases_ms']['step_ms'])"
done
