#!/bin/bash
# round 2, call A (2 GPUs): full GPU suite incl. the W=2 NCCL parity tests, dp_check evidence,
# then the N=1 bench at 20 and 100 steps (timed window now waits for the side-stream plan build)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/a_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/a_pytest.log
rm -f gpurun_out/dp_check_w2.jsonl
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 \
  --master-port=29611 tools/dp_check.py --out gpurun_out/dp_check_w2.jsonl > gpurun_out/a_dpcheck.log 2>&1
echo "dp_check exit $?" >> gpurun_out/a_dpcheck.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/a_bench20.log 2>&1
timeout 600 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/a_bench100.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 \
  --master-port=29612 bench.py --gpus 2 --steps 20 --warmup 5 --no-e2e > gpurun_out/a_bench_n2.log 2>&1
exit 0
