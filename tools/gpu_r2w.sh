#!/bin/bash
# 4 GPUs: full GPU suite (W=2 and W=4 NCCL parity tests run), dp_check W=4 evidence, N=2/N=4 bench lines
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/w_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/w_pytest.log
rm -f gpurun_out/dp_check_w4.jsonl
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
  --master-port=29621 tools/dp_check.py --out gpurun_out/dp_check_w4.jsonl > gpurun_out/w_dpcheck.log 2>&1
echo "dp_check exit $?" >> gpurun_out/w_dpcheck.log
for n in 2 4; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$n --master-addr=127.0.0.1 \
  --master-port=2963$n bench.py --gpus $n --steps 50 --warmup 5 --no-e2e > gpurun_out/w_bench_n$n.log 2>&1
done
exit 0
