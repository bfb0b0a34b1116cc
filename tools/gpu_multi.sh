#!/bin/bash
# N GPUs of one box (gpurun --gpus N): dp_check parity evidence over the NVLink exchange (and one
# NCCL case), bench lines with both exchanges, the multi-GPU pytest.
#   bash tools/gpu_multi.sh N
N=${1:-2}
O=gpurun_out/multi_n$N
mkdir -p $O
rm -f $O/dp_check.jsonl
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
  --master-port=2967$N tools/dp_check.py --out $O/dp_check.jsonl > $O/dp_check.log 2>&1
echo "dp_check exit $?" >> $O/dp_check.log
for ex in p2p nccl; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 \
    --master-port=2968$N bench.py --gpus $N --steps 50 --warmup 5 --no-e2e --exchange $ex > $O/bench_$ex.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > $O/pytest_multi.log 2>&1
exit 0
