#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/dp_check_w2_p2p.jsonl
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 \
  --master-port=29651 tools/dp_check.py --out gpurun_out/dp_check_w2_p2p.jsonl > gpurun_out/zm_dpcheck.log 2>&1
echo "dp_check exit $?" >> gpurun_out/zm_dpcheck.log
for ex in p2p nccl; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=2965$((RANDOM % 9)) \
  bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e --exchange $ex > gpurun_out/zm_bench_$ex.log 2>&1
done
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > gpurun_out/zm_multi.log 2>&1
exit 0
