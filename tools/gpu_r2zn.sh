#!/bin/bash
mkdir -p gpurun_out
rm -f gpurun_out/dp_check_w4_p2p.jsonl
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 \
  --master-port=29661 tools/dp_check.py --out gpurun_out/dp_check_w4_p2p.jsonl > gpurun_out/zn_dpcheck.log 2>&1
echo "dp_check exit $?" >> gpurun_out/zn_dpcheck.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29662 \
  bench.py --gpus 4 --steps 50 --warmup 5 --no-e2e --exchange p2p > gpurun_out/zn_bench_p2p.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29663 \
  bench.py --gpus 4 --steps 50 --warmup 5 --no-e2e --exchange nccl > gpurun_out/zn_bench_nccl.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=4 --master-addr=127.0.0.1 --master-port=29664 \
  bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/zn_bench_default.log 2>&1
timeout 900 python -m pytest tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/zn_multi.log 2>&1
exit 0
