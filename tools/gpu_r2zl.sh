#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python bench.py --model 12.1B --rank 256 --steps 12 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/zl_12b_n1.log 2>&1
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29641 \
  bench.py --gpus 2 --model 12.1B --rank 256 --steps 12 --warmup 2 --no-e2e > gpurun_out/zl_12b_n2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29642 \
  bench.py --gpus 2 --steps 50 --warmup 5 --no-e2e > gpurun_out/zl_n2.log 2>&1
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node=2 --master-addr=127.0.0.1 --master-port=29643 \
  bench.py --gpus 2 --rank 128 --steps 20 --warmup 3 --no-e2e > gpurun_out/zl_n2_r128.log 2>&1
timeout 900 python bench.py --impl reference > gpurun_out/zl_ref.log 2>&1
exit 0
