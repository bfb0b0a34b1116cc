#!/bin/bash
# A/B of the tracker's prefetch start: immediately (default) vs after the queued step work
# (EDGC_PF_AFTER_STEP=1, the earlier behaviour); N = 1 or under torchrun for N > 1
N=${1:-1}
mkdir -p gpurun_out; rm -f gpurun_out/pf_n$N.txt
for rep in 1 2; do
  for v in new old; do
    if [ $v = old ]; then export EDGC_PF_AFTER_STEP=1; else unset EDGC_PF_AFTER_STEP; fi
    if [ $N = 1 ]; then
      L=$(timeout 600 python bench.py --steps 50 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | grep '^{')
    else
      L=$(timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=$N --master-addr=127.0.0.1 --master-port=2977$N bench.py --gpus $N --steps 50 --warmup 5 --no-e2e 2>/dev/null | grep '^{')
    fi
    echo "$v $L" >> gpurun_out/pf_n$N.txt
  done
done
exit 0
