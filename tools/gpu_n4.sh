set -x
nvidia-smi -L
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 4 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/f2_bench_n4.json 2> gpurun_out/f2_bench_n4.err
tail -c 400 gpurun_out/f2_bench_n4.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 4 --impl reference --steps 2 --warmup 1 > gpurun_out/f2_ref_n4.json 2> gpurun_out/f2_ref_n4.err
tail -c 300 gpurun_out/f2_ref_n4.json
