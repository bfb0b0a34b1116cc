set -x
nvidia-smi -L
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q 2>&1 | tail -3
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/final_bench_n2.json 2> gpurun_out/final_bench_n2.err
tail -c 300 gpurun_out/final_bench_n2.json
