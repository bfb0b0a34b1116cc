mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_fused_entropy.py tests/test_gpu_ranks.py tests/test_gpu_dp.py tests/test_gpu_entropy.py tests/test_gpu_sampling.py -x -q -p no:cacheprovider > gpurun_out/a1_pytest.log 2>&1
for b in 0.25 0.05; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --alpha 1 --beta $b > gpurun_out/a1_b$b.log 2>&1; done
timeout 600 python bench.py --steps 40 --warmup 5 --no-cpu-baseline --no-e2e > gpurun_out/a1_default.log 2>&1
