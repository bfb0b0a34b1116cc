# ncu source-level capture of the tcgen05 wide-path kernels (r = 128) + entropy A/B
set -x
timeout 300 python bench.py --steps 30 --warmup 5 --entropy off --no-e2e --no-cpu-baseline > gpurun_out/bench_ent_off.json 2>&1
timeout 300 python bench.py --steps 30 --warmup 5 --entropy inline --no-e2e --no-cpu-baseline > gpurun_out/bench_ent_inline.json 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tc -s 4 -c 4 -o gpurun_out/tc_r128 -f python tools/pass1_ab.py --rank 128 --iters 1 > gpurun_out/ncu_tc.log 2>&1
ls -la gpurun_out
