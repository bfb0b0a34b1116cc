set -x
timeout 1200 python -m pytest tests/test_gpu_engine.py tests/test_gpu_compress.py tests/test_gpu_dp.py tests/test_gpu_recon.py -x -q 2>&1 | tail -2
for r in 64 128 256; do timeout 300 python tools/pass1_ab.py --rank $r --iters 3; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_fx_chol" --csv --log-file gpurun_out/launch_chol.csv python tools/pass1_ab.py --rank 256 --iters 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launch_chol.csv 4
