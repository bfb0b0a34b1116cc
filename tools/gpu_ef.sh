set -x
timeout 900 python -m pytest tests/test_gpu_engine.py tests/test_gpu_recon.py tests/test_gpu_compress.py -x -q 2>&1 | tail -2
for r in 32 128 256; do timeout 300 python tools/pass1_ab.py --rank $r --iters 3; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_tc --csv --log-file gpurun_out/launch_ef.csv python tools/pass1_ab.py --rank 128 --iters 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launch_ef.csv 6
