set -x
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_r256.csv python tools/pass1_ab.py --rank 256 --iters 1 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_r128.csv python tools/pass1_ab.py --rank 128 --iters 1 > /dev/null 2>&1
