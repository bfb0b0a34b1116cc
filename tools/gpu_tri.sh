set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for r in 4 128 256; do timeout 300 python tools/pass1_ab.py --rank $r --iters 3; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_fx --csv --log-file gpurun_out/launch_fx.csv python tools/pass1_ab.py --rank 256 --iters 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launch_fx.csv 6
