set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
for r in 32 64 128 256; do timeout 300 python tools/pass1_ab.py --rank $r --iters 3; done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tc -s 4 -c 4 -o gpurun_out/tc2_r128 -f python tools/pass1_ab.py --rank 128 --iters 1 > gpurun_out/ncu_tc2.log 2>&1
