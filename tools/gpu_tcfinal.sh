set -x
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tc -s 4 -c 4 -o gpurun_out/tc3_r128 -f python tools/pass1_ab.py --rank 128 --iters 1 > gpurun_out/ncu_tc3.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_fx" -s 4 -c 4 -o gpurun_out/fx_r256 -f python tools/pass1_ab.py --rank 256 --iters 1 > gpurun_out/ncu_fx.log 2>&1
