set -x
timeout 600 python -m pytest tests/test_gpu_sampling.py -x -q 2>&1 | tail -2
timeout 300 python tools/plan_prof.py --reps 4
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_walk --csv --log-file gpurun_out/launch_walkev.csv python tools/plan_prof.py --reps 1 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/launch_walkev.csv 3
