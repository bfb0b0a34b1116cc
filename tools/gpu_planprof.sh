set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_bucket_resolve|k_walk" -c 2 -o gpurun_out/plan_src -f python tools/plan_prof.py --reps 1 > gpurun_out/ncu_plan.log 2>&1
tail -2 gpurun_out/ncu_plan.log
