#!/bin/bash
# round 2 final measurements on 1 GPU: smoke, driver-like bench lines, reference arm, ncu evidence, config 5
mkdir -p gpurun_out/final
O=gpurun_out/final
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_default.log 2>&1
timeout 900 python bench.py --steps 100 --warmup 5 --no-e2e > $O/bench_100.log 2>&1
timeout 900 python bench.py --impl reference > $O/bench_reference.log 2>&1
timeout 900 python bench.py --steps 30 --warmup 5 --no-e2e --no-cpu-baseline --entropy off > $O/bench_off.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -c 400 --csv --log-file $O/launches.csv python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline > $O/launches.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pass1t -c 2 \
  -o $O/pass1_full -f python tools/pass1_ab.py --iters 1 > $O/pass1_full.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_walk|k_set_sort|k_set_resolve|k_set_tail|k_gauss_partial" -c 5 \
  -o $O/plan_full -f python tools/plan_prof.py --reps 1 --ahead > $O/plan_full.log 2>&1
timeout 300 python tools/plan_prof.py --reps 5 --ahead > $O/plan_prof.log 2>&1
timeout 300 python tools/plan_prof.py --reps 5 >> $O/plan_prof.log 2>&1
timeout 300 python tools/recon_probe.py --rank 4 > $O/recon_r4.log 2>&1
timeout 300 python tools/api_probe.py > $O/api.log 2>&1
timeout 1200 python bench.py --model 12.1B --rank 256 --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > $O/bench_12b_r256.log 2>&1
for b in 0.25 0.05; do timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --alpha 1 --beta $b > $O/bench_alpha1_b$b.log 2>&1; done
exit 0
