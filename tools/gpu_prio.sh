for cfg in "" "--hi-prio" "PS" "PS --hi-prio" "" "--hi-prio" "PS --hi-prio"; do
  if [[ $cfg == PS* ]]; then export EDGC_PLAN_SHORT=1; a=${cfg#PS}; else unset EDGC_PLAN_SHORT; a=$cfg; fi
  timeout 300 python bench.py --steps 60 --warmup 5 --no-e2e --no-cpu-baseline $a | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('cfg=[$cfg]', round(d['value'],1), round(d['ms_per_step'],3), d['phases_ms']['step_ms'])"
done
