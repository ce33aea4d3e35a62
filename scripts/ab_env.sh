# A/B the step latency over environment settings:
#   bash scripts/ab_env.sh "A=1 B=2" "A=0" ...   (each argument is one setting; "-" = none)
for i in $(seq ${REPS:-2}); do
  for setting in "$@"; do
    env_args=(); [ "$setting" != "-" ] && read -ra env_args <<< "$setting"
    env "${env_args[@]}" python bench.py --steps 500 --warmup 20 --no-cpu-baseline --no-scale-roofline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$setting'.ljust(30), round(d['value']*1e3,2), round(d['median_ms']*1e3,2), round(d['instrumented_step_ms']*1e3,2), round(d['e2e']['value']*1e3,2))"
  done
done
