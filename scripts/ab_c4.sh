# A/B of config-4 throughput over environment settings (see ab_env.sh)
for i in 1 2; do
  for setting in "$@"; do
    env_args=(); [ "$setting" != "-" ] && read -ra env_args <<< "$setting"
    env "${env_args[@]}" python bench.py --workload c4 --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$setting'.ljust(30), '%.3e' % d['value'], {k: round(v, 3) for k, v in d['stage_ms'].items()})"
  done
done
