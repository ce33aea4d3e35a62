#!/bin/bash
# A/B of the rollout -> MLP hand-off: 32-byte position rows (default) vs the
# 64-byte positional encodings (MPPI_MLP_POSENC=1), config 4 and config 2.
OUT=${1:-gpurun_out/ab_handoff}
mkdir -p "$OUT"
for v in q posenc q posenc; do
  if [ $v = posenc ]; then export MPPI_MLP_POSENC=1; else unset MPPI_MLP_POSENC; fi
  python bench.py --workload c4 --steps 20 --warmup 3 > "$OUT/c4_$v.log" 2>&1
  python bench.py --workload c2 --steps 200 --warmup 10 --no-cpu-baseline --no-scale-roofline > "$OUT/c2_$v.log" 2>&1
  python - "$OUT/c4_$v.log" "$OUT/c2_$v.log" $v <<'PY'
import json, sys
for f in sys.argv[1:3]:
    for l in open(f):
        if l.startswith('{'):
            d = json.loads(l)
            print(sys.argv[3], f.split('/')[-1], d['value'], d.get('stage_ms'), d['clocks'])
PY
done
