#!/bin/bash
# A/B of one environment knob on configs 4 and 2, interleaved twice:
#   bash scripts/ab_env.sh OUTDIR VAR "valA valB"
OUT=$1; VAR=$2; VALS=$3
mkdir -p "$OUT"
for rep in 1 2; do
  for v in $VALS; do
    export $VAR=$v
    python bench.py --workload c4 --steps 20 --warmup 3 > "$OUT/c4_${v}_$rep.log" 2>&1
    python bench.py --workload c2 --steps 200 --warmup 10 --no-cpu-baseline --no-scale-roofline > "$OUT/c2_${v}_$rep.log" 2>&1
    python - "$OUT/c4_${v}_$rep.log" "$OUT/c2_${v}_$rep.log" "$VAR=$v" <<'PY'
import json, sys
for f in sys.argv[1:3]:
    for l in open(f):
        if l.startswith('{'):
            d = json.loads(l)
            print(sys.argv[3], f.split('/')[-1], '%.4g' % d['value'], {k: round(v, 4) for k, v in (d.get('stage_ms') or {}).items()}, d['clocks']['sm_mhz'], d['clocks']['reasons'])
PY
  done
done
