#!/bin/bash
# Same-box A/B of an environment knob on config 5 at several N:
#   bash scripts/ab_c5env.sh OUTDIR VAR "valA valB" "N1 N2 ..."
OUT=$1; VAR=$2; VALS=$3; NS=$4
mkdir -p "$OUT"
for rep in 1 2; do
  for n in $NS; do
    for v in $VALS; do
      export $VAR=$v
      python bench.py --workload c5 --particles $n --steps 30 --warmup 5 > "$OUT/c5_${n}_${v}_$rep.log" 2>&1
      python - "$OUT/c5_${n}_${v}_$rep.log" "$VAR=$v N=$n" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d = json.loads(l)
        print(sys.argv[2], '%.4g' % d['value'], 'ms %.4f' % d['ms_per_step'], {k: round(v, 4) for k, v in (d.get('stage_ms') or {}).items()})
PY
    done
  done
done
