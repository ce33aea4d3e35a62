#!/bin/bash
# Same-box A/B of library builds on the config-2 step only:
#   bash scripts/ab_c2.sh OUTDIR "tagA tagB ..." [reps]   (tag "main" = the production _mppi_b200.so)
OUT=$1; TAGS=$2; REPS=${3:-3}
mkdir -p "$OUT"
for rep in $(seq 1 $REPS); do
  for t in $TAGS; do
    if [ "$t" = main ]; then unset MPPI_LIB; else export MPPI_LIB=$PWD/paper_2104_13542_b200/_mppi_b200_$t.so; fi
    python bench.py --workload c2 --steps 300 --warmup 10 --no-cpu-baseline --no-scale-roofline > "$OUT/c2_${t}_$rep.log" 2>&1
    python - "$OUT/c2_${t}_$rep.log" "$t" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d = json.loads(l)
        print(sys.argv[2], '%.3f us' % (d['value'] * 1e3), 'median %.3f' % (d['median_ms'] * 1e3), 'e2e %.3f us' % (d['e2e']['value'] * 1e3), d['clocks']['sm_mhz'])
PY
  done
done
unset MPPI_LIB
