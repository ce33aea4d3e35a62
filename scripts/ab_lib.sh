#!/bin/bash
# Same-box A/B of library builds (MPPI_BUILD_TAG=<tag> python -m paper_2104_13542_b200.build):
#   bash scripts/ab_lib.sh OUTDIR "tagA tagB ..."   (tag "main" = the production _mppi_b200.so)
OUT=$1; TAGS=$2; REPS=${3:-2}
mkdir -p "$OUT"
for rep in $(seq 1 $REPS); do
  for t in $TAGS; do
    if [ "$t" = main ]; then unset MPPI_LIB; else export MPPI_LIB=$PWD/paper_2104_13542_b200/_mppi_b200_$t.so; fi
    python bench.py --workload c4 --steps 20 --warmup 3 > "$OUT/c4_${t}_$rep.log" 2>&1
    python bench.py --workload c2 --steps 200 --warmup 10 --no-cpu-baseline --no-scale-roofline > "$OUT/c2_${t}_$rep.log" 2>&1
    python - "$OUT/c4_${t}_$rep.log" "$OUT/c2_${t}_$rep.log" "$t" <<'PY'
import json, sys
for f in sys.argv[1:3]:
    for l in open(f):
        if l.startswith('{'):
            d = json.loads(l)
            print(sys.argv[3], f.split('/')[-1], '%.4g' % d['value'], {k: round(v, 4) for k, v in (d.get('stage_ms') or {}).items()}, d['clocks']['sm_mhz'], d['clocks']['reasons'])
PY
  done
done
unset MPPI_LIB
