#!/bin/bash
# Same-box A/B of library builds on config 5 at several N:
#   bash scripts/ab_c5.sh OUTDIR "tagA tagB" "N1 N2 ..."
OUT=$1; TAGS=$2; NS=$3
mkdir -p "$OUT"
for rep in 1 2; do
  for n in $NS; do
    for t in $TAGS; do
      if [ "$t" = main ]; then unset MPPI_LIB; else export MPPI_LIB=$PWD/paper_2104_13542_b200/_mppi_b200_$t.so; fi
      python bench.py --workload c5 --particles $n --steps 30 --warmup 5 > "$OUT/c5_${n}_${t}_$rep.log" 2>&1
      python - "$OUT/c5_${n}_${t}_$rep.log" "$t N=$n" <<'PY'
import json, sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d = json.loads(l)
        print(sys.argv[2], '%.4g' % d['value'], 'ms %.4f' % d['ms_per_step'], {k: round(v, 4) for k, v in (d.get('stage_ms') or {}).items()})
PY
    done
  done
done
unset MPPI_LIB
