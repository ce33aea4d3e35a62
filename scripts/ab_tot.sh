#!/bin/bash
# A/B of the MLP-formed particle totals (MPPI_MLP_TOTALS) on the config-2 step
OUT=gpurun_out/ab_tot; mkdir -p $OUT
export MPPI_LIB=$PWD/paper_2104_13542_b200/_mppi_b200_tot.so
for r in 1 2 3 4; do
  for f in 0 1; do
    if [ $f = 1 ]; then export MPPI_MLP_TOTALS=1; else unset MPPI_MLP_TOTALS; fi
    python bench.py --workload c2 --steps 300 --warmup 10 --no-cpu-baseline --no-scale-roofline 2>/dev/null | python -c "import json,sys; [print(\"tot=$f\", \"%.3f %.3f\" % (d[\"value\"]*1e3, d[\"e2e\"][\"value\"]*1e3), d[\"stage_ms\"]) for d in (json.loads(l) for l in sys.stdin if l.startswith(\"{\"))]"
  done
done
