#!/bin/bash
OUT=gpurun_out/ab_fuse; mkdir -p $OUT
export MPPI_LIB=$PWD/paper_2104_13542_b200/_mppi_b200_fe.so
python -m pytest tests/test_gpu_parity.py -x -q -p no:cacheprovider -k "fused_rollout_mlp" 2>&1 | tail -1
for r in 1 2 3; do
  for f in 0 1; do
    if [ $f = 1 ]; then export MPPI_FUSE=1; else unset MPPI_FUSE; fi
    python bench.py --workload c2 --steps 300 --warmup 10 --no-cpu-baseline --no-scale-roofline 2>/dev/null | python -c "import json,sys; [print(\"fuse=$f\", \"%.3f %.3f\" % (d[\"value\"]*1e3, d[\"e2e\"][\"value\"]*1e3)) for d in (json.loads(l) for l in sys.stdin if l.startswith(\"{\"))]"
  done
done
