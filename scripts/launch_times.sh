# Per-kernel device durations of a short bench run under ncu (cold, serialised):
#   bash scripts/launch_times.sh OUT.csv [extra bench args]
OUT=$1; shift
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file "$OUT" \
  python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-scale-roofline "$@" > /dev/null 2>&1
python - "$OUT" <<'PY'
import csv, sys, collections
rows = list(csv.DictReader(l for l in open(sys.argv[1]) if l.startswith('"')))
d = collections.defaultdict(list)
for r in rows:
    if r.get("Metric Name") == "gpu__time_duration.sum":
        d[r["Kernel Name"][:60]].append(float(r["Metric Value"].replace(",", "")))
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    v.sort()
    print(f"{k:60s} n={len(v):4d} median={v[len(v)//2]:9.0f}")
PY
