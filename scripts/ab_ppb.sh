for n in ${NS:-4096 8192 32768}; do for p in ${PS:-0 128 256 512}; do
  if [ $p = 0 ]; then E=""; else E="MPPI_STATS_PPB=$p"; fi
  env $E python bench.py --workload c5 --particles $n --steps 100 --warmup 5 --no-cpu-baseline --no-scale-roofline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print($n, '$p', round(d['ms_per_step']*1000,1), 'us', round(d['e2e']['value']/1e9,3) if isinstance(d['e2e'].get('value'),float) else d['e2e'])"
done; done
