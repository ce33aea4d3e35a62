# Bench lines + ncu evidence for profiles/ (run under gpurun; outputs in gpurun_out/)
#   bash scripts/round_profiles.sh r1
R=${1:-r1}
O=gpurun_out
set -x
python bench.py --steps 300 --warmup 10 > $O/${R}_bench_c2.json 2> $O/${R}_bench_c2.err
python bench.py --workload c4 --steps 20 --warmup 3 --no-cpu-baseline > $O/${R}_bench_c4.json 2> $O/${R}_bench_c4.err
python bench.py --workload c3 --steps 100 --warmup 10 --no-cpu-baseline --no-scale-roofline > $O/${R}_bench_c3.json 2> $O/${R}_bench_c3.err
for n in 4096 32768 262144; do
  python bench.py --workload c5 --particles $n --steps 20 --warmup 3 --no-cpu-baseline > $O/${R}_bench_c5_$n.json 2> $O/${R}_bench_c5_$n.err
done
B="python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-scale-roofline"
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/${R}_bench_launches.csv $B > /dev/null 2>&1
P="python scripts/profile_batched.py 80 3"   # 80 x 500 = 40,000 warps: the many-waves (paired) rollout
$P > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on \
  -k regex:"rollout_pair_kernel|rollout_kernel|mlp_tcgen05|stats_kernel" -s 3 -c 3 -o $O/${R}_full_b80 $P > $O/${R}_full_b80.log 2>&1
S="python scripts/profile_step.py 6 500 2 --flush"
$S > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on \
  -k regex:"rollout_kernel|mlp_tcgen05|stats_cluster" -s 6 -c 3 -o $O/${R}_full_c2 $S > $O/${R}_full_c2.log 2>&1
ls -la $O
