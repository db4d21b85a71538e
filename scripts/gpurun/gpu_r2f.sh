set -u
for c in c2 c3; do
 for cpl in 1 2; do
  r=$(GF_CPL=$cpl timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-layer --no-ablation 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); print('$c cpl$cpl', round(d['value'],3), d['kernels_ms'], round(d['ms_per_step']*1e3,1))" "$r"
 done
done
for cpl in 1 2; do
  r=$(GF_CPL=$cpl timeout 300 python bench.py --config c5gt --steps 10 --warmup 3 --no-cpu-baseline --no-layer --no-ablation 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); print('c5gt cpl$cpl', round(d['value'],3), d['kernels_ms'])" "$r"
done
