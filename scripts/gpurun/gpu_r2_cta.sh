set -u
for thr in 0 1024 2048 8192 16384 0; do
  r=$(timeout 300 python bench.py --config c4 --steps 30 --warmup 5 --no-cpu-baseline --no-layer --no-ablation --no-c5 --no-api --cta-threshold $thr 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); print('thr $thr', d['graph']['cta_threshold'], d['graph']['cta_rows'], round(d['value'],3), d['kernels_ms'])" "$r"
done
