set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unfused_ops.py -q -x 2>&1 | tail -2
for c in c1 c2 c3 c4; do
  r=$(timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline --no-layer --no-ablation --no-c5 --no-api 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); print('$c', round(d['value'],3), d['kernels_ms'], round(d['ms_per_step']*1e3,1),'us', 'step_frac', round(d['step_roofline']['frac'],3))" "$r"
done
