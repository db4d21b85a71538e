set -u
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_unfused_ops.py tests/test_dropin_gpu.py -q -x 2>&1 | tail -2
for c in c1 c2 c3 c4; do
 for pdl in 1 0; do
  r=$(GF_PDL=$pdl timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-layer --no-ablation --no-c5 --no-api 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); print('$c pdl$pdl', round(d['value'],3), d['kernels_ms'], round(d['ms_per_step']*1e3,1),'us')" "$r"
 done
done
