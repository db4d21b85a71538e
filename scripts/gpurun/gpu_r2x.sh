set -u
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2x_t.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r2x_t.log
for c in c1 c2 c3 c4; do
 for pf in 1 0; do
  r=$(GF_L2_PREFETCH=$pf timeout 300 python bench.py --config $c --steps 30 --warmup 5 --no-cpu-baseline --no-layer --no-ablation --no-c5 --no-api 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); print('$c pf$pf', round(d['value'],3), d['kernels_ms'], round(d['ms_per_step']*1e3,1),'us')" "$r"
 done
done
