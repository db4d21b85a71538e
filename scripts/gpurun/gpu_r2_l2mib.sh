set -u
python -c "
import torch; p=torch.cuda.get_device_properties(0); print('L2', p.L2_cache_size/2**20, 'MiB; max persisting', torch.cuda.get_device_properties(0).persisting_l2_cache_max_size/2**20 if hasattr(p,'persisting_l2_cache_max_size') else 'n/a')"
for mib in 32 64 80 96 112; do
  r=$(timeout 300 python bench.py --config c4 --steps 30 --warmup 5 --no-cpu-baseline --no-layer --no-ablation --no-c5 --no-api --l2-persist-mib $mib 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); print('mib $mib', round(d['value'],3), d['kernels_ms'], 'without', round(d['l2_carveout']['value_without'],3))" "$r"
done
