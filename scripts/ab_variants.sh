#!/bin/bash
# A/B kernel build variants: ab_variants.sh <config> <variant|default>...
cfg=$1; shift
for v in "$@"; do
  if [ "$v" = default ]; then unset GF_CUDA_LIB; else export GF_CUDA_LIB=variants/$v/libgraphfuse_cuda.so; fi
  r=$(timeout 300 python bench.py --config $cfg --steps 20 --warmup 3 --no-cpu-baseline --no-layer --no-ablation --no-c5 --no-api 2>/dev/null | tail -1)
  python -c "import json,sys; d=json.loads(sys.argv[1]); print('$cfg $v', round(d['value'],3), d['kernels_ms'], 'no-setaside', round((d.get('l2_carveout') or {}).get('value_without', 0),3), 'table', round((d.get('gat_table_form') or {}).get('value', 0),3), (d.get('gat_table_form') or {}).get('kernels_ms'))" "$r" || echo "$cfg $v FAILED"
done
