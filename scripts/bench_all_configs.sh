# Every config's bench line (bench.py defaults: --steps 50 --warmup 3), tag $1.
set -u
tag=${1:-r2}
for c in c1 c2 c3 c4 c5gat c5gt; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_$tag.json 2> gpurun_out/bench_${c}_$tag.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value'],3), d['kernels_ms'], round(d['e2e']['value'],3), d['layer'] and round(d['layer']['value'],3), round(d['roofline']['frac'],3), d['roofline']['bound'])" gpurun_out/bench_${c}_$tag.json || tail -3 gpurun_out/bench_${c}_$tag.err
done
