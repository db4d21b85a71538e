set -u
for c in c1 c2 c3 c4 c5gat c5gt; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${c}_r1l.json 2> gpurun_out/bench_${c}_r1l.err
  python -c "import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1]); print(sys.argv[1], round(d['value'],3), d['kernels_ms'], round(d['e2e']['value'],3), d['layer'] and round(d['layer']['value'],3))" gpurun_out/bench_${c}_r1l.json || tail -3 gpurun_out/bench_${c}_r1l.err
done
