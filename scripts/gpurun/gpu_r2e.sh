set -u
mkdir -p gpurun_out
for c in c1 c2 c3; do
  timeout 300 python bench.py --config $c --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2e_bench_$c.json 2> gpurun_out/r2e_bench_$c.err
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"fwd_fast|bwd_rows_fast|bwd_cols_fast" -c 30 --csv --log-file gpurun_out/r2e_launches_$c.csv python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-layer --no-ablation > /dev/null 2>&1
done
