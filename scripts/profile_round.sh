#!/bin/bash
# Evidence pass (run under gpurun): default bench line, launch list, and
# ncu --set full of the attention kernels on C4.  Outputs in gpurun_out/.
# gpurun copies back <= 64 MiB per call, so split the captures across calls:
#   bash scripts/profile_round.sh r1f bench fwd_fast
#   bash scripts/profile_round.sh r1f bwd_rows_fast bwd_cols_fast
set -u
tag=$1
shift
for k in "$@"; do
  if [ "$k" = bench ]; then
    timeout 900 python bench.py > gpurun_out/bench_c4_$tag.json 2> gpurun_out/bench_c4_$tag.err
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$tag.csv \
      timeout 600 python bench.py --steps 2 --warmup 3 --no-layer --no-ablation --no-cpu-baseline > /dev/null 2>&1
  else
    ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_${k}_$tag \
      timeout 900 python bench.py --steps 2 --warmup 3 --no-layer --no-ablation --no-cpu-baseline > /dev/null 2>&1
  fi
done
ls -la gpurun_out/*_$tag*
