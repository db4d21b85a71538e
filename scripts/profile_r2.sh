#!/bin/bash
# Round-2 evidence pass (under gpurun): bench line, launch list of the same
# command, ncu --set full of the three attention kernels on C4.
set -u
tag=$1; shift
for k in "$@"; do
  if [ "$k" = bench ]; then
    timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/bench_c4_$tag.json 2> gpurun_out/bench_c4_$tag.err
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$tag.csv \
      timeout 900 python bench.py --gpus 1 --steps 3 --warmup 3 --no-layer --no-ablation --no-cpu-baseline --no-c5 --no-api > /dev/null 2>&1
  else
    ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_${k}_$tag \
      timeout 900 python bench.py --steps 2 --warmup 3 --no-layer --no-ablation --no-cpu-baseline --no-c5 --no-api > /dev/null 2>&1
  fi
done
ls -la gpurun_out/*_$tag*
