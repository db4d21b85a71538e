#!/bin/bash
# Evidence pass (run under gpurun): default bench line, launch list, ncu --set full
# of the three attention kernels on C4 and of the tcgen05 projection.  Outputs in gpurun_out/.
set -u
tag=${1:-r1c}
timeout 900 python bench.py > gpurun_out/bench_c4_$tag.json 2> gpurun_out/bench_c4_$tag.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c4_$tag.csv \
  timeout 600 python bench.py --steps 2 --warmup 3 --no-layer --no-ablation --no-cpu-baseline > /dev/null 2>&1
for k in fwd_fast bwd_rows_fast bwd_cols_fast; do
  ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_${k}_$tag \
    timeout 900 python bench.py --steps 2 --warmup 3 --no-layer --no-ablation --no-cpu-baseline > /dev/null 2>&1
done
ncu --set full --clock-control none --import-source on -k regex:tc_gemm_3xtf32 -s 6 -c 1 -o gpurun_out/prof_gemm_$tag \
  timeout 600 python scripts/bench_gemm.py > /dev/null 2>&1
ls -la gpurun_out/*_$tag*
