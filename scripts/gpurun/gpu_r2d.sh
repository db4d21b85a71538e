set -u
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -k "bench_graph or symmetric or c4_scale or fullsize" --durations=15 > gpurun_out/r2d_t.log 2>&1; echo "rc=$?" >> gpurun_out/r2d_t.log
tail -25 gpurun_out/r2d_t.log
