set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_dropin_gpu.py tests/test_gpu_state.py tests/test_reference_suites.py -q -x > gpurun_out/r2g_t.log 2>&1; echo "rc=$?" >> gpurun_out/r2g_t.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2g_bench_c4.json 2> gpurun_out/r2g_bench_c4.err; echo "rc=$?" >> gpurun_out/r2g_bench_c4.err
tail -3 gpurun_out/r2g_t.log
