set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2a_gpu.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2a_t.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2a_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2a_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r2a_bench_c4.json 2> gpurun_out/r2a_bench_c4.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2a_ref_c4.json 2> gpurun_out/r2a_ref_c4.err
tail -3 gpurun_out/r2a_t.log
