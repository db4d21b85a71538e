# Round-end rehearsal: what the driver runs on a fresh box.
set -u
mkdir -p gpurun_out
t0=$(date +%s)
timeout 1500 python -m pytest tests/ -x -q -m gpu > gpurun_out/rh_t.log 2>&1; echo "pytest rc=$? $(( $(date +%s) - t0 ))s" >> gpurun_out/rh_t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rh_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rh_smoke.log
t1=$(date +%s); timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/rh_bench.json 2> gpurun_out/rh_bench.err; echo "bench rc=$? $(( $(date +%s) - t1 ))s" >> gpurun_out/rh_bench.err
t2=$(date +%s); timeout 900 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/rh_ref.json 2> gpurun_out/rh_ref.err; echo "ref rc=$? $(( $(date +%s) - t2 ))s" >> gpurun_out/rh_ref.err
tail -2 gpurun_out/rh_t.log; tail -2 gpurun_out/rh_smoke.log; tail -1 gpurun_out/rh_bench.err; tail -1 gpurun_out/rh_ref.err
