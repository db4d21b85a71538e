set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_generators.py tests/test_capi.py -x -q > gpurun_out/r2b_t.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2b_t.log
timeout 900 python bench.py --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2b_bench_c4.json 2> gpurun_out/r2b_bench_c4.err; echo "rc=$?" >> gpurun_out/r2b_bench_c4.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --gpus 1 --force-shard --steps 10 --warmup 3 --no-ablation > gpurun_out/r2b_bench_c4_fs.json 2> gpurun_out/r2b_bench_c4_fs.err; echo "rc=$?" >> gpurun_out/r2b_bench_c4_fs.err
timeout 600 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 > gpurun_out/r2b_ref_c4.json 2> gpurun_out/r2b_ref_c4.err
tail -3 gpurun_out/r2b_t.log
