set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.log 2>&1; echo "pytest rc=$?" >> gpurun_out/t.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_c4_r1e.json 2> gpurun_out/bench_c4_r1e.err
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29555 bench.py --force-shard --steps 10 --warmup 3 --no-ablation > gpurun_out/bench_c4_fs_r1e.json 2> gpurun_out/bench_c4_fs_r1e.err
tail -3 gpurun_out/t.log; cat gpurun_out/smoke.log | tail -2
