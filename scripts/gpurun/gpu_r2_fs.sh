set -u
for a in "--config c5gat" "--config c5gt --phased on" "--config c4 --phased on"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29556 bench.py --gpus 1 --force-shard --steps 5 --warmup 3 --no-ablation --no-c5 --no-api $a > gpurun_out/fs.json 2> gpurun_out/fs.err
  echo "[$a] rc=$?"; python -c "import json;d=json.loads([l for l in open('gpurun_out/fs.json') if l.startswith('{')][-1]);print(round(d['value'],3), d['phased_forward'], d['allgather_ms'], d['layer']['exchange'][:40], round(d['layer']['value'],3))" || grep -n "Error" gpurun_out/fs.err | head -3
done
