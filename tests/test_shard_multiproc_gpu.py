"""GPU, multi-process: the row-sharded layer step with 2 and 3 real ranks
(torch.distributed.run, gloo process group over CUDA tensors, every rank on
the one B200 this environment has).  Each rank starts with only its own block
of the source-side tables and gets the others through the exchanges the
sharded step uses; all ranks check the result against the unsharded 1-GPU
step bitwise (tests/mp_shard_worker.py).  NCCL cannot put two ranks on one
GPU, so this is the closest on-hardware check of the multi-GPU data path."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("world,model", [(2, "gat"), (2, "gat_layer"), (2, "gt"), (2, "agnn"),
                                         (3, "gat_layer"), (3, "gt")])
def test_sharded_step_across_processes(cuda, world, model):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "tests", "mp_shard_worker.py"), "--model", model]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count("SHARD-OK") == world, out[-4000:]


@pytest.mark.parametrize("world,model", [(2, "gt"), (3, "gat_layer")])
def test_phased_forward_across_processes(cuda, world, model):
    """The source-phased forward (per-owner broadcasts, one forward per source
    block, gf_attn_merge_parts) across real ranks == 1 GPU up to the merge's
    fp32 rounding (2e-5), backward included."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={world}", "--master-addr", "127.0.0.1", f"--master-port={port}",
           os.path.join(ROOT, "tests", "mp_shard_worker.py"), "--model", model, "--phased"]
    env = dict(os.environ, OMP_NUM_THREADS="1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-4000:]
    assert out.count("SHARD-OK") == world, out[-4000:]
