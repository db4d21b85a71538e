"""GPU: device-wide state the library touches only on request:
the persisting-L2 set-aside is opt-in (gf_l2_persist), never raised by an
attention call on its own, works as the first CUDA call of a process, and
gf_l2_persist(0) gives it back; scratch comes from a private pool
(gf_scratch_trim releases it)."""
import ctypes as C
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_l2_persist_is_opt_in(cuda):
    code = r"""
import ctypes as C, sys
sys.path.insert(0, %r)
from paper_2411_16127_b200._capi import lib, check
L = lib()
check(L.gf_l2_persist(0), "first call of the process")   # no context yet
got = C.c_size_t()
check(L.gf_l2_persist_get(C.byref(got)), "get")
assert got.value == 0, got.value
import numpy as np, torch
from paper_2411_16127_b200 import fused
import oracle
rng = np.random.default_rng(0)
key = np.unique(rng.integers(0, 500, 3000) * 500 + rng.integers(0, 500, 3000))
g = oracle.from_coo(500, key %% 500, key // 500)
dg = fused.DeviceGraph.from_host_csr(g.n, g.row_ptr, g.col, g.csc_ptr, g.csc_row)
spec = fused.AttnSpec("add", 8, 8)
t = [torch.rand(500, w, device="cuda") for w in (8, 8, 64, 64)]
O, st = fused.attn_forward(dg, spec, t[0], t[1], t[2])
fused.attn_backward(dg, spec, t[0], t[1], t[2], O, st, t[3])
torch.cuda.synchronize()
check(L.gf_l2_persist_get(C.byref(got)), "get")
assert got.value == 0, "an attention call changed the persisting-L2 limit"
check(L.gf_l2_persist(64 << 20), "set")
check(L.gf_l2_persist_get(C.byref(got)), "get")
assert got.value > 0
check(L.gf_l2_reset_persisting(), "reset")
check(L.gf_l2_persist(0), "release")
check(L.gf_l2_persist_get(C.byref(got)), "get")
assert got.value == 0
check(L.gf_scratch_trim(), "trim")
print("ok")
""" % ROOT
    env = dict(os.environ)
    env.pop("GF_L2_SETASIDE", None)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                       cwd=ROOT, timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("ok"), r.stdout + r.stderr


def test_pdl_and_split_overrides_keep_results(cuda):
    """Programmatic dependent launch (default) vs GF_PDL=0, and a forced
    multi-CTA split (GF_SPLIT_LEN=100) vs the default: forward and backward
    results are bitwise equal for PDL and oracle-equal for the split."""
    code = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r)
sys.path.insert(0, %r + "/tests")
from test_gpu_parity import make_graph, make_inputs, run_device
from paper_2411_16127_b200.fused import AttnSpec
g = make_graph("hub")
spec = AttnSpec(variant="dot", heads=8, head_dim=16, scale=0.25)
Q, K, V, dO = make_inputs(g, "dot", 8, 16, np.float32, 3)
r = run_device(g, spec, Q, K, V, dO)
np.savez(sys.argv[1], **r)
""" % (ROOT, ROOT)
    outs = {}
    for name, env_extra in (("pdl", {}), ("nopdl", {"GF_PDL": "0"}), ("split", {"GF_SPLIT_LEN": "100"})):
        env = dict(os.environ, **env_extra)
        path = os.path.join(ROOT, "gpurun_out", f"_state_{name}.npz")
        os.makedirs(os.path.dirname(path), exist_ok=True)
        r = subprocess.run([sys.executable, "-c", code, path], capture_output=True, text=True,
                           env=env, cwd=ROOT, timeout=300)
        assert r.returncode == 0, r.stderr[-3000:]
        import numpy as np

        outs[name] = dict(np.load(path))
    for k in ("O", "dQ", "dK", "dV"):
        assert (outs["pdl"][k] == outs["nopdl"][k]).all(), k
        a, b = outs["pdl"][k], outs["split"][k]
        assert float(abs(a - b).max() / max(1.0, float(abs(a).max()))) < 1e-5, k


def test_l2_policy_word_matches_device(cuda):
    """The backward passes receive the evict_last policy word as a kernel
    argument (csrc/gf_policy.h); it must equal what createpolicy yields."""
    from paper_2411_16127_b200._capi import check, lib

    dev, host = C.c_uint64(), C.c_uint64()
    check(lib().gf_l2_policy_word(C.byref(dev), C.byref(host)), "gf_l2_policy_word")
    assert dev.value == host.value, (hex(dev.value), hex(host.value))
