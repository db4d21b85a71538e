"""CPU: bench.py's launcher, reference arm and host graph generators (no GPU).

* `--gpus N` re-launches itself under torch.distributed.run when no launcher
  set WORLD_SIZE, and refuses a WORLD_SIZE that disagrees with --gpus;
* the reference arm (oracle/_ref, the reference compiled from its sources)
  prints one JSON line whose `config` equals the GPU arm's, timing whole
  steps of every head;
* the numpy restatements of the device generators keep their contracts
  (the bit-exact host == device check is tests/test_gpu_generators.py).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402


def test_gpus_flag_spawns_ranks(monkeypatch):
    calls = []
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd, env=None: calls.append((cmd, env)) or 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    assert bench.main(["--gpus", "4", "--steps", "2"]) == 0
    (cmd, env), = calls
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]
    assert env["NCCL_DEBUG"] == "INFO"


def test_gpus_flag_must_match_world(monkeypatch, capsys):
    monkeypatch.setenv("WORLD_SIZE", "2")
    monkeypatch.setenv("RANK", "1")
    assert bench.main(["--gpus", "4"]) == 2
    assert "WORLD_SIZE=2" in capsys.readouterr().err


def _ref_available():
    import oracle

    return oracle.ref_available()


@pytest.mark.skipif(not _ref_available(), reason="oracle/_ref not built")
def test_reference_arm_line(capsys, monkeypatch):
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    assert bench.main(["--impl", "reference", "--config", "c1", "--steps", "2",
                       "--warmup", "3"]) == 0
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "GEdges/s"
    assert line["config"] == bench.config_key("c1")
    n, src, _ = bench.gen_graph_host("cora")
    assert line["sample"]["edges"] == len(src) and line["sample"]["nodes"] == n
    assert line["steps"] == 2 and line["ms_per_step"] > 0
    assert line["value"] == pytest.approx(len(src) / (line["ms_per_step"] / 1e3) / 1e9)
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["kind"] == "reference"


@pytest.mark.skipif(not _ref_available(), reason="oracle/_ref not built")
def test_reference_arm_under_launcher():
    """`bench.py --impl reference --gpus 2` on CPU: the launcher starts two
    ranks (gloo-free: the reference arm needs no process group), rank 0 prints
    the only JSON line, rank 1 exits 0."""
    env = dict(os.environ)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--gpus", "2", "--config", "c1", "--steps", "1", "--warmup", "3"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    out = json.loads(lines[0])
    assert out["n_gpus"] == 2 and out["impl"] == "reference"


def test_host_power_law_slice_equals_full_filtered():
    n = 5_000
    s, d = bench.host_power_law(n, 600, 0.34, seed=3)
    rows = n // 7
    s2, d2 = bench.host_power_law(n, 600, 0.34, seed=3, rows=rows)
    keep = d < rows
    np.testing.assert_array_equal(s[keep], s2)
    np.testing.assert_array_equal(d[keep], d2)
    k = d * n + s
    assert np.all(np.diff(k) > 0)  # distinct, (dst, src) order
    deg = np.sort(np.bincount(d, minlength=n))[::-1]
    want = np.sort(bench.power_law_degrees(n, 600, 0.34))[::-1]
    assert np.all(deg <= want) and deg[0] >= 600 - 600 * 600 // n - 5


def test_host_random_contract():
    s, d = bench.host_random(3000, 3.5, seed=7)
    assert len(s) == int(3.5 * 3000 + 0.5)
    k = d * 3000 + s
    assert np.all(np.diff(k) > 0) and s.min() >= 0 and s.max() < 3000
    s2, _ = bench.host_random(3000, 3.5, seed=8)
    assert not np.array_equal(s, s2)


def test_host_molecules_contract():
    s, d = bench.host_molecules(50, 26, 3, seed=3)
    n = 50 * 26
    k = d * n + s
    assert np.all(np.diff(k) > 0) and not np.any(s == d)
    assert np.all(s // 26 == d // 26)
    assert set((d * n + s).tolist()) == set((s * n + d).tolist())


def test_row_slice_sample_is_the_row_prefix():
    import oracle

    n, src, dst = bench.gen_graph_host("cora")
    g = oracle.from_coo(n, src, dst)
    rows = 700
    sub = bench.row_slice_sample(n, g.row_ptr, g.col, rows)
    keep = dst < rows
    ref = oracle.from_coo(n, src[keep], dst[keep])
    for a in ("row_ptr", "col", "csc_ptr", "csc_row", "csc_perm"):
        np.testing.assert_array_equal(getattr(sub, a), getattr(ref, a))
