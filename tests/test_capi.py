"""CPU: the C-ABI library loads and exports every symbol include/gf_cuda.h
declares (no compute calls), the ctypes binding covers them, and the build
targets sm_100a only."""
import os
import re
import subprocess

import pytest

from paper_2411_16127_b200 import _capi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gf_cuda.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\**(gf_\w+)\s*\(", src, flags=re.M)))


def test_header_parses():
    names = declared_functions()
    assert "gf_attn_fwd" in names and "gf_attn_bwd" in names and "gf_graph_create" in names
    assert len(names) >= 20


def test_library_exports_every_declared_symbol():
    lib = _capi.lib()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_ctypes_binding_covers_header():
    assert set(declared_functions()) == set(_capi.SIGNATURES)


def test_cubin_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _capi.LIB_PATH], capture_output=True,
                         text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
    assert archs == {"100a"}, archs


def test_error_reporting_without_device():
    """Argument validation happens before any device work and is reported."""
    import ctypes as C

    lib = _capi.lib()
    d = _capi.AttnDesc(0, 1, 1, 1, 8, 0, 1.0, 0.2)  # add + l2 is invalid
    rc = lib.gf_attn_fwd(C.c_void_p(1), C.byref(d), None, None, None, None, None, None, None)
    assert rc == 1
    assert b"invalid descriptor" in lib.gf_last_error()
    rc = lib.gf_graph_create(-1, 0, None, None, None, None, 0, None, C.byref(C.c_void_p()))
    assert rc == 1


def test_descriptor_flags_validated_without_device():
    """GF_FLAG_LOGITS_FROM_V is only valid with the additive variant; unknown
    flag bits are rejected; the single-step ops take no flags."""
    import ctypes as C

    lib = _capi.lib()
    dot_flag = _capi.AttnDesc(0, 0, 0, 8, 8, _capi.GF_FLAG_LOGITS_FROM_V, 1.0, 0.2)
    rc = lib.gf_attn_fwd(C.c_void_p(1), C.byref(dot_flag), None, None, None, None, None, None,
                         None)
    assert rc == 1 and b"flags" in lib.gf_last_error()
    bad_bits = _capi.AttnDesc(0, 1, 0, 8, 8, 6, 1.0, 0.2)
    assert lib.gf_attn_bwd(C.c_void_p(1), C.byref(bad_bits), *([None] * 10)) == 1
    ok_flag = _capi.AttnDesc(0, 1, 0, 8, 8, _capi.GF_FLAG_LOGITS_FROM_V, 1.0, 0.2)
    assert lib.gf_sddmm(C.c_void_p(1), C.byref(ok_flag), None, None, None, None) == 1
    assert b"no descriptor flags" in lib.gf_last_error()
