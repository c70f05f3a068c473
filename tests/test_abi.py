"""The C-ABI library loads and exports every symbol include/rbs.h declares (no GPU needed)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "rbs.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(rbs_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def rbs():
    from paper_1804_06363_b200 import build
    build.build()
    import paper_1804_06363_b200 as r
    r.lib()
    return r


def test_header_declares_expected_calls():
    syms = declared_symbols()
    for s in ("rbs_create", "rbs_set_operator_blocks", "rbs_set_rhs_constant", "rbs_load_basis",
              "rbs_solve_batch", "rbs_build_greedy"):
        assert s in syms


def test_library_exports_every_declared_symbol(rbs):
    out = subprocess.check_output(["nm", "-D", "--defined-only", rbs._SO]).decode()
    exported = set(re.findall(r" T (rbs_\w+)", out))
    missing = [s for s in declared_symbols() if s not in exported]
    assert not missing, missing
    # the Python binding binds exactly the declared calls
    assert sorted(rbs.EXPORTED) == declared_symbols()


def test_library_is_sm100a_only(rbs):
    out = subprocess.check_output(["cuobjdump", "--list-elf", rbs._SO]).decode()
    assert "sm_100a" in out
    sass = subprocess.check_output(["cuobjdump", "-sass", rbs._SO]).decode()
    assert "DMMA" in sass  # FP64 tensor-core projection / prolongation


def test_host_logic_without_gpu(rbs):
    import ctypes as C
    assert rbs.lib().rbs_version() == 1
    assert rbs.lib().rbs_status_string(0).decode() == "RBS_OK"
    h = C.c_void_p()
    st = rbs.lib().rbs_create(0, C.byref(h))
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if not has_gpu:
        assert st != 0 and not h.value  # no device -> error status, never an abort
    o = rbs.rbs_default_opts()
    assert o.method == rbs.RBS_RBCG and o.tol == 1e-10 and o.sweeps == 1 and o.graph_chunk % 2 == 0


def test_binding_has_no_fallback(rbs, monkeypatch):
    monkeypatch.setattr(rbs, "_lib", None)
    monkeypatch.setattr(rbs, "_SO", "/nonexistent/librbs.so")
    with pytest.raises(rbs.RbsError):
        rbs.lib()
