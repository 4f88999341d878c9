"""The C-ABI library builds for sm_100a, loads, and exports every symbol
include/somf.h declares (no compute calls: runs without a GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "somf.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(somf_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_1701_05363_b200 import _lib
    return _lib.build()


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ("somf_create", "somf_partial_fit", "somf_transform", "somf_components", "somf_objective"):
        assert n in names


def test_every_declared_symbol_is_exported(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (somf_[a-z0-9_]+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    # nothing else leaks (kernels and helpers are hidden)
    extra = [n for n in exported if n not in _declared()]
    assert not extra, extra


def test_sass_is_sm100a(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_library_loads_and_binding_matches(libpath):
    from paper_1701_05363_b200 import _lib
    L = _lib.load(libpath)
    assert L.somf_abi_version() == 3
    names = {n for n, _, _ in _lib.SIGNATURES}
    assert names == set(_declared())
    import ctypes as C
    cfg = _lib.SomfConfig()
    L.somf_config_default(C.byref(cfg))
    assert cfg.u == pytest.approx(0.917) and cfg.r == 1.0 and cfg.b_mode == 0


def test_invalid_config_rejected_without_gpu(libpath):
    """Argument validation happens before any device call."""
    import ctypes as C
    from paper_1701_05363_b200 import _lib
    L = _lib.load(libpath)
    cfg = _lib.SomfConfig()
    L.somf_config_default(C.byref(cfg))
    cfg.p, cfg.k, cfg.eta = 100, 4, 8
    h = C.c_void_p()
    for field, bad in (("r", 0.5), ("k", 0), ("k", 300), ("nu", 1.5), ("mu", -0.1), ("u", 0.0),
                       ("lambda_", -1.0), ("eta", 0), ("b_mode", 7)):
        old = getattr(cfg, field)
        setattr(cfg, field, bad)
        assert L.somf_create(C.byref(cfg), C.byref(h)) == 1, field
        setattr(cfg, field, old)
