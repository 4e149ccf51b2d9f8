"""C-ABI library (no GPU needed): it builds for sm_100a, loads, exports every symbol that
include/bipb.h declares, implements the host-side partition, and fails loudly (status
code, no fallback) when no CUDA device is present."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HDR = os.path.join(ROOT, "include", "bipb.h")


def _declared():
    txt = open(HDR).read()
    return sorted(set(re.findall(r"\b(bipb_[a-z_0-9]+)\s*\(", txt)))


@pytest.fixture(scope="module")
def lib():
    import importlib.util
    spec = importlib.util.spec_from_file_location("b", os.path.join(ROOT, "paper_1301_5885_b200", "build.py"))
    b = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(b)
    path = b.build()
    return ctypes.CDLL(path), path


def test_exports_every_declared_symbol(lib):
    L, path = lib
    names = _declared()
    assert {"bipb_setup", "bipb_source", "bipb_matvec", "bipb_gmres_solve", "bipb_energy"} <= set(names)
    for nm in names:
        assert hasattr(L, nm), nm
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
    for nm in names:
        assert re.search(rf"\bT {nm}\b", out), nm


def test_sass_is_sm100a(lib):
    _, path = lib
    out = subprocess.run(["cuobjdump", "--list-elf", path], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", path], capture_output=True, text=True).stdout
    assert "DFMA" in sass and "MUFU.RSQ64H" in sass and "UBLKCP" in sass  # FP64 pipe, RSQ64H seed, TMA bulk copy


def test_binding_names_match_abi():
    import paper_1301_5885_b200 as bp
    for nm in _declared():
        assert nm in bp.EXPORTS
        assert hasattr(bp, nm) or nm in ("bipb_last_error", "bipb_timing_enable", "bipb_timing_get",
                                         "bipb_timing_reset", "bipb_version")


@pytest.mark.parametrize("n,world", [(1, 1), (10, 3), (327680, 8), (5, 8), (1310720, 7)])
def test_partition(n, world):
    import paper_1301_5885_b200 as bp
    rows = [bp.bipb_partition(n, world, r) for r in range(world)]
    np_pad = -(-n // world)
    cover = []
    for r, (a, b) in enumerate(rows):
        assert 0 <= a <= b <= n and b - a <= np_pad
        assert a == min(r * np_pad, n)
        cover.extend(range(a, b))
    assert cover == list(range(n))


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import bipb_inputs as g
    import paper_1301_5885_b200 as bp
    p = g.config("C1")
    with pytest.raises(bp.BipbError) as ei:
        bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, 1.0, 80.0, 0.1257)
    assert ei.value.status == bp.ERR_CUDA
    with pytest.raises(bp.BipbError) as ei:
        bp.bipb_setup(p.centroids[:0], p.normals[:0], p.areas[:0], p.charges, 1.0, 80.0, 0.1)
    assert ei.value.status == bp.ERR_ARG


def test_header_documents_citations():
    txt = open(HDR).read()
    for cite in ("Eq. (11)", "Eqs. (12)-(13)", "Eq. (14)", "P:271-272", "eps2/eps1"):
        assert cite in txt


def test_binding_rejects_wrong_sizes():
    """The C ABI takes bare pointers: the binding checks every array's element count first."""
    import paper_1301_5885_b200 as bp
    ctx = bp.Context(ctypes.c_void_p(0), 4, 1, None)  # never reaches the library
    with pytest.raises(ValueError):
        bp.bipb_matvec(ctx, np.zeros(7))
    with pytest.raises(ValueError):
        bp.bipb_matvec(ctx, np.zeros(8), np.zeros(9))
    with pytest.raises(ValueError):
        bp.bipb_energy(ctx, np.zeros(8), np.zeros(2))
    with pytest.raises(ValueError):
        bp.bipb_gmres_solve(ctx, np.zeros(6))
    with pytest.raises(ValueError):
        bp.bipb_matvec_batch(ctx, np.zeros((2, 7)))
    with pytest.raises(ValueError):
        bp.bipb_setup(np.zeros((4, 3)), np.zeros((4, 3)), np.zeros(3), np.zeros((1, 4)), 1.0, 80.0, 0.1)
    with pytest.raises(ValueError):
        bp.bipb_setup(np.zeros((4, 3)), np.zeros((4, 3)), np.zeros(4), np.zeros((1, 3)), 1.0, 80.0, 0.1)
    with pytest.raises(ValueError):
        bp.bipb_matvec(ctx, np.zeros(8, dtype=np.float32))
    ctx._h = None
