"""Device math routines of the pair kernels (bipb_kernels.cuh: rsqrt_fp64 = MUFU.RSQ64H seed +
cubic correction, exp_neg = 2^(-j/2048) table + degree-3 Taylor) against long-double libm on the
host (tools/math_accuracy.cu, 4M random arguments per routine): the error bounds DESIGN.md §6
states, pinned directly rather than only through the matvec parity."""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("defs", [[], ["-DBIPB_RSQ_INT=1", "-DBIPB_EXP_F32K=1"]], ids=["default", "int_fp32_variants"])
def test_device_math_error_bounds(tmp_path, defs):
    exe = str(tmp_path / "math_accuracy")
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    subprocess.check_call([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-fmad=false", *defs, "-o", exe,
                           os.path.join(ROOT, "tools", "math_accuracy.cu")])
    r = json.loads(subprocess.check_output([exe], text=True).strip().splitlines()[-1])
    assert r["err"] == "no error"
    assert r["rsqrt_max_ulp"] <= 1.0
    assert r["exp_max_ulp_t_lt_0.2"] <= 1.5
    assert r["exp_max_ulp_t_0.2_10"] <= 4.5
    assert r["exp_max_abs_t_10_690"] <= 1e-19
