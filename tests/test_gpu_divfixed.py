"""pp::div_fixed (a hoisted-reciprocal split of the compiler's fp64 division,
common.cuh) against '/' bit for bit on the device: random operands over the
whole exponent range and near 1, all-ones / power-of-two / short mantissas,
small integers (the DP's stage-term and chan divisions use it)."""

import ctypes
import os
import shutil
import subprocess
import struct

import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def lib(tmp_path_factory):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    out = str(tmp_path_factory.mktemp("divfixed") / "divfixed.so")
    subprocess.run([nvcc, "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-fmad=false", "-std=c++17",
                    "-Xcompiler", "-fPIC", "-shared", "-o", out, os.path.join(HERE, "cuda", "divfixed_check.cu")],
                   check=True)
    return ctypes.CDLL(out)


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_div_fixed_matches_ieee_division(lib, seed):
    out = (ctypes.c_ulonglong * 9)()
    rc = lib.run_divfixed(ctypes.c_ulonglong(seed), ctypes.c_longlong(1 << 22), ctypes.c_int(64), out)
    assert rc == 0
    bad = [(struct.unpack("<d", struct.pack("<Q", out[1 + 2 * k]))[0],
            struct.unpack("<d", struct.pack("<Q", out[2 + 2 * k]))[0]) for k in range(min(out[0], 4))]
    assert out[0] == 0, f"{out[0]} mismatches, e.g. (a, b) = {bad}"
