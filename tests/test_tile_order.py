"""The GEMM CTA raster (tile_order in csrc/tile.cuh) must visit every output tile of a launch
exactly once; compiled as host code with nvcc, no GPU needed."""

import os
import shutil
import subprocess

import pytest

from conftest import REPO


def test_tile_order_is_bijective(tmp_path):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not os.path.exists(nvcc):
        pytest.skip("nvcc not available")
    exe = tmp_path / "check"
    src = os.path.join(REPO, "tests", "native", "check_tile_order.cu")
    subprocess.run([nvcc, "-std=c++17", "-O1", "-o", str(exe), src], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout
    assert " 0 bad" in out.stdout
