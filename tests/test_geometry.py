"""Launch geometry at p = 2, 4, 8 without a GPU: tests/geometry_check.cpp is
compiled with g++ against csrc/geometry.h — the very functions the kernels
(device) and launchers (host) use — and proves that every byte of every
BASELINE-size message (cfg1-cfg4, the cfg2 sweep 8 B - 1 GiB) is covered
exactly once by one share, chunk and round, and that every flag step fits its
12-bit field."""

import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def test_geometry_covers_every_byte_once(tmp_path):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("g++ not available")
    exe = tmp_path / "geometry_check"
    subprocess.run([gxx, "-O2", "-std=c++17", "-I", str(ROOT / "paper_2303_08374_b200" / "csrc"),
                    str(ROOT / "tests" / "geometry_check.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and out.stdout.startswith("OK"), out.stdout + out.stderr
    assert int(out.stdout.split()[1]) > 6000
