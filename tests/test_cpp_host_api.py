"""The host C++ API (include/q8p.hpp) compiled into a standalone program, as a
latq caller would link it: QSHP round trip, typed errors, planner (CPU), and
DeviceLayer::infer / q8p::infer against the reference goldens (GPU)."""
from __future__ import annotations

import os
import subprocess

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

LIBDIR = os.path.join(ROOT, "paper_2402_04396_b200")
NAMES = ["e8p2_96x160", "rvq3_56x112", "rvq4_64x64", "rfft2_344x512", "rfft3_56x112"]


@pytest.fixture(scope="module")
def exe(tmp_path_factory):
    if not os.path.exists(os.path.join(LIBDIR, "libq8p.so")):
        pytest.fail("libq8p.so not built")
    out = str(tmp_path_factory.mktemp("cpp") / "host_api")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "host_api.cpp"), "-o", out, f"-L{LIBDIR}", "-l:libq8p.so",
                    f"-Wl,-rpath,{LIBDIR}"], check=True)
    return out


@pytest.mark.parametrize("name", NAMES)
def test_cpp_host_api_cpu(exe, name):
    r = subprocess.run([exe, "cpu", os.path.join(GOLDEN, f"{name}.qshp")], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_cpp_device_layer_infer(exe, tmp_path, name):
    x = np.load(os.path.join(GOLDEN, f"{name}.x.npy"))
    y = np.load(os.path.join(GOLDEN, f"{name}.y.npy"))
    x.astype(np.float64).tofile(tmp_path / "x.f64")
    y.astype(np.float64).tofile(tmp_path / "y.f64")
    r = subprocess.run([exe, "gpu", os.path.join(GOLDEN, f"{name}.qshp"), str(tmp_path / "x.f64"),
                        str(tmp_path / "y.f64"), str(x.shape[0])], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
