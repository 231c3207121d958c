"""Shared pytest setup.  `-m gpu` tests need a B200 and call through the
C ABI (libq8p.so); everything else runs on CPU (oracle vs golden vectors,
host logic, C-ABI symbol exports, multi-process gloo tests)."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a real B200 (sm_100a) GPU")
    # Build the checker (C restatement) and the product library if absent.
    if not os.path.exists(os.path.join(ROOT, "oracle", "build", "liblatq_oracle.so")):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    if not os.path.exists(os.path.join(ROOT, "paper_2402_04396_b200", "libq8p.so")):
        subprocess.run(["make", "-s", "-j8", "-C", os.path.join(ROOT, "paper_2402_04396_b200", "csrc")], check=True)


@pytest.fixture(scope="session")
def kat():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def oracle():
    from oracle.refpy import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle.refpy import Ref, REF_SO
    if not os.path.exists(REF_SO):
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return Ref()


def load_case(name: str):
    with open(os.path.join(GOLDEN, f"{name}.qshp"), "rb") as f:
        art = f.read()
    x = np.load(os.path.join(GOLDEN, f"{name}.x.npy"))
    y = np.load(os.path.join(GOLDEN, f"{name}.y.npy"))
    return art, x, y


def golden_names():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return [c["name"] for c in json.load(f)["cases"]]


def rel_err(a, b) -> float:
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def random_artifact(m, n, stages, seed, codes=None, transform=0):
    """A structurally valid QSHP artifact with random codes (acceptance.cpp:438-450 style);
    transform 0 = rht (random sign bytes), 1 = rfft (random f32 phases in [0, 2 pi))."""
    import struct
    rng = np.random.default_rng(seed)
    body = b"QSHP" + struct.pack("<HIIBB", 1, m, n, transform, len(stages))
    for cid, scale in stages:
        body += bytes([len(cid)]) + cid.encode() + struct.pack("<f", scale)
    if transform == 0:
        body += rng.integers(0, 256, (m + 7) // 8, dtype=np.uint8).tobytes()
        body += rng.integers(0, 256, (n + 7) // 8, dtype=np.uint8).tobytes()
    else:
        body += rng.uniform(0, 2 * np.pi, m // 2).astype("<f4").tobytes()
        body += rng.uniform(0, 2 * np.pi, n // 2).astype("<f4").tobytes()
    words = m * n // 8
    for s, (cid, _) in enumerate(stages):
        if codes is not None and codes[s] is not None:
            c = codes[s]
        elif cid == "e8p-2bit":
            c = rng.integers(0, 65536, words, dtype=np.uint16)
        else:
            c = rng.integers(0, 256, words, dtype=np.uint8)
        body += np.ascontiguousarray(c).tobytes()
    return body
