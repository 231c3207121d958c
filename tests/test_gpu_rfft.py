"""rfft transform artifacts (SideTransform kind rfft, core/src/rfft.cpp:39-71):
GPU forward vs the oracle (relative L2 error <= TC, the same bound as the rht
parity tests; the DFT passes run in fp32) at the config shapes, incl. n = 11008 (DFT length
5504 = 64 x 86) and n = 28672 (14336 = 112 x 128); artifact validation on CPU.
The golden rfft fixtures (tests/golden/rfft*) run through test_gpu_parity.py."""
from __future__ import annotations

import numpy as np
import pytest

from conftest import random_artifact, rel_err

TC = 1e-5


@pytest.fixture(scope="module")
def dev():
    import torch

    assert torch.cuda.is_available(), "gpu tests need a B200"
    return torch.device("cuda:0")

STAGES = {2: [("e8p-2bit", 1.11)], 3: [("e8p-2bit", 1.02), ("e8-1bit", 0.49)],
          4: [("e8p-2bit", 0.97), ("e8p-2bit", 0.29)]}


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,bits", [(4096, 4096, 2), (11008, 4096, 2), (4096, 11008, 2), (8192, 8192, 3),
                                      (2048, 28672, 4), (28672, 8192, 2), (1030, 512, 2)])
def test_rfft_forward_vs_oracle(dev, oracle, m, n, bits):
    import torch

    import paper_2402_04396_b200 as q8p

    art = random_artifact(m, n, STAGES[bits], 31 * m + n + bits, transform=1)
    L = q8p.Layer.from_qshp(art)
    assert L.info["m"] == m
    batch = 1 if m * n > 1e8 else 2
    x = np.random.default_rng(5).standard_normal((batch, n)).astype(np.float32).astype(np.float64)
    want = oracle.infer(art, x, threads=8)
    got = L.forward(torch.from_numpy(x.astype(np.float32)).to(dev)).cpu().numpy()
    for b in range(batch):
        assert rel_err(got[b], want[b]) < TC, (m, n, bits, rel_err(got[b], want[b]))


@pytest.mark.gpu
def test_rfft_batches_and_portable_path(dev, oracle):
    # batch 1..64 (17-32: MMA N = 128, 64: two chunks) and an e8-1bit-first artifact
    # (no tensor-core path: the portable GEMV between the rfft passes)
    import torch

    import paper_2402_04396_b200 as q8p

    art = random_artifact(256, 512, STAGES[3], 7, transform=1)
    x = np.random.default_rng(6).standard_normal((64, 512)).astype(np.float32).astype(np.float64)
    want = oracle.infer(art, x)
    L = q8p.Layer.from_qshp(art)
    for nb in (1, 3, 8, 16, 17, 32, 64):  # 32: MMA N = 128; 64: 32-vector chunks
        got = L.forward(torch.from_numpy(x[:nb].astype(np.float32)).to(dev)).cpu().numpy()
        assert rel_err(got, want[:nb]) < TC, (nb, rel_err(got, want[:nb]))
    art2 = random_artifact(128, 256, [("e8-1bit", 0.7)], 8, transform=1)
    x2 = np.random.default_rng(7).standard_normal((2, 256)).astype(np.float32).astype(np.float64)
    got = q8p.Layer.from_qshp(art2).forward(torch.from_numpy(x2.astype(np.float32)).to(dev)).cpu().numpy()
    assert rel_err(got, oracle.infer(art2, x2)) < TC


@pytest.mark.gpu
def test_rfft_linearity_70b(dev):
    # size-independent property at the 70B down-projection shape (n = 28672)
    import torch

    import paper_2402_04396_b200 as q8p

    L = q8p.Layer.from_qshp(random_artifact(8192, 28672, STAGES[2], 3, transform=1))
    g = torch.Generator().manual_seed(1)
    x1, x2 = torch.randn(28672, generator=g).cuda(), torch.randn(28672, generator=g).cuda()
    y1, y2, y12 = L.forward(x1), L.forward(x2), L.forward(0.75 * x1 - 1.5 * x2)
    ref = 0.75 * y1 - 1.5 * y2
    assert float((y12 - ref).norm() / ref.norm()) < 1e-4


def test_rfft_artifact_validation():
    import paper_2402_04396_b200 as q8p

    # DFT length 4 * 7919 (prime): no factorization fits the two-pass kernels
    with pytest.raises(q8p.UnsupportedError):
        q8p.Layer.from_qshp(random_artifact(8, 8 * 7919, STAGES[2], 1, transform=1))
    # odd m cannot carry phases (pipeline.cpp:353-355)
    with pytest.raises(q8p.FormatError):
        q8p.Layer.from_qshp(random_artifact(7, 64, STAGES[2], 1, transform=1))
