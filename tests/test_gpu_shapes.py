"""GPU parity across the batch sizes and shapes of BASELINE.json's configs:
every tensor-core variant (N = 8/16/32/48/64 columns of activation limbs,
1- and 2-stage codebooks, 2/3 decode groups) and the 16-vector chunking
beyond batch 16, against the CPU oracle (oracle/latq_oracle.c restating
core/src/pipeline.cpp:151-197), plus the 70B-shaped layers at batch 1."""
import numpy as np
import pytest

import paper_2402_04396_b200 as q8p
from conftest import random_artifact, rel_err

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

TC = 1e-5    # tensor-core path: 25-bit integer activations (see test_gpu_parity.py)
PREFILL = 1e-4  # K4 prefill (batch >= 64): 16-bit fixed-point activations per vector (two s8 limbs), exact s32 accumulation
TOL = 1e-3   # portable fp32 path / north-star bar

STAGES = {2: [("e8p-2bit", 1.11)], 3: [("e8p-2bit", 1.02), ("e8-1bit", 0.49)],
          4: [("e8p-2bit", 0.97), ("e8p-2bit", 0.29)]}


@pytest.fixture(scope="module")
def dev():
    assert torch.cuda.is_available(), "gpu tests need a B200"
    return torch.device("cuda:0")


@pytest.mark.parametrize("bits", [2, 3, 4])
@pytest.mark.parametrize("batch", [1, 2, 3, 4, 8, 13, 16, 17, 24, 32, 40, 64, 70, 96])
def test_batches_vs_oracle(dev, oracle, bits, batch):
    m, n = 1024, 2048
    art = random_artifact(m, n, STAGES[bits], 100 * bits + batch)
    L = q8p.Layer.from_qshp(art)
    x = np.random.default_rng(batch).standard_normal((batch, n)).astype(np.float32).astype(np.float64)
    want = oracle.infer(art, x, threads=8)
    got = L.forward(torch.from_numpy(x.astype(np.float32)).to(dev)).cpu().numpy()
    bar = TC if batch < 64 else PREFILL  # batches 17..32: MMA N = 128; 33..63: 32-vector chunks; >= 64: K4
    for b in range(batch):
        assert rel_err(got[b], want[b]) < bar, (b, rel_err(got[b], want[b]))


@pytest.mark.parametrize("m,n", [(8192, 8192), (28672, 8192), (8192, 28672)])
def test_70b_shapes_vs_oracle(dev, oracle, m, n):
    art = random_artifact(m, n, STAGES[2], m ^ n)
    L = q8p.Layer.from_qshp(art)
    x = np.random.default_rng(7).standard_normal((1, n)).astype(np.float32).astype(np.float64)
    want = oracle.infer(art, x, threads=16)
    got = L.forward(torch.from_numpy(x.astype(np.float32)).to(dev)).cpu().numpy()
    assert rel_err(got[0], want[0]) < TC, rel_err(got[0], want[0])


def test_batched_equals_single_all_variants(dev):
    # per-vector activation scales: every row of a batched call equals the
    # single-vector call bit for bit, whatever N / group variant the batch picks
    art = random_artifact(512, 1024, STAGES[3], 5)
    L = q8p.Layer.from_qshp(art)
    x = torch.randn(96, 1024, generator=torch.Generator().manual_seed(1)).to(dev)
    for batch in (2, 4, 8, 16, 20, 32, 40):  # tensor-core GEMV variants and the 32-vector chunks
        y = L.forward(x[:batch].contiguous())
        for b in (0, batch - 1):
            assert torch.equal(y[b], L.forward(x[b:b + 1].contiguous())[0])


@pytest.mark.parametrize("batch", [4, 8, 16, 32, 40, 64])
def test_large_layer_all_batch_variants(dev, oracle, batch):
    # many items per CTA at every N variant (the B-image ring wraps several times)
    m, n = 4096, 8192
    art = random_artifact(m, n, STAGES[2], 31 + batch)
    L = q8p.Layer.from_qshp(art)
    x = np.random.default_rng(batch).standard_normal((batch, n)).astype(np.float32).astype(np.float64)
    want = oracle.infer(art, x, threads=16)
    got = L.forward(torch.from_numpy(x.astype(np.float32)).to(dev)).cpu().numpy()
    bar = TC if batch < 64 else PREFILL
    for b in range(batch):
        assert rel_err(got[b], want[b]) < bar, (b, rel_err(got[b], want[b]))


@pytest.mark.parametrize("bits", [3, 4])
@pytest.mark.parametrize("m,n", [(11008, 4096), (4096, 11008), (28672, 8192)])
def test_rvq_big_shapes_vs_oracle(dev, oracle, m, n, bits):
    # BASELINE configs[3] (3/4-bit RVQ) on the 7B MLP and 70B MLP shapes, batch 1 and 2
    art = random_artifact(m, n, STAGES[bits], m + 3 * n + bits)
    L = q8p.Layer.from_qshp(art)
    x = np.random.default_rng(bits).standard_normal((2, n)).astype(np.float32).astype(np.float64)
    want = oracle.infer(art, x, threads=16)
    got = L.forward(torch.from_numpy(x.astype(np.float32)).to(dev)).cpu().numpy()
    for b in range(2):
        assert rel_err(got[b], want[b]) < TC, (b, rel_err(got[b], want[b]))
    assert rel_err(L.forward(torch.from_numpy(x[:1].astype(np.float32)).to(dev)).cpu().numpy()[0], want[0]) < TC


@pytest.mark.parametrize("m,n,batch", [(8192, 8192, 1024), (8192, 8192, 2048), (28672, 8192, 1024),
                                       (28672, 8192, 2048)])
def test_prefill_configs(dev, oracle, m, n, batch):
    # BASELINE configs[4] (prefill batch 128-2048) at the 70B shapes through K4:
    # sampled rows match the oracle (and the batch-1 tensor-core GEMV) within the
    # prefill bar, and a repeated call gives the same bits.
    art = random_artifact(m, n, STAGES[2], m + batch)
    L = q8p.Layer.from_qshp(art)
    x = torch.randn(batch, n, generator=torch.Generator().manual_seed(batch)).to(dev)
    y = L.forward(x)
    assert y.shape == (batch, m) and bool(torch.isfinite(y).all())
    assert torch.equal(L.forward(x), y)
    for b in [0, 255, 256, batch - 1]:
        assert rel_err(y[b].cpu().numpy(), L.forward(x[b:b + 1].contiguous())[0].cpu().numpy()) < PREFILL, b
    sample = [0, batch // 2 + 7, batch - 1]
    xs = x[sample].cpu().numpy().astype(np.float64)
    want = oracle.infer(art, xs, threads=16)
    for i, b in enumerate(sample):
        assert rel_err(y[b].cpu().numpy(), want[i]) < PREFILL, (b, rel_err(y[b].cpu().numpy(), want[i]))


@pytest.mark.parametrize("n", [16384, 28672])
def test_repeatable_code_ring_wrap(dev, n):
    # Long-k layers wrap K2's shared-memory code ring several times per CTA; the
    # same input must give the same integer accumulators every time (regression:
    # a decoder released its ring slot before its shared-memory loads completed,
    # and the producer's bulk copy for item i + S overwrote the slot under them).
    art = random_artifact(4096, n, STAGES[2], n)
    L = q8p.Layer.from_qshp(art)
    for batch in (1, 2, 3, 5, 9, 16):
        x = torch.randn(batch, n, generator=torch.Generator().manual_seed(batch)).to(dev)
        z0 = L.rows_z(x)
        for _ in range(6):
            assert torch.equal(L.rows_z(x), z0), batch
