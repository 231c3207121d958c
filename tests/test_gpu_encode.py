"""GPU E8P encoder (q8p_e8p_encode) vs the reference e8p_encode
(core/src/e8p.cpp:114-156, compiled in place): bit-identical words, including
inputs on the quarter-integer grid where distance ties decide by the smaller word."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2402_04396_b200 as q8p

pytestmark = pytest.mark.gpu


def _inputs():
    rng = np.random.default_rng(0)
    parts = [rng.standard_normal((4000, 8)) * s for s in (0.3, 1.0, 2.0, 4.0)]
    parts.append(rng.integers(-12, 13, (4000, 8)) / 4.0)   # quarter-integer grid: exact ties
    parts.append(rng.integers(-6, 7, (2000, 8)) / 2.0)
    parts.append(np.zeros((4, 8)))
    return np.concatenate(parts)


def test_encode_bit_identical_to_reference(ref):
    v = _inputs()
    got = q8p.e8p_encode(torch.from_numpy(v).cuda()).cpu().numpy()
    want = np.array([ref.e8p_encode(b) for b in v], dtype=np.int64)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, (bad[:5], got[bad[:5]], want[bad[:5]])


def test_encode_decode_round_trip():
    # encoding an exactly representable codeword returns it (its distance is 0)
    words = np.random.default_rng(1).integers(0, 65536, 5000)
    pts = np.stack([q8p.e8p_decode_host(int(w)) for w in words]).astype(np.float64)
    got = q8p.e8p_encode(torch.from_numpy(pts).cuda()).cpu().numpy()
    back = np.stack([q8p.e8p_decode_host(int(w)) for w in got]).astype(np.float64)
    assert np.array_equal(back, pts)


@pytest.mark.parametrize("bits", [2, 3, 4])
def test_rvq_quantize_bit_identical_to_reference(ref, bits):
    # default_scheme(bits) (rvq.cpp:9-21) with f32-frozen scales as the producer uses them
    cbs = {2: [q8p.CB_E8P_2BIT], 3: [q8p.CB_E8P_2BIT, q8p.CB_E8_1BIT], 4: [q8p.CB_E8P_2BIT, q8p.CB_E8P_2BIT]}[bits]
    rho = {2: [0.9], 3: [0.98, 2.04], 4: [1.03, 3.45]}[bits]
    scales = [float(np.float32(1.0 / r)) for r in rho]
    v = _inputs()[:12000]
    got = q8p.rvq_quantize(torch.from_numpy(v).cuda(), list(zip(cbs, scales))).cpu().numpy()
    want = ref.rvq_quantize(bits, scales, v).astype(np.int64)
    assert np.array_equal(got, want), np.argwhere(got != want)[:5]


@pytest.mark.parametrize("m,n,bits,seed", [(64, 128, 2, 11), (96, 160, 3, 6), (56, 112, 4, 7), (256, 512, 2, 3)])
def test_gpu_producer_equals_reference_quantize(ref, m, n, bits, seed):
    # The H = I producer route (ref_quantize_hi == quantize_layer(W, I, cfg)) with
    # every numeric step on the GPU: W~ = T_u W T_v^T in f64 (q8p_rht_cols_f64),
    # RVQ codes (q8p_rvq_quantize); the artifact bytes must equal the reference's.
    w = ref.gen_weights(m, n, ref.substream_seed(seed, 10))
    su = ref.random_signs(m, ref.substream_seed(seed, 0))
    sv = ref.random_signs(n, ref.substream_seed(seed, 1))
    body = q8p.produce_artifact(torch.from_numpy(w).cuda(), su, sv, bits)
    want = ref.quantize_hi(m, n, bits, seed)
    assert body == want


def test_reference_quantized_4096_batch1(ref, oracle):
    # BASELINE configs[0]: a single 4096 x 4096 E8P 2-bit layer of Gaussian weights
    # quantized by the reference route (gen_weights, harness.cpp:136-146; H = I
    # quantize_layer) -- the GPU producer's artifact is byte-identical to the
    # reference's, and its batch-1 forward matches the reference infer.
    m = n = 4096
    seed = 0
    w = ref.gen_weights(m, n, ref.substream_seed(seed, 10))
    su = ref.random_signs(m, ref.substream_seed(seed, 0))
    sv = ref.random_signs(n, ref.substream_seed(seed, 1))
    art = q8p.produce_artifact(torch.from_numpy(w).cuda(), su, sv, 2)
    assert art == ref.quantize_hi(m, n, 2, seed, threads=16)
    x = ref.gen_weights(1, n, ref.substream_seed(seed, 12)).astype(np.float32).astype(np.float64)
    L = q8p.Layer.from_qshp(art)
    got = L.forward(torch.from_numpy(x.astype(np.float32)).cuda()).cpu().numpy()
    want = ref.infer(art, x, threads=16)
    err = np.linalg.norm(got[0] - want[0]) / np.linalg.norm(want[0])
    assert err < 1e-5, err
