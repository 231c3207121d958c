"""Layer sets (q8p_forward_set / q8p_forward_set_host): several independent
layer forwards per call; the host variant replays H2D + kernels + D2H as one
cached CUDA graph when the host buffers are pinned.  Results must equal the
per-layer q8p_forward bit for bit (same kernels, deterministic arithmetic)."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2402_04396_b200 as q8p
from conftest import random_artifact

pytestmark = pytest.mark.gpu

SHAPES = [(256, 512, [("e8p-2bit", 1.1)], 0), (512, 256, [("e8p-2bit", 1.0), ("e8-1bit", 0.5)], 0),
          (128, 1024, [("e8p-2bit", 0.9)], 1), (384, 768, [("e8p-2bit", 0.97), ("e8p-2bit", 0.3)], 0)]


def _layers():
    return [q8p.Layer.from_qshp(random_artifact(m, n, st, 11 * i + 3, transform=tr))
            for i, (m, n, st, tr) in enumerate(SHAPES)]


@pytest.mark.parametrize("concurrent", [False, True])
@pytest.mark.parametrize("batch", [1, 4, 17])
def test_forward_set_equals_per_layer(batch, concurrent):
    layers = _layers()
    S = q8p.LayerSet(layers, concurrent=concurrent)
    g = torch.Generator().manual_seed(batch)
    xs = [torch.randn(batch, L.info["n"], generator=g).cuda() for L in layers]
    want = [L.forward(x) for L, x in zip(layers, xs)]
    got = S.forward(xs)
    for a, b in zip(got, want):
        assert torch.equal(a, b)


@pytest.mark.parametrize("concurrent", [False, True])
@pytest.mark.parametrize("pinned", [True, False])
def test_forward_set_host_graph_replays(pinned, concurrent):
    layers = _layers()
    S = q8p.LayerSet(layers, concurrent=concurrent)
    batch = 2
    nsum = sum(L.info["n"] for L in layers)
    msum = sum(L.info["m"] for L in layers)
    hx = torch.empty(batch * nsum).pin_memory() if pinned else torch.empty(batch * nsum)
    hy = torch.empty(batch * msum).pin_memory() if pinned else torch.empty(batch * msum)
    ws = S.workspace(batch)
    for it in range(3):  # capture, then replays re-reading the host inputs
        hx.copy_(torch.randn(batch * nsum, generator=torch.Generator().manual_seed(it)))
        k0 = q8p.kernel_launches()
        S.forward_host(hx, hy, batch, workspace=ws)
        assert q8p.kernel_launches() > k0  # the library's kernels ran (also on graph replays)
        xo = yo = 0
        for L in layers:
            m, n = L.info["m"], L.info["n"]
            x = hx[xo:xo + batch * n].view(batch, n).cuda()
            assert torch.equal(hy[yo:yo + batch * m].view(batch, m), L.forward(x).cpu()), (it, m, n)
            xo += batch * n
            yo += batch * m


def test_layer_destroy_drops_cached_graphs():
    layers = _layers()
    S = q8p.LayerSet(layers)
    nsum = sum(L.info["n"] for L in layers)
    msum = sum(L.info["m"] for L in layers)
    hx, hy = torch.randn(nsum).pin_memory(), torch.empty(msum).pin_memory()
    S.forward_host(hx, hy, 1)
    y0 = hy.clone()
    del S
    for L in layers:
        L.close()
    layers2 = _layers()  # may reuse the freed handles' addresses
    S2 = q8p.LayerSet(layers2)
    S2.forward_host(hx, hy, 1)
    assert torch.equal(hy, y0)  # same artifacts, same inputs: same results through a fresh graph


def test_concurrent_set_under_caller_graph_capture():
    # the caller captures the concurrent set into its own graph: forked lanes become branches
    layers = _layers()
    S = q8p.LayerSet(layers, concurrent=True)
    xs = [torch.randn(2, L.info["n"]).cuda() for L in layers]
    ys = [torch.empty(2, L.info["m"]).cuda() for L in layers]
    ws = S.workspace(2)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        S.forward(xs, ys, stream=s, workspace=ws)
    torch.cuda.synchronize()
    want = [y.clone() for y in ys]
    for y in ys:
        y.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        S.forward(xs, ys, stream=s, workspace=ws)
    g.replay()
    torch.cuda.synchronize()
    for a, b in zip(ys, want):
        assert torch.equal(a, b)


def test_forward_set_validation():
    layers = _layers()
    S = q8p.LayerSet(layers)
    with pytest.raises(q8p.ValidationError):
        S.forward([torch.randn(1, 7).cuda()] * len(layers))
    with pytest.raises(q8p.SizeError):
        S.forward_host(torch.empty(3), torch.empty(3), 1)
