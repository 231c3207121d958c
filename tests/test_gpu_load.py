"""Multi-layer loading: q8p_layers_from_qshp parses and
uploads a model's artifacts concurrently; every layer must be the one
q8p_layer_from_qshp builds (bit-identical forwards), and a malformed artifact in
the list fails the whole call with the reference's typed error."""
import numpy as np
import pytest

from conftest import random_artifact


@pytest.mark.gpu
def test_layers_from_qshp_equal_single_loads():
    import torch

    import paper_2402_04396_b200 as q8p

    shapes = [(1024, 2048, [("e8p-2bit", 1.11)]), (2048, 1024, [("e8p-2bit", 1.02), ("e8-1bit", 0.49)]),
              (4096, 4096, [("e8p-2bit", 0.97), ("e8p-2bit", 0.29)]), (8192, 8192, [("e8p-2bit", 1.11)]),
              (512, 512, [("e8p-2bit", 1.11)]), (1024, 1024, [("e8p-2bit", 1.11)])]
    arts = [random_artifact(m, n, st, 40 + i) for i, (m, n, st) in enumerate(shapes)]
    many = q8p.Layer.many_from_qshp(arts, device=0)
    assert len(many) == len(arts)
    for (m, n, _), art, L in zip(shapes, arts, many):
        x = torch.randn(3, n, generator=torch.Generator().manual_seed(m + n)).cuda()
        assert torch.equal(L.forward(x), q8p.Layer.from_qshp(art, device=0).forward(x)), (m, n)


@pytest.mark.gpu
def test_layers_from_qshp_bad_artifact_fails_whole_call():
    import paper_2402_04396_b200 as q8p

    good = random_artifact(512, 512, [("e8p-2bit", 1.11)], 3)
    with pytest.raises(q8p.FormatError):
        q8p.Layer.many_from_qshp([good, good[:100], good], device=0)
    assert q8p.Layer.many_from_qshp([], device=0) == []
