"""Row-sharded forward: rank g holds rows shard_rows(m, G, g),
computes its z slice, the slices are all-gathered (NCCL on the GPU path),
then every rank applies the output transform T_u^T to the full z.

CPU (gloo, world 2): the decomposition itself, checked against the oracle
infer (oracle/latq_oracle.c, which restates core/src/pipeline.cpp:151-197).
GPU: q8p_forward_sharded through the C ABI over a real NCCL communicator
(world 1 on the single-GPU box) is bit-identical to q8p_forward; multi-GPU
runs (torchrun) go through bench.py --gpus N.
"""
from __future__ import annotations

import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN


def _qshp_signs_scales(art: bytes):
    """QSHP v1 header fields (README.md:118-136 / pipeline.cpp:323-383)."""
    assert art[:4] == b"QSHP"
    _ver, m, n, kind, S = struct.unpack_from("<HIIBB", art, 4)
    off = 4 + 2 + 4 + 4 + 1 + 1
    scales = []
    for _ in range(S):
        ln = art[off]
        off += 1 + ln
        scales.append(struct.unpack_from("<f", art, off)[0])
        off += 4
    su = np.frombuffer(art, np.uint8, (m + 7) // 8, off)
    off += (m + 7) // 8
    sv = np.frombuffer(art, np.uint8, (n + 7) // 8, off)
    return m, n, scales, su, sv


def test_shard_rows_partition():
    import paper_2402_04396_b200 as q8p
    for m, world in [(8192, 2), (28672, 8), (4096, 4), (128, 1)]:
        spans = [q8p.shard_rows(m, world, r) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == m
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        assert len({hi - lo for lo, hi in spans}) == 1
    with pytest.raises(q8p.ValidationError):
        q8p.shard_rows(11008, 3, 0)
    with pytest.raises(q8p.ValidationError):
        q8p.shard_rows(64, 2, 2)


def _rank_main(rank: int, world: int, port: int, name: str, q):
    import torch
    import torch.distributed as dist

    import paper_2402_04396_b200 as q8p
    from oracle.refpy import Oracle

    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        art = open(os.path.join(GOLDEN, f"{name}.qshp"), "rb").read()
        x = np.load(os.path.join(GOLDEN, f"{name}.x.npy"))[:2]
        orc = Oracle()
        m, n, scales, su, sv = _qshp_signs_scales(art)
        lo, hi = q8p.shard_rows(m, world, rank)
        w_loc = sum(np.float64(sc) * orc.decode_stage(art, s)[lo:hi] for s, sc in enumerate(scales))
        z_loc = np.stack([w_loc @ orc.side_apply(sv, xb) for xb in x])  # [B][m/G]
        parts = [torch.zeros(z_loc.shape, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(parts, torch.from_numpy(z_loc))
        z = torch.cat(parts, dim=1).numpy()
        y = np.stack([orc.side_apply(su, zb, transpose=True) for zb in z])
        want = orc.infer(art, x)
        q.put((rank, float(np.max(np.abs(y - want)) / np.max(np.abs(want)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["e8p2_128x256", "rvq3_256x128", "rvq4_128x128"])
def test_row_sharded_decomposition_gloo(name):
    import socket

    import torch.multiprocessing as mp

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    res = dict(q.get(timeout=5) for _ in range(2))
    assert set(res) == {0, 1}
    for r, err in res.items():
        assert err < 1e-12, (r, err)


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["e8p2_1024x1024", "rvq3_256x128", "rvq4_128x128", "rfft2_344x512"])
def test_forward_sharded_world1_bit_exact(name):
    import torch

    import paper_2402_04396_b200 as q8p

    art = open(os.path.join(GOLDEN, f"{name}.qshp"), "rb").read()
    x = torch.from_numpy(np.load(os.path.join(GOLDEN, f"{name}.x.npy")).astype(np.float32)).cuda()
    comm = q8p.NcclComm(q8p.NcclComm.unique_id(), 1, 0, 0)
    try:
        L = q8p.Layer.from_qshp(art, device=0)
        y0 = L.forward(x)
        before = q8p.kernel_launches()
        y1 = L.forward_sharded(x, comm)
        torch.cuda.synchronize()
        assert q8p.kernel_launches() > before
        assert torch.equal(y0, y1)
    finally:
        comm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [3, 16, 20])
def test_forward_sharded_world1_batches(batch):
    import torch

    import paper_2402_04396_b200 as q8p

    art = open(os.path.join(GOLDEN, "rvq4_128x128.qshp"), "rb").read()
    x = torch.randn(batch, 128, generator=torch.Generator().manual_seed(batch)).cuda()
    comm = q8p.NcclComm(q8p.NcclComm.unique_id(), 1, 0, 0)
    try:
        L = q8p.Layer.from_qshp(art, device=0)
        assert torch.equal(L.forward(x), L.forward_sharded(x, comm))
    finally:
        comm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [64, 200])
def test_forward_sharded_world1_prefill(batch):
    # batches >= 64 take K4 on the rank's rows + K3 pass 1 on them + one all-gather:
    # at world 1 that is the unsharded prefill forward, bit for bit
    import torch

    import paper_2402_04396_b200 as q8p
    from conftest import random_artifact

    art = random_artifact(8192, 4096, [("e8p-2bit", 1.11)], 77)
    x = torch.randn(batch, 4096, generator=torch.Generator().manual_seed(batch)).cuda()
    comm = q8p.NcclComm(q8p.NcclComm.unique_id(), 1, 0, 0)
    try:
        L = q8p.Layer.from_qshp(art, device=0)
        assert torch.equal(L.forward(x), L.forward_sharded(x, comm))
    finally:
        comm.close()


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("bits", [2, 3])
def test_row_shards_on_one_gpu(world, bits):
    # What q8p_forward_sharded computes at G ranks, run on one GPU without NCCL:
    # every shard handle's z rows (K1 -> K2 on its rows -> combine) concatenate to
    # the full layer's z bit for bit (row sharding leaves each row's integer
    # accumulation unchanged), and T_u^T of that z is the layer's forward.
    import torch

    import paper_2402_04396_b200 as q8p
    from conftest import random_artifact

    m, n = 2048, 1024
    stages = {2: [("e8p-2bit", 1.11)], 3: [("e8p-2bit", 1.02), ("e8-1bit", 0.49)]}[bits]
    art = random_artifact(m, n, stages, 17 * world + bits)
    x = torch.randn(2, n, generator=torch.Generator().manual_seed(world)).cuda()
    full = q8p.Layer.from_qshp(art, device=0)
    z_full = full.rows_z(x)
    parts = [q8p.Layer.from_qshp(art, device=0, rows=q8p.shard_rows(m, world, r)).rows_z(x) for r in range(world)]
    assert torch.equal(torch.cat(parts, dim=1), z_full)
    _m, _n, _scales, su, _sv = _qshp_signs_scales(art)
    y = full.forward(x)
    y_from_z = q8p.rht(z_full, torch.from_numpy(su.copy()).cuda(), transpose=True)
    rel = float((y_from_z - y).norm() / y.norm())
    assert rel < 1e-5, rel


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("m,n,bits", [(8192, 8192, 2), (28672, 8192, 2), (8192, 28672, 2), (4096, 11008, 3),
                                      (11008, 4096, 4)])
@pytest.mark.parametrize("batch", [1, 3])
def test_sharded_forward_sim_bit_exact(world, m, n, bits, batch):
    # q8p_forward_sharded's data path at G ranks on one GPU (all-gather replaced by
    # copies): per-rank K1 -> K2 on its rows -> K3 pass 1 on its rows into the send
    # buffer, the rank-major gather, K3 pass 2 -> y equals the unsharded forward bit
    # for bit (70B shapes incl. base 28, the 7B MLP shapes incl. base 172).
    import torch

    import paper_2402_04396_b200 as q8p
    from conftest import random_artifact

    stages = {2: [("e8p-2bit", 1.11)], 3: [("e8p-2bit", 1.02), ("e8-1bit", 0.49)],
              4: [("e8p-2bit", 0.97), ("e8p-2bit", 0.29)]}[bits]
    art = random_artifact(m, n, stages, m + n + world)
    x = torch.randn(batch, n, generator=torch.Generator().manual_seed(world + batch)).cuda()
    full = q8p.Layer.from_qshp(art, device=0)
    shards = [q8p.Layer.from_qshp(art, device=0, rows=q8p.shard_rows(m, world, r)) for r in range(world)]
    assert torch.equal(q8p.forward_sharded_sim(shards, x), full.forward(x))
