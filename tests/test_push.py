"""Push all-gather: q8p_forward_sharded_push fuses the
z all-gather into K3 pass 1 -- every rank stores its rows straight into every
rank's window (peer memory over NVLink, CUDA IPC mappings) as {value, call tag}
words; K3 pass 2 reads its own window as the tagged words arrive.  The rows are
independent in the reference (core/src/pipeline.cpp:176-191), so every rank's y
must equal the unsharded forward bit for bit.

GPU (one B200): (1) the whole group in one process, wired directly, every rank's
forward in stream order (data placement, call tags / window parity over repeated
calls and multi-chunk batches); (2) world 1 through the public API;
(3) two processes on the same GPU exchanging CUDA IPC handles over gloo -- the
real cross-process protocol, with the two ranks' kernels time-sliced.
"""
from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
STAGES = {2: [("e8p-2bit", 1.11)], 3: [("e8p-2bit", 1.02), ("e8-1bit", 0.49)],
          4: [("e8p-2bit", 0.97), ("e8p-2bit", 0.29)]}


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("m,n,bits", [(8192, 8192, 2), (28672, 8192, 2), (4096, 11008, 3), (11008, 4096, 4)])
def test_push_sim_bit_exact_repeated(world, m, n, bits):
    import torch

    import paper_2402_04396_b200 as q8p
    from conftest import random_artifact

    art = random_artifact(m, n, STAGES[bits], m + n + 3 * world)
    full = q8p.Layer.from_qshp(art, device=0)
    shards = [q8p.Layer.from_qshp(art, device=0, rows=q8p.shard_rows(m, world, r)) for r in range(world)]
    ml = m // world
    group = [q8p.PeerGroup(0, world, r, 32 * ml) for r in range(world)]
    q8p.PeerGroup.connect_local(group)
    # 5 calls: both window parities twice; batch 40 = two chunks = two epochs in one call
    for it, batch in enumerate([1, 3, 40, 2, 1]):
        x = torch.randn(batch, n, generator=torch.Generator().manual_seed(it + world)).cuda()
        ys = q8p.forward_sharded_push_sim(shards, group, x)
        want = full.forward(x)
        for r in range(world):
            assert torch.equal(ys[r], want), (it, r)
    assert [g.state() for g in group] == [6] * world  # K3 chunks (push calls) completed per rank


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("m,n,bits,batch", [(8192, 8192, 2, 96), (28672, 8192, 2, 256), (4096, 4096, 3, 64)])
def test_push_sim_prefill(world, m, n, bits, batch):
    # batches >= 64: K1 -> K4 on each rank's rows -> K3 pass 1 summing the rank's K-split
    # partials and pushing -> pass 2.  The K split is chosen per shard, so the fp32
    # partial sums may round differently from the unsharded forward: prefill bar 1e-4.
    import torch

    import paper_2402_04396_b200 as q8p
    from conftest import random_artifact

    art = random_artifact(m, n, STAGES[bits], m + n + world)
    full = q8p.Layer.from_qshp(art, device=0)
    shards = [q8p.Layer.from_qshp(art, device=0, rows=q8p.shard_rows(m, world, r)) for r in range(world)]
    group = [q8p.PeerGroup(0, world, r, batch * (m // world)) for r in range(world)]
    q8p.PeerGroup.connect_local(group)
    for it in range(3):  # both window parities
        x = torch.randn(batch, n, generator=torch.Generator().manual_seed(it)).cuda()
        ys = q8p.forward_sharded_push_sim(shards, group, x)
        want = full.forward(x)
        for r in range(world):
            assert torch.equal(ys[r], ys[0])
        rel = float((ys[0] - want).norm() / want.norm())
        assert rel < 1e-4, (it, rel)


@pytest.mark.gpu
def test_push_world1_public_api():
    import torch

    import paper_2402_04396_b200 as q8p
    from conftest import random_artifact

    m, n = 4096, 4096
    art = random_artifact(m, n, STAGES[2], 11)
    L = q8p.Layer.from_qshp(art, device=0)
    g = q8p.PeerGroup(0, 1, 0, 128 * m)
    g.connect([g.handle])
    for it, batch in enumerate([1, 7, 1, 33, 128, 2]):  # 128: the K4 prefill chain
        x = torch.randn(batch, n, generator=torch.Generator().manual_seed(it)).cuda()
        assert torch.equal(L.forward_sharded_push(x, g), L.forward(x)), it


@pytest.mark.gpu
def test_push_rejects_bad_setup():
    import torch

    import paper_2402_04396_b200 as q8p
    from conftest import random_artifact

    m, n = 4096, 4096
    art = random_artifact(m, n, STAGES[2], 12)
    shard = q8p.Layer.from_qshp(art, device=0, rows=q8p.shard_rows(m, 2, 1))
    g = q8p.PeerGroup(0, 2, 1, 1024)
    x = torch.randn(1, n).cuda()
    with pytest.raises(q8p.ValidationError):  # not connected
        shard.forward_sharded_push(x, g)
    with pytest.raises(q8p.ValidationError):
        g.connect([g.handle])  # wrong count
    with pytest.raises(q8p.ValidationError):
        q8p.PeerGroup(0, 2, 2, 1024)
    small = [q8p.PeerGroup(0, 2, r, 1024) for r in range(2)]
    q8p.PeerGroup.connect_local(small)
    shards = [q8p.Layer.from_qshp(art, device=0, rows=q8p.shard_rows(m, 2, r)) for r in range(2)]
    with pytest.raises(q8p.SizeError):  # window slice < m_local
        q8p.forward_sharded_push_sim(shards, small, x)


_RANK_SCRIPT = r"""
import os, sys
sys.path.insert(0, {root!r}); sys.path.insert(0, os.path.join({root!r}, "tests"))
import torch, torch.distributed as dist
import paper_2402_04396_b200 as q8p
from conftest import random_artifact
rank, world, port = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{{port}}", rank=rank, world_size=world)
m, n = 8192, 8192
art = random_artifact(m, n, [("e8p-2bit", 1.11)], 5)
full = q8p.Layer.from_qshp(art, device=0)
shard = q8p.Layer.from_qshp(art, device=0, rows=q8p.shard_rows(m, world, rank))
g = q8p.PeerGroup(0, world, rank, 32 * (m // world))
handles = [None] * world
dist.all_gather_object(handles, g.handle)
g.connect(handles)
dist.barrier()
ok = True
for it, batch in enumerate([1, 4, 1, 2]):
    x = torch.randn(batch, n, generator=torch.Generator().manual_seed(it)).cuda()
    y = shard.forward_sharded_push(x, g)
    torch.cuda.synchronize()
    ok &= bool(torch.equal(y, full.forward(x)))
dist.barrier()
g.close()
print("PUSH_OK" if ok else "PUSH_MISMATCH", flush=True)
dist.destroy_process_group()
"""


@pytest.mark.gpu
def test_push_two_processes_one_gpu(tmp_path):
    import subprocess

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    script = tmp_path / "rank.py"
    script.write_text(_RANK_SCRIPT.format(root=ROOT))
    procs = [subprocess.Popen([sys.executable, str(script), str(r), "2", str(port)], stdout=subprocess.PIPE,
                              stderr=subprocess.STDOUT, text=True) for r in range(2)]
    outs = []
    for p in procs:
        try:
            out, _ = p.communicate(timeout=300)
        except subprocess.TimeoutExpired:
            for q in procs:
                q.kill()
            raise
        outs.append(out)
    for r, (p, out) in enumerate(zip(procs, outs)):
        assert p.returncode == 0 and "PUSH_OK" in out, (r, out[-2000:])
