import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_2402_04396_b200 as q8p
from conftest import random_artifact
for (m, n) in [(8192, 8192), (28672, 8192), (8192, 28672)]:
    art = random_artifact(m, n, [("e8p-2bit", 1.11)], 3)
    L = q8p.Layer.from_qshp(art, device=0, rows=(0, m))
    g = q8p.PeerGroup(0, 1, 0, 32 * m)
    g.connect([g.handle])
    comm = q8p.NcclComm(q8p.NcclComm.unique_id(), 1, 0, 0)
    x = torch.randn(1, n, device="cuda")
    ws = L.workspace(1)
    y = torch.empty(1, m, device="cuda")
    s = torch.cuda.Stream()
    res = {}
    for name, fn in [("nccl", lambda: L.forward_sharded(x, comm, out=y, stream=s, workspace=ws)),
                     ("push", lambda: L.forward_sharded_push(x, g, out=y, stream=s, workspace=ws)),
                     ("plain", lambda: L.forward(x, out=y, stream=s, workspace=ws))]:
        with torch.cuda.stream(s):
            for _ in range(5): fn()
            s.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            for _ in range(50): fn()
            e1.record(s)
            s.synchronize()
        res[name] = e0.elapsed_time(e1) / 50 * 1e3
    print(m, n, {k: round(v, 1) for k, v in res.items()}, "state", g.state(), flush=True)
    g.close(); comm.close()
