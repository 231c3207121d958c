import os, sys, statistics
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import torch, paper_2402_04396_b200 as q8p
from conftest import random_artifact
for bits, st in [(3, [("e8p-2bit", 1.0), ("e8-1bit", 0.5)]), (4, [("e8p-2bit", 0.97), ("e8p-2bit", 0.3)])]:
    L = q8p.Layer.from_qshp(random_artifact(8192, 8192, st, 3))
    for batch in (16, 32, 512):
        x = torch.randn(batch, 8192, device="cuda"); y = torch.empty(batch, 8192, device="cuda"); ws = L.workspace(batch)
        for _ in range(2): L.forward(x, out=y, workspace=ws)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for _ in range(5):
            a.record(); L.forward(x, out=y, workspace=ws); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b))
        print(f"{bits}-bit 8192^2 batch {batch}: {statistics.median(ts):.3f} ms", flush=True)
