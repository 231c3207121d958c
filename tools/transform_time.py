"""Per-layer forward time, rht vs rfft artifacts (batch 1 and 16), CUDA graph of
R forwards over two layer copies, CUDA events.  Usage: python tools/transform_time.py"""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_2402_04396_b200 as q8p
from conftest import random_artifact

R = 20
for (m, n) in [(8192, 8192), (28672, 8192), (8192, 28672), (4096, 11008)]:
    for tr in (0, 1):
        Ls = [q8p.Layer.from_qshp(random_artifact(m, n, [("e8p-2bit", 1.1)], 7 + c, transform=tr)) for c in range(2)]
        for batch in (1, 16):
            x = torch.randn(batch, n, device="cuda")
            y = torch.empty(batch, m, device="cuda")
            ws = Ls[0].workspace(batch)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for L in Ls:
                    L.forward(x, out=y, workspace=ws, stream=s)
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for i in range(R):
                    Ls[i % 2].forward(x, out=y, workspace=ws, stream=s)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts = []
            for _ in range(5):
                g.replay()
                a.record(); g.replay(); b.record(); torch.cuda.synchronize()
                ts.append(a.elapsed_time(b) * 1e3 / R)
            print(f"{m}x{n} {'rfft' if tr else 'rht '} batch {batch:2d}: {statistics.median(ts):7.1f} us/layer",
                  flush=True)
