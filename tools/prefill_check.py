"""Prefill K4: accuracy vs the oracle and timing vs the 32-vector-chunk path (Q8P_PREFILL=0 in a subprocess)."""
import os, subprocess, sys, time
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_2402_04396_b200 as q8p
from conftest import random_artifact
from oracle.refpy import Oracle
orc = Oracle()
STAGES = {2: [("e8p-2bit", 1.11)], 3: [("e8p-2bit", 1.02), ("e8-1bit", 0.49)], 4: [("e8p-2bit", 0.97), ("e8p-2bit", 0.29)]}
mode = os.environ.get("Q8P_PREFILL", "1")
for (m, n, batch, bits) in [(1024, 2048, 64, 2), (1024, 2048, 300, 3), (1024, 2048, 96, 4), (8192, 8192, 512, 2),
                            (28672, 8192, 512, 2), (8192, 28672, 512, 2), (8192, 8192, 2048, 2)]:
    art = random_artifact(m, n, STAGES[bits], m + n + batch)
    L = q8p.Layer.from_qshp(art)
    x = torch.randn(batch, n, generator=torch.Generator().manual_seed(batch)).cuda()
    y = L.forward(x)
    idx = [0, batch // 2, batch - 1]
    want = orc.infer(art, x[idx].cpu().numpy().astype(np.float64), threads=16)
    err = max(float(np.linalg.norm(y[i].cpu().numpy() - want[k]) / np.linalg.norm(want[k])) for k, i in enumerate(idx))
    ws = L.workspace(batch)
    for _ in range(3):
        L.forward(x, out=y, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        L.forward(x, out=y, workspace=ws)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    tf = 2.0 * m * n * batch / (ms * 1e-3) / 1e12
    print(f"prefill={mode} {m}x{n} b{batch} {bits}bit: rel err {err:.2e}  forward {ms:.3f} ms  {tf:.0f} TFLOP/s-equiv")
