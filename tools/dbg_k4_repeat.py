"""Debug: run-to-run repeatability of the K4 prefill path (deterministic by design:
any difference between repeats is a race).  Prints per case the number of repeats
that differ bitwise from the first, and the first repeat's error vs the oracle."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_2402_04396_b200 as q8p
from conftest import random_artifact, rel_err
from oracle.refpy import Oracle

STAGES = {2: [("e8p-2bit", 1.11)], 3: [("e8p-2bit", 1.02), ("e8-1bit", 0.49)],
          4: [("e8p-2bit", 0.97), ("e8p-2bit", 0.29)]}
R = int(os.environ.get("REPS", "30"))
orc = Oracle()
for (m, n, bits, batch) in [(1024, 2048, 3, 64), (1024, 2048, 2, 64), (1024, 2048, 4, 96), (4096, 4096, 3, 300),
                            (4096, 8192, 2, 512)]:
    art = random_artifact(m, n, STAGES[bits], 7 * bits + batch)
    L = q8p.Layer.from_qshp(art)
    x = np.random.default_rng(batch).standard_normal((batch, n)).astype(np.float32)
    xd = torch.from_numpy(x).cuda()
    ref = L.forward(xd).clone()
    diff = 0
    for r in range(R):
        y = L.forward(xd)
        if not torch.equal(y, ref):
            diff += 1
    torch.cuda.synchronize()
    err = ""
    if m * n <= 4096 * 4096 and batch <= 300:
        want = orc.infer(art, x[:4].astype(np.float64), threads=8)
        got = ref[:4].cpu().numpy()
        err = max(rel_err(got[b], want[b]) for b in range(4))
    print(f"{m}x{n} bits {bits} batch {batch}: {diff}/{R} repeats differ; err {err}", flush=True)
