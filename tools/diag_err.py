"""Diagnose per-element deviations of the GPU forward vs the oracle on one shape."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np, torch
import paper_2402_04396_b200 as q8p
from conftest import random_artifact
from oracle.refpy import Oracle
m, n = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "8192x28672").split("x"))
art = random_artifact(m, n, [("e8p-2bit", 1.11)], m ^ n)
L = q8p.Layer.from_qshp(art)
x = np.random.default_rng(7).standard_normal((1, n)).astype(np.float32).astype(np.float64)
want = Oracle().infer(art, x, threads=16)[0]
got = L.forward(torch.from_numpy(x.astype(np.float32)).cuda()).cpu().numpy()[0].astype(np.float64)
d = np.abs(got - want)
print("rel", np.linalg.norm(got - want) / np.linalg.norm(want), "max abs", d.max(), "median abs", np.median(d),
      "rms y", np.sqrt(np.mean(want ** 2)))
idx = np.argsort(-d)[:12]
print("worst idx", idx, d[idx])
# is the error in z (before K3)?  compare y-domain errors' structure: transform back
