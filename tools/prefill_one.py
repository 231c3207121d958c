import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_2402_04396_b200 as q8p
from conftest import random_artifact
m, n, batch = (int(v) for v in os.environ.get("SHAPE", "28672x8192x512").split("x"))
L = q8p.Layer.from_qshp(random_artifact(m, n, [("e8p-2bit", 1.11)], 3))
x = torch.randn(batch, n, device="cuda")
for _ in range(2):
    L.forward(x)
torch.cuda.synchronize()
print("ok")
