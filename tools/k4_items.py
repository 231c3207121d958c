"""Debug: K4 per-item timeline (CTA 0; build with NVEXTRA=-DQ8P_K4_TRACE, run with Q8P_TRACE)."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
out = os.path.join(ROOT, "gpurun_out", "tl", "k4")
os.makedirs(os.path.dirname(out), exist_ok=True)
os.environ["Q8P_TRACE"] = out
import torch
import paper_2402_04396_b200 as q8p
from conftest import random_artifact
m, n, batch = (int(v) for v in os.environ.get("SHAPE", "28672x8192x512").split("x"))
L = q8p.Layer.from_qshp(random_artifact(m, n, [("e8p-2bit", 1.11)], 3))
x = torch.randn(batch, n, device="cuda")
for _ in range(2):
    L.forward(x)
torch.cuda.synchronize()
K = 512
t = np.fromfile(out + ".k4.bin", dtype=np.uint64).astype(np.int64).reshape(18, K, 8)
base = t[t > 0].min()
iss = t[0][:, :4]; iss = iss[(iss > 0).all(axis=1)] - base
ph = np.diff(iss, axis=1)
per = np.diff(iss[:, 0])
print(f"issuer: items {len(iss)} | A wait {np.median(ph[:,0]):.0f} (mean {ph[:,0].mean():.0f}) | B wait {np.median(ph[:,1]):.0f} (mean {ph[:,1].mean():.0f}) | issue {np.median(ph[:,2]):.0f} | per item median {np.median(per):.0f} mean {per.mean():.0f} cyc")
big = per > 3 * np.median(per)
print("  long gaps (> 3x median):", int(big.sum()), "total cyc", int(per[big].sum()), "of", int(per.sum()))
for w in range(16):
    d = t[2 + w][:, [0, 2, 2, 4, 3]]; d = d[(d[:, [0, 2, 3, 4]] > 0).all(axis=1)] - base
    if len(d) < 3: continue
    ph = np.diff(d, axis=1); per = np.diff(d[:, 0])
    print(f"   w{w}: decode+sts {np.median(ph[:,2]):.0f} | fence+syncwarp {np.median(ph[:,3]):.0f}")
    print(f"dec w{w}: items {len(d)} | code wait {np.median(ph[:,0]):.0f} (mean {ph[:,0].mean():.0f}) | A-empty wait {np.median(ph[:,1]):.0f} (mean {ph[:,1].mean():.0f}) | decode+store {np.median(ph[:,2]):.0f} | per item {np.median(per):.0f} mean {per.mean():.0f}")
