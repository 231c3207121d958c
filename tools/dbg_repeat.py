"""Repeatability probe: the same forward twice must give identical y (exact integer path)."""
import sys, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2402_04396_b200 as q8p
from conftest import random_artifact
bad = tot = 0
for it in range(8):
    for (m, n, batch) in [(8192, 28672, 3), (8192, 28672, 1), (28672, 8192, 3), (8192, 8192, 3), (4096, 28672, 4)]:
        art = random_artifact(m, n, [("e8p-2bit", 1.11)], m + n + it)
        x = torch.randn(batch, n, generator=torch.Generator().manual_seed(it)).cuda()
        L = q8p.Layer.from_qshp(art, device=0)
        y0 = L.forward(x)
        for k in range(4):
            tot += 1
            if not torch.equal(L.forward(x), y0):
                bad += 1
                print("MISMATCH", it, m, n, batch, k)
print("bad", bad, "of", tot)
