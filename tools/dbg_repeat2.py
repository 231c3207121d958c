import sys, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2402_04396_b200 as q8p
from conftest import random_artifact
bad = tot = 0
for it in range(10):
    for (m, n, batch) in [(4096, 28672, 4), (8192, 28672, 3)]:
        art = random_artifact(m, n, [("e8p-2bit", 1.11)], m + n + it)
        x = torch.randn(batch, n, generator=torch.Generator().manual_seed(it)).cuda()
        L = q8p.Layer.from_qshp(art, device=0)
        z0 = L.rows_z(x)
        y0 = L.forward(x)
        for k in range(4):
            tot += 1
            z = L.rows_z(x)
            y = L.forward(x)
            if not torch.equal(y, y0) or not torch.equal(z, z0):
                bad += 1
                for b in range(batch):
                    d = (y[b] - y0[b]); dz = (z[b] - z0[b])
                    c = float((d @ y0[b]) / (y0[b] @ y0[b]))
                    print(f"MISMATCH it{it} {m}x{n} b{batch} k{k} vec{b}: y relerr {float(d.norm()/y0[b].norm()):.3e} proj {c:.3f} | z relerr {float(dz.norm()/z0[b].norm()):.3e} zproj {float((dz @ z0[b])/(z0[b] @ z0[b])):.3f}")
print("bad", bad, "of", tot)
