import sys, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2402_04396_b200 as q8p
from conftest import random_artifact
n, batch = 28672, 9
art = random_artifact(4096, n, [("e8p-2bit", 1.11)], 5)
L = q8p.Layer.from_qshp(art, device=0)
x = torch.randn(batch, n, generator=torch.Generator().manual_seed(1)).cuda()
z0 = L.rows_z(x)
bad = sum(0 if torch.equal(L.rows_z(x), z0) else 1 for _ in range(3))
print("bad", bad)
