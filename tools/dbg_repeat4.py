import sys, torch, collections
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2402_04396_b200 as q8p
from conftest import random_artifact
res = collections.Counter(); tot = collections.Counter()
for it in range(6):
    for n in (16384, 28672):
        art = random_artifact(4096, n, [("e8p-2bit", 1.11)], n + it)
        L = q8p.Layer.from_qshp(art, device=0)
        for batch in (9, 12, 13, 16):
            x = torch.randn(batch, n, generator=torch.Generator().manual_seed(it)).cuda()
            z0 = L.rows_z(x)
            for k in range(4):
                tot[(n, batch)] += 1
                if not torch.equal(L.rows_z(x), z0):
                    res[(n, batch)] += 1
print(" ".join(f"{key}:{res[key]}/{tot[key]}" for key in sorted(tot)))
