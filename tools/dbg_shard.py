import sys, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import paper_2402_04396_b200 as q8p
from conftest import random_artifact
bad = 0
for it in range(6):
  for (m, n, world, batch) in [(8192, 28672, 2, 3), (28672, 8192, 4, 3), (8192, 28672, 8, 3), (8192, 8192, 2, 3)]:
    art = random_artifact(m, n, [("e8p-2bit", 1.11)], m + n + world)
    x = torch.randn(batch, n, generator=torch.Generator().manual_seed(world + batch)).cuda()
    full = q8p.Layer.from_qshp(art, device=0)
    shards = [q8p.Layer.from_qshp(art, device=0, rows=q8p.shard_rows(m, world, r)) for r in range(world)]
    yf = full.forward(x)
    for k in range(3):
        ys = q8p.forward_sharded_sim(shards, x); yf2 = full.forward(x)
        if not torch.equal(ys, yf) or not torch.equal(yf2, yf):
            bad += 1
            print("MISMATCH", it, m, n, world, batch, k, "sim==full", torch.equal(ys, yf), "full==full", torch.equal(yf, yf2),
                  "rows bad", [int(((ys[b]-yf[b]).abs() > 0).sum()) for b in range(batch)], float((ys-yf).abs().max()))
print("bad", bad)
