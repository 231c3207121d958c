import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_2402_04396_b200 as q8p
from conftest import random_artifact
m, n, world = 8192, 8192, 2
art = random_artifact(m, n, [("e8p-2bit", 1.11)], 3)
full = q8p.Layer.from_qshp(art, device=0)
shards = [q8p.Layer.from_qshp(art, device=0, rows=q8p.shard_rows(m, world, r)) for r in range(world)]
group = [q8p.PeerGroup(0, world, r, 32 * m // world) for r in range(world)]
q8p.PeerGroup.connect_local(group)
print("state0", [g.state() for g in group], flush=True)
x = torch.randn(1, n).cuda()
ys = q8p.forward_sharded_push_sim(shards, group, x)
torch.cuda.synchronize()
print("state1", [g.state() for g in group], flush=True)
print("eq", [bool(torch.equal(ys[r], full.forward(x))) for r in range(world)])
