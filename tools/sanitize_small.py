"""Small forwards through every path for compute-sanitizer (memcheck / initcheck):
rht 2/3/4-bit at batch 1/5/20/40/64/300 (K2 paths and the K4 prefill), rfft,
sharded rows_z, the push all-gather (one-process group of 2), large-batch
transforms, concurrent multi-layer loading, layer sets, the producer kernels."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_2402_04396_b200 as q8p
from conftest import random_artifact

ST = {2: [("e8p-2bit", 1.1)], 3: [("e8p-2bit", 1.0), ("e8-1bit", 0.5)], 4: [("e8p-2bit", 0.97), ("e8p-2bit", 0.3)]}
for tr in (0, 1):
    for bits in (2, 3, 4):
        art = random_artifact(384, 512, ST[bits], bits, transform=tr)
        L = q8p.Layer.from_qshp(art)
        for b in (1, 5, 20, 40, 64, 300):
            y = L.forward(torch.randn(b, 512).cuda())
        z = q8p.Layer.from_qshp(art, rows=(128, 256)).rows_z(torch.randn(3, 512).cuda())
torch.cuda.synchronize()
Ls = [q8p.Layer.from_qshp(random_artifact(256, 256, ST[2], 9 + i)) for i in range(3)]
for conc in (False, True):
    S = q8p.LayerSet(Ls, concurrent=conc)
    S.forward([torch.randn(2, 256).cuda() for _ in Ls])
    hx, hy = torch.randn(2 * 768).pin_memory(), torch.empty(2 * 768).pin_memory()
    S.forward_host(hx, hy, 2)
torch.cuda.synchronize()
art = random_artifact(1024, 512, ST[2], 21)
sh = [q8p.Layer.from_qshp(art, rows=q8p.shard_rows(1024, 2, r)) for r in range(2)]
grp = [q8p.PeerGroup(0, 2, r, 32 * 512) for r in range(2)]
q8p.PeerGroup.connect_local(grp)
for b in (1, 3):
    q8p.forward_sharded_push_sim(sh, grp, torch.randn(b, 512).cuda())
q8p.rht(torch.randn(70, 4096).cuda(), torch.randint(0, 256, (512,), dtype=torch.uint8, device="cuda"), transpose=True)
many = q8p.Layer.many_from_qshp([random_artifact(256, 512, ST[b], 30 + b) for b in (2, 3, 4)])
for L in many:
    L.forward(torch.randn(2, 512).cuda())
torch.cuda.synchronize()
print("sanitize run ok")
v = torch.randn(5000, 8, dtype=torch.float64, device="cuda")
q8p.e8p_encode(v)
q8p.rvq_quantize(v, [(q8p.CB_E8P_2BIT, 1.0), (q8p.CB_E8_1BIT, 0.5)])
w = torch.randn(96, 160, dtype=torch.float64, device="cuda")
q8p.rht_cols_f64(w, torch.randint(0, 256, (12,), dtype=torch.uint8, device="cuda"))
torch.cuda.synchronize()
print("sanitize producer ok")
