"""Small forwards through every path for compute-sanitizer (memcheck):
rht 2/3/4-bit at batch 1/5/20/40, rfft, sharded rows_z, layer sets."""
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
        for b in (1, 5, 20, 40, 64):
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
print("sanitize run ok")
v = torch.randn(5000, 8, dtype=torch.float64, device="cuda")
q8p.e8p_encode(v)
q8p.rvq_quantize(v, [(q8p.CB_E8P_2BIT, 1.0), (q8p.CB_E8_1BIT, 0.5)])
w = torch.randn(96, 160, dtype=torch.float64, device="cuda")
q8p.rht_cols_f64(w, torch.randint(0, 256, (12,), dtype=torch.uint8, device="cuda"))
torch.cuda.synchronize()
print("sanitize producer ok")
