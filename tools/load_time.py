"""Load time of the 70B layer set (3 layers, 134.6 MB of codes): one q8p_layer_from_qshp
per layer vs q8p_layers_from_qshp (concurrent parse / upload / transcode)."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch
import paper_2402_04396_b200 as q8p
from conftest import random_artifact
arts = [random_artifact(m, n, [("e8p-2bit", 1.11)], i) for i, (m, n) in enumerate([(8192, 8192), (28672, 8192), (8192, 28672)])]
torch.zeros(1, device="cuda"); torch.cuda.synchronize()
q8p.Layer.from_qshp(arts[0]).close()  # warm (tables, context)
seq, many = [], []
for rep in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); Ls = [q8p.Layer.from_qshp(a) for a in arts]; torch.cuda.synchronize(); t1 = time.perf_counter()
    for L in Ls: L.close()
    torch.cuda.synchronize()
    t2 = time.perf_counter(); Ms = q8p.Layer.many_from_qshp(arts); torch.cuda.synchronize(); t3 = time.perf_counter()
    for L in Ms: L.close()
    seq.append(1e3 * (t1 - t0)); many.append(1e3 * (t3 - t2))
print("sequential ms", [round(v, 1) for v in seq], "min", round(min(seq), 1))
print("layers_from_qshp ms", [round(v, 1) for v in many], "min", round(min(many), 1))
