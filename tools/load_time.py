"""Layer upload time (QSHP bytes -> device layer) at the 70B MLP shape."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2402_04396_b200 as q8p
art = bench.make_artifact(28672, 8192, 1)
torch.cuda.init()
q8p.Layer.from_qshp(bench.make_artifact(256, 256, 2))
for _ in range(2):
    t0 = time.perf_counter(); L = q8p.Layer.from_qshp(art); torch.cuda.synchronize(); t1 = time.perf_counter()
    print(f"from_qshp 28672x8192 ({len(art) / 1e6:.1f} MB): {1e3 * (t1 - t0):.0f} ms")
    del L
