"""Debug: dump K2's CTA-0 timeline (Q8P_TRACE) for one big layer."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "trace", "t")
os.makedirs(os.path.dirname(out), exist_ok=True)
os.environ["Q8P_TRACE"] = out
import torch
import bench
import paper_2402_04396_b200 as q8p
m, n = (int(v) for v in (sys.argv[2] if len(sys.argv) > 2 else os.environ.get("SHAPE", "28672x8192")).split("x"))
# 3 distinct copies (> L2 for the big layers) so the traced launch streams from HBM
Ls = [q8p.Layer.from_qshp(bench.make_artifact(m, n, 7 + c), device=0) for c in range(3)]
x = torch.randn(int(os.environ.get("BATCH", "1")), n, device="cuda")
for c in range(3):
    y = Ls[c].forward(x)
torch.cuda.synchronize()
print("ok", y.shape)
