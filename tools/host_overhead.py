"""Host-side cost of one Layer.forward call (no sync) and the e2e step pattern."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, bench
import paper_2402_04396_b200 as q8p
L = q8p.Layer.from_qshp(bench.make_artifact(8192, 8192, 3), device=0)
x = torch.randn(1, 8192, device="cuda"); y = torch.empty(1, 8192, device="cuda"); ws = L.workspace(1)
s = torch.cuda.Stream()
for _ in range(20):
    L.forward(x, out=y, workspace=ws, stream=s)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(200):
    L.forward(x, out=y, workspace=ws, stream=s)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host per Layer.forward: {(t1 - t0) / 200 * 1e6:.1f} us")
hx = torch.randn(1, 8192).pin_memory(); hy = torch.empty(1, 8192).pin_memory()
t0 = time.perf_counter()
for _ in range(200):
    with torch.cuda.stream(s):
        x.copy_(hx, non_blocking=True); L.forward(x, out=y, workspace=ws, stream=s); hy.copy_(y, non_blocking=True)
t1 = time.perf_counter()
torch.cuda.synchronize()
print(f"host per copy+forward+copy: {(t1 - t0) / 200 * 1e6:.1f} us")
