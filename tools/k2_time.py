"""Time K2 (CUDA events around the GEMV inside forward) on one layer shape, 2 copies (cold L2)."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2402_04396_b200 as q8p
shapes = sys.argv[1:] or ["28672x8192"]
for sh in shapes:
    m, n = (int(v) for v in sh.split("x"))
    Ls = [q8p.Layer.from_qshp(bench.make_artifact(m, n, 7 + c), device=0) for c in range(2)]
    x = torch.randn(1, n, device="cuda")
    y = torch.empty(1, m, device="cuda")
    ws = torch.empty(Ls[0].workspace_bytes(1) + (1 << 20), dtype=torch.uint8, device="cuda")
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(2)]
    for a, b in ev:
        a.record(); b.record()
    ts = []
    for it in range(60):
        c = it % 2
        Ls[c].forward(x, out=y, workspace=ws, gemv_events=ev[c])
        torch.cuda.synchronize()
        if it >= 10:
            ts.append(ev[c][0].elapsed_time(ev[c][1]) * 1e3)
    b = m * n // 4 + 4 * (m + n)
    t = statistics.median(ts)
    print(f"{sh}: K2 {t:.2f} us  {b / t / 1e3:.0f} GB/s", flush=True)
