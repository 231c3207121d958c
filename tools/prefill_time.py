"""Time one layer forward at prefill batch sizes (graph-free, CUDA events)."""
import os, sys, statistics
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch, bench
import paper_2402_04396_b200 as q8p
m, n = (int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "8192x8192").split("x"))
L = q8p.Layer.from_qshp(bench.make_artifact(m, n, 3), device=0)
for batch in [int(b) for b in (sys.argv[2] if len(sys.argv) > 2 else "16,128,512").split(",")]:
    x = torch.randn(batch, n, device="cuda")
    y = torch.empty(batch, m, device="cuda")
    ws = L.workspace(batch)
    for _ in range(2):
        L.forward(x, out=y, workspace=ws)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(5):
        a.record(); L.forward(x, out=y, workspace=ws); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    t = statistics.median(ts)
    ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
    ev[0].record(); ev[1].record()
    L.forward(x, out=y, workspace=ws, gemv_events=ev)  # K2 of the first chunk
    torch.cuda.synchronize()
    k2 = ev[0].elapsed_time(ev[1])
    print(f"{m}x{n} batch {batch}: {t:.3f} ms  {2 * m * n * batch / (t * 1e-3) / 1e12:.2f} TFLOP/s-equiv  "
          f"{batch / (t * 1e-3):.0f} tokens/s  (K2 of the first chunk {k2 * 1e3:.1f} us)", flush=True)
