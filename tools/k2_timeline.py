"""Debug: per-CTA globaltimer timeline of the warp-MMA K2 (Q8P_TRACE) next to its
event-timed duration, on a few layer shapes (three copies each, so the traced
launch streams from HBM).  Prints, per launch: event us, CTA entry spread,
setup (entry -> LUT/barriers done), first B image, last CTA done."""
import glob, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
out = os.path.join(ROOT, "gpurun_out", "tl", "t")
os.makedirs(os.path.dirname(out), exist_ok=True)
if not os.environ.get("NO_TRACE"): os.environ["Q8P_TRACE"] = out
import torch
import bench
import paper_2402_04396_b200 as q8p
shapes = [s for s in os.environ.get("SHAPES", "4096x4096,8192x8192,28672x8192").split(",")]
for sh in shapes:
    m, n = (int(v) for v in sh.split("x"))
    Ls = [q8p.Layer.from_qshp(bench.make_artifact(m, n, 7 + c), device=0) for c in range(3)]
    x = torch.randn(1, n, device="cuda")
    for rep in range(3):
        for c in range(3):
            e = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            e[0].record(); e[1].record()
            for f in glob.glob(out + ".mma.*"):
                os.remove(f)
            y = Ls[c].forward(x, gemv_events=e)
            torch.cuda.synchronize()
            us = e[0].elapsed_time(e[1]) * 1e3
            f = glob.glob(out + ".mma.*")
            if not f or rep < 2:
                continue
            t = np.fromfile(f[0], dtype=np.uint64).reshape(-1, 4)
            t = t[t[:, 0] > 0].astype(np.int64)
            t0 = t[:, 0].min()
            r = (t - t0) / 1e3
            print(f"{sh} copy{c}: event {us:.1f} us | ctas {len(t)} entry max {r[:,0].max():.2f} | setup med {np.median(r[:,1]-r[:,0]):.2f} "
                  f"| firstB med {np.median(r[:,2]):.2f} max {r[:,2].max():.2f} | end min {r[:,3].min():.2f} med {np.median(r[:,3]):.2f} max {r[:,3].max():.2f}")
