"""Debug: per-CTA globaltimer span of the tcgen05 K2 (build with NVEXTRA=-DQ8P_K2_TRACE,
run with Q8P_TRACE): entry spread, setup, work-done, next to the event time."""
import glob, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
out = os.path.join(ROOT, "gpurun_out", "tl", "tc")
os.makedirs(os.path.dirname(out), exist_ok=True)
os.environ["Q8P_TRACE"] = out
import torch
import bench
import paper_2402_04396_b200 as q8p
for sh in os.environ.get("SHAPES", "4096x4096,8192x8192,28672x8192").split(","):
    m, n = (int(v) for v in sh.split("x"))
    Ls = [q8p.Layer.from_qshp(bench.make_artifact(m, n, 7 + c), device=0) for c in range(3)]
    x = torch.randn(1, n, device="cuda")
    for rep in range(2):
        for c in range(3):
            for f in glob.glob(out + ".*"):
                os.remove(f)
            Ls[c].forward(x)
            torch.cuda.synchronize()
            f = [g for g in glob.glob(out + ".*") if ".fused." not in g]
            if not f or rep < 1:
                continue
            t = np.fromfile(f[0], dtype=np.uint64)
            g = t[11 * 128 * 4: 11 * 128 * 4 + 148 * 4].reshape(-1, 4).astype(np.int64)
            g = g[g[:, 0] > 0]
            t0 = g[:, 0].min()
            r = (g - t0) / 1e3
            print(f"TC {sh} copy{c}: ctas {len(g)} entry max {r[:,0].max():.2f} | setup med {np.median(r[:,1]):.2f} | end min {r[:,2].min():.2f} med {np.median(r[:,2]):.2f} max {r[:,2].max():.2f}")
