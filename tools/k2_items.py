"""Debug: per-item phase breakdown of the tcgen05 K2 decoder groups and MMA issuers
(CTA 0 clock64 stamps; build with NVEXTRA=-DQ8P_K2_TRACE, run with Q8P_TRACE).
Decoder stamps per item: 0 before the code-slab wait, 1 slab landed, 2 A buffer free
(after the decode), 3 A tile stored + arrived.  Issuer: 0 start, 1 A full, 2 B full, 3 issued."""
import glob, os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
out = os.path.join(ROOT, "gpurun_out", "tl", "it")
os.makedirs(os.path.dirname(out), exist_ok=True)
os.environ["Q8P_TRACE"] = out
import torch
import bench
import paper_2402_04396_b200 as q8p
K = 128
for sh in os.environ.get("SHAPES", "28672x8192").split(","):
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
    t = np.fromfile(f[0], dtype=np.uint64).astype(np.int64)
    tr = t[: 16 * K * 4].reshape(16, K, 4)  # roles 0-10, 11-12 = per-CTA globaltimer, 13-14 = issuers g1, g2
    base = tr[tr > 0].min()
    print(f"== {sh}")
    for g in range(3):
        d = tr[g]
        d = d[(d > 0).all(axis=1)]
        if len(d) < 3: continue
        d = d - base
        ph = np.diff(d, axis=1)
        gap = d[1:, 0] - d[:-1, 3]
        per = np.diff(d[:, 0])
        print(f"dec g{g}: items {len(d)} | slab wait {np.median(ph[:,0]):6.0f} | decode+A wait {np.median(ph[:,1]):6.0f} | "
              f"store+arrive {np.median(ph[:,2]):6.0f} | gap {np.median(gap):6.0f} | per item {np.median(per):6.0f} cyc")
    for g, role in [(0, 8), (1, 13), (2, 14)]:
        d = tr[role]
        d = d[(d > 0).all(axis=1)]
        if len(d) < 3: continue
        d = d - base
        ph = np.diff(d, axis=1)
        per = np.diff(d[:, 0])
        print(f"mma g{g}: items {len(d)} | A wait {np.median(ph[:,0]):6.0f} | B wait {np.median(ph[:,1]):6.0f} | "
              f"issue {np.median(ph[:,2]):6.0f} | per item {np.median(per):6.0f} cyc")
    d = tr[9]; d = d[(d > 0).all(axis=1)] - base
    if len(d) > 3:
        print(f"producer: items {len(d)} | slot wait median {np.median(d[:,1]-d[:,0]):.0f} cyc")
    if len(tr[10]) and tr[10][0][1] > 0:
        print("setup (cyc from entry):", tr[10][0][1] - tr[10][0][0], "first decode ready:", tr[10][1][0] - tr[10][0][0])
