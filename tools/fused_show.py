import sys, numpy as np
raw = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64)
p = raw[12 * 128 * 4: 12 * 128 * 4 + 148 * 12].reshape(148, 12)
g = raw[11 * 128 * 4: 11 * 128 * 4 + 148 * 4].reshape(148, 4)
t0 = g[:, 0][g[:, 0] > 0].min()
names = ["start", "pdl_ok", "p1_done", "bar1", "p2_done", "bar2", "loop_end", "bar3", "p3_done", "bar4", "p4_done"]
for k, nm in enumerate(names):
    v = p[:, k]
    v = v[v > 0] - t0
    if len(v):
        print(f"{nm:9s} min {v.min():7d} med {int(np.median(v)):7d} max {v.max():7d} ns")
e = g[:, 2][g[:, 2] > 0] - t0
print(f"{'cta_end':9s} min {e.min():7d} med {int(np.median(e)):7d} max {e.max():7d} ns")
