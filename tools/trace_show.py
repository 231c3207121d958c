import sys, numpy as np
t = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(16, 128, 4).astype(np.int64)
G = int(sys.argv[2]) if len(sys.argv) > 2 else 3
nz = t[t > 0]
t0 = nz.min()
t = np.where(t > 0, t - t0, -1)
print("role item: [ev0 ev1 ev2 ev3] (cycles from first stamp)")
print("kernel: start/after-setup/loop-end/end", t[10,0], " lut-ready", t[10,1,0])
for i in list(range(int(sys.argv[3]) if len(sys.argv) > 3 else 24)) + list(range(40, 60)):
    g = i % G
    print(f"item {i:3d} dec{g}: {t[g, i]}  mma: {t[8, i]}  prod: {t[9, i]}")
m = t[8]
v = m[m[:, 3] >= 0]
print("mma items", len(v), "span", v[-1, 3] - v[0, 0] if len(v) else 0, "per item", np.diff(v[:, 3]).mean() if len(v) > 1 else 0)
raw = np.fromfile(sys.argv[1], dtype=np.uint64).astype(np.int64)
g = raw[11 * 128 * 4: 11 * 128 * 4 + 148 * 4].reshape(148, 4)
if (g[:, 0] > 0).all():
    t0 = g[:, 0].min()
    print("globaltimer ns: entry min/max", 0, g[:, 0].max() - t0, " setup done max", g[:, 1].max() - t0,
          " end min/med/max", g[:, 2].min() - t0, int(np.median(g[:, 2] - t0)), g[:, 2].max() - t0)
