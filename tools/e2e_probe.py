"""Where does the e2e step time go?  70B layer set, batch 1, host-timed loops."""
import os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import bench
import paper_2402_04396_b200 as q8p

shapes = [(8192, 8192), (28672, 8192), (8192, 28672)]
copies = [[q8p.Layer.from_qshp(bench.make_artifact(m, n, 7 + 3 * c + i)) for i, (m, n) in enumerate(shapes)]
          for c in range(2)]
sets = [q8p.LayerSet(r) for r in copies]
nsum, msum = sum(n for _, n in shapes), sum(m for m, _ in shapes)
hx, hy = torch.randn(nsum).pin_memory(), torch.empty(msum).pin_memory()
dx, dy = torch.empty(nsum, device="cuda"), torch.empty(msum, device="cuda")
ws = torch.empty(max(S.workspace_bytes(1) for S in sets), dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
K = 200


def timeit(name, fn):
    for i in range(10):
        fn(i)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(K):
        fn(i)
    torch.cuda.synchronize()
    print(f"{name:48s} {(time.perf_counter() - t0) / K * 1e6:7.1f} us/step", flush=True)


timeit("set.forward_host (graph, pinned)", lambda i: sets[i % 2].forward_host(hx, hy, 1, stream=s, workspace=ws))
fn = q8p.lib().q8p_forward_set_host
args = [(S._arr, 3, hx.data_ptr(), hy.data_ptr(), 1, ws.data_ptr(), ws.numel(), s.cuda_stream) for S in sets]
timeit("raw ctypes q8p_forward_set_host", lambda i: fn(*args[i % 2]))
os.environ["Q8P_NO_SET_GRAPH"] = "1"  # read once per process: no effect after first call; kept for symmetry


def memcpy_only(i):
    dx.copy_(hx, non_blocking=True)
    hy.copy_(dy, non_blocking=True)
    s.synchronize()


with torch.cuda.stream(s):
    timeit("H2D + D2H + sync only", memcpy_only)
    g = torch.cuda.CUDAGraph()
    xs = [dx[:n].view(1, n) for _, n in shapes]
    ys = [dy[:m].view(1, m) for m, _ in shapes]
    for r in copies:
        for L, x, y in zip(r, xs, ys):
            L.forward(x, out=y, stream=s, workspace=ws)
    torch.cuda.synchronize()
    graphs = []
    for r in copies:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for L, x, y in zip(r, xs, ys):
                L.forward(x, out=y, stream=s, workspace=ws)
        graphs.append(g)
    timeit("device graph replay + sync each step", lambda i: (graphs[i % 2].replay(), s.synchronize()))
    timeit("device graph replay, no sync", lambda i: graphs[i % 2].replay())
    e = torch.cuda.CUDAGraph()
    with torch.cuda.graph(e, stream=s):
        dx.add_(0)
    timeit("tiny graph replay + sync (latency floor)", lambda i: (e.replay(), s.synchronize()))

    def eager(i):
        dx.copy_(hx, non_blocking=True)
        for L, x, y in zip(copies[i % 2], xs, ys):
            L.forward(x, out=y, stream=s, workspace=ws)
        hy.copy_(dy, non_blocking=True)
        s.synchronize()
    timeit("eager per-layer API + copies + sync", eager)

    # torch-captured graph of the per-layer C calls with x / y in pinned host memory (zero-copy)
    fwd = q8p.lib().q8p_forward
    gz = []
    for r in copies:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            xo = yo = 0
            for L, (m, n) in zip(r, shapes):
                assert fwd(L._h, hx.data_ptr() + 4 * xo, hy.data_ptr() + 4 * yo, 1, ws.data_ptr(), ws.numel(),
                           s.cuda_stream) == 0
                xo += n
                yo += m
        gz.append(g)
    timeit("torch graph, zero-copy x/y in pinned host memory", lambda i: (gz[i % 2].replay(), s.synchronize()))
    os.environ["Q8P_NO_SET_GRAPH"] = "1"
