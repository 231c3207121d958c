#!/usr/bin/env python
"""Benchmark: QuIP# E8P 2-bit quantized linear layers at batch 1 on B200.

Metric (BASELINE.json): "E8P 2-bit quantized matvec: achieved HBM GB/s vs
peak; layer tokens/s at batch 1".  One step = one batch-1 token through the
Llama-2-70B-shaped layer set (8192x8192, 28672x8192, 8192x28672; configs[2]),
each layer y = S_U H^T W_hat H S_V x (K1 -> K2 -> K3).

  value    tokens/s of the layer set, inputs already in HBM (CUDA graph of
           the step, replayed K times, CUDA events on the launching stream,
           max over ranks).
  e2e      the same metric through the public API with HOST buffers: per
           step one q8p_forward_set_host call (H2D of every layer's x, the
           layer forwards, D2H of every y, stream sync; pinned buffers, so the
           library replays the step as one cached CUDA graph).  Sharded runs
           loop q8p_forward_sharded per layer between the two copies.
  roofline the decode-GEMV kernel (K2): algorithmic bytes
           (codes + 4 B x activations in + 4 B x outputs)
           / average kernel time from CUDA events recorded around K2.
  cpu_baseline  the reference latq::infer (oracle/_ref, compiled from the
           reference sources) on the box's host cores, bounded sample.

N > 1 (torchrun): the layers are row-sharded across ranks (each rank holds
m/N rows); by default K3 pass 1 pushes every rank's rows straight into every
rank's window over NVLink (q8p_forward_sharded_push, after a bit-exact self-check
against the NCCL all-gather path; --allgather nccl selects q8p_forward_sharded);
total work is fixed -> "scaling": "strong".

`--impl reference` times the reference CPU implementation instead (rank 0
only; other ranks exit 0).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import struct
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LAYERS_70B = [(8192, 8192), (28672, 8192), (8192, 28672)]
LAYERS_7B = [(4096, 4096)] * 4 + [(11008, 4096)] * 2 + [(4096, 11008)]
LAYERS_4096 = [(4096, 4096)]  # BASELINE configs[0]: one 4096 x 4096 layer
WORKLOADS = {"70b": LAYERS_70B, "7b": LAYERS_7B, "4096": LAYERS_4096}
METRIC = "E8P 2-bit quantized matvec: achieved HBM GB/s vs peak; layer tokens/s at batch 1"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


# default_scheme(bits) (rvq.cpp:9-21) stage codebooks, with the scales a unit-RMS
# layer gets (s = r1 / rho, r1 ~ 1)
SCHEMES = {2: [("e8p-2bit", 1.11)], 3: [("e8p-2bit", 1.02), ("e8-1bit", 0.49)],
           4: [("e8p-2bit", 0.97), ("e8p-2bit", 0.29)]}
CODE_BYTES = {"e8p-2bit": 2, "e8-1bit": 1}


def make_artifact(m: int, n: int, seed: int, scale: float = 1.11, bits: int = 2) -> bytes:
    """QSHP v1 with default_scheme(bits) stages, seeded synthetic codes and signs."""
    rng = np.random.default_rng(seed)
    stages = SCHEMES[bits] if bits != 2 else [("e8p-2bit", scale)]
    body = b"QSHP" + struct.pack("<HIIBB", 1, m, n, 0, len(stages))
    for cid, sc in stages:
        body += bytes([len(cid)]) + cid.encode() + struct.pack("<f", sc)
    body += rng.integers(0, 256, (m + 7) // 8, dtype=np.uint8).tobytes()
    body += rng.integers(0, 256, (n + 7) // 8, dtype=np.uint8).tobytes()
    for cid, _ in stages:
        if cid == "e8p-2bit":
            body += rng.integers(0, 65536, m * n // 8, dtype=np.uint16).tobytes()
        else:
            body += rng.integers(0, 256, m * n // 8, dtype=np.uint8).tobytes()
    return body


def make_artifact_gaussian(m: int, n: int, seed: int, bits: int = 2) -> bytes:
    """North-star weights: synthetic Gaussian W (N(0,1), seeded torch generator on the
    device) quantized by the reference's H = I producer route on the GPU
    (q8p.produce_artifact: RHT incoherence, r1, f32-frozen default_scheme(bits)
    scales, RVQ codes -- byte-identical to quantize_layer(W, I) for the same W,
    tests/test_gpu_encode.py)."""
    import torch
    import paper_2402_04396_b200 as q8p
    g = torch.Generator(device="cuda").manual_seed(seed)
    w = torch.randn(m, n, generator=g, device="cuda", dtype=torch.float64)
    rng = np.random.default_rng(seed)
    su = rng.integers(0, 256, (m + 7) // 8, dtype=np.uint8)
    sv = rng.integers(0, 256, (n + 7) // 8, dtype=np.uint8)
    if m % 8:
        su[-1] &= (1 << (m % 8)) - 1
    if n % 8:
        sv[-1] &= (1 << (n % 8)) - 1
    art = q8p.produce_artifact(w, su, sv, bits, exact_r1=False)
    del w
    torch.cuda.empty_cache()
    return art


def cpu_info():
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"cpu_model": model, "host_threads": os.cpu_count(), "compiler_flags": "-O2 (reference Release default, "
            "proj/CMakeLists.txt:7-9), unmodified reference sources built in place by oracle/Makefile"}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown," \
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown," \
             "clocks_event_reasons.sw_power_cap"

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.proc:
            time.sleep(0.2)
            self.proc.terminate()
            try:
                self.out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = []
        for line in (self.out or "").strip().splitlines():
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                rows.append((float(parts[0]), float(parts[1]), parts[3:7]))
            except ValueError:
                continue
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v.lower() == "active"})
        loaded = [c for c, _, _ in rows]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": max(m for _, m, _ in rows), "reasons": reasons,
                "samples": len(rows)}


def cpu_reference(layers, tokens_per_step: int, threads: int, sample_div: int, steps: int, warmup: int, bits: int = 2):
    """Time the reference latq::infer (oracle/_ref) on the host: each step runs
    `threads` vectors concurrently (one std::thread each, the reference's own
    re-entrant infer) through the layer set (sample_div > 1: the first
    m/sample_div rows, scaled; the decode loop is linear in m).  Returns tokens/s.
    The CPU reads uniform-random codes of the same shapes (its decode cost is
    independent of the code values)."""
    from oracle.refpy import Ref
    ref = Ref()
    arts = []
    for i, (m, n) in enumerate(layers):
        ms = m // sample_div
        arts.append((make_artifact(ms, n, 1000 + i, bits=bits), n))
    times = []
    for it in range(warmup + steps):
        t0 = time.perf_counter()
        for art, n in arts:
            x = np.random.default_rng(it).standard_normal((threads * tokens_per_step, n))
            ref.infer(art, x, threads=threads)
        dt = time.perf_counter() - t0
        if it >= warmup:
            times.append(dt)
    step = statistics.median(times)
    # full-layer time per step = sampled time * sample_div (decode loop is linear in m)
    return threads * tokens_per_step / (step * sample_div), step


def cpu_latency_1core(layers, sample_div: int, bits: int = 2):
    """Single-thread latency of one token through the layer set (the reference's
    infer is single-threaded by construction, pipeline.cpp:151-197), on the first
    m/sample_div rows of each layer scaled x sample_div (bounded sample)."""
    from oracle.refpy import Ref
    ref = Ref()
    t = 0.0
    for i, (m, n) in enumerate(layers):
        art = make_artifact(max(m // sample_div, 8), n, 2000 + i, bits=bits)
        x = np.random.default_rng(i).standard_normal((1, n))
        ref.infer(art, x, threads=1)
        t0 = time.perf_counter()
        ref.infer(art, x, threads=1)
        t += (time.perf_counter() - t0) * sample_div
    return t


def workload_name(args) -> str:
    if args.workload == "4096":
        return f"single-4096x4096-{args.bits}bit-b{args.batch}"
    return f"llama2-{args.workload}-layer-set-{args.bits}bit-b{args.batch}"


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    layers = WORKLOADS[args.workload]
    threads = args.cpu_threads or min(os.cpu_count() or 1, 64)
    tps, step = cpu_reference(layers, 1, threads, args.sample_div, args.steps, args.warmup, args.bits)
    line = {
        "impl": "reference", "metric": METRIC, "value": tps, "unit": "tokens/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / tps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args), "batch": 1,
                   "layers": [f"{m}x{n}" for m, n in layers]},
        "cpu_baseline": dict({"value": tps, "unit": "tokens/s", "cores": threads, "kind": "reference",
                         "sample": f"per step {threads} concurrent latq::infer calls (1 thread each, one token "
                                   f"each) through " + ("the full layers" if args.sample_div == 1 else
                                   f"the first m/{args.sample_div} rows of each layer, scaled x{args.sample_div}")},
                             **cpu_info()),
        "e2e": {"value": tps, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import torch
    import torch.distributed as dist

    import paper_2402_04396_b200 as q8p

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    layers = WORKLOADS[args.workload]
    hbm_peak, peak_kind = peaks()
    sharded = world > 1 or args.sharded  # --sharded at N=1: the row-sharded path over a 1-rank NCCL comm

    comm = None
    peers = None
    if sharded:
        uid = torch.zeros(128, dtype=torch.uint8, device=dev)
        if rank == 0:
            uid.copy_(torch.frombuffer(bytearray(q8p.NcclComm.unique_id()), dtype=torch.uint8))
        if world > 1:
            dist.broadcast(uid, 0)
        comm = q8p.NcclComm(bytes(uid.cpu().numpy()), world, rank, local)
        if args.allgather == "push":
            # push all-gather group: one window per rank, IPC handles exchanged over the process group
            peers = q8p.PeerGroup(local, world, rank, args.batch * max(m // world for m, _ in layers))
            handles = [None] * world
            if world > 1:
                dist.all_gather_object(handles, peers.handle)
            else:
                handles = [peers.handle]
            peers.connect(handles)

    # `copies` full copies of the layer set (distinct device buffers) rotate so
    # every step streams its codes from HBM: at least 4x the L2 capacity of codes
    # (70B set, 2 bits: 4 x 134.6 MB; 7B set: 10 copies; one 4096^2 layer: 120).
    set_code_bytes = sum(m * n // 8 * sum(CODE_BYTES[c] for c, _ in SCHEMES[args.bits]) for m, n in layers)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    args.copies = max(args.copies, -(-4 * l2_bytes // set_code_bytes))
    copies = []
    if args.codes == "gaussian":
        arts = [make_artifact_gaussian(m, n, 1000 + i, bits=args.bits) for i, (m, n) in enumerate(layers)]
    else:
        arts = [make_artifact(m, n, 1000 + i, bits=args.bits) for i, (m, n) in enumerate(layers)]
    for c in range(args.copies):
        row = []
        for (m, n), art in zip(layers, arts):
            if sharded:
                row.append(q8p.Layer.from_qshp(art, device=local, rows=q8p.shard_rows(m, world, rank)))
            else:
                row.append(q8p.Layer.from_qshp(art, device=local))
        copies.append(row)
    maxn = max(n for _, n in layers)
    maxm = max(m for m, _ in layers)
    B = args.batch
    ws = torch.empty(max(L.workspace_bytes(B) for L in copies[0]) + (1 << 20), dtype=torch.uint8, device=dev)
    xs = [torch.randn(B, n, device=dev) for _, n in layers]
    ys = [torch.empty(B, m, device=dev) for m, _ in layers]
    stream = torch.cuda.Stream(device=dev)

    n_gemv = len(layers)
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n_gemv)]
          for _ in range(args.copies)]

    def sharded_forward(L, x, y):
        if peers is not None:
            L.forward_sharded_push(x, peers, out=y, stream=stream, workspace=ws)
        else:
            L.forward_sharded(x, comm, out=y, stream=stream, workspace=ws)

    allgather = None
    if sharded and peers is not None:
        # self-check: the push all-gather's y equals the NCCL all-gather's bit for bit
        ok = True
        with torch.cuda.stream(stream):
            for li, L in enumerate(copies[0]):
                ya = L.forward_sharded_push(xs[li], peers, stream=stream, workspace=ws)
                yb = L.forward_sharded(xs[li], comm, stream=stream, workspace=ws)
                stream.synchronize()
                ok &= bool(torch.equal(ya, yb))
        flag = torch.tensor([1 if ok else 0], device=dev)
        if world > 1:
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
        if int(flag.item()) == 0:
            peers = None
            allgather = "nccl (push all-gather self-check failed)"
        else:
            allgather = "push (K3 pass 1 stores into peers' windows over NVLink)"
    elif sharded:
        allgather = "nccl"

    def step(c, events=True):
        for li, L in enumerate(copies[c]):
            e = ev[c][li] if events else None
            if sharded:
                sharded_forward(L, xs[li], ys[li])
            else:
                L.forward(xs[li], out=ys[li], stream=stream, workspace=ws, gemv_events=e)

    # Mark the GEMV events as recorded for torch's bookkeeping; the library
    # re-records them (cudaEventRecord) around K2, also inside graphs.
    for row in ev:
        for a, b in row:
            a.record(stream)
            b.record(stream)
    # Warm-up (eager), then capture one graph per copy.
    with torch.cuda.stream(stream):
        for _ in range(max(args.warmup, 3)):
            for c in range(args.copies):
                step(c, events=False)
    torch.cuda.synchronize()
    graphs, ev_graphs = [], []
    use_graph = not args.no_graph  # sharded too: the NCCL all-gather captures as a graph node
    tc_path = B <= 32  # one K2 launch per forward (larger batches run in 32-vector chunks)
    if use_graph:
        # headline graphs: no event nodes (they would break the programmatic
        # dependent launch edges between kernels); instrumented twins time K2.
        for c in range(args.copies):
            g = torch.cuda.CUDAGraph()
            k0 = q8p.kernel_launches()
            with torch.cuda.graph(g, stream=stream):
                step(c, events=False)
            launches_per_step = q8p.kernel_launches() - k0  # q8p kernels captured per step
            graphs.append(g)
            if not sharded:
                g2 = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g2, stream=stream):
                    step(c, events=True)
                ev_graphs.append(g2)
        torch.cuda.synchronize()
        for c in range(args.copies):
            graphs[c].replay()
            if ev_graphs:
                ev_graphs[c].replay()
        torch.cuda.synchronize()

    launches0 = q8p.kernel_launches()
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gemv_ms = {li: [] for li in range(n_gemv)}
    with ClockSampler(local) as clocks:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            t0.record(stream)
            for s in range(args.steps):
                c = s % args.copies
                if use_graph:
                    graphs[c].replay()
                else:
                    step(c)
            t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        # gather GEMV durations of the last replay of each copy
    total_ms = t0.elapsed_time(t1)
    launches = (q8p.kernel_launches() - launches0) if not use_graph else launches_per_step * args.steps
    if not sharded:
        # Re-run the timed steps once more collecting every GEMV event pair.
        with torch.cuda.stream(stream):
            for s in range(args.steps):
                c = s % args.copies
                if use_graph:
                    ev_graphs[c].replay()
                else:
                    step(c)
                stream.synchronize()
                for li in range(n_gemv):
                    gemv_ms[li].append(ev[c][li][0].elapsed_time(ev[c][li][1]))
    ms = total_ms / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    tokens_per_s = B * 1e3 / ms

    # e2e through the public API with host buffers: per step, one H2D copy of all
    # layers' inputs from pinned memory, the layer forwards, one D2H copy of all
    # outputs, and a stream sync (the result is on the host when the step ends).
    nsum, msum = sum(n for _, n in layers), sum(m for m, _ in layers)
    hx = torch.randn(B * nsum).pin_memory()
    hy = torch.empty(B * msum).pin_memory()
    dx = torch.empty(B * nsum, device=dev)
    dy = torch.empty(B * msum, device=dev)
    xo = np.cumsum([0] + [B * n for _, n in layers])
    yo = np.cumsum([0] + [B * m for m, _ in layers])
    xv = [dx[xo[i]:xo[i + 1]].view(B, n) for i, (_, n) in enumerate(layers)]
    yv = [dy[yo[i]:yo[i + 1]].view(B, m) for i, (m, _) in enumerate(layers)]
    h2d, d2h = 4 * B * nsum, 4 * B * msum
    sets = None if sharded else [q8p.LayerSet(row) for row in copies]
    ws_set = None if sharded else torch.empty(max(S.workspace_bytes(B) for S in sets), dtype=torch.uint8, device=dev)

    def e2e_step(c):
        if sharded:
            dx.copy_(hx, non_blocking=True)
            for li, L in enumerate(copies[c]):
                sharded_forward(L, xv[li], yv[li])
            hy.copy_(dy, non_blocking=True)
            stream.synchronize()
        else:
            sets[c].forward_host(hx, hy, B, stream=stream, workspace=ws_set)

    with torch.cuda.stream(stream):
        for c in range(args.copies):  # warm-up (the set path captures its graphs here)
            e2e_step(c)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        e0.record(stream)
        for s in range(args.steps):
            e2e_step(s % args.copies)
        e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        t = torch.tensor([e2e_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())

    # The same layer set with the layers declared independent (Q8P_SET_CONCURRENT:
    # each reads only its own input, as the q/k/v or gate/up projections do): they
    # run on parallel streams, so one layer's transforms overlap another's GEMV.
    # Reported beside the sequential headline, not instead of it.
    conc = None
    if not sharded and use_graph:
        csets = [q8p.LayerSet(row, concurrent=True) for row in copies]
        ws_c = torch.empty(max(S.workspace_bytes(B) for S in csets), dtype=torch.uint8, device=dev)
        cgraphs = []
        with torch.cuda.stream(stream):
            for S in csets:
                S.forward(xs, ys, stream=stream, workspace=ws_c)
        torch.cuda.synchronize()
        for S in csets:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                S.forward(xs, ys, stream=stream, workspace=ws_c)
            cgraphs.append(g)
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            for g in cgraphs:
                g.replay()
            torch.cuda.synchronize()
            t0.record(stream)
            for s in range(args.steps):
                cgraphs[s % args.copies].replay()
            t1.record(stream)
        torch.cuda.synchronize()
        conc_ms = t0.elapsed_time(t1) / args.steps
        with torch.cuda.stream(stream):
            for c in range(args.copies):
                csets[c].forward_host(hx, hy, B, stream=stream, workspace=ws_c)
        torch.cuda.synchronize()
        e0.record(stream)
        with torch.cuda.stream(stream):
            for s in range(args.steps):
                csets[s % args.copies].forward_host(hx, hy, B, stream=stream, workspace=ws_c)
        e1.record(stream)
        torch.cuda.synchronize()
        conc_e2e_ms = e0.elapsed_time(e1) / args.steps
        conc = {"value": B * 1e3 / conc_ms, "ms_per_step": conc_ms,
                "e2e": {"value": B * 1e3 / conc_e2e_ms, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h},
                "note": "layers declared independent (Q8P_SET_CONCURRENT): parallel streams, same kernels, "
                        "bit-identical outputs; the headline value/e2e above run them in sequence"}

    # K2 chained: each layer's decode-GEMV launched back to back over the rotating
    # copies (q8p_bench_gemv; PDL-chained as inside a forward, so a launch's
    # prologue overlaps its predecessor's tail as K2's overlaps K1's), CUDA events
    # around the whole sequence on the launching stream / launches.  The stream
    # ceiling: a plain bulk-copy read of the same code-slab bytes, same harness.
    chained, ceiling = {}, {}
    if tc_path:
        reps = 5
        for li, (m, n) in enumerate(layers):
            with torch.cuda.stream(stream):
                copies[0][li].forward(xs[li], out=ys[li], stream=stream, workspace=ws)  # B images for this n
                for c in range(args.copies):
                    copies[c][li].bench_gemv(B, ws, 1, stream=stream)  # warm
                torch.cuda.synchronize()
                t0.record(stream)
                for r in range(reps):
                    for c in range(args.copies):
                        copies[c][li].bench_gemv(B, ws, 1, stream=stream)
                t1.record(stream)
                torch.cuda.synchronize()
                chained[li] = t0.elapsed_time(t1) / (reps * args.copies)
                regions = [copies[c][li].code_region(0) for c in range(args.copies)]
                for addr, nb in regions:
                    q8p.bench_stream(addr, nb, 1, stream=stream)
                torch.cuda.synchronize()
                t0.record(stream)
                for r in range(reps):
                    for addr, nb in regions:
                        q8p.bench_stream(addr, nb, 1, stream=stream)
                t1.record(stream)
                torch.cuda.synchronize()
                ceiling[li] = (t0.elapsed_time(t1) / (reps * args.copies), regions[0][1])
        if world > 1:  # per-rank kernel times: the max over ranks
            keys = sorted(chained)
            t = torch.tensor([chained[k] for k in keys] + [ceiling[k][0] for k in keys], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            for i, k in enumerate(keys):
                chained[k] = float(t[i])
                ceiling[k] = (float(t[len(keys) + i]), ceiling[k][1])

    # Roofline of the dominant kernel (K2) on the largest layer.
    roof = None
    if chained or all(gemv_ms[li] for li in range(n_gemv)):
        per = []
        for li, (m, n) in enumerate(layers):
            ml = m // world  # this rank's rows (row-sharded: the per-rank K2)
            b = ml * n // 8 * sum(CODE_BYTES[c] for c, _ in SCHEMES[args.bits]) + 4 * B * n + 4 * B * ml
            t_iso = statistics.mean(gemv_ms[li]) if gemv_ms[li] else None
            t = chained.get(li, t_iso)
            e = {"layer": f"{m}x{n}" + (f" rows/{world}" if world > 1 else ""), "bytes": b, "us": t * 1e3,
                 "gbs": b / (t * 1e-3) / 1e9, "isolated_us": t_iso * 1e3 if t_iso is not None else None}
            if li in ceiling:
                cms, cb = ceiling[li]
                e["stream_ceiling"] = {"us": cms * 1e3, "slab_bytes": cb, "gbs": cb / (cms * 1e-3) / 1e9}
            per.append(e)
        # dominant kernel: K2 on the largest layer(s) (both 70B MLP shapes move the same bytes)
        bmax = max(p["bytes"] for p in per)
        dom = [p for p in per if p["bytes"] == bmax]
        dom_us = statistics.mean(p["us"] for p in dom)
        achieved = bmax / (dom_us * 1e-6) / 1e9
        traffic = None
        try:  # dram bytes per launch of the same kernel from the committed ncu --set full capture
            with open(os.path.join(ROOT, "profiles", "r02", "k2_traffic.json")) as f:
                tj = json.load(f)
            if int(tj.get("algorithmic_bytes_per_launch", -1)) == bmax and world == 1:
                traffic = float(tj["dram_bytes_per_launch"])
        except Exception:
            traffic = None
        tot_t = sum(p["us"] for p in per) * 1e-6
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak,
                "peak_kind": peak_kind, "traffic": traffic,
                "kernel": f"q8p gemv (K2) on {dom[0]['layer']}: algorithmic bytes (m*n/8)*2 + 4n + 4m per launch "
                          f"/ mean launch duration from CUDA events around {args.copies}x5 back-to-back launches "
                          f"(PDL-chained, rotating copies); isolated_us = events recorded right around one "
                          f"launch inside the forward (includes its launch latency)",
                "stream_ceiling": dom[0].get("stream_ceiling"),
                "per_layer": per, "gemv_share_of_step": (tot_t * 1e3) / ms}

    if B >= 64 and all(gemv_ms[li] for li in range(n_gemv)):  # prefill: the K4 decode-GEMM is tensor-bound
        tf_peak = None
        try:
            with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
                tf_peak = float(json.load(f)["bf16_tflops"])
        except Exception:
            tf_peak = 2250.0
        per = []
        for li, (m, n) in enumerate(layers):
            t = statistics.mean(gemv_ms[li]) * 1e-3
            fl = 2.0 * m * n * B  # one effective matrix; the s8 MMAs issued are 2x per stage (2 limbs)
            per.append({"layer": f"{m}x{n}", "flops": fl, "us": t * 1e6, "tflops": fl / t / 1e12,
                        "tflops_issued": 2 * fl * sum(1 for _ in SCHEMES[args.bits]) / t / 1e12})
        dom = max(per, key=lambda p: p["flops"])
        roof = {"bound": "tensor", "achieved": dom["tflops"], "peak": tf_peak, "unit": "TFLOP/s",
                "frac": dom["tflops"] / tf_peak, "traffic": None,
                "kernel": f"q8p prefill decode-GEMM (pack + K4) on {dom['layer']} at batch {B}: 2 m n B flops / "
                          f"mean CUDA-event duration vs the measured bf16 peak (K4 runs kind::i8 MMAs: tflops_issued counts "
                          f"the s8 ops actually run, 2 activation limbs per stage, against an s8 peak of 2x bf16)",
                "per_layer": per}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            threads = args.cpu_threads or min(os.cpu_count() or 1, 64)
            tps, step_s = cpu_reference(layers, 1, threads, args.cpu_sample_div, 2, 0, args.bits)
            lat = cpu_latency_1core(layers, 8, args.bits)
            cpu = dict({"value": tps, "unit": "tokens/s", "cores": threads, "kind": "reference",
                        "sample": f"{threads} concurrent latq::infer calls (1 thread each, one token each) through "
                                  + ("the full layers" if args.cpu_sample_div == 1 else
                                     f"the first m/{args.cpu_sample_div} rows of each layer, scaled x{args.cpu_sample_div}")
                                  + f"; median of 2 steps, {step_s:.1f} s per step",
                        "latency_1core_s": lat,
                        "latency_1core_sample": "one token, one thread, first m/8 rows of each layer scaled x8"},
                       **cpu_info())
        except Exception as e:  # reference .so missing etc.
            cpu = {"value": None, "unit": "tokens/s", "cores": 0, "kind": "reference", "sample": f"unavailable: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": tokens_per_s, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "s8xs8->s32 (K2 tensor cores) + fp32 (RHT, I/O)", "data": "synthetic",
            "config": {"workload": workload_name(args), "batch": B,
                       "layers": [f"{m}x{n}" for m, n in layers],
                       "parallelism": f"row-shard tp{world}" if world > 1 else ("row-shard tp1" if sharded else "single-gpu"),
                       **({"allgather": allgather} if sharded else {}),
                       "l2": f"{args.copies} rotating copies of the layer set (distinct buffers, "
                             f"{args.copies * set_code_bytes / 1e6:.0f} MB of codes >= 4x the {l2_bytes / 1e6:.0f} MB L2)",
                       "codes": (f"synthetic Gaussian W quantized by the reference H = I route on the GPU "
                                 f"(q8p.produce_artifact), default_scheme({args.bits})" if args.codes == "gaussian" else
                                 f"uniform-random codes, default_scheme({args.bits}) stages (perf variant, "
                                 f"test_pipeline.cpp:256-273)"),
                       "cuda_graph": use_graph},
            "e2e": {"value": B * 1e3 / e2e_ms, "unit": "tokens/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
            "gpu_launches": int(launches),
            "concurrent_set": conc,
            "roofline": roof,
            "cpu_baseline": cpu,
            "clocks": clocks.summary(),
        }
        print(json.dumps(line), flush=True)
    if comm is not None:
        comm.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="70b", choices=["70b", "7b", "4096"])
    ap.add_argument("--copies", type=int, default=4)
    ap.add_argument("--codes", default="gaussian", choices=["gaussian", "random"],
                    help="gaussian: reference-route quantized N(0,1) weights (GPU producer); random: uniform codes")
    ap.add_argument("--batch", type=int, default=1, help="vectors per layer call (BASELINE configs[1]: 1..16)")
    ap.add_argument("--bits", type=int, default=2, choices=[2, 3, 4],
                    help="2: E8P (headline); 3 / 4: RVQ variants (BASELINE configs[3])")
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--sharded", action="store_true", help="use the row-sharded path even at N=1 (1-rank group)")
    ap.add_argument("--allgather", choices=["push", "nccl"], default="push",
                    help="sharded z exchange: push = q8p_forward_sharded_push (K3 pass 1 stores into the peers' "
                         "windows), nccl = q8p_forward_sharded (ncclAllGather between the K3 passes)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-threads", type=int, default=0)
    ap.add_argument("--sample-div", type=int, default=1, help="row sampling of --impl reference steps (1: full rows)")
    ap.add_argument("--cpu-sample-div", type=int, default=1, help="row sampling of our line's cpu_baseline")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
