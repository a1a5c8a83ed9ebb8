#!/usr/bin/env python
"""Benchmark of the GraphPy sparse hot path on B200 (BASELINE.json metric:
"gSpMM GE/s & HBM GB/s (% of 8 TB/s), Reddit-shape F=64, 1/2/4/8 B200").

One STEP = one pass of the whole hot path over the Reddit-shaped graph
(A9 at N > 1):
    out1 = gspmm(X,  BOTH, fwd)            GCN forward          (A3)
    out2 = gspmm(dY, BOTH, rev)            GCN backward         (A4)
    s    = gsddmm(Z, Z)        [E, H]      GAT scores           (A5)
    a    = edge_softmax(s)     in place    GAT attention        (A6)
    out3 = gspmm_weighted(Z, a, fwd)       GAT aggregate        (A7)
    out4 = gspmm_weighted(dO, a, rev)      GAT backward dZ      (A8)
With --chain fused (the default) A5-A7 run as ONE kernel (gsp_gat_forward,
NEXT-2) that leaves the same state behind: a = alpha [E, H] in the same buffer,
out3 the aggregate -- 4 launches per step; --chain separate runs the six
calls above.  The separate A5-A7 calls are then timed outside the step
(per_op, "in_step": false) so every row keeps its own number.
value = edge visits per second over the step = 6 * E / t_step (GE/s), whole job.
At N > 1 every rank runs the same step on its destination-row partition and
all-gathers each vertex-level output over NCCL (A9); scaling is "strong"
(the graph is fixed).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl gsp|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402

L2_FLUSH_BYTES = 512 << 20          # > 126 MB L2: written between timed steps
N_OPS = 6                           # sparse ops per step (edge visits = N_OPS * E)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["gsp", "reference"], default="gsp")
    ap.add_argument("--config", default="reddit", choices=sorted(datagen.CONFIGS))
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e / cpu baseline / clocks)")
    ap.add_argument("--check", action="store_true", help="N > 1: compare the exchanged outputs with the full graph")
    ap.add_argument("--chain", choices=["fused", "separate"], default="fused",
                    help="GAT forward A5-A7 as one fused kernel (default) or three calls")
    return ap.parse_args()


# ------------------------------------------------------------- byte models
def step_config(cfg, V, E, P, fused):
    """The workload description both arms print (the reference arm runs the same step)."""
    F, H = cfg.H * cfg.Fh, cfg.H
    return {"workload": f"{cfg.name}-shaped GCN gSpMM fwd+bwd (BOTH norm) + GAT chain "
                        f"(gSDDMM u.v, edge softmax, weighted gSpMM fwd+rev), F={F}, H={H}x{cfg.Fh}",
            "gat_chain": ("fused: gSDDMM + edge softmax + weighted gSpMM fwd in one kernel "
                          "(gsp_gat_forward; alpha still written)") if fused else "separate: 3 kernels",
            "V": V, "E": E, "F": F, "H": H, "Fh": cfg.Fh,
            "graph": f"Chung-Lu beta={cfg.beta}, seed={cfg.seed:#x}" if cfg.kind == "chung_lu"
            else f"R-MAT scale {cfg.scale}, seed={cfg.seed:#x}",
            "parallelism": f"row-partition x{P}" if P > 1 else "single GPU",
            "l2": f"flushed between timed steps ({L2_FLUSH_BYTES >> 20} MiB write); "
                  f"per-step inputs (col ids {4 * E / 1e9:.2f} GB, alpha {4 * E * H / 1e9:.2f} GB) exceed L2",
            "edge_visits_per_step": N_OPS * E}


def alg_bytes(op, V, E, F, H):
    """Algorithmic (compulsory) bytes per launch: every
    gathered feature row counted once per edge, indices/values/outputs once."""
    base = 8 * (V + 1) + 4 * E                      # offsets + column ids
    if op == "gspmm":
        return base + 4 * E * F + 4 * V * F + 8 * V
    if op == "gspmm_weighted_fwd":
        return base + 4 * E * F + 4 * V * F + 4 * E * H
    if op == "gspmm_weighted_rev":
        return base + 4 * E * F + 4 * V * F + 4 * E * H + 4 * E
    if op == "gsddmm":
        return base + 4 * V * F + 4 * E * F + 4 * E * H
    if op == "edge_softmax":
        return 8 * (V + 1) + 4 * E * H + 4 * E * H
    if op == "gat_forward":      # fused A5-A7 (Y == Vt gathered once): alpha written once
        return base + 4 * V * F + 4 * E * F + 4 * E * H + 4 * V * F
    raise KeyError(op)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def load_l2_ceiling():
    """Best random 256-B row-gather rate from an L2-resident table of the Reddit F=64
    size (tools/l2bench.cu; committed output profiles/r01_l2bench.txt), GB/s."""
    p = os.path.join(ROOT, "profiles", "r01_l2bench.txt")
    if not os.path.exists(p):
        return None
    best = None
    for line in open(p):
        if line.startswith("table") and best is not None:
            break                       # first table only (59.6 MB = the Reddit F=64 table)
        if "GB/s" in line:
            v = float(line.split("ms")[1].split("GB/s")[0])
            best = v if best is None else max(best, v)
    return best


def load_traffic(config):
    """ncu DRAM bytes (read + write) per launch of each op's kernel, from the committed
    full-capture summaries (profiles/ncu_traffic.json, written by tools/ncu_traffic.py)."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        d = json.load(f)
    return {k: float(v["dram_bytes"]) for k, v in d.get(config, {}).items()}


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# --------------------------------------------------------------- CPU oracle
def oracle_sample(V, src, dst, cfg, target_edges):
    """A bounded sample of the workload for the CPU oracle: all edges whose
    destination falls in a random row subset holding ~target_edges edges
    (same graph shape per edge)."""
    rng = np.random.default_rng(cfg.seed)
    frac = min(1.0, target_edges / max(1, len(src)))
    keep_rows = rng.random(V) < frac
    m = keep_rows[dst]
    return src[m], dst[m]


def run_oracle_step(og, V, cfg, inputs):
    """The step's six ops, by the oracle (fp64)."""
    X, dY, Z, dO = inputs
    H = cfg.H
    og.gspmm(X, 2, False)
    og.gspmm(dY, 2, True)
    s, _ = og.gsddmm(Z, Z, H)
    a = og.edge_softmax(s.astype(np.float32))
    a32 = a.astype(np.float32)
    og.gspmm_weighted(Z, a32, False)
    og.gspmm_weighted(dO, a32, True)


def cpu_oracle_bench(V, src, dst, cfg, target_edges, steps=1, warmup=0):
    import oracle
    ssrc, sdst = oracle_sample(V, src, dst, cfg, target_edges)
    t0 = time.perf_counter()
    og = oracle.Graph(V, ssrc, sdst)
    t_build = time.perf_counter() - t0
    F = cfg.H * cfg.Fh
    inputs = [datagen.uniform(cfg.seed + k, V, F) for k in range(4)]
    for _ in range(warmup):
        run_oracle_step(og, V, cfg, inputs)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        run_oracle_step(og, V, cfg, inputs)
        times.append(time.perf_counter() - t0)
    t = sum(times) / len(times)
    return {"E_sample": int(len(ssrc)), "t_step": t, "t_build": t_build,
            "value": N_OPS * len(ssrc) / t / 1e9}


# ------------------------------------------------------------------ GPU arm
def small_config_latency(gsp, torch):
    """Cora GCN fwd+bwd (F=16) and the Pubmed GAT forward (8x8, as three calls and
    as the fused kernel): microseconds per step, eager vs the same calls captured
    in one CUDA graph (the launch-bound regime of P:1632-1688)."""
    res = {}
    st = torch.cuda.Stream()

    def timed(stepf, reps=200):
        with torch.cuda.stream(st):
            for _ in range(5):
                stepf()
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(st)
        with torch.cuda.stream(st):
            for _ in range(reps):
                stepf()
        a1.record(st)
        torch.cuda.synchronize()
        eager = a0.elapsed_time(a1) * 1e3 / reps
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            stepf()
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        a0.record(st)
        with torch.cuda.stream(st):
            for _ in range(reps):
                gr.replay()
        a1.record(st)
        torch.cuda.synchronize()
        return round(eager, 2), round(a0.elapsed_time(a1) * 1e3 / reps, 2)

    for name in ("cora", "pubmed"):
        cfg = datagen.CONFIGS[name]
        V, src, dst = datagen.make_graph(cfg)
        G = gsp.Graph(V, src, dst, device=torch.cuda.current_device())
        F = cfg.F
        X = torch.from_numpy(datagen.uniform(1, V, F)).cuda()
        o1 = torch.empty((V, F), device="cuda")
        o2 = torch.empty((V, F), device="cuda")
        if name == "cora":
            def stepf():
                G.gspmm(X, gsp.NORM_BOTH, out=o1, stream=st)
                G.gspmm(o1, gsp.NORM_BOTH, out=o2, reverse=True, stream=st)
            eager, graph = timed(stepf)
            res[name] = {"ops": "gspmm fwd+rev (BOTH), F=16", "n_kernels": 2, "eager_us_per_step": eager,
                         "cuda_graph_us_per_step": graph, "V": V, "E": int(G.E)}
        else:
            s = torch.empty((G.E, cfg.H), device="cuda")
            def stepf():
                G.gsddmm(X, X, out=s, stream=st)
                G.edge_softmax(s, out=s, stream=st)
                G.gspmm_weighted(X, s, out=o1, stream=st)
            def fusedf():
                G.gat_forward(X, X, X, cfg.H, alpha=s, out=o1, stream=st)
            eager, graph = timed(stepf)
            feager, fgraph = timed(fusedf)
            res[name] = {"ops": "GAT forward 8x8: gsddmm+softmax+weighted (3 kernels) / fused (1 kernel)",
                         "n_kernels": 3, "eager_us_per_step": eager, "cuda_graph_us_per_step": graph,
                         "fused_eager_us_per_step": feager, "fused_cuda_graph_us_per_step": fgraph,
                         "V": V, "E": int(G.E)}
    return res


def main_gsp(args):
    import torch
    import torch.distributed as dist

    import paper_2402_03548_b200 as gsp

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # one process per GPU; GSP_BENCH_BACKEND=gloo lets a 1-GPU box run N ranks on one device
    # (validation only: the exchange then goes through host copies)
    backend = os.environ.get("GSP_BENCH_BACKEND", "nccl")
    local = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    cfg = datagen.CONFIGS[args.config]
    assert cfg.H > 0, "bench step needs a config with the GAT chain (reddit / pubmed)"
    F, H = cfg.H * cfg.Fh, cfg.H
    if cfg.F != F:
        raise SystemExit("config F must equal H*Fh for the step")

    t0 = time.time()
    V, src, dst = datagen.make_graph(cfg)
    t_gen = time.time() - t0
    t0 = time.time()
    G = gsp.Graph(V, src, dst, device=local)
    t_create = time.time() - t0
    E = G.E
    stream = torch.cuda.current_stream()

    P = world
    if P > 1:
        part = G.partition(P, rank, device=local)
        b = G.partition_bounds(P)
        R = part.R
        rows_lo, rows_hi = b[rank], b[rank + 1]
    else:
        part = G
        R = V
        b = np.array([0, V])
    ncols = P * R

    def padded_input(seed):
        Xh = datagen.uniform(seed, V, F)
        if P == 1:
            return torch.from_numpy(Xh).cuda()
        Xp = torch.zeros((ncols, F), device="cuda")
        for p in range(P):
            Xp[p * R:p * R + b[p + 1] - b[p]] = torch.from_numpy(Xh[b[p]:b[p + 1]]).cuda()
        return Xp

    X, dY, Z, dO = (padded_input(cfg.seed + k) for k in range(4))
    X_, dY_, Z_, dO_ = X, dY, Z, dO
    Ep = part.E
    s = torch.empty((Ep, H), device="cuda")
    outs = [torch.empty((R, F), device="cuda") for _ in range(4)]
    gathered = [torch.empty((ncols, F), device="cuda") for _ in range(3)] if P > 1 else None
    partial = torch.empty((ncols, F), device="cuda") if P > 1 else None
    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")

    fused = args.chain == "fused"
    op_names = (["gspmm_fwd", "gspmm_rev", "gat_forward", "gspmm_weighted_rev"] if fused else
                ["gspmm_fwd", "gspmm_rev", "gsddmm", "edge_softmax", "gspmm_weighted_fwd", "gspmm_weighted_rev"])
    ev = {k: [] for k in op_names + ["exchange"]}

    # the step as a list of (name, launch, input index into (X, dY, Z, dO) or None, output index or None)
    def op_list(ins=None, outs=outs):
        X, dY, Z, dO = ins if ins is not None else (X_, dY_, Z_, dO_)
        L = [("gspmm_fwd", lambda: part.gspmm(X, gsp.NORM_BOTH, out=outs[0], stream=stream), 0, 0),
             ("gspmm_rev", lambda: part.gspmm(dY, gsp.NORM_BOTH, out=outs[1], reverse=True, stream=stream), 1, 1)]
        if fused:   # A5-A7 in one pass per destination row; s ends up holding alpha, as below
            L.append(("gat_forward", lambda: part.gat_forward(Z, Z, Z, H, alpha=s, out=outs[2], stream=stream), 2, 2))
        else:
            L += [("gsddmm", lambda: part.gsddmm(Z, Z, out=s, stream=stream), 2, None),
                  ("edge_softmax", lambda: part.edge_softmax(s, out=s, stream=stream), None, None),
                  ("gspmm_weighted_fwd", lambda: part.gspmm_weighted(Z, s, out=outs[2], stream=stream), None, 2)]
        if P == 1:
            L.append(("gspmm_weighted_rev",
                      lambda: part.gspmm_weighted(dO, s, out=outs[3], reverse=True, stream=stream), 3, 3))
        else:
            # alpha of an edge lives on its destination's rank: each rank sums its own
            # edges per (padded) source row; one reduce-scatter completes dZ
            L.append(("gspmm_weighted_rev",
                      lambda: part.gspmm_weighted(dO, s, out=partial, reverse=True, stream=stream), 3, None))
        return L
    OPS = op_list()

    def exchange():
        if backend == "nccl":
            for o, gbuf in zip(outs[:3], gathered[:3]):
                dist.all_gather_into_tensor(gbuf, o)
            dist.reduce_scatter_tensor(outs[3], partial)
        else:   # host-staged equivalent (validation on a 1-GPU box)
            for o, gbuf in zip(outs[:3], gathered[:3]):
                parts = [torch.empty((R, F)) for _ in range(P)]
                dist.all_gather(parts, o.cpu())
                gbuf.copy_(torch.cat(parts))
            t = partial.cpu()
            dist.all_reduce(t)
            outs[3].copy_(t[rank * R:(rank + 1) * R])

    # NCCL: each op's collective is issued (async) as soon as the op is enqueued, so
    # the all-gather of one op's output runs beside the next op's kernel; the step
    # ends by making the compute stream wait for all of them.  gloo (validation on a
    # 1-GPU box): the host-staged exchange() after the last op.
    overlap = P > 1 and backend == "nccl"

    def issue_collective(name, i_out, pending, outs=outs):
        if not overlap:
            return
        if name == "gspmm_weighted_rev":
            pending.append(dist.reduce_scatter_tensor(outs[3], partial, async_op=True))
        elif i_out is not None:
            pending.append(dist.all_gather_into_tensor(gathered[i_out], outs[i_out], async_op=True))

    def finish_exchange(pending):
        if overlap:
            for w in pending:
                w.wait()          # stream-ordered: the compute stream waits for the NCCL stream
        elif P > 1:
            exchange()

    def allreduce_max(v):
        t = torch.tensor([float(v)], device="cuda" if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def step(record):
        def mark():
            e = torch.cuda.Event(enable_timing=True)
            e.record(stream)
            return e
        marks = [mark()] if record else None
        pending = []
        for name, fn, _, i_out in OPS:
            fn()
            issue_collective(name, i_out, pending)
            if record:
                marks.append(mark())
        if P > 1:
            finish_exchange(pending)
            if record:
                marks.append(mark())
        return marks

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()

    clocks = ClockSampler(local) if (rank == 0 and not args.profile) else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    if P > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    step_ms = []
    host_launch_ms = []
    for _ in range(args.steps):
        flush.fill_(1.0)                      # L2 flush between timed steps (outside the events)
        h0 = time.perf_counter()
        marks = step(True)
        host_launch_ms.append((time.perf_counter() - h0) * 1e3)
        torch.cuda.synchronize()
        names = op_names + (["exchange"] if P > 1 else [])
        for i, n in enumerate(names):
            ev[n].append(marks[i].elapsed_time(marks[i + 1]))
        step_ms.append(marks[0].elapsed_time(marks[-1]))
    torch.cuda.synchronize()
    if P > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    clk = clocks.stop() if clocks else None

    t_step = sum(step_ms) / len(step_ms)
    if P > 1:
        t_step = allreduce_max(t_step)
    value = N_OPS * E / (t_step * 1e-3) / 1e9

    # ------------------------------------------- N > 1: check vs the full graph
    check = None
    if P > 1 and args.check:
        step(False)
        torch.cuda.synchronize()
        def unpad(t):
            return torch.cat([t[p * R:p * R + b[p + 1] - b[p]] for p in range(P)])
        Xf, dYf, Zf, dOf = (unpad(t) for t in (X, dY, Z, dO))
        ref1 = G.gspmm(Xf, gsp.NORM_BOTH)
        ref2 = G.gspmm(dYf, gsp.NORM_BOTH, reverse=True)
        sf = G.gsddmm(Zf, Zf, H=H)
        G.edge_softmax(sf, out=sf)
        ref3 = G.gspmm_weighted(Zf, sf)
        ref4 = G.gspmm_weighted(dOf, sf, reverse=True)
        def rel(a, ref):
            return float((a - ref).abs().max() / (ref.abs().max() + 1e-30))
        lo, hi = b[rank], b[rank + 1]
        errs = [rel(unpad(gathered[0]), ref1), rel(unpad(gathered[1]), ref2), rel(unpad(gathered[2]), ref3),
                rel(outs[3][:hi - lo], ref4[lo:hi])]
        m = allreduce_max(max(errs))
        check = {"max_rel_err_vs_single_gpu": m, "ok": bool(m < 1e-5)}
        del ref1, ref2, ref3, ref4, sf, Xf, dYf, Zf, dOf

    # ---------------------------------------------------------------- e2e
    # The same step through the C ABI with HOST buffers: every step copies its four
    # input tables from pinned host memory (H2D engine) and reads its four outputs
    # back (D2H engine), inside the timed region.  Steps are pipelined the way a
    # stream of batches runs: two device buffer sets, so step k+1's inputs upload
    # while step k computes and step k's outputs download while step k+1 computes;
    # each op waits only for its own input, each output leaves as soon as it is
    # final.  No L2 flush between steps: each step's inputs (4 x 59.6 MB tables +
    # 3.67 GB of alpha) exceed the 126 MB L2.  gloo ranks (validation): no e2e.
    e2e = None
    if not args.no_e2e and not args.profile and (P == 1 or overlap):
        hin = [torch.empty((ncols, F), dtype=torch.float32).pin_memory() for _ in range(4)]
        for h, d in zip(hin, (X, dY, Z, dO)):
            h.copy_(d.cpu())
        sets = [((X, dY, Z, dO), outs),
                (tuple(torch.empty_like(t) for t in (X, dY, Z, dO)), [torch.empty_like(o) for o in outs])]
        ops_of = [op_list(*sets[0]), op_list(*sets[1])]
        hout = [[torch.empty((R, F), dtype=torch.float32).pin_memory() for _ in range(4)] for _ in range(2)]
        h2d = torch.cuda.Stream()
        d2h = torch.cuda.Stream()
        in_free, out_free = [None, None], [None, None]

        def e2e_step(k):
            j = k % 2
            ins, outs_j = sets[j]
            if in_free[j] is not None:          # step k-2 is done reading this input set
                h2d.wait_event(in_free[j])
            ready = []
            with torch.cuda.stream(h2d):
                for h, d in zip(hin, ins):
                    d.copy_(h, non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(h2d)
                    ready.append(e)
            if out_free[j] is not None:         # step k-2's outputs have left this set
                stream.wait_event(out_free[j])
            done, pending = [], []
            for name, fn, i_in, i_out in ops_of[j]:
                if i_in is not None:
                    stream.wait_event(ready[i_in])
                fn()
                issue_collective(name, i_out, pending, outs_j)
                if i_out is not None and P == 1:
                    e = torch.cuda.Event()
                    e.record(stream)
                    done.append((e, i_out))
            if P > 1:
                finish_exchange(pending)
                e = torch.cuda.Event()
                e.record(stream)
                done = [(e, i) for i in range(4)]
            f = torch.cuda.Event()
            f.record(stream)
            in_free[j] = f
            with torch.cuda.stream(d2h):
                for e, i in done:
                    d2h.wait_event(e)
                    hout[j][i].copy_(outs_j[i], non_blocking=True)
            g = torch.cuda.Event()
            g.record(d2h)
            out_free[j] = g

        for k in range(2):
            e2e_step(k)
        torch.cuda.synchronize()
        if P > 1:
            dist.barrier()
        K = max(4, args.steps)
        a0 = torch.cuda.Event(enable_timing=True)
        a1 = torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        h2d.wait_event(a0)
        d2h.wait_event(a0)
        for k in range(K):
            e2e_step(k)
        stream.wait_stream(h2d)
        stream.wait_stream(d2h)
        a1.record(stream)
        torch.cuda.synchronize()
        t_e2e = a0.elapsed_time(a1) / K
        if P > 1:
            t_e2e = allreduce_max(t_e2e)
        # the host copies hold what the device computed
        assert torch.equal(hout[(K - 1) % 2][0], sets[(K - 1) % 2][1][0].cpu())
        e2e = {"value": round(N_OPS * E / (t_e2e * 1e-3) / 1e9, 4), "unit": "GE/s",
               "ms_per_step": round(t_e2e, 4), "steps": K,
               "h2d_bytes_per_step": int(sum(h.numel() * 4 for h in hin)),
               "d2h_bytes_per_step": int(sum(h.numel() * 4 for h in hout[0])),
               "how": "pinned host buffers, H2D / D2H engines overlapped with the kernels and pipelined across "
                      "steps (two device buffer sets); no L2 flush (per-step inputs exceed L2)"}
        del sets, ops_of

    # ------------------------- launch-bound configs (BASELINE configs[0], [1])
    latency = None
    if rank == 0 and not args.profile:
        latency = small_config_latency(gsp, torch)

    # ----------------------------------------------------------- roofline
    peak, peak_kind = load_peaks()
    avg = {k: (sum(v) / len(v) if v else None) for k, v in ev.items()}
    Vloc, Eloc = (R, Ep) if P > 1 else (V, E)
    def time_op(fn, reps=5, flush_l2=True):
        """median event time of one call (L2 flushed before each), outside the step"""
        for _ in range(2):
            fn()
        ts = []
        for _ in range(reps):
            if flush_l2:
                flush.fill_(1.0)
            a0 = torch.cuda.Event(enable_timing=True)
            a1 = torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            fn()
            a1.record(stream)
            torch.cuda.synchronize()
            ts.append(a0.elapsed_time(a1))
        return sorted(ts)[len(ts) // 2]

    # rows the step does not launch on their own: timed one by one outside it
    outside = {}
    if not args.profile:
        if fused:   # the unfused A5-A7 calls, each on its own (same graph, same inputs)
            s2 = torch.empty((Ep, H), device="cuda")
            g2 = torch.empty((R, F), device="cuda")
            part.gsddmm(Z, Z, out=s2, stream=stream)
            outside["gsddmm"] = time_op(lambda: part.gsddmm(Z, Z, out=s2, stream=stream))
            raw = s2.clone()              # out of place: the same logits every call
            outside["edge_softmax"] = time_op(lambda: part.edge_softmax(raw, out=s2, stream=stream))
            outside["gspmm_weighted_fwd"] = time_op(lambda: part.gspmm_weighted(Z, s2, out=g2, stream=stream))
            del s2, g2, raw
        else:
            g2 = torch.empty((R, F), device="cuda")
            outside["gat_forward"] = time_op(lambda: part.gat_forward(Z, Z, Z, H, alpha=torch.empty_like(s),
                                                                      out=g2, stream=stream))
            del g2

    # ------------------------------------------- NEXT rows (outside the step)
    next_rows = None
    if not args.profile:
        alpha2 = torch.empty((Ep, H), device="cuda")
        gout = torch.empty((R, F), device="cuda")
        dal = torch.rand((Ep, H), device="cuda")
        ms_gat = avg["gat_forward"] if fused else outside["gat_forward"]
        ms_max = time_op(lambda: part.gspmm_reduce(X, gsp.REDUCE_MAX, out=gout, stream=stream))
        hout = torch.empty((R, H), device="cuda")
        ms_e = time_op(lambda: part.gspmm_e(s, gsp.REDUCE_SUM, out=hout, stream=stream))
        ms_ve = time_op(lambda: part.gsddmm_ve(Z[:, :H], dal, gsp.OP_ADD, gsp.SIDE_SRC, out=alpha2, stream=stream))
        ms_sbw = time_op(lambda: part.edge_softmax_backward(s, dal, out=dal, stream=stream))
        # NEXT-1 fused: gSDDMM(dO, Z) + softmax backward in one pass (vs the two calls)
        ms_gbw = time_op(lambda: part.gat_backward_scores(dO, Z, s, out=alpha2, stream=stream))
        ms_gbw_sep = time_op(lambda: part.gsddmm(dO, Z, out=alpha2, stream=stream)) + ms_sbw
        sep = sum((outside if fused else avg)[k] for k in ("gsddmm", "edge_softmax", "gspmm_weighted_fwd"))
        next_rows = {
            "gat_forward_fused": {"row": "NEXT-2", "ms": round(ms_gat, 4), "in_step": fused,
                                  "vs_separate_chain_ms": round(sep, 4),
                                  "GE_s": round(Eloc / (ms_gat * 1e-3) / 1e9, 3)},
            "gspmm_reduce_max": {"row": "NEXT-3", "ms": round(ms_max, 4),
                                 "GB_s": round(alg_bytes("gspmm", Vloc, Eloc, F, H) / (ms_max * 1e-3) / 1e9, 1)},
            # algorithmic bytes: w read once (+ row offsets, out) / w read + out
            # written + col indices + the gathered X table read once
            "gspmm_e_sum": {"row": "NEXT-3", "ms": round(ms_e, 4),
                            "GB_s": round((Eloc * H * 4 + (Vloc + 1) * 8 + Vloc * H * 4) / (ms_e * 1e-3) / 1e9, 1)},
            "gsddmm_ve_add_src": {"row": "NEXT-3", "ms": round(ms_ve, 4),
                                  "GB_s": round((2 * Eloc * H * 4 + Eloc * 4 + (Vloc + 1) * 8 + V * H * 4)
                                                / (ms_ve * 1e-3) / 1e9, 1)},
            "gat_backward_scores_fused": {"row": "NEXT-1", "ms": round(ms_gbw, 4),
                                          "vs_gsddmm_plus_softmax_backward_ms": round(ms_gbw_sep, 4)},
            "edge_softmax_backward": {"row": "NEXT-1", "ms": round(ms_sbw, 4),
                                      "GB_s": round(alg_bytes("edge_softmax", Vloc, Eloc, F, H) * 1.5 / (ms_sbw * 1e-3) / 1e9, 1)},
        }
        del alpha2, gout, dal, hout
        # context: warm-L2 times of the headline op (no flush:
        # steady state layer to layer) and the paper's kernel-plot shapes
        # (F = 32, one head: P:2308) on the same graph
        warm_ms = time_op(lambda: part.gspmm(X, gsp.NORM_BOTH, out=outs[0], stream=stream), flush_l2=False)
        X32 = torch.rand((part.ncols, 32), device="cuda") - 0.5
        w1 = torch.rand((Ep, 1), device="cuda")
        o32 = torch.empty((R, 32), device="cuda")
        shapes = {
            "gspmm_fwd_F32": time_op(lambda: part.gspmm(X32, gsp.NORM_BOTH, out=o32, stream=stream)),
            "gspmm_weighted_rev_F32_H1": time_op(lambda: part.gspmm_weighted(X32, w1, out=o32, reverse=True,
                                                                             stream=stream)) if P == 1 else None,
            "gsddmm_F32_H1": time_op(lambda: part.gsddmm(X32, X32, H=1, out=w1, stream=stream)),
        }
        next_rows["context"] = {"gspmm_fwd_warm_l2_ms": round(warm_ms, 4),
                                "paper_plot_shapes_ms": {k: (round(v, 4) if v is not None else None)
                                                         for k, v in shapes.items()}}
        del X32, w1, o32

    per_op = {}
    traffic = load_traffic(args.config) if P == 1 else {}
    bytes_of = {"gspmm_fwd": alg_bytes("gspmm", Vloc, Eloc, F, H), "gspmm_rev": alg_bytes("gspmm", Vloc, Eloc, F, H),
                "gsddmm": alg_bytes("gsddmm", Vloc, Eloc, F, H),
                "edge_softmax": alg_bytes("edge_softmax", Vloc, Eloc, F, H),
                "gspmm_weighted_fwd": alg_bytes("gspmm_weighted_fwd", Vloc, Eloc, F, H),
                "gspmm_weighted_rev": alg_bytes("gspmm_weighted_rev", Vloc, Eloc, F, H),
                "gat_forward": alg_bytes("gat_forward", Vloc, Eloc, F, H)}
    for k, ms in [(k, avg[k]) for k in op_names] + list(outside.items()):
        gbs = bytes_of[k] / (ms * 1e-3) / 1e9
        per_op[k] = {"ms": round(ms, 4), "GE_s": round(Eloc / (ms * 1e-3) / 1e9, 3), "alg_GB": round(bytes_of[k] / 1e9, 3),
                     "GB_s": round(gbs, 1), "frac_of_peak": round(gbs / peak, 4),
                     "frac_of_8TBs": round(gbs / 8000.0, 4), "in_step": k in op_names,
                     "traffic_GB": round(traffic[k] / 1e9, 3) if k in traffic else None,
                     # SURVEY §8(d) "reuse = B_alg / DRAM bytes" (> 1: the gathers are L2-served)
                     "reuse": round(bytes_of[k] / traffic[k], 2) if traffic.get(k) else None}
    if P > 1:
        per_op["exchange"] = {"ms": round(avg["exchange"], 4),
                              "what": "3 x all_gather_into_tensor [R,F] + reduce_scatter_tensor [P*R,F] "
                                      + ("(NCCL, each issued async right after its op and overlapped with the "
                                         "next ops; ms = the residual wait after the last op)"
                                         if backend == "nccl" else "(host-staged gloo: validation only)")}
    dom = "gspmm_fwd"
    achieved = per_op[dom]["GB_s"]
    roofline = {"bound": "hbm", "kernel": "spmm_kernel<VEC=8,LPE=8,CPL=1,scaled,U=4,3 CTAs/SM> (gspmm fwd, BOTH norm)",
                "achieved": achieved, "peak": peak, "peak_kind": f"{peak_kind} hbm_gbs (MEASURED_PEAKS.json)",
                "unit": "GB/s", "frac": round(achieved / peak, 4),
                "alg_bytes_per_launch": bytes_of[dom],
                "traffic": traffic.get(dom)}
    l2c = load_l2_ceiling() if args.config == "reddit" else None
    if l2c:
        # the gathered rows are L2-served (table 59.6 MB < L2), so the kernel's real ceiling is
        # the L2 gather rate, not HBM: context beside the HBM-peak fraction the contract asks for
        roofline["l2_gather_ceiling"] = {"GB_s": l2c, "frac": round(achieved / l2c, 4),
                                         "source": "tools/l2bench.cu -> profiles/r01_l2bench.txt: 114.6M random "
                                                   "256-B row gathers (LDG.256) from a 59.6 MB table"}

    cpu = None
    if rank == 0 and P == 1 and not args.no_cpu_baseline and not args.profile:
        r = cpu_oracle_bench(V, src, dst, cfg, target_edges=3_000_000, steps=1)
        cpu = {"value": round(r["value"], 6), "unit": "GE/s", "cores": 1, "kind": "oracle",
               "sample": f"the step's 6 ops by the fp64 C oracle (1 thread) on the edges of a random "
                         f"{r['E_sample'] / E:.1%} of destination rows ({r['E_sample']} edges, same graph); "
                         f"oracle build {r['t_build']:.1f}s not included"}

    if rank == 0:
        line = {
            "metric": "gSpMM GE/s & HBM GB/s (% of 8 TB/s), Reddit-shape F=64, 1/2/4/8 B200",
            "value": round(value, 4), "unit": "GE/s",
            "n_gpus": P, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": step_config(cfg, V, E, P, fused),
            "per_op": per_op,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "next_rows": next_rows,
            "multi_gpu_check": check,
            "small_config_latency": latency,
            "e2e": e2e,
            "gpu_launches": (len(OPS) * args.steps),
            "clocks": clk,
            "timing": {"wall_s_timed_region": round(wall, 3),
                       "host_launch_ms_per_step": round(sum(host_launch_ms) / len(host_launch_ms), 3), "graph_gen_s": round(t_gen, 2),
                       "graph_create_s": round(t_create, 2), "device_graph_bytes": G.device_bytes},
        }
        print(json.dumps(line), flush=True)
    if P > 1:
        dist.destroy_process_group()


# ------------------------------------------------------------ reference arm
def main_reference(args):
    """The oracle (as it stands) timed on the host cores on a bounded sample of
    the same workload.  Under torchrun only rank 0 works."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = datagen.CONFIGS[args.config]
    V, src, dst = datagen.make_graph(cfg)
    target = 1_000_000
    r = cpu_oracle_bench(V, src, dst, cfg, target_edges=target, steps=args.steps, warmup=args.warmup)
    sample = (f"per step: the 6 ops by the fp64 C oracle (1 thread; C4 x2, C6, C7, C5 x2: the state the "
              f"fused chain leaves) on the edges of a random {r['E_sample'] / len(src):.2%} of destination rows "
              f"({r['E_sample']} of {len(src)} edges); value = 6 x sampled edges / step time")
    line = {
        "impl": "reference",
        "metric": "gSpMM GE/s & HBM GB/s (% of 8 TB/s), Reddit-shape F=64, 1/2/4/8 B200",
        "value": round(r["value"], 6), "unit": "GE/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(r["t_step"] * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": step_config(cfg, V, int(len(src)), args.gpus, args.chain == "fused"),
        "cpu_baseline": {"value": round(r["value"], 6), "unit": "GE/s", "cores": 1, "kind": "oracle",
                         "sample": sample},
        "e2e": {"value": round(r["value"], 6), "unit": "GE/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.impl == "reference":
        main_reference(args)
    else:
        main_gsp(args)


if __name__ == "__main__":
    main()
