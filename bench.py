#!/usr/bin/env python
"""Benchmark of the GraphPy sparse hot path on B200 (BASELINE.json metric:
"gSpMM GE/s & HBM GB/s (% of 8 TB/s), Reddit-shape F=64, 1/2/4/8 B200").

One STEP = one pass of the whole hot path over a BASELINE config's graph
(A9 at N > 1):
  --config reddit (default) / pubmed -- GCN + GAT:
    out1 = gspmm(X,  BOTH, fwd)            GCN forward          (A3)
    out2 = gspmm(dY, BOTH, rev)            GCN backward         (A4)
    s    = gsddmm(Z, Z)        [E, H]      GAT scores           (A5)
    a    = edge_softmax(s)     in place    GAT attention        (A6)
    out3 = gspmm_weighted(Z, a, fwd)       GAT aggregate        (A7)
    out4 = gspmm_weighted(dO, a, rev)      GAT backward dZ      (A8)
  With --chain fused (default) A5-A7 run as ONE kernel (gsp_gat_forward, NEXT-2)
  that leaves the same state behind (s holds alpha): 4 launches per step.
  --config arxiv / products / cora -- GCN only: out1 and out2 (2 launches).

value = the METRIC: gSpMM GE/s = E / t of the GCN forward layer (A3; at N > 1
the layer ends when its output is all-gathered on every rank, max over ranks),
measured inside the timed steps.  The whole step's edge-visit rate is
`step.GE_s`.  N > 1: every rank runs the step on its destination-row partition
and exchanges each vertex-level output over NCCL (A9): all-gathers (chunked for
ogbn-products, each chunk's all-gather overlapping the next chunk's kernel),
reduce-scatters of per-source partials (GAT backward; GCN backward on a
directed graph).  Scaling is "strong" (the graph is fixed).

At N = 1 the default run also reports, beside the headline: an in-run gather
ceiling for the metric's kernel (tools/probe.cu: the same row gathers with no
sparse bookkeeping), the other BASELINE configs (`configs`: arxiv F=128,
products F=100, Reddit F=602, Cora / Pubmed latency), the CPU oracle on a
bounded sample (`cpu_baseline`, core count stated) and per-element parity of
sampled rows against that oracle (`parity`).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--config NAME] [--impl gsp|reference]
"""
from __future__ import annotations

import argparse
import ctypes
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
METRIC = "gSpMM GE/s & HBM GB/s (% of 8 TB/s), Reddit-shape F=64, 1/2/4/8 B200"
# paper's own numbers for context (A100-40GB, relative only: no absolute kernel rates)
PAPER_CONTEXT = {"hardware": "NVIDIA A100 40GB (P:1409, P:2165), precision unstated (fp32 implied, P:998)",
                 "gspmmv_vs_gnnadvisor": "2.87x faster (P:2375-2376)",
                 "gspmmve_T_vs_cusparse": "1.16x faster (P:2373)",
                 "gsddmm_vs_dgl": "2.99x faster on average (P:2299)",
                 "absolute_rates": "none published (kernel plots are [FIGURE] placeholders in PAPER.md)"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["gsp", "reference"], default="gsp")
    ap.add_argument("--config", default="reddit", choices=[k for k in sorted(datagen.CONFIGS) if k != "kron25"])
    ap.add_argument("--chunks", type=int, default=0,
                    help="N > 1: row chunks per rank for the all-gather overlap (0: 4 for products, else 1)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-configs", action="store_true", help="skip the other BASELINE configs' rows")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no e2e / cpu baseline / extras)")
    ap.add_argument("--check", action="store_true",
                    help="N > 1: compare every exchanged output with the oracle on sampled rows")
    ap.add_argument("--chain", choices=["fused", "separate"], default="fused",
                    help="GAT forward A5-A7 as one fused kernel (default) or three calls")
    return ap.parse_args()


# ------------------------------------------------------------- byte models
def alg_bytes(op, V, E, F, H):
    """Algorithmic (compulsory) bytes per launch: every gathered
    feature row counted once per edge, indices/values/outputs once."""
    base = 8 * (V + 1) + 4 * E                      # offsets + column ids
    if op in ("gspmm", "gspmm_fwd", "gspmm_rev"):
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


def uniq_bytes(op, V, E, F, H, edge_scales=True):
    """B_uniq: every array the op touches counted ONCE -- the
    gathered table once instead of once per edge; alg_bytes / uniq_bytes is the
    reuse the L2 must supply."""
    base = 8 * (V + 1) + 4 * E                      # offsets + column ids
    if op in ("gspmm", "gspmm_fwd", "gspmm_rev"):
        return base + 4 * V * F + 4 * V * F + 8 * V + (4 * E if edge_scales else 0)
    if op == "gspmm_weighted_fwd":
        return base + 4 * V * F + 4 * V * F + 4 * E * H
    if op == "gspmm_weighted_rev":
        return base + 4 * V * F + 4 * V * F + 4 * E * H + 4 * E
    if op == "gsddmm":           # X == Y (the bench's gsddmm(Z, Z)): one table
        return base + 4 * V * F + 4 * E * H
    if op == "edge_softmax":
        return 8 * (V + 1) + 4 * E * H + 4 * E * H
    if op == "gat_forward":
        return base + 4 * V * F + 4 * E * H + 4 * V * F
    raise KeyError(op)


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured hbm_gbs (MEASURED_PEAKS.json, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def load_traffic(config):
    """ncu DRAM bytes (read + write) per launch of each op's kernel, from the COMMITTED
    full-capture summaries (profiles/ncu_traffic.json, tools/ncu_traffic.py): ncu cannot
    run inside a timed bench process, so this is labelled as committed, not in-run."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return {}, None
    with open(p) as f:
        d = json.load(f)
    c = d.get(config, {})
    return {k: float(v["dram_bytes"]) for k, v in c.items()}, (c.get("gspmm_fwd") or {}).get("source")


def load_l2_traffic(config):
    """L2 -> L1 bytes per launch (ncu l1tex__m_xbar2l1tex_read_bytes.sum) of each op's
    kernel from the same committed captures: what the L2 actually served."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        c = json.load(f).get(config, {})
    return {k: float(v["l2_read_bytes"]) for k, v in c.items() if v.get("l2_read_bytes")}


class Probe:
    """tools/libgspprobe.so: the gather-ceiling probe (measurement only)."""

    def __init__(self):
        so = os.path.join(ROOT, "tools", "libgspprobe.so")
        self.lib = None
        if os.path.exists(so):
            self.lib = ctypes.CDLL(so)
            self.lib.gsp_probe_gather.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                                  ctypes.c_int64, ctypes.c_int, ctypes.c_void_p,
                                                  ctypes.POINTER(ctypes.c_float)]
            self.lib.gsp_probe_gather.restype = ctypes.c_int

    def gather_ms(self, X, col, stream, reps=5):
        if self.lib is None:
            return None
        ms = ctypes.c_float()
        rc = self.lib.gsp_probe_gather(X.data_ptr(), X.stride(0), X.shape[1], col.data_ptr(), col.numel(), reps,
                                       ctypes.c_void_p(stream.cuda_stream), ctypes.byref(ms))
        return float(ms.value) if rc == 0 else None


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
def host_cpu():
    """Core count and model of this host."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        avail = sorted(os.sched_getaffinity(0))
    except AttributeError:
        avail = list(range(os.cpu_count() or 1))
    return {"cpu_count": os.cpu_count(), "available": len(avail), "model": model}, avail


class pinned_core:
    """Run the oracle single-threaded pinned to one core (the last available one,
    away from core 0 where the launching thread usually runs); restores the mask."""

    def __enter__(self):
        self.info, avail = host_cpu()
        self.old = set(avail)
        self.core = avail[-1]
        try:
            os.sched_setaffinity(0, {self.core})
        except (AttributeError, OSError):
            self.core = None
        return self

    def __exit__(self, *a):
        try:
            os.sched_setaffinity(0, self.old)
        except (AttributeError, OSError):
            pass

    def describe(self):
        return {"cores": 1, "host_cores": self.info["cpu_count"], "cpu_model": self.info["model"],
                "used": f"1 of {self.info['available']} cores (single-threaded oracle, "
                        f"sched_setaffinity pinned to core {self.core})"}


def oracle_sample(V, src, dst, seed, target_edges):
    """A bounded sample of the workload for the CPU oracle: all edges whose
    destination falls in a random row subset holding ~target_edges edges."""
    rng = np.random.default_rng(seed)
    frac = min(1.0, target_edges / max(1, len(src)))
    keep_rows = rng.random(V) < frac
    m = keep_rows[dst]
    return src[m], dst[m]


def run_oracle_step(og, kind, cfg, inputs):
    """The step's ops by the oracle (fp64): C4 x2 (+ C6, C7, C5 x2 for the GAT step).
    Returns the time of the GCN forward (C4 fwd: the metric's op) and of the step."""
    X, dY, Z, dO = inputs[0], inputs[1], inputs[2], inputs[3]
    t0 = time.perf_counter()
    og.gspmm(X, 2, False)
    t_fwd = time.perf_counter() - t0
    og.gspmm(dY, 2, True)
    if kind == "gat":
        s, _ = og.gsddmm(Z, Z, cfg.H)
        a = og.edge_softmax(s.astype(np.float32)).astype(np.float32)
        og.gspmm_weighted(Z, a, False)
        og.gspmm_weighted(dO, a, True)
    return t_fwd, time.perf_counter() - t0


def cpu_oracle_bench(V, src, dst, cfg, kind, F, target_edges, steps=1, warmup=0):
    import oracle
    ssrc, sdst = oracle_sample(V, src, dst, cfg.seed, target_edges)
    with pinned_core() as pc:
        t0 = time.perf_counter()
        og = oracle.Graph(V, ssrc, sdst)
        t_build = time.perf_counter() - t0
        inputs = [datagen.uniform(cfg.seed + k, V, F) for k in range(4)]
        for _ in range(warmup):
            run_oracle_step(og, kind, cfg, inputs)
        tf, ts = [], []
        for _ in range(steps):
            a, b = run_oracle_step(og, kind, cfg, inputs)
            tf.append(a)
            ts.append(b)
    t_fwd, t = sum(tf) / len(tf), sum(ts) / len(ts)
    nops = 6 if kind == "gat" else 2
    # value in the metric's unit: GCN forward (C4) edges per second on the sample
    return {"E_sample": int(len(ssrc)), "t_step": t, "t_fwd": t_fwd, "t_build": t_build, "nops": nops,
            "value": len(ssrc) / t_fwd / 1e9, "step_GE_s": nops * len(ssrc) / t / 1e9, "cpu": pc.describe()}


def sample_rows(off, seed, n_heavy=8, n_rand=24, n_light=8):
    """Rows for per-element parity: the heaviest (CTA-split path), random, the lightest non-empty."""
    deg = np.diff(off)
    order = np.argsort(-deg, kind="stable")
    nz = order[deg[order] > 0]
    rng = np.random.default_rng(seed)
    rows = np.concatenate([order[:n_heavy], rng.choice(len(deg), n_rand, replace=False), nz[-n_light:]])
    return np.unique(rows).astype(np.int64)


def ratio(gpu, ref, bound):
    err = np.abs(np.asarray(gpu, np.float64) - ref)
    return float(np.max(err / bound)) if err.size else 0.0


def parity_gspmm(V, src, dst, fwd_off, rev_off, X, out_fwd, out_rev, F, seed):
    """Max err / bound of sampled rows of the GCN forward / backward outputs against
    oracle C4 evaluated straight from the COO list (north_star bound 1e-5 (T + 1))."""
    import oracle
    res = {}
    for name, off, out, rev in (("gspmm_fwd", fwd_off, out_fwd, False), ("gspmm_rev", rev_off, out_rev, True)):
        if out is None:
            continue
        rows = sample_rows(off, seed + int(rev))
        ref, T = oracle.gspmm_rows_coo(V, src, dst, X[int(rev)], 2, rows, reverse=rev, F=F)
        res[name] = round(ratio(out[rows], ref, oracle.bound(T)), 5)
    return res


def parity_gat(V, src, dst, fwd_off, Zh, dOh, H, alpha_rows, out_gat, out_wrev, seed):
    """Sampled-row parity of the GAT outputs the step leaves behind:
    alpha and the aggregate of sampled destination rows against oracle C10 on the
    sub-graph of those rows' in-edges (a row depends only on its own in-edges);
    the weighted reverse of sampled source rows against oracle C5 with the
    ORACLE's alpha (sub-graph of every in-edge of the sources' destinations), the
    bound widened by alpha's own bound propagated: 1e-5 (T + 1) + 2e-5 sum|dO|."""
    import oracle
    res = {}
    rows = sample_rows(fwd_off, seed)
    deg = np.diff(fwd_off)
    sel = np.isin(dst, rows)
    sub = oracle.Graph(V, src[sel], dst[sel])
    a_ref, o_ref, T = sub.gat_forward(Zh, Zh, Zh, H)
    eids = np.concatenate([np.arange(fwd_off[r], fwd_off[r + 1]) for r in rows]) if len(rows) else np.zeros(0, int)
    res["gat_alpha"] = round(ratio(alpha_rows(eids), a_ref, 2e-5), 5)
    res["gat_out"] = round(ratio(out_gat[rows], o_ref[rows], oracle.bound(T[rows])), 5)
    if out_wrev is not None:
        rng = np.random.default_rng(seed + 1)
        light = np.argsort(deg, kind="stable")
        light = light[deg[light] > 0][:4]
        us = np.unique(np.concatenate([light, rng.choice(V, 4, replace=False)])).astype(np.int64)
        dsts = np.unique(dst[np.isin(src, us)])
        sel = np.isin(dst, dsts)
        sub = oracle.Graph(V, src[sel], dst[sel])
        a_sub = sub.gat_forward(Zh, Zh, Zh, H)[0].astype(np.float32)
        ref, T = sub.gspmm_weighted(dOh, a_sub, True, rows=us)
        absd, _ = sub.gspmm(np.abs(dOh).astype(np.float32), 0, True, rows=us)
        res["gspmm_weighted_rev"] = round(ratio(out_wrev[us], ref, oracle.bound(T) + 2e-5 * absd), 5)
    return res


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


def make_time_op(torch, stream, flush):
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
    return time_op


def gspmm_row(name, V, E, F, ms, peak, probe_ms, extra=None):
    """One per-config / per-op line: ms, GE/s, algorithmic GB/s and its fraction of the
    HBM peak and of the in-run gather ceiling (probe: same gathers, no bookkeeping)."""
    b = alg_bytes("gspmm", V, E, F, 0)
    gbs = b / (ms * 1e-3) / 1e9
    row = {"op": name, "ms": round(ms, 4), "GE_s": round(E / (ms * 1e-3) / 1e9, 3), "alg_GB": round(b / 1e9, 3),
           "GB_s": round(gbs, 1), "frac_of_hbm_peak": round(gbs / peak, 4)}
    if probe_ms:
        ceil = (4 * E * F + 4 * E) / (probe_ms * 1e-3) / 1e9
        row["gather_ceiling_GB_s"] = round(ceil, 1)
        row["frac_of_gather_ceiling"] = round(gbs / ceil, 4)
    if extra:
        row.update(extra)
    return row


def other_configs(gsp, torch, stream, flush, probe, peak, G_main, cfg_main, oracle_parity):
    """BASELINE configs beside the headline (N = 1): gSpMM BOTH fwd / rev at
    arxiv F=128, products F=100, Reddit F=602 (ld 604); Cora / Pubmed latency."""
    time_op = make_time_op(torch, stream, flush)
    rows = {}
    traffic, _ = load_traffic("products")
    for name in ("arxiv", "products"):
        cfg = datagen.CONFIGS[name]
        V, src, dst = datagen.make_graph(cfg)
        G = gsp.Graph(V, src, dst, device=torch.cuda.current_device())
        F = cfg.F
        Xh = [datagen.uniform(cfg.seed + k, V, F) for k in range(2)]
        X = [torch.from_numpy(x).cuda() for x in Xh]
        outs = [torch.empty((V, F), device="cuda") for _ in range(2)]
        ms_f = time_op(lambda: G.gspmm(X[0], gsp.NORM_BOTH, out=outs[0], stream=stream))
        ms_r = time_op(lambda: G.gspmm(X[1], gsp.NORM_BOTH, out=outs[1], reverse=True, stream=stream))
        ex = G.export(rev=True, coo=False)
        col = torch.from_numpy(ex["fwd_col"]).cuda()
        pms = probe.gather_ms(X[0], col, stream)
        del col
        extra = {"table_MB": round(V * F * 4 / 1e6, 1), "graph": "R-MAT, directed" if cfg.kind == "rmat"
                 else "Chung-Lu, symmetric", "V": V, "E": int(G.E)}
        if name == "products" and traffic.get("gspmm_fwd"):
            extra["ncu_dram_GB_per_launch"] = round(traffic["gspmm_fwd"] / 1e9, 3)
            extra["ncu_dram_GB_s"] = round(traffic["gspmm_fwd"] / (ms_f * 1e-3) / 1e9, 1)
            extra["ncu_dram_frac_of_hbm_peak"] = round(traffic["gspmm_fwd"] / (ms_f * 1e-3) / 1e9 / peak, 4)
        r = {"fwd": gspmm_row("gspmm_fwd", V, G.E, F, ms_f, peak, pms, extra),
             "rev": gspmm_row("gspmm_rev", V, G.E, F, ms_r, peak, None)}
        if oracle_parity:
            outs_h = [o.cpu().numpy() for o in outs]
            r["parity_max_err_over_bound"] = parity_gspmm(V, src, dst, ex["fwd_off"], ex["rev_off"], Xh,
                                                           outs_h[0], outs_h[1], F, cfg.seed)
        rows[f"{name}_F{F}"] = r
        del G, X, outs, ex
        torch.cuda.empty_cache()
    # Reddit F = 602 (the input layer width; ld 604): a 561 MB table that misses L2
    V = G_main.V
    Xh = datagen.uniform(0x2EDD + 602, V, 602, ld=604)
    X = torch.from_numpy(Xh).cuda()[:, :602]
    out = torch.empty((V, 602), device="cuda")
    ms_f = time_op(lambda: G_main.gspmm(X, gsp.NORM_BOTH, out=out, stream=stream), reps=3)
    ms_r = time_op(lambda: G_main.gspmm(X, gsp.NORM_BOTH, out=out, reverse=True, stream=stream), reps=3)
    r = {"fwd": gspmm_row("gspmm_fwd", V, G_main.E, 602, ms_f, peak, None,
                          {"table_MB": round(V * 604 * 4 / 1e6, 1), "ld": 604}),
         "rev": gspmm_row("gspmm_rev", V, G_main.E, 602, ms_r, peak, None)}
    if oracle_parity:
        src, dst = oracle_parity
        ex = G_main.export(rev=True, coo=False)
        o = out.cpu().numpy()   # holds the reverse result (last call)
        rows_r = sample_rows(ex["rev_off"], 602)
        import oracle
        ref, T = oracle.gspmm_rows_coo(V, src, dst, Xh, 2, rows_r, reverse=True, F=602)
        r["parity_max_err_over_bound"] = {"gspmm_rev": round(ratio(o[rows_r], ref, oracle.bound(T)), 5)}
    rows["reddit_F602"] = r
    del X, out
    torch.cuda.empty_cache()
    rows["latency"] = small_config_latency(gsp, torch)
    return rows


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
        elif backend == "fake":
            # control-flow check of the NCCL path on a 1-GPU box: one process plays rank RANK of
            # WORLD_SIZE; collectives are shape-checked no-ops (no data moves, no --check)
            from torch.testing._internal.distributed.fake_pg import FakeStore
            dist.init_process_group("fake", store=FakeStore(), rank=rank, world_size=world)
        else:
            dist.init_process_group(backend)
    cfg = datagen.CONFIGS[args.config]
    kind = "gat" if cfg.H > 0 else "gcn"
    F = cfg.F
    H = cfg.H
    if kind == "gat" and cfg.F != cfg.H * cfg.Fh:
        raise SystemExit("GAT config F must equal H*Fh")

    t0 = time.time()
    V, src, dst = datagen.make_graph(cfg)
    t_gen = time.time() - t0
    t0 = time.time()
    G = gsp.Graph(V, src, dst, device=local)
    t_create = time.time() - t0
    E = G.E
    stream = torch.cuda.current_stream()

    P = world

    class Layout:
        """one padded table layout of the N > 1 step: this rank's C chunk
        partitions (chunk-major slots; C = 1 is the plain rank-major layout)"""

        def __init__(self, C):
            self.C = C
            if P > 1:
                self.parts = [G.partition(P, rank, device=local, nchunks=C, chunk=c) for c in range(C)]
                self.R = self.parts[0].R
                self.bq = G.partition_bounds(P * C)
            else:
                self.parts, self.R, self.bq = [G], V, np.array([0, V])
            self.ncols = self.parts[0].ncols
            self.E = sum(pg.E for pg in self.parts)
            self.lo, self.hi = int(self.bq[rank * C]), int(self.bq[(rank + 1) * C])   # this rank's rows

        def slot(self, q):
            return (q % self.C) * P + q // self.C

        def padded(self, Xh):
            if P == 1:
                return torch.from_numpy(Xh).cuda()
            Xp = torch.zeros((self.ncols, F), device="cuda")
            for q in range(P * self.C):
                s0 = self.slot(q) * self.R
                Xp[s0:s0 + self.bq[q + 1] - self.bq[q]] = torch.from_numpy(Xh[self.bq[q]:self.bq[q + 1]]).cuda()
            return Xp

        def unpad(self, t):
            if P == 1:
                return t
            return torch.cat([t[self.slot(q) * self.R:self.slot(q) * self.R + self.bq[q + 1] - self.bq[q]]
                              for q in range(P * self.C)])

    # GCN ops: chunked all-gathers on symmetric graphs (each chunk's all-gather overlaps the
    # next chunk's kernel); a directed graph's reverse and the GAT ops (alpha, per-source
    # partials + reduce-scatter) use the unchunked layout.  The all-gather moves the whole
    # [V, F] table while the kernel moves ~E rows, so it only matters next to the compute on
    # low-degree graphs (ogbn-products, mean 50: 0.95 ms vs 1.3 ms at P = 8);
    # on Reddit (mean 492: ~60 us vs 0.2 ms) chunks would only add launches
    # (tools/part_cost.py: P = 8 rank compute 0.22 / 0.23 / 0.32 ms at C = 1 / 2 / 4)
    Cg = 1
    if P > 1 and G.symmetric:
        Cg = args.chunks or (4 if G.E < 128 * V else 1)
    lay_gcn = Layout(Cg)
    fused = args.chain == "fused"
    rev_partial = P > 1 and not G.symmetric                     # directed GCN backward at N > 1
    # the unchunked layout: only built when an op needs it (GAT ops, directed reverse)
    lay_one = lay_gcn if (Cg == 1 or (kind == "gcn" and not rev_partial)) else Layout(1)
    # op: (name, input index, output index, exchange, layout)
    if kind == "gcn":
        op_defs = [("gspmm_fwd", 0, 0, "ag", lay_gcn),
                   ("gspmm_rev", 1, 1, "rs", lay_one) if rev_partial else ("gspmm_rev", 1, 1, "ag", lay_gcn)]
    else:
        op_defs = [("gspmm_fwd", 0, 0, "ag", lay_gcn), ("gspmm_rev", 1, 1, "ag", lay_gcn)]
        if fused:
            op_defs.append(("gat_forward", 2, 2, "ag", lay_one))
        else:
            op_defs += [("gsddmm", 2, None, None, lay_one), ("edge_softmax", None, None, None, lay_one),
                        ("gspmm_weighted_fwd", None, 2, "ag", lay_one)]
        op_defs.append(("gspmm_weighted_rev", 3, 3, "rs", lay_one))
    op_names = [d[0] for d in op_defs]
    nout = 1 + max(d[2] for d in op_defs if d[2] is not None)
    in_lay = {d[1]: d[4] for d in op_defs if d[1] is not None}     # the layout of each input table
    out_lay = {d[2]: d[4] for d in op_defs if d[2] is not None}
    ins0 = tuple(in_lay[k].padded(datagen.uniform(cfg.seed + k, V, F)) for k in range(4 if kind == "gat" else 2))
    Eloc = lay_one.E                                     # this rank's edges (alpha rows)
    R, ncols = lay_one.R, lay_one.ncols                  # per-op figures below use the unchunked layout
    s = torch.empty((Eloc, H), device="cuda") if kind == "gat" else None

    def new_set(ins):
        outs = [torch.empty((out_lay[i].C * out_lay[i].R if P > 1 else V, F), device="cuda") for i in range(nout)]
        partial = {d[2]: torch.empty((d[4].ncols, F), device="cuda") for d in op_defs if d[3] == "rs" and P > 1}
        gathered = {d[2]: torch.empty((d[4].ncols, F), device="cuda") for d in op_defs if d[3] == "ag" and P > 1}
        return {"ins": ins, "outs": outs, "partial": partial, "gathered": gathered}

    set0 = new_set(ins0)

    def launch(name, c, st, L):
        """kernel of op `name` for chunk c of layout L with the buffers of set st"""
        pg = L.parts[c]
        ins, outs = st["ins"], st["outs"]
        o = (lambda i: outs[i][c * L.R:(c + 1) * L.R]) if P > 1 else (lambda i: outs[i])
        if name == "gspmm_fwd":
            pg.gspmm(ins[0], gsp.NORM_BOTH, out=o(0), stream=stream)
        elif name == "gspmm_rev":
            if rev_partial:
                pg.gspmm(ins[1], gsp.NORM_BOTH, out=st["partial"][1], reverse=True, stream=stream)
            else:
                pg.gspmm(ins[1], gsp.NORM_BOTH, out=o(1), reverse=True, stream=stream)
        elif name == "gat_forward":
            pg.gat_forward(ins[2], ins[2], ins[2], H, alpha=s, out=o(2), stream=stream)
        elif name == "gsddmm":
            pg.gsddmm(ins[2], ins[2], out=s, stream=stream)
        elif name == "edge_softmax":
            pg.edge_softmax(s, out=s, stream=stream)
        elif name == "gspmm_weighted_fwd":
            pg.gspmm_weighted(ins[2], s, out=o(2), stream=stream)
        elif name == "gspmm_weighted_rev":
            if P == 1:
                pg.gspmm_weighted(ins[3], s, out=o(3), reverse=True, stream=stream)
            else:   # alpha lives on the destination's rank: per-source partials
                pg.gspmm_weighted(ins[3], s, out=st["partial"][3], reverse=True, stream=stream)
        else:
            raise KeyError(name)

    overlap = P > 1 and backend in ("nccl", "fake")
    obs = torch.cuda.Stream() if overlap else None

    def issue(name, i_out, exch, c, st, pending, L):
        """NCCL: the op's collective for chunk c, issued async right after its kernel"""
        if not overlap or exch is None:
            return
        if exch == "ag":
            w = dist.all_gather_into_tensor(st["gathered"][i_out][c * P * L.R:(c + 1) * P * L.R],
                                            st["outs"][i_out][c * L.R:(c + 1) * L.R], async_op=True)
        else:
            w = dist.reduce_scatter_tensor(st["outs"][i_out], st["partial"][i_out], async_op=True)
        pending.setdefault(name, []).append(w)

    def host_exchange(st):
        """gloo (validation on a 1-GPU box): host-staged equivalent after the step"""
        for name, _, i_out, exch, L in op_defs:
            if exch == "ag":
                for c in range(L.C):
                    blk = [torch.empty((L.R, F)) for _ in range(P)]
                    dist.all_gather(blk, st["outs"][i_out][c * L.R:(c + 1) * L.R].cpu())
                    st["gathered"][i_out][c * P * L.R:(c + 1) * P * L.R].copy_(torch.cat(blk))
            elif exch == "rs":
                t = st["partial"][i_out].cpu()
                dist.all_reduce(t)
                st["outs"][i_out].copy_(t[rank * L.R:(rank + 1) * L.R])

    def allreduce_max(v):
        t = torch.tensor([float(v)], device="cuda" if backend in ("nccl", "fake") else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def mark(st_=None):
        e = torch.cuda.Event(enable_timing=True)
        e.record(st_ or stream)
        return e

    def step(record, st=set0):
        """one step; returns (marks after each op, layer-done event)"""
        marks = [mark()] if record else None
        pending = {}
        layer = None
        for name, _, i_out, exch, L in op_defs:
            for c in range(L.C):
                launch(name, c, st, L)
                issue(name, i_out, exch, c, st, pending, L)
            if record:
                marks.append(mark())
            if record and name == "gspmm_fwd":
                if overlap:      # the layer ends when its all-gathers land (observer stream)
                    with torch.cuda.stream(obs):
                        for w in pending.get(name, []):
                            w.wait()
                    layer = mark(obs)
                else:
                    layer = marks[-1]
        if P > 1:
            if overlap:
                for ws in pending.values():
                    for w in ws:
                        w.wait()          # stream-ordered: the compute stream waits for NCCL
            else:
                host_exchange(st)
            if record:
                marks.append(mark())
        return marks, layer

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()

    flush = torch.empty(L2_FLUSH_BYTES // 4, dtype=torch.float32, device="cuda")
    clocks = ClockSampler(local) if (rank == 0 and not args.profile) else None
    if clocks:
        clocks.start()
        time.sleep(0.3)
    if P > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    ev = {k: [] for k in op_names + ["exchange"]}
    step_ms, layer_ms, host_launch_ms = [], [], []
    for _ in range(args.steps):
        flush.fill_(1.0)                      # L2 flush between timed steps (outside the events)
        h0 = time.perf_counter()
        marks, layer = step(True)
        host_launch_ms.append((time.perf_counter() - h0) * 1e3)
        torch.cuda.synchronize()
        names = op_names + (["exchange"] if P > 1 else [])
        for i, n in enumerate(names):
            ev[n].append(marks[i].elapsed_time(marks[i + 1]))
        step_ms.append(marks[0].elapsed_time(marks[-1]))
        layer_ms.append(marks[0].elapsed_time(layer))
    torch.cuda.synchronize()
    if P > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    clk = clocks.stop() if clocks else None

    t_step = sum(step_ms) / len(step_ms)
    t_layer = sum(layer_ms) / len(layer_ms)
    if P > 1:
        t_step = allreduce_max(t_step)
        t_layer = allreduce_max(t_layer)
    value = E / (t_layer * 1e-3) / 1e9
    visits = (6 if kind == "gat" else 2) * E
    avg = {k: (sum(v) / len(v) if v else None) for k, v in ev.items()}

    # ------------------------------------------- N > 1: check vs the oracle
    check = None
    if P > 1 and args.check and backend != "fake":
        check = multi_gpu_check(args, gsp, torch, dist, rank, P, cfg, kind, V, src, dst, G, new_set, in_lay,
                                step, op_defs, allreduce_max)

    # ---------------------------------------------------------------- e2e
    # The same step through the C ABI with HOST buffers: every step copies its input
    # tables from pinned host memory (H2D engine) and reads its vertex outputs back
    # (D2H engine), inside the timed region.  Steps are pipelined the way a stream of
    # batches runs: two device buffer sets (each with its own outputs, partials and
    # gathered tables), so step k+1's inputs upload while step k computes; each op
    # waits only for its own input, each output leaves as soon as it is final.  No L2
    # flush between steps: each step's inputs exceed L2.  gloo ranks: no e2e.
    e2e = None
    if not args.no_e2e and not args.profile and (P == 1 or overlap):
        nin = len(ins0)
        hin = [torch.empty(tuple(t.shape), dtype=torch.float32).pin_memory() for t in ins0]
        for h, d in zip(hin, ins0):
            h.copy_(d.cpu())
        sets = [set0, new_set(tuple(torch.empty_like(t) for t in ins0))]
        h2d = torch.cuda.Stream()
        d2h = torch.cuda.Stream()

        def run_e2e(defs):
            """K pipelined steps of the ops `defs` (inputs uploaded / outputs read back
            every step); returns (ms per step, H2D bytes, D2H bytes per step)"""
            used_in = sorted({d[1] for d in defs if d[1] is not None})
            used_out = sorted({d[2] for d in defs if d[2] is not None})
            hout = [{i: torch.empty(tuple(sets[j]["outs"][i].shape), dtype=torch.float32).pin_memory()
                     for i in used_out} for j in range(2)]
            in_free, out_free = [None, None], [None, None]

            def e2e_step(k):
                j = k % 2
                st = sets[j]
                if in_free[j] is not None:          # step k-2 is done reading this input set
                    h2d.wait_event(in_free[j])
                ready = {}
                with torch.cuda.stream(h2d):
                    for i in used_in:
                        st["ins"][i].copy_(hin[i], non_blocking=True)
                        e = torch.cuda.Event()
                        e.record(h2d)
                        ready[i] = e
                if out_free[j] is not None:         # step k-2's outputs have left this set
                    stream.wait_event(out_free[j])
                done, pending = [], {}
                for name, i_in, i_out, exch, L in defs:
                    if i_in is not None:
                        stream.wait_event(ready[i_in])
                    for c in range(L.C):
                        launch(name, c, st, L)
                        issue(name, i_out, exch, c, st, pending, L)
                    if i_out is not None and P == 1:
                        e = torch.cuda.Event()
                        e.record(stream)
                        done.append((e, i_out))
                if P > 1:
                    for ws in pending.values():
                        for w in ws:
                            w.wait()
                    e = torch.cuda.Event()
                    e.record(stream)
                    done = [(e, i) for i in used_out]
                f = torch.cuda.Event()
                f.record(stream)
                in_free[j] = f
                with torch.cuda.stream(d2h):
                    for e, i in done:
                        d2h.wait_event(e)
                        hout[j][i].copy_(st["outs"][i], non_blocking=True)   # each rank: its own rows
                g = torch.cuda.Event()
                g.record(d2h)
                out_free[j] = g

            for k in range(2):
                e2e_step(k)
            torch.cuda.synchronize()
            if P > 1:
                dist.barrier()
            # a pipelined run pays one upload (fill) and one read-back (drain) that no
            # compute hides; >= 32 steps keep that one-time cost to a few % of the figure
            K = max(32, args.steps)
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
            t = a0.elapsed_time(a1) / K
            if P > 1:
                t = allreduce_max(t)
            jl = (K - 1) % 2      # the host copies hold what the device computed
            assert torch.equal(hout[jl][used_out[0]], sets[jl]["outs"][used_out[0]].cpu())
            return t, K, sum(hin[i].numel() * 4 for i in used_in), sum(h.numel() * 4 for h in hout[0].values())

        # the metric end to end: the GCN forward layer (A3, + its all-gather at N > 1) as a
        # user runs it layer after layer -- X uploaded from pinned host memory, the layer's
        # output read back, every step
        def link_gbs(dst, src, st_):
            """this box's host link: GB/s of one pinned copy of the layer's table, alone"""
            ts = []
            for _ in range(3):
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                with torch.cuda.stream(st_):
                    a0.record(st_)
                    dst.copy_(src, non_blocking=True)
                    a1.record(st_)
                torch.cuda.synchronize()
                ts.append(a0.elapsed_time(a1))
            return round(src.numel() * 4 / (min(ts) * 1e-3) / 1e9, 1)
        link = {"h2d_GB_s": link_gbs(sets[1]["ins"][0], hin[0], h2d),
                "d2h_GB_s": link_gbs(hin[0], sets[1]["ins"][0], d2h)}
        # both directions at once (what the pipelined layer does every step)
        hscratch = torch.empty_like(hin[0]).pin_memory()
        tb = []
        for _ in range(3):
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            h2d.wait_event(a0)
            d2h.wait_event(a0)
            with torch.cuda.stream(h2d):
                sets[1]["ins"][0].copy_(hin[0], non_blocking=True)
            with torch.cuda.stream(d2h):
                hscratch.copy_(set0["ins"][0], non_blocking=True)
            stream.wait_stream(h2d)
            stream.wait_stream(d2h)
            a1.record(stream)
            torch.cuda.synchronize()
            tb.append(a0.elapsed_time(a1))
        link["both_directions_ms"] = round(min(tb), 4)
        del hscratch
        hin[0].copy_(ins0[0].cpu())
        t_l, K, bi, bo = run_e2e([d for d in op_defs if d[0] == "gspmm_fwd"])
        # and the whole step the same way (all inputs up, all vertex outputs back)
        t_s, _, bis, bos = run_e2e(op_defs)
        e2e = {"value": round(E / (t_l * 1e-3) / 1e9, 4), "unit": "GE/s",
               "what": "E / t of the GCN forward layer through the C ABI with host buffers: every step uploads "
                       "X from pinned host memory and reads the layer's output back (the metric end to end)",
               "ms_per_step": round(t_l, 4), "steps": K, "h2d_bytes_per_step": int(bi), "d2h_bytes_per_step": int(bo),
               "step": {"ops": op_names, "ms": round(t_s, 4), "GE_s": round(visits / (t_s * 1e-3) / 1e9, 4),
                        "h2d_bytes_per_step": int(bis), "d2h_bytes_per_step": int(bos)},
               "how": "pinned host buffers, H2D / D2H engines overlapped with the kernels and pipelined across "
                      "steps (two device buffer sets); no L2 flush (per-step inputs exceed L2)",
               # the host link of this box, measured alone: the layer's e2e floor is
               # max(kernel, bytes / link) -- box-dependent (PCIe / NUMA placement)
               "link": link, "link_floor_ms": link["both_directions_ms"] if bi == bo else
               round(max(bi / link["h2d_GB_s"], bo / link["d2h_GB_s"]) / 1e6, 4)}
        del sets
        torch.cuda.empty_cache()

    # ----------------------------------------------------------- roofline
    peak, peak_kind = load_peaks()
    time_op = make_time_op(torch, stream, flush)
    Vloc = (lay_one.hi - lay_one.lo) if P > 1 else V   # this rank's rows
    per_op = {}
    traffic, traffic_src = load_traffic(args.config) if P == 1 else ({}, None)

    # rows the step does not launch on their own: timed one by one outside it
    outside = {}
    if not args.profile and kind == "gat" and P == 1:
        if fused:   # the unfused A5-A7 calls, each on its own (same graph, same inputs)
            Z = ins0[2]
            s2 = torch.empty((Eloc, H), device="cuda")
            g2 = torch.empty((Vloc, F), device="cuda")
            G.gsddmm(Z, Z, out=s2, stream=stream)
            outside["gsddmm"] = time_op(lambda: G.gsddmm(Z, Z, out=s2, stream=stream))
            raw = s2.clone()              # out of place: the same logits every call
            outside["edge_softmax"] = time_op(lambda: G.edge_softmax(raw, out=s2, stream=stream))
            outside["gspmm_weighted_fwd"] = time_op(lambda: G.gspmm_weighted(Z, s2, out=g2, stream=stream))
            del s2, g2, raw
        else:
            g2 = torch.empty((Vloc, F), device="cuda")
            outside["gat_forward"] = time_op(lambda: G.gat_forward(ins0[2], ins0[2], ins0[2], H,
                                                                   alpha=torch.empty_like(s), out=g2, stream=stream))
            del g2

    # ------------------------------------------- NEXT rows (outside the step)
    next_rows = None
    if not args.profile and kind == "gat" and P == 1:
        X, dY, Z, dO = ins0
        alpha2 = torch.empty((Eloc, H), device="cuda")
        gout = torch.empty((Vloc, F), device="cuda")
        dal = torch.rand((Eloc, H), device="cuda")
        ms_gat = avg["gat_forward"] if fused else outside["gat_forward"]
        ms_max = time_op(lambda: G.gspmm_reduce(X, gsp.REDUCE_MAX, out=gout, stream=stream))
        hout_ = torch.empty((Vloc, H), device="cuda")
        ms_e = time_op(lambda: G.gspmm_e(s, gsp.REDUCE_SUM, out=hout_, stream=stream))
        ms_ve = time_op(lambda: G.gsddmm_ve(Z[:, :H], dal, gsp.OP_ADD, gsp.SIDE_SRC, out=alpha2, stream=stream))
        ms_sbw = time_op(lambda: G.edge_softmax_backward(s, dal, out=dal, stream=stream))
        ms_gbw = time_op(lambda: G.gat_backward_scores(dO, Z, s, out=alpha2, stream=stream))
        ms_gbw_sep = time_op(lambda: G.gsddmm(dO, Z, out=alpha2, stream=stream)) + ms_sbw
        # NEXT-3 additive GAT attention: scores alone and the fused forward (alpha + aggregate)
        el = Z[:, :H].contiguous()
        er = dO[:, :H].contiguous()
        ms_add = time_op(lambda: G.gsddmm_add_leaky(el, er, 0.2, out=alpha2, stream=stream))
        ms_gat_add = time_op(lambda: G.gat_forward_additive(el, er, Z, 0.2, alpha=alpha2, out=gout, stream=stream))
        sep = sum((outside if fused else avg)[k] for k in ("gsddmm", "edge_softmax", "gspmm_weighted_fwd"))
        next_rows = {
            "gat_forward_fused": {"row": "NEXT-2", "ms": round(ms_gat, 4), "in_step": fused,
                                  "vs_separate_chain_ms": round(sep, 4),
                                  "GE_s": round(Eloc / (ms_gat * 1e-3) / 1e9, 3)},
            "gspmm_reduce_max": {"row": "NEXT-3", "ms": round(ms_max, 4),
                                 "GB_s": round(alg_bytes("gspmm", Vloc, Eloc, F, H) / (ms_max * 1e-3) / 1e9, 1)},
            "gspmm_e_sum": {"row": "NEXT-3", "ms": round(ms_e, 4),
                            "GB_s": round((Eloc * H * 4 + (Vloc + 1) * 8 + Vloc * H * 4) / (ms_e * 1e-3) / 1e9, 1)},
            "gsddmm_ve_add_src": {"row": "NEXT-3", "ms": round(ms_ve, 4),
                                  "GB_s": round((2 * Eloc * H * 4 + Eloc * 4 + (Vloc + 1) * 8 + V * H * 4)
                                                / (ms_ve * 1e-3) / 1e9, 1)},
            "gsddmm_add_leaky": {"row": "NEXT-3", "ms": round(ms_add, 4),
                                 "GB_s": round((Eloc * 4 + Eloc * H * 4 + Eloc * H * 4 + (Vloc + 1) * 8 + V * H * 4)
                                               / (ms_add * 1e-3) / 1e9, 1),
                                 "what": "additive GAT scores lrelu(el[u] + er[v]), H = 8"},
            "gat_forward_additive_fused": {"row": "NEXT-3", "ms": round(ms_gat_add, 4),
                                           "GE_s": round(Eloc / (ms_gat_add * 1e-3) / 1e9, 3),
                                           "what": "alpha = softmax(lrelu(el[u] + er[v])), out = sum alpha Z[u], "
                                                   "one pass, alpha written (H = 8, Fh = 8)"},
            "gat_backward_scores_fused": {"row": "NEXT-1", "ms": round(ms_gbw, 4),
                                          "vs_gsddmm_plus_softmax_backward_ms": round(ms_gbw_sep, 4)},
            "edge_softmax_backward": {"row": "NEXT-1", "ms": round(ms_sbw, 4),
                                      "GB_s": round(alg_bytes("edge_softmax", Vloc, Eloc, F, H) * 1.5
                                                    / (ms_sbw * 1e-3) / 1e9, 1)},
        }
        del alpha2, gout, dal, hout_, el, er
        # context: warm-L2 time of the headline op (no flush: steady
        # state layer to layer) and the paper's kernel-plot shapes (F = 32, one head:
        # P:2308) on the same graph
        o0 = set0["outs"][0]
        warm_ms = time_op(lambda: G.gspmm(X, gsp.NORM_BOTH, out=o0, stream=stream), flush_l2=False)
        X32 = torch.rand((V, 32), device="cuda") - 0.5
        w1 = torch.rand((Eloc, 1), device="cuda")
        o32 = torch.empty((V, 32), device="cuda")
        shapes = {
            "gspmm_fwd_F32": time_op(lambda: G.gspmm(X32, gsp.NORM_BOTH, out=o32, stream=stream)),
            "gspmm_weighted_rev_F32_H1": time_op(lambda: G.gspmm_weighted(X32, w1, out=o32, reverse=True,
                                                                          stream=stream)),
            "gsddmm_F32_H1": time_op(lambda: G.gsddmm(X32, X32, H=1, out=w1, stream=stream)),
        }
        next_rows["context"] = {"gspmm_fwd_warm_l2_ms": round(warm_ms, 4),
                                "paper_plot_shapes_ms": {k: round(v, 4) for k, v in shapes.items()}}
        del X32, w1, o32

    bytes_of = {k: alg_bytes(k, Vloc, Eloc, F, H) for k in
                ("gspmm_fwd", "gspmm_rev", "gsddmm", "edge_softmax", "gspmm_weighted_fwd", "gspmm_weighted_rev",
                 "gat_forward")}
    uniq_of = {k: uniq_bytes(k, Vloc, Eloc, F, H, edge_scales=G.memory()["edge_scales"] > 0) for k in bytes_of}
    l2traffic = load_l2_traffic(args.config) if P == 1 else {}
    for k, ms in [(k, avg[k]) for k in op_names] + list(outside.items()):
        gbs = bytes_of[k] / (ms * 1e-3) / 1e9
        per_op[k] = {"ms": round(ms, 4), "GE_s": round(Eloc / (ms * 1e-3) / 1e9, 3),
                     "alg_GB": round(bytes_of[k] / 1e9, 3), "alg_GB_s": round(gbs, 1),
                     "in_step": k in op_names,
                     "ncu_dram_GB": round(traffic[k] / 1e9, 3) if k in traffic else None,
                     # measured DRAM traffic (committed ncu capture) over this run's time
                     "dram_GB_s": round(traffic[k] / (ms * 1e-3) / 1e9, 1) if k in traffic else None,
                     "dram_frac_of_hbm_peak": round(traffic[k] / (ms * 1e-3) / 1e9 / peak, 4) if k in traffic else None,
                     # SURVEY §8(d) "reuse = B_alg / DRAM bytes" (> 1: the gathers are L2-served)
                     "reuse": round(bytes_of[k] / traffic[k], 2) if traffic.get(k) else None,
                     "uniq_GB": round(uniq_of[k] / 1e9, 3),
                     "ncu_l2_to_l1_GB": round(l2traffic[k] / 1e9, 3) if k in l2traffic else None}
    if P > 1:
        per_op["exchange"] = {"ms": round(avg["exchange"], 4),
                              "what": f"GCN ops {Cg} chunk(s) per all-gather; all-gathers / reduce-scatters "
                                      + ("(NCCL, each issued async right after its kernel and overlapped with the "
                                         "next kernels; ms = the residual wait after the last op)"
                                         if backend == "nccl" else
                                         "(fake process group: control-flow check, no data moved)" if backend == "fake"
                                         else "(host-staged gloo: validation only)")}

    # the metric's kernel against its ceilings: the gathered table of Reddit F = 64 is
    # L2-resident, so the bound is the L2 gather rate, measured in this run by the probe
    # (the same row gathers with no sparse bookkeeping); HBM beside it in measured bytes
    probe = Probe()
    dom = "gspmm_fwd"
    achieved = per_op[dom]["alg_GB_s"]
    roofline = {"kernel": "spmm_kernel<VEC=8,LPE=8,CPL=1,scaled,U=4,3 CTAs/SM> (gspmm fwd, BOTH norm)",
                "unit": "GB/s", "achieved": achieved, "alg_bytes_per_launch": bytes_of[dom],
                "achieved_definition": "algorithmic bytes (gathered rows once per edge, SURVEY §8(d)) / the "
                                       "kernel's event-timed duration inside the step"}
    pms = None
    if not args.profile and P == 1 and probe.lib is not None:
        col = torch.from_numpy(G.export(rev=False, coo=False)["fwd_col"]).cuda()
        pms = probe.gather_ms(ins0[0], col, stream)
        del col
    table_mb = ncols * F * 4 / 1e6
    if pms:
        ceil = (4 * Eloc * F + 4 * Eloc) / (pms * 1e-3) / 1e9
        roofline.update({"bound": "l2" if table_mb < 100 else "hbm",
                         "peak": round(ceil, 1),
                         "peak_kind": "in-run gather ceiling (tools/probe.cu: this graph's fwd_col row gathers "
                                      "from this table, LDG.256, no sparse bookkeeping; rows + column ids)",
                         "frac": round(achieved / ceil, 4)})
    else:
        roofline.update({"bound": "hbm", "peak": peak, "peak_kind": peak_kind, "frac": round(achieved / peak, 4)})
    tr = traffic.get(dom)
    roofline["traffic"] = tr
    roofline["traffic_source"] = (f"committed ncu --set full capture ({traffic_src or 'profiles/ncu_traffic.json'}): "
                                  "dram__bytes_read.sum + dram__bytes_write.sum per launch (not measured in-run)"
                                  if tr else None)
    roofline["hbm"] = {"peak": peak, "peak_kind": peak_kind,
                       "alg_frac": round(achieved / peak, 4),
                       "dram_GB_s": round(tr / (avg[dom] * 1e-3) / 1e9, 1) if tr else None,
                       "dram_frac": round(tr / (avg[dom] * 1e-3) / 1e9 / peak, 4) if tr else None,
                       "note": "algorithmic bytes exceed HBM peak because the gathers are L2-served "
                               "(table fits L2); dram_* = measured DRAM bytes over time"}

    # ---------------------------------- CPU oracle: baseline + sampled parity
    cpu = None
    parity = None
    oracle_ok = rank == 0 and P == 1 and not args.no_cpu_baseline and not args.profile
    if oracle_ok:
        r = cpu_oracle_bench(V, src, dst, cfg, kind, F, target_edges=3_000_000 if kind == "gat" else 6_000_000)
        cpu = {"value": round(r["value"], 6), "unit": "GE/s", "kind": "oracle", **r["cpu"],
               "sample": f"the step's {r['nops']} ops by the fp64 C oracle (1 thread) on the edges of a random "
                         f"{r['E_sample'] / E:.1%} of destination rows ({r['E_sample']} edges, same graph); "
                         f"value = sampled edges / time of the GCN forward (C4, the metric's op); "
                         f"oracle build {r['t_build']:.1f}s not included",
               "step_GE_s": round(r["step_GE_s"], 6), "t_step_s": round(r["t_step"], 3)}
        ex = G.export(rev=True, coo=False)
        Xh = [datagen.uniform(cfg.seed + k, V, F) for k in range(4 if kind == "gat" else 2)]
        outs_h = [o.cpu().numpy() for o in set0["outs"]]
        parity = {"bound": "1e-5 (T + 1) per element (north_star); alpha 2e-5 absolute",
                  "rows": "sampled: 8 heaviest, 24 random, 8 lightest non-empty per output",
                  **parity_gspmm(V, src, dst, ex["fwd_off"], ex["rev_off"], Xh, outs_h[0], outs_h[1], F, cfg.seed)}
        if kind == "gat":
            alpha_rows = lambda ei: s[torch.from_numpy(ei).cuda()].cpu().numpy()
            parity.update(parity_gat(V, src, dst, ex["fwd_off"], Xh[2], Xh[3], H, alpha_rows,
                                     outs_h[2], outs_h[3], cfg.seed + 3))
        parity["max"] = max(v for k, v in parity.items() if isinstance(v, float))
        del ex, outs_h

    # ------------------------------------ other BASELINE configs (N = 1 only)
    configs = None
    if rank == 0 and P == 1 and not args.profile and not args.no_configs and args.config == "reddit":
        for k in ("outs", "partial", "gathered"):
            set0[k] = None
        torch.cuda.empty_cache()
        configs = other_configs(gsp, torch, stream, flush, probe, peak, G, cfg,
                                (src, dst) if oracle_ok else None)

    if rank == 0:
        launches = sum(d[4].C for d in op_defs) * args.steps
        line = {
            "metric": METRIC,
            "value": round(value, 4), "unit": "GE/s",
            "value_definition": ("E / t of the GCN forward layer (gspmm fwd, BOTH norm, A3)"
                                 + (" incl. its all-gather, max over ranks" if P > 1 else "")
                                 + ", averaged over the timed steps (CUDA events on the launching stream)"),
            "n_gpus": P, "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step, 4),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": "f32", "data": "synthetic",
            "config": {"workload": f"{cfg.name}-shaped " + (
                "GCN gSpMM fwd+bwd (BOTH norm) + GAT chain (gSDDMM u.v, edge softmax, weighted gSpMM fwd+rev), "
                f"F={F}, H={H}x{cfg.Fh}" if kind == "gat" else f"GCN gSpMM fwd+bwd (BOTH norm), F={F}"),
                       "gat_chain": (("fused: gSDDMM + edge softmax + weighted gSpMM fwd in one kernel "
                                      "(gsp_gat_forward; alpha still written)") if fused else "separate: 3 kernels")
                       if kind == "gat" else None,
                       "V": V, "E": E, "F": F, "H": H or None, "Fh": cfg.Fh or None,
                       "graph": f"Chung-Lu beta={cfg.beta}, seed={cfg.seed:#x}" if cfg.kind == "chung_lu"
                       else f"R-MAT scale {cfg.scale}, seed={cfg.seed:#x}",
                       "parallelism": (f"row-partition x{P}" + (f", {Cg} chunks per rank for the GCN ops"
                                                                 if Cg > 1 else "")) if P > 1 else "single GPU",
                       "l2": f"flushed between timed steps ({L2_FLUSH_BYTES >> 20} MiB write)",
                       "edge_visits_per_step": visits},
            "step": {"ops": op_names, "ms": round(t_step, 4), "GE_s": round(visits / (t_step * 1e-3) / 1e9, 4),
                     "what": "edge visits of all the step's ops / step time",
                     "layer_ms": round(t_layer, 4)},
            "per_op": per_op,
            "roofline": roofline,
            "cpu_baseline": cpu,
            "parity": parity,
            "configs": configs,
            "next_rows": next_rows,
            "multi_gpu_check": check,
            "paper_context": PAPER_CONTEXT,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "timing": {"wall_s_timed_region": round(wall, 3),
                       "host_launch_ms_per_step": round(sum(host_launch_ms) / len(host_launch_ms), 3),
                       "graph_gen_s": round(t_gen, 2), "graph_create_s": round(t_create, 2),
                       "device_graph_bytes": G.device_bytes, "device_graph_bytes_by_kind": G.memory()},
        }
        print(json.dumps(line), flush=True)
    if P > 1:
        dist.destroy_process_group()


def multi_gpu_check(args, gsp, torch, dist, rank, P, cfg, kind, V, src, dst, G, new_set, in_lay, step, op_defs,
                    allreduce_max):
    """N > 1 --check: one step on seeded inputs, then every exchanged output of
    sampled rows against the oracle per element (north_star bound).  The GAT
    weighted reverse gets seeded weights w (the oracle's C5 input) instead of alpha;
    each rank holds w for its own edge-id range."""
    import oracle
    F, H = cfg.F, cfg.H
    nin = 4 if kind == "gat" else 2
    Xh = [datagen.uniform(cfg.seed + 100 + k, V, F) for k in range(nin)]
    st = new_set(tuple(in_lay[k].padded(Xh[k]) for k in range(nin)))
    step(False, st)
    torch.cuda.synchronize()
    res = {}
    ex = G.export(rev=True, coo=False)
    fin, lay = {}, {}
    for name, _, i_out, exch, L in op_defs:
        if i_out is None:
            continue
        lay[name] = L
        if exch == "ag":
            fin[name] = L.unpad(st["gathered"][i_out]).cpu().numpy()
        else:   # rs: this rank's own rows of the rank-major layout
            fin[name] = st["outs"][i_out].cpu().numpy()
    for name, off, rev in (("gspmm_fwd", ex["fwd_off"], False), ("gspmm_rev", ex["rev_off"], True)):
        rows = sample_rows(off, 7 + int(rev))
        ref, T = oracle.gspmm_rows_coo(V, src, dst, Xh[int(rev)], 2, rows, reverse=rev, F=F)
        got = fin[name]
        if got.shape[0] != V:            # reduce-scatter output: only this rank's rows
            lo, hi = lay[name].lo, lay[name].hi
            rows_m = rows[(rows >= lo) & (rows < hi)]
            sel = np.isin(rows, rows_m)
            got, ref, T, rows = got[rows_m - lo], ref[sel], T[sel], rows_m
        else:
            got = got[rows]
        res[name] = ratio(got, ref, oracle.bound(T))
    if kind == "gat":
        og = oracle.Graph(V, src, dst)
        rows = sample_rows(og.fwd_off, 9)
        sel = np.isin(dst, rows)
        sub = oracle.Graph(V, src[sel], dst[sel])
        a_ref, o_ref, T = sub.gat_forward(Xh[2], Xh[2], Xh[2], H)
        res["gat_forward"] = ratio(fin.get("gat_forward", fin.get("gspmm_weighted_fwd"))[rows], o_ref[rows],
                                   oracle.bound(T[rows]))
        # weighted reverse with seeded weights: this rank's w rows = its edge-id range
        L = lay["gspmm_weighted_rev"]
        lo, hi = L.lo, L.hi
        wh = datagen.uniform(cfg.seed + 200, og.E, H, lo=0, hi=1)
        e0, e1 = og.fwd_off[lo], og.fwd_off[hi]
        wloc = torch.from_numpy(wh[e0:e1]).cuda()
        part = st["partial"][3]
        L.parts[0].gspmm_weighted(st["ins"][3], wloc, out=part, reverse=True)
        tot = part.cpu()
        dist.all_reduce(tot)
        mine = tot.numpy()[rank * L.R:rank * L.R + hi - lo]
        rows = np.arange(lo, hi)
        rows = rows[np.random.default_rng(11).choice(len(rows), min(48, len(rows)), replace=False)] if len(rows) else rows
        ref, T = og.gspmm_weighted(Xh[3], wh, True, rows=rows)
        res["gspmm_weighted_rev"] = ratio(mine[rows - lo], ref, oracle.bound(T))
    m = allreduce_max(max(res.values()))
    return {"max_err_over_bound": m, "per_output": {k: round(v, 5) for k, v in res.items()},
            "bound": "1e-5 (T + 1) per element vs the oracle on sampled rows", "ok": bool(m <= 1.0)}


# ------------------------------------------------------------ reference arm
def main_reference(args):
    """The oracle (as it stands) timed on the host cores on a bounded sample of
    the same workload.  Under torchrun only rank 0 works."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = datagen.CONFIGS[args.config]
    kind = "gat" if cfg.H > 0 else "gcn"
    V, src, dst = datagen.make_graph(cfg)
    r = cpu_oracle_bench(V, src, dst, cfg, kind, cfg.F, target_edges=1_000_000, steps=args.steps,
                         warmup=args.warmup)
    # the metric's unit: gSpMM (A3) edges per second = sampled edges / time of the GCN forward
    value = r["value"]
    sample = (f"per step: the {r['nops']} ops by the fp64 C oracle (1 thread, pinned) on the edges of a random "
              f"{r['E_sample'] / len(src):.2%} of destination rows ({r['E_sample']} of {len(src)} edges); "
              f"value = sampled edges / time of the GCN forward (C4) in the step")
    line = {
        "impl": "reference",
        "metric": METRIC,
        "value": round(value, 6), "unit": "GE/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(r["t_step"] * 1e3, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{cfg.name}-shaped, the same step as the gsp arm, CPU oracle", "V": V,
                   "E": int(len(src)), "F": cfg.F},
        "cpu_baseline": {"value": round(value, 6), "unit": "GE/s", "kind": "oracle", **r["cpu"], "sample": sample},
        "e2e": {"value": round(value, 6), "unit": "GE/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
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
