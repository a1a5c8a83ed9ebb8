"""Compute cost of one rank's share of the N > 1 step: gSpMM fwd (BOTH) over rank 0's
C chunk partitions of P (Reddit-shaped by default), launched back to back on one
GPU (L2 flushed first), against the ideal t_full / P.  Shows what chunking and
the heavy rows cost once a launch holds 1/(P C) of the graph.

usage: python tools/part_cost.py [--config reddit] [--P 2,4,8] [--C 1,2,4] [--reps 7]"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen  # noqa: E402
import paper_2402_03548_b200 as gsp  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="reddit")
ap.add_argument("--P", default="2,4,8")
ap.add_argument("--C", default="1,2,4")
ap.add_argument("--reps", type=int, default=7)
args = ap.parse_args()
cfg = datagen.CONFIGS[args.config]
V, src, dst = datagen.make_graph(cfg)
G = gsp.Graph(V, src, dst, device=0)
F = cfg.F
flush = torch.empty(512 << 18, device="cuda")


def timed(fn):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(args.reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return float(np.median(ts))


X = torch.rand((V, F), device="cuda")
out = torch.empty((V, F), device="cuda")
t_full = timed(lambda: G.gspmm(X, gsp.NORM_BOTH, out=out))
res = {"config": args.config, "t_full_ms": round(t_full, 4), "runs": []}
for P in [int(x) for x in args.P.split(",")]:
    for C in [int(x) for x in args.C.split(",")]:
        parts = [G.partition(P, 0, device=0, nchunks=C, chunk=c) for c in range(C)]
        R = parts[0].R
        Xp = torch.rand((parts[0].ncols, F), device="cuda")
        o = torch.empty((C * R, F), device="cuda")

        def run():
            for c, pg in enumerate(parts):
                pg.gspmm(Xp, gsp.NORM_BOTH, out=o[c * R:(c + 1) * R])
        t = timed(run)
        res["runs"].append({"P": P, "C": C, "ms": round(t, 4), "ideal_ms": round(t_full / P, 4),
                            "efficiency": round(t_full / P / t, 3), "rank0_edges": int(sum(pg.E for pg in parts))})
        del parts, Xp, o
        torch.cuda.empty_cache()
print(json.dumps(res))
