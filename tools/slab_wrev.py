"""Experiment: the edge-ID indirected weighted reverse (A8) split into destination
slabs.  alpha is stored by edge ID = fwd slot, i.e. destination-major, so the
edges of destinations [v0, v1) own one contiguous range of alpha; a reverse pass
restricted to one slab touches only that range (a smaller L2 working set per id
window).  Emulated with sub-graphs holding only the slab's edges (same vertex
ids, same relative orders, the slab's alpha range as their own alpha): the
question is whether S slab launches beat one full launch.

usage: python tools/slab_wrev.py [--slabs 1,2,4] [--reps 7]"""
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
ap.add_argument("--slabs", default="1,2,4")
ap.add_argument("--reps", type=int, default=7)
args = ap.parse_args()
cfg = datagen.CONFIGS["reddit"]
V, src, dst = datagen.make_graph(cfg)
H, F = 8, 64
Z = torch.from_numpy(datagen.uniform(2, V, F)).cuda()
flush = torch.empty(512 << 18, device="cuda")
res = {}
for S in [int(x) for x in args.slabs.split(",")]:
    # slab bounds: equal edge counts by destination (in-degree prefix)
    indeg = np.bincount(dst, minlength=V)
    cum = np.cumsum(indeg)
    bounds = [0] + [int(np.searchsorted(cum, len(src) * k / S)) + 1 for k in range(1, S)] + [V]
    graphs, alphas, outs = [], [], []
    for k in range(S):
        m = (dst >= bounds[k]) & (dst < bounds[k + 1])
        G = gsp.Graph(V, src[m], dst[m], device=0, share_symmetric=False)
        graphs.append(G)
        alphas.append(torch.rand((G.E, H), device="cuda"))
        outs.append(torch.empty((V, F), device="cuda"))

    def run():
        for G, a, o in zip(graphs, alphas, outs):
            G.gspmm_weighted(Z, a, out=o, reverse=True)
    for _ in range(2):
        run()
    ts = []
    for _ in range(args.reps):
        flush.fill_(1.0)
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        run()
        a1.record()
        torch.cuda.synchronize()
        ts.append(a0.elapsed_time(a1))
    res[S] = {"ms": round(float(np.median(ts)), 4), "E_per_slab": [int(G.E) for G in graphs]}
    del graphs, alphas, outs
    torch.cuda.empty_cache()
print(json.dumps(res))
