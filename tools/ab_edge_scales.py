"""Isolated A/B of the per-edge column scales (GSP_BUILD_EDGE_SCALES) and of the
GCN-lean device format (GSP_BUILD_NO_EDGE_IDS): the same gSpMM (BOTH norm)
launches on graphs that differ only in these flags, interleaved A/B/C rounds
(CUDA events, L2 flushed before every call, median per variant).

usage: python tools/ab_edge_scales.py [--configs reddit,products] [--rounds 7] [--out profiles/x.json]"""
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
ap.add_argument("--configs", default="reddit,products")
ap.add_argument("--rounds", type=int, default=7)
ap.add_argument("--out", default="")
args = ap.parse_args()

flush = torch.empty(512 << 18, device="cuda")
res = {}
for name in args.configs.split(","):
    cfg = datagen.CONFIGS[name]
    V, src, dst = datagen.make_graph(cfg)
    variants = {"edge_scales": dict(edge_scales=True), "gathered_scales": dict(edge_scales=False),
                "lean_no_edge_ids": dict(edge_scales=False, edge_ids=False)}
    graphs = {k: gsp.Graph(V, src, dst, device=0, **kw) for k, kw in variants.items()}
    X = torch.from_numpy(datagen.uniform(1, V, cfg.F)).cuda()
    out = torch.empty((V, cfg.F), device="cuda")
    ref = {}
    t = {k: {"fwd": [], "rev": []} for k in variants}
    for r in range(args.rounds + 1):
        for k, G in graphs.items():
            for d in ("fwd", "rev"):
                flush.fill_(1.0)
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record()
                G.gspmm(X, gsp.NORM_BOTH, out=out, reverse=(d == "rev"))
                a1.record()
                torch.cuda.synchronize()
                if r > 0:
                    t[k][d].append(a0.elapsed_time(a1))
                if r == 0:
                    if d not in ref:
                        ref[d] = out.clone()
                    else:   # identical results up to summation rounding
                        assert float((out - ref[d]).abs().max()) <= 1e-5 * float(ref[d].abs().max() + 1)
    res[name] = {k: {"ms_fwd": round(float(np.median(v["fwd"])), 4), "ms_rev": round(float(np.median(v["rev"])), 4),
                     "device_bytes": graphs[k].device_bytes, "by_kind": graphs[k].memory()}
                 for k, v in t.items()}
    res[name]["E"] = int(graphs["edge_scales"].E)
    res[name]["paper_accounting_bytes_|V|+|E|_words"] = 8 * (V + 1) + 4 * int(graphs["edge_scales"].E)
    del graphs, X, out
    torch.cuda.empty_cache()
print(json.dumps(res, indent=1))
if args.out:
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
