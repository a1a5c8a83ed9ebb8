import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import datagen, oracle, paper_2402_03548_b200 as gsp
for (V, E, seed) in [(4, 8, 0), (50, 300, 1), (300, 5000, 2)]:
    src, dst = datagen.random_multigraph(V, E, seed)
    G = gsp.Graph(V, src, dst, device=0); og = oracle.Graph(V, src, dst)
    H = 8
    Z = datagen.uniform(seed + 1, V, 64)
    a_ref, o_ref, T = og.gat_forward(Z, Z, Z, H)
    alpha, out = G.gat_forward(torch.from_numpy(Z).cuda(), torch.from_numpy(Z).cuda(), torch.from_numpy(Z).cuda(), H)
    a = alpha.cpu().numpy(); o = out.cpu().numpy()
    bad = np.argwhere(np.abs(a - a_ref) > 1e-4)
    print("V", V, "E", og.E, "bad alpha", len(bad), "of", a.size, "out err", float(np.abs(o - o_ref).max()))
    rows = np.repeat(np.arange(V), np.diff(og.fwd_off))
    for j, h in bad[:12]:
        r = rows[j]
        print("  edge", j, "head", h, "row", r, "slot", j - og.fwd_off[r], "deg", og.fwd_off[r+1]-og.fwd_off[r], "gpu", a[j, h], "ref", a_ref[j, h])
