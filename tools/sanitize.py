"""Run every kernel family once on small graphs (for compute-sanitizer)."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2402_03548_b200 as gsp

def run(V, src, dst, F=64, H=8):
    g = gsp.Graph(V, src, dst, device=0)
    X = torch.from_numpy(datagen.uniform(1, V, F)).cuda()
    for norm in (0, 1, 2):
        for rev in (0, 1):
            g.gspmm(X, norm, reverse=rev)
    for red in (1, 2):
        g.gspmm_reduce(X, red)
    s = g.gsddmm(X, X, H=H)
    g.edge_softmax(s, out=s)
    g.gspmm_weighted(X, s)
    g.gspmm_weighted(X, s, reverse=True)
    g.edge_softmax_backward(s, s.clone())
    a, _ = g.gat_forward(X, X, X, H)
    g.gat_backward_scores(X, X, a)
    g.gspmm_e(s, 0)
    g.gspmm_e(s, 2, reverse=True)
    g.gsddmm_ve(X[:, :H], s, 0, 1)
    for red in (0, 1, 2):                      # vector gSpMMe paths (H = 4, 8, 16; fwd + rev)
        for hh in (4, 16):
            w = torch.rand((g.E, hh), device="cuda")
            g.gspmm_e(w, red)
            g.gspmm_e(w, red, reverse=True)
        g.gspmm_e(s, red)
    for op in range(4):                        # vector gSDDMMve, both sides, in place
        for side in (0, 1):
            g.gsddmm_ve(X[:, :H], s, op, side)
            t = s.clone()
            g.gsddmm_ve(X[:, :H], t, op, side, out=t)
    wp = torch.rand((g.E, 12), device="cuda")[:, :8]   # padded rows (ld 12)
    g.gspmm_e(wp, 0)
    g.gsddmm_ve(X[:, :8], wp, 0, 1, out=wp)
    # odd shapes (generic / scalar paths)
    X3 = torch.from_numpy(datagen.uniform(2, V, 15)).cuda()
    g.gspmm(X3, 2)
    s3 = g.gsddmm(X3, X3, H=3)
    g.edge_softmax(s3)
    g.gspmm_weighted(X3, s3)
    g.gspmm_weighted(X3, s3, reverse=True)
    P = 3
    parts = [g.partition(P, p, device=0) for p in range(P)]
    R = parts[0].R
    Xp = torch.zeros((P * R, F), device="cuda")
    for pg in parts:
        pg.gspmm(Xp, 2)
        a = pg.gsddmm(Xp, Xp, H=H)
        pg.gspmm_weighted(Xp, a)
        pg.gspmm_weighted(Xp, a, reverse=True)
    # round 2: additive GAT (one-pass H = 8 and the 3-kernel fallback H = 3), chunked
    # chunk-major partitions, directed-partition reverse partials, GCN-lean graph
    el = torch.rand((V, H), device="cuda") - 0.5
    er = torch.rand((V, H), device="cuda") - 0.5
    g.gsddmm_add_leaky(el, er, 0.2)
    g.gat_forward_additive(el, er, X, 0.2)
    g.gat_forward_additive(el[:, :3].contiguous(), er[:, :3].contiguous(), X3[:, :12].contiguous(), 0.01)
    C = 3
    cparts = [g.partition(2, p, device=0, nchunks=C, chunk=c) for p in range(2) for c in range(C)]
    Xc = torch.zeros((cparts[0].ncols, F), device="cuda")
    for pg in cparts:
        pg.gspmm(Xc, 2)
        pg.gspmm(Xc, 2, reverse=True)
        pg.gat_forward(Xc, Xc, Xc, H)
    rs, rd = datagen.rmat(int(np.ceil(np.log2(V))), V, min(10 * V, 30000), 7)   # directed: reverse partials
    gd = gsp.Graph(V, rs, rd, device=0)
    for pg in [gd.partition(2, p, device=0) for p in range(2)]:
        pg.gspmm(torch.zeros((pg.ncols, F), device="cuda"), 2, reverse=True)
    gl = gsp.Graph(V, src, dst, device=0, edge_ids=False, edge_scales=False)
    gl.gspmm(X, 2)
    gl.gspmm(X, 1, reverse=True)
    torch.cuda.synchronize()

V, src, dst = datagen.make_graph("cora")
run(V, src, dst)
src, dst = datagen.skewed_multigraph(1500, 60000, 3, alpha=1.6)   # heavy (CTA-split) rows
run(1500, src, dst)
print("sanitize workload done")
