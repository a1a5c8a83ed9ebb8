import sys, numpy as np, torch
sys.path.insert(0, '.')
import datagen, oracle, paper_2402_03548_b200 as gsp
V, E = 4000, 600_000
src, dst = datagen.skewed_multigraph(V, E, 3, alpha=1.6)
G = gsp.Graph(V, src, dst, device=0); og = oracle.Graph(V, src, dst)
deg = np.diff(og.fwd_off)
print("max deg", deg.max(), "n>1024", (deg > 1024).sum())
for F in (16, 64):
    Xh = datagen.uniform(5, V, F, lo=0.0, hi=1.0)
    out = G.gspmm(torch.from_numpy(Xh).cuda(), 0).cpu().numpy().astype(np.float64)
    ref, T = og.gspmm(Xh, 0, False)
    r = np.abs(out - ref) / (1e-5 * (T + 1))
    worst = np.argsort(-r.max(1))[:8]
    for v in worst:
        f = int(np.argmax(r[v]))
        print(F, "row", v, "deg", deg[v], "ratio", r[v, f], "err", out[v, f] - ref[v, f], "T", T[v, f])
    # f64 sum emulating fp32 sequential accumulation for the worst row
    v = worst[0]
    cols = og.fwd_col[og.fwd_off[v]:og.fwd_off[v+1]]
    xs = Xh[cols, 0]
    acc = np.float32(0)
    for x in xs: acc = np.float32(acc + x)
    print("seq fp32 err", float(acc) - xs.astype(np.float64).sum())
