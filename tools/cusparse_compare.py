"""Library context for the paper's relative claims (GraphPy vs
cuSPARSE on A100): the same Reddit-shaped ops through torch's cuSPARSE bindings
on this B200, timed like the bench (CUDA events, L2 flushed, median), beside
libgsp.  Context only -- the paper's comparison systems are out of scope.
usage: python tools/cusparse_compare.py [--config reddit] [--reps 7]"""
import argparse, json, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2402_03548_b200 as gsp

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="reddit")
ap.add_argument("--reps", type=int, default=7)
args = ap.parse_args()
cfg = datagen.CONFIGS[args.config]
V, src, dst = datagen.make_graph(cfg)
G = gsp.Graph(V, src, dst, device=0)
E = G.E
ex = G.export(rev=False, coo=False)
crow = torch.from_numpy(ex["fwd_off"]).cuda()
colt = torch.from_numpy(ex["fwd_col"].astype(np.int64)).cuda()
flush = torch.empty(512 << 18, device="cuda")


def t(fn):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(args.reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return round(float(np.median(ts)), 4)


def check(a, b):
    return float((a - b).abs().max() / (b.abs().max() + 1e-30))


res = {"config": args.config, "V": V, "E": E, "torch": torch.__version__}
ones = torch.ones(E, device="cuda")
A1 = torch.sparse_csr_tensor(crow, colt, ones, (V, V))
for F in (64, 32):
    X = torch.rand((V, F), device="cuda") - 0.5
    out = torch.empty((V, F), device="cuda")
    ref = torch.sparse.mm(A1, X)
    G.gspmm(X, gsp.NORM_NONE, out=out)
    res[f"spmm_F{F}"] = {"gsp_ms": t(lambda: G.gspmm(X, gsp.NORM_NONE, out=out)),
                         "cusparse_ms": t(lambda: torch.sparse.mm(A1, X)), "max_rel_diff": check(out, ref)}
# weighted, one head, F = 32 (the paper's exp-gpu-gspmmve shape): forward and reverse (A^T)
w = torch.rand((E, 1), device="cuda")
Aw = torch.sparse_csr_tensor(crow, colt, w[:, 0].contiguous(), (V, V))
X = torch.rand((V, 32), device="cuda") - 0.5
out = torch.empty((V, 32), device="cuda")
ref = torch.sparse.mm(Aw, X)
G.gspmm_weighted(X, w, out=out)
res["weighted_fwd_F32_H1"] = {"gsp_ms": t(lambda: G.gspmm_weighted(X, w, out=out)),
                              "cusparse_ms": t(lambda: torch.sparse.mm(Aw, X)), "max_rel_diff": check(out, ref)}
AwT = Aw.t()   # transposed operand: cuSPARSE op(A) = A^T (no explicit csr2csc here)
try:
    refT = torch.sparse.mm(AwT, X)
    G.gspmm_weighted(X, w, out=out, reverse=True)
    res["weighted_rev_F32_H1"] = {"gsp_ms": t(lambda: G.gspmm_weighted(X, w, out=out, reverse=True)),
                                  "cusparse_ms": t(lambda: torch.sparse.mm(AwT, X)), "max_rel_diff": check(out, refT)}
except Exception as e:   # noqa: BLE001
    res["weighted_rev_F32_H1"] = {"error": repr(e)[:200]}
# gSDDMM, one head, F = 32 (exp-sddmm shape): cuSPARSE SDDMM via sampled_addmm
Y = torch.rand((V, 32), device="cuda") - 0.5
s = torch.empty((E, 1), device="cuda")
try:
    S = torch.sparse.sampled_addmm(A1, X, Y.t().contiguous(), beta=0.0, alpha=1.0)
    G.gsddmm(X, Y, out=s)
    res["sddmm_F32_H1"] = {"gsp_ms": t(lambda: G.gsddmm(X, Y, out=s)),
                           "cusparse_ms": t(lambda: torch.sparse.sampled_addmm(A1, X, Y.t().contiguous(), beta=0.0,
                                                                               alpha=1.0)),
                           "max_rel_diff": check(s[:, 0], S.values())}
except Exception as e:   # noqa: BLE001
    res["sddmm_F32_H1"] = {"error": repr(e)[:200]}
for k, v in res.items():
    if isinstance(v, dict) and "gsp_ms" in v:
        v["speedup"] = round(v["cusparse_ms"] / v["gsp_ms"], 2)
print(json.dumps(res))
