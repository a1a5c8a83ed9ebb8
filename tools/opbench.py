"""Per-op timing on a BASELINE config (CUDA events, L2 flushed between reps).
usage: python tools/opbench.py [--config reddit] [--reps 10] [--ops gspmm_fwd,...] [--F 64]"""
import argparse, json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2402_03548_b200 as gsp

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="reddit")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--ops", default="gspmm_fwd,gspmm_rev,gsddmm,edge_softmax,wfwd,wrev,gat_fused,softmax_bwd")
ap.add_argument("--F", type=int, default=0)
ap.add_argument("--ld", type=int, default=0)
ap.add_argument("--tag", default=os.environ.get("GSP_TUNE_SPMM", ""))
args = ap.parse_args()
cfg = datagen.CONFIGS[args.config]
if os.environ.get("GSP_PERSIST_MB"):   # experiment: L2 set-aside for persisting (evict_last) lines
    import ctypes
    torch.cuda.init(); torch.empty(1, device="cuda")
    rt = ctypes.CDLL(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib", "libcudart.so.12"))
    mb = int(os.environ["GSP_PERSIST_MB"])
    st = rt.cudaDeviceSetLimit(6, ctypes.c_size_t(mb << 20))
    got = ctypes.c_size_t(0); rt.cudaDeviceGetLimit(ctypes.byref(got), 6)
    print("persist limit", st, got.value >> 20, "MB", file=sys.stderr)
V, src, dst = datagen.make_graph(cfg)
G = gsp.Graph(V, src, dst, device=0)
E = G.E
F = args.F or cfg.F
ld = args.ld or max(F, cfg.ld if not args.F else F)
H = cfg.H or 8
Fg = H * int(os.environ.get("GSP_OPBENCH_FH", 0) or cfg.Fh or 8)   # env: other head widths (experiments)
X = torch.from_numpy(datagen.uniform(1, V, F, ld=ld)).cuda()[:, :F]
Z = torch.from_numpy(datagen.uniform(2, V, Fg)).cuda()
out = torch.empty((V, F), device="cuda")
outg = torch.empty((V, Fg), device="cuda")
s = torch.empty((E, H), device="cuda")
s2 = torch.rand((E, H), device="cuda")
outh = torch.empty((V, H), device="cuda")
flush = torch.empty(512 << 18, device="cuda")
el = Z[:, :H].contiguous()
er = Z[:, H:2 * H].contiguous()
ops = {
    "gspmm_fwd": lambda: G.gspmm(X, 2, out=out),
    "gspmm_rev": lambda: G.gspmm(X, 2, out=out, reverse=True),
    "gspmm_none": lambda: G.gspmm(X, 0, out=out),
    "gspmm_right": lambda: G.gspmm(X, 1, out=out),
    "gspmm_max": lambda: G.gspmm_reduce(X, 2, out=out),
    "gsddmm": lambda: G.gsddmm(Z, Z, out=s),
    "edge_softmax": lambda: G.edge_softmax(s, out=s),
    "wfwd": lambda: G.gspmm_weighted(Z, s, out=outg),
    "wrev": lambda: G.gspmm_weighted(Z, s, out=outg, reverse=True),
    "gat_fused": lambda: G.gat_forward(Z, Z, Z, H, alpha=s, out=outg),
    "gat_add": lambda: G.gat_forward_additive(el, er, Z, 0.2, alpha=s, out=outg),
    "add_leaky": lambda: G.gsddmm_add_leaky(el, er, 0.2, out=s),
    "gat_bwd": lambda: G.gat_backward_scores(Z, Z, s, out=s2),
    "softmax_bwd": lambda: G.edge_softmax_backward(s, s2, out=s2),
    "e_sum": lambda: G.gspmm_e(s, 0, out=outh),
    "e_sum_rev": lambda: G.gspmm_e(s, 0, out=outh, reverse=True),
    "ve_src": lambda: G.gsddmm_ve(Z[:, :H], s2, 0, 1, out=s),
    "ve_dst": lambda: G.gsddmm_ve(Z[:, :H], s2, 0, 0, out=s),
}
G.gsddmm(Z, Z, out=s); G.edge_softmax(s, out=s)
res = {}
for name in args.ops.split(","):
    f = ops[name]
    for _ in range(3):
        f()
    ts = []
    for _ in range(args.reps):
        flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    res[name] = round(float(np.median(ts)), 4)
print(json.dumps({"tag": args.tag, "config": args.config, "F": F, "ms": res}))
