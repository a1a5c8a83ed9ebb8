"""NEXT-4 demo: billion-edge Kron-25 GCN aggregation on one B200 (P:2152, P:2272:
the paper fits it in 29.8 GB on an A100-40GB).  Prints one JSON line: build
time, device bytes, gspmm fwd (BOTH, F=150) time and throughput."""
import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2402_03548_b200 as gsp

# --lean: the GCN-lean device format (GSP_BUILD_NO_EDGE_IDS, no per-edge scales):
# the paper's (|V|+|E|) words of topology + O(V) arrays
lean = "--lean" in sys.argv
cfg = datagen.CONFIGS["kron25"]
t0 = time.time(); V, src, dst = datagen.make_graph(cfg); t_gen = time.time() - t0
t0 = time.time()
G = gsp.Graph(V, src, dst, device=0, **(dict(edge_ids=False, edge_scales=False) if lean else {}))
t_build = time.time() - t0
del src, dst
X = torch.from_numpy(datagen.uniform(1, V, cfg.F, ld=cfg.ld)).cuda()[:, :cfg.F]
out = torch.empty((V, cfg.F), device="cuda")
for _ in range(2):
    G.gspmm(X, gsp.NORM_BOTH, out=out)
torch.cuda.synchronize()
ts = []
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); G.gspmm(X, gsp.NORM_BOTH, out=out); b.record(); torch.cuda.synchronize()
    ts.append(a.elapsed_time(b))
ms = float(np.median(ts))
E, F = G.E, cfg.F
alg = 8 * (V + 1) + 4 * E + 4 * E * F + 4 * V * F + 8 * V
print(json.dumps({"workload": "kron25 GCN gSpMM fwd BOTH", "format": "GCN-lean (no edge ids / edge scales)" if lean
                  else "default (rev_eid + per-edge scales)", "V": V, "E": E, "F": F, "gen_s": round(t_gen, 1),
                  "build_s": round(t_build, 1), "device_graph_GB": round(G.device_bytes / 1e9, 2),
                  "device_graph_bytes_by_kind": G.memory(),
                  "paper_accounting_GB": round((8 * (V + 1) + 4 * G.E) / 1e9, 2),
                  "features_GB": round(2 * V * cfg.ld * 4 / 1e9, 2),
                  "peak_device_GB": round(torch.cuda.max_memory_allocated() / 1e9 + G.device_bytes / 1e9, 2),
                  "gspmm_ms": round(ms, 3), "GE_s": round(E / ms / 1e6, 2), "alg_GB_s": round(alg / ms / 1e6, 1)}))
