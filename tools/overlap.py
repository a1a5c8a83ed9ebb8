"""How much do independent ops of the step overlap on two streams?"""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import datagen, paper_2402_03548_b200 as gsp
cfg = datagen.CONFIGS["reddit"]
V, src, dst = datagen.make_graph(cfg)
G = gsp.Graph(V, src, dst, device=0)
E, F, H = G.E, 64, 8
mk = lambda k: torch.from_numpy(datagen.uniform(k, V, F)).cuda()
X, dY, Z, dO = mk(1), mk(2), mk(3), mk(4)
o = [torch.empty((V, F), device="cuda") for _ in range(4)]
s = torch.empty((E, H), device="cuda")
flush = torch.empty(512 << 18, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
def serial():
    G.gspmm(X, 2, out=o[0], stream=sa); G.gspmm(dY, 2, out=o[1], reverse=True, stream=sa)
    G.gsddmm(Z, Z, out=s, stream=sa); G.edge_softmax(s, out=s, stream=sa)
    G.gspmm_weighted(Z, s, out=o[2], stream=sa); G.gspmm_weighted(dO, s, out=o[3], reverse=True, stream=sa)
def overlapped():
    ev = torch.cuda.Event(); ev.record(sa); sb.wait_event(ev)
    G.gsddmm(Z, Z, out=s, stream=sb); G.edge_softmax(s, out=s, stream=sb)
    G.gspmm_weighted(Z, s, out=o[2], stream=sb); G.gspmm_weighted(dO, s, out=o[3], reverse=True, stream=sb)
    G.gspmm(X, 2, out=o[0], stream=sa); G.gspmm(dY, 2, out=o[1], reverse=True, stream=sa)
    e2 = torch.cuda.Event(); e2.record(sb); sa.wait_event(e2)
for name, fn in [("serial", serial), ("overlapped", overlapped)]:
    ts = []
    for r in range(8):
        with torch.cuda.stream(sa):
            flush.fill_(1.0)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(sa); fn(); b.record(sa); torch.cuda.synchronize()
        if r >= 2: ts.append(a.elapsed_time(b))
    print(name, round(float(np.median(ts)), 3))
