"""Line-reuse model of the edge-ID indirected weighted reverse (A8, gSpMMve^T via
rev_eid) on the Reddit-shaped graph: replays the alpha-row reads of
a rev-row schedule through an LRU cache of 128-B lines (4 alpha rows of H = 8)
and reports the DRAM bytes an ideal LRU L2 of the given capacity would fetch.

Model: W rows in flight (the warps resident on the GPU); each slot walks its row
one edge per tick and pulls the next row of the schedule when it finishes
(tools/lru_sim.c, simulate2).  Used in DESIGN.md §6 to compare schedules and to
show how far the measured DRAM traffic is from an LRU cache.

usage: python tools/lru_sim.py [--caps 30,60,100] [--W 2368]"""
import argparse
import ctypes
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import datagen  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--caps", default="30,60,100")
ap.add_argument("--W", type=int, default=2368)
args = ap.parse_args()

so = "/tmp/gsp_lru_sim.so"
subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", os.path.join(ROOT, "tools", "lru_sim.c"), "-o", so])
lib = ctypes.CDLL(so)
lib.simulate2.restype = ctypes.c_int64

cfg = datagen.CONFIGS["reddit"]
V, src, dst = datagen.make_graph(cfg)
E = len(src)
# fwd slots: rows = dst sorted by (dst, src, input position); rev: rows = src sorted by (src, dst, eid)
order_f = np.lexsort((np.arange(E), src, dst))
eid_of = np.empty(E, np.int64)
eid_of[order_f] = np.arange(E)
rev_eid = np.ascontiguousarray(eid_of[np.lexsort((eid_of, dst, src))].astype(np.int32))
deg = np.bincount(src, minlength=V)
rev_off = np.zeros(V + 1, np.int64)
rev_off[1:] = np.cumsum(deg)

lpt = np.lexsort((np.arange(V), -deg))
nh = int((deg > 2048).sum())


def win_order(win):   # the library's task_id schedule: heavy rows (LPT), then id windows by degree
    light = lpt[nh:]
    return np.concatenate([lpt[:nh], light[np.lexsort((light, -deg[light], light // win))]])


schedules = {"LPT (degree order)": lpt, "id windows of 2048 (library)": win_order(2048),
             "id windows of 512": win_order(512), "pure id order": np.arange(V)}
for cap in [int(c) for c in args.caps.split(",")]:
    for name, order in schedules.items():
        order = np.ascontiguousarray(order, np.int32)
        m = lib.simulate2(ctypes.c_int64(V), order.ctypes.data_as(ctypes.c_void_p),
                          rev_off.ctypes.data_as(ctypes.c_void_p), rev_eid.ctypes.data_as(ctypes.c_void_p),
                          ctypes.c_int64(args.W), ctypes.c_int64(cap * 8192), ctypes.c_int(4))
        print(f"cap {cap:4d} MB  {name:30s} alpha lines fetched {m / 1e6:7.2f} M = {m * 128 / 1e9:5.2f} GB "
              f"({m * 128 / (E * 32):.2f} x the alpha array)", flush=True)
