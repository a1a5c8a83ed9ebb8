"""Same-box A/B of library builds / env knobs: runs tools/opbench.py once per
variant per round, alternating variants (A B C A B C ...), and reports the
median over rounds per op.  A variant is NAME=LIB[;ENV=V;ENV=V] where LIB is a
path to a libgsp build (empty: the in-tree libgsp.so).

usage: python tools/ab.py --variants 'base=_ab/libgsp_base.so' 'new=' --ops gat_fused,wrev [--config reddit]
       [--rounds 3] [--reps 7]"""
import argparse
import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ap = argparse.ArgumentParser()
ap.add_argument("--variants", nargs="+", required=True)
ap.add_argument("--ops", required=True)
ap.add_argument("--config", default="reddit")
ap.add_argument("--rounds", type=int, default=3)
ap.add_argument("--reps", type=int, default=7)
ap.add_argument("--F", type=int, default=0)
ap.add_argument("--ld", type=int, default=0)
args = ap.parse_args()
vs = []
for v in args.variants:
    name, spec = v.split("=", 1)
    parts = spec.split(";")
    env = dict(os.environ)
    if parts[0]:
        env["GSP_LIB_OVERRIDE"] = os.path.abspath(os.path.join(ROOT, parts[0]))
    for kv in parts[1:]:
        k, val = kv.split("=", 1)
        env[k] = val
    vs.append((name, env))
res = {n: {} for n, _ in vs}
for r in range(args.rounds):
    for name, env in vs:
        out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "opbench.py"), "--config", args.config,
                              "--ops", args.ops, "--reps", str(args.reps), "--F", str(args.F), "--ld", str(args.ld)],
                             capture_output=True, text=True, env=env,
                             timeout=600)
        line = json.loads(out.stdout.strip().splitlines()[-1])
        for op, ms in line["ms"].items():
            res[name].setdefault(op, []).append(ms)
summary = {n: {op: round(float(np.median(v)), 4) for op, v in d.items()} for n, d in res.items()}
print(json.dumps({"config": args.config, "rounds": args.rounds, "median_ms": summary, "all": res}))
