"""Per-op DRAM traffic from ncu --set full summaries (tools/ncu_summary.py
output) of bench.py steps -> profiles/ncu_traffic.json, read by bench.py for
the roofline "traffic" key and per_op "traffic_GB".

usage: python tools/ncu_traffic.py CONFIG OUT.json SUMMARY.csv [SUMMARY.csv ...]
Kernels map to ops by name; the gspmm kernel of mode 0 (scaled) appears twice
per step, forward first.  Later files / launches override earlier ones."""
import csv
import json
import os
import re
import sys

config, out, srcs = sys.argv[1], sys.argv[2], sys.argv[3:]


def op_of(name, seen_scaled):
    if "gat_fused_kernel" in name:
        return "gat_forward"
    if "sddmm_kernel" in name:
        return "gsddmm"
    if "softmax_kernel" in name:
        return "edge_softmax"
    m = re.search(r"spmm_kernel<(\d+), (\d+), (\d+), (\d+)", name)
    if m:
        mode = int(m.group(4))
        if mode == 0:
            return "gspmm_rev" if seen_scaled % 2 else "gspmm_fwd"
        return {1: "gspmm_weighted_fwd", 2: "gspmm_weighted_rev"}.get(mode)
    return None


d = json.load(open(out)) if os.path.exists(out) else {}
cfg = d.setdefault(config, {})
for src in srcs:
    rows = list(csv.reader(open(src)))
    hdr = rows[0]
    col = {k: hdr.index(k) for k in hdr}
    n_scaled = 0
    for r in rows[2:]:
        name = r[col["Kernel Name"]]
        op = op_of(name, n_scaled)
        if op is None:
            continue
        if op in ("gspmm_fwd", "gspmm_rev"):
            n_scaled += 1
        gb = float(r[col["dram__bytes_read.sum"]]) + float(r[col["dram__bytes_write.sum"]])
        cfg[op] = {"dram_bytes": gb * 1e9, "ms": float(r[col["gpu__time_duration.sum"]]),
                   "l2_hit_pct": float(r[col["lts__t_sector_hit_rate.pct"]]),
                   "l2_read_bytes": float(r[col["l1tex__m_xbar2l1tex_read_bytes.sum"]]) * 1e9
                   if "l1tex__m_xbar2l1tex_read_bytes.sum" in col else None,
                   "kernel": name, "source": os.path.relpath(src)}
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d, indent=1))
