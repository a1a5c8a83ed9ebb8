"""Print registers / spills per kernel from `nvcc -Xptxas=-v` output (stdin)."""
import re, subprocess, sys
name = regs = None
rows = []
for l in sys.stdin.read().split("\n"):
    m = re.search(r"entry function '(\S+)'", l)
    if m:
        name = m.group(1); continue
    m = re.search(r"(\d+) bytes spill stores", l)
    if m and name:
        sp = int(m.group(1))
    m = re.search(r"Used (\d+) registers", l)
    if m and name:
        dn = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        rows.append((sp, int(m.group(1)), dn[:120]))
        name = None
for r in sorted(rows, reverse=True)[: int(sys.argv[1]) if len(sys.argv) > 1 else 15]:
    print(*r)
