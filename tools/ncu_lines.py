"""Aggregate an ncu source-page column per CUDA source line (needs -lineinfo).

  python tools/ncu_lines.py <report> <kernel-regex> [top] [column]

column defaults to "# Samples" (warp-stall samples); e.g. "L1 Wavefronts Shared"
gives the shared-memory wavefronts issued by each source line.
"""
import collections
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
col = sys.argv[4] if len(sys.argv) > 4 else "# Samples"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source=cuda,sass"], capture_output=True, text=True).stdout
agg = collections.Counter()
src = {}
fname = None
line = None
ci = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No" or r[0] == "Address":
        if col in r:
            ci = r.index(col)
        continue
    if r[0] == "Function Name":
        continue
    val = r[ci] if ci is not None and len(r) > ci else ""
    if r[0].isdigit():  # a source line row
        line = (fname, int(r[0]))
        src[line] = r[1].strip()[:90]
        continue
    try:
        v = float(val)
    except ValueError:
        continue
    if line:
        agg[line] += v
tot = sum(agg.values()) or 1
for k, v in agg.most_common(top):
    print(f"{v:12.0f} {100 * v / tot:5.1f}% {k[0]}:{k[1]:<4d} {src.get(k, '')}")
print(f"total {tot:.0f}")
