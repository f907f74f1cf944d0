"""Aggregate ncu warp-stall samples per CUDA source line (needs -lineinfo)."""
import csv, subprocess, sys, collections
rep, kern = sys.argv[1], sys.argv[2]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}",
                      "--print-source=cuda,sass"], capture_output=True, text=True).stdout
agg = collections.Counter(); src = {}
fname = None; line = None
for r in csv.reader(out.splitlines()):
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] in ("Function Name", "Line No"): continue
    if r[0] and r[0].isdigit():
        line = (fname, int(r[0])); src[line] = r[1].strip()[:90]
        if len(r) > 4 and r[4].isdigit(): agg[line] += int(r[4])
        continue
    if len(r) > 4 and r[4].isdigit() and line: agg[line] += int(r[4])
tot = sum(agg.values()) or 1
for k, v in agg.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 25):
    print(f"{v:8d} {100*v/tot:5.1f}% {k[0]}:{k[1]:<4d} {src.get(k,'')}")
