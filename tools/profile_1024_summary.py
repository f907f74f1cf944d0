"""Summary of the n = 1024 ncu capture (tools/profile_1024.sh) into
profiles/r2_ncu_full_1024.md:  python tools/profile_1024_summary.py [report]"""
import csv
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
rep = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "full1024.ncu-rep")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
cols = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "ms"),
        ("dram__bytes_read.sum", "DRAM read GB"), ("dram__bytes_write.sum", "DRAM write GB"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("launch__registers_per_thread", "regs"), ("launch__block_size", "block"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
        ("l1tex__throughput.avg.pct_of_peak_sustained_active", "L1/shared %"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
        ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_sb"),
        ("smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio", "stall mio"),
        ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_sb"),
        ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier")]
L = []
L.append("# r2: ncu --set full, n = 1024 one-GPU RK4 step (slab p = 1, ~155 GB), one launch per kernel, "
         "--clock-control none\n")
L.append("Command: `tools/profile_1024.sh` (bench.py --size 1024 --steps 1 --warmup 1 under ncu); this "
         "summary: `tools/profile_1024_summary.py`. Work fields in the in-place chunk-major layout "
         "[kz chunk][x][y][8] (DESIGN.md §3). Stall columns are warps stalled per issue-active cycle.\n")
L.append("| " + " | ".join(c[1] for c in cols) + " |")
L.append("|" + "---|" * len(cols))
seen = set()
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")].replace("(int)", "").replace("void ", "").split("(")[0]
    if name in seen:
        continue
    seen.add(name)
    vals = []
    for c, _ in cols:
        v = r[hdr.index(c)]
        if c == "Kernel Name":
            v = "`" + name + "`"
        else:
            try:
                f = float(v)
                v = ("%.3f" % f) if f < 1000 else ("%d" % f)
            except ValueError:
                pass
        vals.append(v)
    L.append("| " + " | ".join(vals) + " |")
lines = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "ncu_lines.py"), rep, "k_pipe_xinv1", "8"],
                       capture_output=True, text=True).stdout.strip()
L.append("\nPer source line, `k_pipe_xinv1<1024, 9, 1>` (P1; warp-stall samples, `tools/ncu_lines.py`):\n")
L.append("```\n" + lines + "\n```\n")
notes = os.path.join(ROOT, "profiles", "r2_ncu_full_1024.notes.md")
if os.path.exists(notes):
    L.append(open(notes).read())
open(os.path.join(ROOT, "profiles", "r2_ncu_full_1024.md"), "w").write("\n".join(L))
print("\n".join(L[:12]))
