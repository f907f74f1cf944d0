"""Summarise ncu captures into profiles/ (tracked).

  python tools/profile_summary.py <round-tag> <n> <launches.csv> <full.ncu-rep> [more.ncu-rep ...]

Writes profiles/<tag>_launches_<n>.md (per-kernel share of the launch list),
profiles/<tag>_ncu_full_<n>.md (per-kernel counters of the full capture) and
merges per-launch DRAM traffic into profiles/ncu_traffic.json, which bench.py
reports as roofline.traffic.
"""
import collections
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PASS_OF = [("k_pipe_xinv", "x_inv_curl"), ("k_pipe_yinv", "y_inv"), ("k_z_fused", "z_fused"),
           ("k_rk_update<1>", "x_fwd_rk0"), ("k_rk_update<2>", "x_fwd_rk12"),
           ("k_rk_update<3>", "x_fwd_rk3"), ("k_rk_update<0>", "x_fwd_tail")]


def short(name):
    name = name.replace("(int)", "").replace("void ", "").replace("sdns_dev::", "")
    return name.split("(")[0]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    tot = collections.defaultdict(float)
    cnt = collections.Counter()
    for r in rows:
        if r[-3] != "gpu__time_duration.sum":
            continue
        k = short(r[4])
        v = float(r[-1])
        unit = r[-2]
        ns = v * {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(unit, 1)
        tot[k] += ns
        cnt[k] += 1
    return tot, cnt


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "launch__shared_mem_per_block_dynamic", "launch__block_size",
            "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
            "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]
    units = rows[1]
    res = []
    for r in rows[2:]:
        d = {}
        for w in want:
            if w in h:
                i = h.index(w)
                d[w] = (r[i], units[i])
        res.append(d)
    return res


def to_bytes(v, unit):
    return float(v) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def main():
    tag, n, lpath, fpaths = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4:]
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    tot, cnt = launches(lpath)
    allns = sum(tot.values())
    lines = [f"# {tag}: ncu launch list, n = {n} (`ncu --metrics gpu__time_duration.sum "
             f"--clock-control none`, bench.py --steps 2 --warmup 3)", "",
             "Cold-cache, serialised per-launch times: compare shares, not absolutes.", "",
             "| kernel | launches | total ms | share |", "|---|---|---|---|"]
    for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
        lines.append(f"| `{k}` | {cnt[k]} | {v / 1e6:.3f} | {100 * v / allns:.1f}% |")
    open(os.path.join(ROOT, "profiles", f"{tag}_launches_{n}.md"), "w").write("\n".join(lines) + "\n")

    res = [d for fp in fpaths for d in full(fp)]
    lines = [f"# {tag}: ncu --set full, n = {n} (one launch per kernel, --clock-control none)", "",
             "| kernel | ms | DRAM read GB | DRAM write GB | DRAM % | warps active % | regs | smem KB |"
             " block | fp64 pipe % | issue % | smem bank conflicts | smem wavefronts |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    traffic_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    traffic = json.load(open(traffic_path)) if os.path.exists(traffic_path) else {}
    tr = traffic.setdefault(str(n), {})
    acc = {}  # pass -> [bytes per launch, ...]
    plain_order = ["y_fwd", "x_fwd_fft"]  # the step's k_pipe_plain launches, in capture order
    for d in res:
        name = d["Kernel Name"][0]
        rd = to_bytes(*d["dram__bytes_read.sum"])
        wr = to_bytes(*d["dram__bytes_write.sum"])
        g = lambda k: d.get(k, ("", ""))[0]  # noqa: E731
        lines.append(f"| `{short(name)}` | {float(g('gpu__time_duration.sum')):.3f} | {rd / 1e9:.3f} | "
                     f"{wr / 1e9:.3f} | {float(g('gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed')):.1f} | "
                     f"{float(g('sm__warps_active.avg.pct_of_peak_sustained_active')):.1f} | "
                     f"{g('launch__registers_per_thread')} | {g('launch__shared_mem_per_block_dynamic')} | "
                     f"{g('launch__block_size')} | "
                     f"{float(g('sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active')):.1f} | "
                     f"{float(g('smsp__issue_active.avg.pct_of_peak_sustained_active')):.1f} | "
                     f"{g('l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum')} | "
                     f"{g('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum')} |")
        for key, pname in PASS_OF:
            if key in name.replace("(int)", ""):
                acc.setdefault(pname, []).append(rd + wr)
        if "k_pipe_plain" in name and plain_order:
            acc.setdefault(plain_order.pop(0), []).append(rd + wr)
    for pname, v in acc.items():
        tr[pname] = sum(v) / len(v)
    open(os.path.join(ROOT, "profiles", f"{tag}_ncu_full_{n}.md"), "w").write("\n".join(lines) + "\n")
    json.dump(traffic, open(traffic_path, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
