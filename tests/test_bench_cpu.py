"""CPU checks of bench.py's reporting: the step roofline formula reproduces
BASELINE.md §3's table, the per-pass NVLink split, and the
reference arm's JSON line at a small size (it runs without a GPU)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402

# BASELINE.md §3, spec peaks 8.0 TB/s HBM, 900 GB/s NVLink per direction
TABLE = [
    ((512, "slab", 1, 1, 1), 28.70, "hbm"),
    ((512, "slab", 8, 1, 8), 4.72, "nvlink"),
    ((1024, "pencil", 8, 2, 4), 53.79, "nvlink"),
    ((1024, "slab", 8, 1, 8), 37.65, "nvlink"),
    ((256, "slab", 1, 1, 1), 3.60, "hbm"),
]


@pytest.mark.parametrize("geom,ms,bound", TABLE)
def test_step_roofline_reproduces_baseline_table(geom, ms, bound):
    r = bench.step_roofline(*geom, 8000.0, 900.0)
    assert round(r["roofline_ms"], 2) == ms
    assert r["bound"] == bound


def test_survey_8d_rows():
    # 512^3 slab p2 / p4 t_HBM and t_NVL columns
    r2 = bench.step_roofline(512, "slab", 2, 1, 2, 8000.0, 900.0)
    r4 = bench.step_roofline(512, "slab", 4, 1, 4, 8000.0, 900.0)
    assert round(r2["t_hbm_ms"], 2) == 14.35 and round(r2["t_nvlink_ms"], 2) == 10.78
    assert abs(r4["t_nvlink_ms"] - 8.09) <= 0.01 and r4["bound"] == "nvlink"
    assert round(r2["a2a_bytes_per_step"] / 1e9, 2) == 9.70


def test_pass_nvlink_split_sums_to_transposed_fields():
    # slab: 5 inverse + 3 forward fields per RHS leave the GPU with f=(p-1)/p
    s = sum(bench.pass_a2a_c(k, "slab", 8, 1, 8) for k in bench.PASS_BYTES_C)
    assert abs(s - 8 * 7 / 8) < 1e-12
    assert bench.pass_a2a_c("z_fused", "slab", 8, 1, 8) == 0.0
    assert bench.pass_a2a_c("x_inv_curl", "slab", 1, 1, 1) == 0.0
    pen = {k: bench.pass_a2a_c(k, "pencil", 8, 2, 4) for k in bench.PASS_BYTES_C}
    assert pen["z_fused"] == 3 * 0.75 and pen["x_inv_curl"] == 5 * 0.5


def test_resolve_workloads():
    class A:
        n, decomp, p1, p2 = 1024, "pencil", 0, 0
    c = bench.resolve(A, 8)
    assert (c["p1"], c["p2"]) == (2, 4) and c["workload"].startswith("configs[3]")
    A.decomp = "slab"
    assert "slab 1x8" in bench.resolve(A, 8)["workload"]
    A.n, A.decomp = 512, None
    c = bench.resolve(A, 1)
    assert c["workload"].startswith("configs[2]") and c["nu"] == 5e-4


def test_reference_arm_line_small(ref):
    """The reference arm runs the compiled reference (whole rk4_step + project
    steps on the iso field) and reports exactly the steps it timed."""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--n", "16", "--steps", "3", "--warmup", "1"],
                         capture_output=True, text=True, timeout=300, check=True)
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["steps"] == 3 and line["warmup"] == 1
    assert line["value"] > 0 and line["e2e"]["value"] == line["value"]
    assert line["cpu_baseline"]["kind"] == "reference" and "whole RK4 steps" in line["cpu_baseline"]["sample"]
    assert line["config"]["n"] == 16 and line["config"]["seed"] == 1607
    assert line["cpu_p1"]["cores"] == 1
