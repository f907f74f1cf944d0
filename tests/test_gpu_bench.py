"""GPU: bench.py's JSON line keeps the driver's contract at a small size
(one rank): metric/value/unit, the device-timed steps, roofline with its
bound and peak source, step roofline, e2e through the host-buffer API with
its byte counts, clocks sampled during the timed region, and the number of
the library's own kernel launches."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_line_contract():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--size", "64", "--steps", "2",
                          "--warmup", "3", "--no-cpu-baseline", "--no-other-configs"],
                         capture_output=True, text=True, timeout=600, check=True)
    line = json.loads([x for x in out.stdout.splitlines() if x.startswith("{")][-1])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "step_roofline", "e2e", "clocks", "gpu_launches"):
        assert k in line, k
    assert line["n_gpus"] == 1 and line["steps"] == 2 and line["warmup"] == 3
    assert line["value"] > 0 and abs(line["value"] - 1e3 / line["ms_per_step"]) < 1e-6 * line["value"]
    assert line["roofline"]["bound"] in ("hbm", "nvlink")
    assert 0 < line["roofline"]["frac"] and line["roofline"]["peak"] > 0
    assert line["step_roofline"]["bound"] == "hbm" and line["step_roofline"]["a2a_bytes_per_step"] == 0
    e = line["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] == e["d2h_bytes_per_step"] > 0
    assert line["gpu_launches"] >= 2 * 24  # ~24 of our kernels per RK4 step
    assert line["config"]["n"] == 64 and line["check"]["finite"]
