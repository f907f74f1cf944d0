"""The reference-side binding shown in INTEGRATION.md (integration/
run_worker_gpu.cpp) compiles against the reference's own headers and links
against the product library and the reference core with no undefined
symbols (needs /root/reference; CPU only, nothing runs)."""
import glob
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_INC = "/root/reference/proj/core/include"


@pytest.mark.skipif(not os.path.isdir(REF_INC), reason="reference headers not present")
def test_integration_snippet_compiles_and_links(tmp_path):
    src = os.path.join(ROOT, "integration", "run_worker_gpu.cpp")
    obj = tmp_path / "rw.o"
    subprocess.run(["g++", "-std=c++20", "-O1", "-fPIC", "-Wall", "-Wextra", "-Werror",
                    f"-I{REF_INC}", f"-I{os.path.join(ROOT, 'include')}", "-c", src, "-o", str(obj)],
                   check=True)
    core = sorted(glob.glob(os.path.join(ROOT, "oracle", "_ref", "obj", "core_*.o")))
    shim = os.path.join(ROOT, "oracle", "_ref", "obj", "fftw_shim.o")
    if not core or not os.path.exists(shim):
        pytest.skip("oracle/_ref objects not built (make -C oracle)")
    pkg = os.path.join(ROOT, "paper_1607_00850_b200")
    subprocess.run(["g++", "-shared", "-pthread", "-Wl,--no-undefined", "-o", str(tmp_path / "rw.so"),
                    str(obj)] + core + [shim, f"-L{pkg}", "-l:libsdns_cuda.so"], check=True)
    assert (tmp_path / "rw.so").exists()
