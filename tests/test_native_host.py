"""Host-only native checks (no GPU): tests/native/*.cu are compiled with nvcc for sm_100a and their host
main() run.  item_sched_check.cu covers the persistent kernels' work-item order (item_sched.cuh) and the
host-made division magics (FastDiv) it decodes with."""
import os
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.mark.skipif(not (os.path.exists(NVCC) or shutil.which("nvcc")), reason="nvcc not available")
def test_item_sched_and_fastdiv():
    with tempfile.TemporaryDirectory() as tmp:
        exe = os.path.join(tmp, "item_sched_check")
        subprocess.run([NVCC if os.path.exists(NVCC) else "nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O2",
                        "-std=c++17", "-I", os.path.join(ROOT, "paper_2510_25979_b200", "csrc"), "-I",
                        os.path.join(ROOT, "include"), "-o", exe, os.path.join(ROOT, "tests", "native", "item_sched_check.cu")],
                       check=True, capture_output=True, timeout=300)
        r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
        assert r.returncode == 0 and "item_sched_check ok" in r.stdout, r.stdout + r.stderr
