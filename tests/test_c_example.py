"""examples/c_api_step.c: the step through the C ABI alone (no Python binding).  CPU: it compiles and links
against the built libattncache.so with the header as the only interface.  GPU: it runs and passes its own
checks (planted hits, a miss, cached O against full attention)."""
import os
import shutil
import subprocess
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
LIBDIR = os.path.join(ROOT, "paper_2510_25979_b200", "lib")


def _build(out):
    if not os.path.exists(os.path.join(LIBDIR, "libattncache.so")):
        pytest.skip("libattncache.so not built")
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    subprocess.run(["gcc", "-O2", "-std=c11", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I",
                    os.path.join(CUDA, "include"), os.path.join(ROOT, "examples", "c_api_step.c"), "-L", LIBDIR,
                    "-lattncache", "-L", os.path.join(CUDA, "lib64"), "-lcudart", "-lm", f"-Wl,-rpath,{LIBDIR}",
                    "-o", out], check=True)


def test_c_example_compiles_and_links():
    with tempfile.TemporaryDirectory() as d:
        _build(os.path.join(d, "c_api_step"))
        assert os.path.getsize(os.path.join(d, "c_api_step")) > 0


@pytest.mark.gpu
def test_c_example_runs():
    with tempfile.TemporaryDirectory() as d:
        exe = os.path.join(d, "c_api_step")
        _build(exe)
        r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, (r.stdout, r.stderr)
        assert ": ok" in r.stdout
