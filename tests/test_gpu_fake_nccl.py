"""The library's collective code at world 2 and 3 on ONE GPU (this pool grants one): every rank is a process on
GPU 0 and the library's NCCL calls go to tests/native/fake_nccl.cpp (ATTNCACHE_NCCL_LIB), a functional stand-in
that moves the bytes through host memory between host barriers.  tests/workers/multi_gpu_step.py then checks
the collective step (routed and owner-affinity placements, skewed ownership; search, search_all, count
exchanges, routed V / O, relocation) bitwise against the single-GPU step.  A correctness
check of collective.cu's logic only: no timing is taken here."""
import os
import socket
import subprocess
import sys
import tempfile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def fake_nccl():
    out = os.path.join(tempfile.mkdtemp(), "libfake_nccl.so")
    cuda = os.environ.get("CUDA_HOME", "/usr/local/cuda")
    subprocess.run(["g++", "-shared", "-fPIC", "-O2", "-I", os.path.join(cuda, "include"), "-o", out,
                    os.path.join(ROOT, "tests", "native", "fake_nccl.cpp"), "-L", os.path.join(cuda, "lib64"),
                    "-L", os.path.join(cuda, "lib64", "stubs"), "-lcudart", "-lcuda"], check=True)
    return out


@pytest.mark.gpu
@pytest.mark.parametrize("g", [2, 3, 4])
def test_collective_step_fake_nccl_one_gpu(fake_nccl, g):
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    env = dict(os.environ, ATTNCACHE_NCCL_LIB=fake_nccl, ATTNCACHE_TEST_SINGLE_DEVICE="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={g}",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "workers", "multi_gpu_step.py")],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert f"world {g} ok" in r.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("placement,gpus,scaling", [("affinity", 2, "weak"), ("routed", 2, "weak"),
                                                    ("affinity", 4, "strong")])
def test_bench_n2_line_fake_nccl_one_gpu(fake_nccl, placement, gpus, scaling):
    """`bench.py --gpus 2` (self-launched ranks) runs its N > 1 path end to end and prints one well-formed JSON line
    (the driver's SCALE run uses this path on a multi-GPU box); the numbers of this one-GPU run mean nothing."""
    import json
    env = dict(os.environ, ATTNCACHE_NCCL_LIB=fake_nccl, ATTNCACHE_TEST_SINGLE_DEVICE="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(gpus), "--steps", "2", "--warmup",
                        "3", "--placement", placement, "--scaling", scaling, "--no-cpu-baseline"],
                       cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    line = json.loads([s for s in r.stdout.splitlines() if s.startswith("{")][-1])
    assert line["n_gpus"] == gpus and line["value"] > 0 and line["scaling"] == scaling
    assert line["other_scaling"]["ms_per_step"] > 0 and line["gpu_launches"] > 0
    assert line["config"]["placement"] == placement
    assert line["e2e"]["value"] > 0 and line["e2e"]["h2d_bytes_per_step"] > 0 and line["e2e"]["d2h_bytes_per_step"] > 0


@pytest.mark.gpu
def test_bench_reference_arm_n2(fake_nccl):
    """`bench.py --impl reference --gpus 2`: rank 0 alone times the oracle and prints the line, the other rank exits
    0 without work (the driver launches the reference arm the same way as ours)."""
    import json
    env = dict(os.environ, ATTNCACHE_NCCL_LIB=fake_nccl, ATTNCACHE_TEST_SINGLE_DEVICE="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2", "--steps",
                        "1", "--warmup", "3"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    lines = [json.loads(s) for s in r.stdout.splitlines() if s.startswith("{")]
    assert len(lines) == 1 and lines[0]["impl"] == "reference" and lines[0]["value"] > 0


_ABORT_SCRIPT = r"""
import ctypes, os, torch
import paper_2510_25979_b200 as ac
ctx = ac.Context(0, 0, 1, ac.attncache_get_unique_id())            # collective ctx at world 1 (fake NCCL)
x = torch.randn(4, 128, device="cuda")
x = (x / x.norm(dim=1, keepdim=True)).to(torch.bfloat16)
db = ac.Database(ctx, x)
idx, score, hit = ac.attncache_search(db, x[:2], 0.5)
ctx.sync()
assert idx.tolist() == [0, 1], idx
os.environ["FAKE_NCCL_ASYNC_ERROR"] = "1"                          # the communicator reports an async error
codes = []
for call in (ctx.sync, lambda: ac.attncache_search(db, x[:2], 0.5), ctx.sync):
    try:
        call()
        codes.append(0)
    except ac.AttnCacheError as e:
        codes.append(e.status)
    os.environ["FAKE_NCCL_ASYNC_ERROR"] = "0"                      # sticky: later calls fail without a new error
fake = ctypes.CDLL(os.environ["ATTNCACHE_NCCL_LIB"])
print("codes", codes, "aborts", fake.fake_nccl_abort_count())
db.close()
ctx.close()
print("abort ok")
"""


@pytest.mark.gpu
def test_async_nccl_error_aborts_the_communicator(fake_nccl):
    """SURVEY.md §5 failure detection: an asynchronous NCCL error seen by attncache_ctx_sync aborts the
    communicator (ncclCommAbort, once) and every later collective call returns ATTNCACHE_ERR_NCCL (11) instead of
    waiting on it; the ctx and db can still be destroyed."""
    env = dict(os.environ, ATTNCACHE_NCCL_LIB=fake_nccl)
    r = subprocess.run([sys.executable, "-c", _ABORT_SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "codes [11, 11, 11] aborts 1" in r.stdout and "abort ok" in r.stdout, r.stdout


_HANG_SCRIPT = r"""
import ctypes, os, time, torch
import paper_2510_25979_b200 as ac
ctx = ac.Context(0, 0, 1, ac.attncache_get_unique_id())
x = torch.randn(4, 128, device="cuda")
x = (x / x.norm(dim=1, keepdim=True)).to(torch.bfloat16)
db = ac.Database(ctx, x)
os.environ["FAKE_NCCL_HANG_ON"] = "allgather"    # the next all-gather's stream never finishes on its own
os.environ["FAKE_NCCL_ASYNC_ERROR"] = "1"        # ... and the communicator reports an async error
t0 = time.time()
try:
    ac.attncache_search(db, x[:2], 0.5)          # its batch-size exchange waits on the host
    code = 0
except ac.AttnCacheError as e:
    code = e.status
dt = time.time() - t0
torch.cuda.synchronize()                         # the abort released the stream
fake = ctypes.CDLL(os.environ["ATTNCACHE_NCCL_LIB"])
print("hang code", code, "aborts", fake.fake_nccl_abort_count(), "returned", dt < 60)
db.close()
ctx.close()
"""


@pytest.mark.gpu
def test_collective_wait_on_a_dead_peer_returns_err_nccl(fake_nccl):
    """A collective whose stream never completes (the stand-in's all-gather leaves its stream waiting on a flag,
    as NCCL's kernels wait for a peer that died) while NCCL reports an async error: the library's host wait polls
    ncclCommGetAsyncError, aborts the communicator (which releases the stream) and returns ATTNCACHE_ERR_NCCL
    instead of waiting forever."""
    env = dict(os.environ, ATTNCACHE_NCCL_LIB=fake_nccl)
    r = subprocess.run([sys.executable, "-c", _HANG_SCRIPT], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=180)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert "hang code 11 aborts 1 returned True" in r.stdout, r.stdout
