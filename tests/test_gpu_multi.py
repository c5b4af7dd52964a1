"""the collective step on g GPUs (one process per GPU under torch.distributed.run, the
library's own NCCL communicator) equals the single-GPU step bitwise under skewed ownership, for both
placements.  Skipped where the box has fewer than g GPUs (this pool grants one; world 1 is covered by
test_gpu_parity.py::test_collective_ctx_world1_matches_single_gpu_step)."""
import os
import socket
import subprocess
import sys

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
@pytest.mark.parametrize("g", [2, 4, 8])
def test_torchrun_world(g):
    if torch.cuda.device_count() < g:
        pytest.skip(f"needs {g} GPUs, the box has {torch.cuda.device_count()}")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={g}",
                        "--master-addr", "127.0.0.1", "--master-port", str(port),
                        os.path.join(ROOT, "tests", "workers", "multi_gpu_step.py")],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, (r.stdout[-3000:], r.stderr[-3000:])
    assert f"world {g} ok" in r.stdout
