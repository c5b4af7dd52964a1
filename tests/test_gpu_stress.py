"""Schedule stress: the library rebuilt with -DAC_STRESS (random warp-uniform sleeps at the top of every role
loop of the persistent tcgen05 kernels, sm100.cuh AC_STRESS_DELAY) must finish and reproduce the normal
build's outputs bit for bit on every kernel family (scripts/stress_check.py).  The delays change only the
interleaving of loader, MMA, softmax and epilogue roles, so any difference or hang is a synchronisation
bug (e.g. an mbarrier parity wait that can see its barrier two phases ahead).  Checked against an injected
bug: dropping the attention MMA's wait for the epilogue's o_free hung the stress run (and mismatched two
cases even without the delays)."""
import os
import subprocess
import sys
import tempfile

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_stress_build_is_bitwise_identical():
    with tempfile.TemporaryDirectory() as tmp:
        env = dict(os.environ, ATTNCACHE_BUILD_ROOT=os.path.join(tmp, "stress"), ATTNCACHE_EXTRA_FLAGS="-DAC_STRESS")
        subprocess.run([sys.executable, "-m", "paper_2510_25979_b200.build"], cwd=ROOT, env=env, check=True,
                       stdout=subprocess.DEVNULL, timeout=900)
        stress_lib = os.path.join(tmp, "stress", "lib", "libattncache.so")
        ref_out, stress_out = os.path.join(tmp, "ref.pt"), os.path.join(tmp, "stress.pt")
        script = os.path.join(ROOT, "scripts", "stress_check.py")
        base_env = {k: v for k, v in os.environ.items() if k not in ("ATTNCACHE_LIB", "ATTNCACHE_EXTRA_FLAGS",
                                                                      "ATTNCACHE_BUILD_ROOT")}
        subprocess.run([sys.executable, script, ref_out, "1"], cwd=ROOT, env=base_env, check=True, timeout=600)
        subprocess.run([sys.executable, script, stress_out, "3"], cwd=ROOT, env=dict(base_env, ATTNCACHE_LIB=stress_lib),
                       check=True, timeout=300)
        ref, got = torch.load(ref_out), torch.load(stress_out)
        assert set(ref) == set(got) and len(ref) >= 10
        for name, (r,) in ref.items():
            for i, g in enumerate(got[name]):
                assert torch.equal(r, g), f"{name} repeat {i}"
