"""Host-side checks that need no GPU: the C-ABI library loads and exports every declared symbol,
status plumbing works, the product path never touches the oracle, and it fails loudly without
an sm_100a device."""
import os
import re
import subprocess

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2510_25979_b200 import build
    build.build()
    import paper_2510_25979_b200 as ac
    return ac.load_library()


def _declared():
    src = open(os.path.join(ROOT, "include", "attncache.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(attncache_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_all_exported(lib):
    declared = _declared()
    assert len(declared) >= 19
    out = subprocess.run(["nm", "-D", "--defined-only", lib._name], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\bT (attncache_\w+)", out))
    missing = [s for s in declared if s not in exported]
    assert not missing, f"declared but not exported: {missing}"
    import paper_2510_25979_b200 as ac
    assert sorted(ac.ABI_FUNCTIONS) == declared  # the binding wraps every ABI call


def test_library_is_sm100a_only(lib):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", lib._name], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_status_strings(lib):
    import paper_2510_25979_b200 as ac
    assert lib.attncache_status_string(0) == b"ATTNCACHE_OK"
    assert lib.attncache_status_string(5) == b"ATTNCACHE_ERR_NOT_FOUND"
    assert ac.attncache_version() >= 100
    assert ac.attncache_launch_count() >= 0


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure mode")
def test_no_gpu_fails_loudly(lib):
    import paper_2510_25979_b200 as ac
    with pytest.raises(ac.AttnCacheError) as e:
        ac.Context(0)
    assert e.value.name == "ATTNCACHE_ERR_UNSUPPORTED"


def test_product_path_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2510_25979_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "oracle." not in txt and "liboracle" not in txt, \
                    f"{f} references the oracle"
    synth_src = open(os.path.join(ROOT, "synth", "__init__.py")).read()
    assert "import oracle" not in synth_src and "paper_2510_25979_b200" not in synth_src
    orc = open(os.path.join(ROOT, "oracle", "attncache_oracle.c")).read()
    includes = re.findall(r"#include\s*[<\"]([^>\"]+)", orc)
    assert includes and all(i in ("math.h", "stdint.h", "stdlib.h", "string.h", "omp.h") for i in includes), includes


def test_keys_are_order_preserving():
    """Reading R3 packed key, re-derived in Python: max key <=> (max score, min index)."""
    import struct

    def key(s, i):
        s = s + 0.0
        b = struct.unpack("<I", struct.pack("<f", s))[0]
        o = (~b & 0xFFFFFFFF) if b & 0x80000000 else (b | 0x80000000)
        return (o << 32) | (0xFFFFFFFF - i)

    vals = [(-1.0, 3), (-0.0, 2), (0.0, 5), (1e-30, 9), (0.5, 1), (0.5, 0), (1.0, 7), (float("-inf"), 0)]
    keys = [key(s, i) for s, i in vals]
    order = sorted(range(len(vals)), key=lambda k: keys[k])
    ranked = sorted(range(len(vals)), key=lambda k: (vals[k][0], -vals[k][1]))
    assert order == ranked
    assert key(-0.0, 4) == key(0.0, 4)
    assert all(k > 0 for k in keys)


def test_packed_layout_size_formula(lib):
    """PACKED layout (include/attncache.h): row i keeps 8*(i//8 + 1) elements, rows back to back."""
    import paper_2510_25979_b200 as ac
    for S in (8, 32, 128, 256, 1024):
        assert ac.attncache_packed_map_elems(S) == sum(8 * (i // 8 + 1) for i in range(S))
        assert ac.attncache_packed_map_elems(S) >= S * (S + 1) // 2      # holds the whole triangle
    assert ac.attncache_packed_map_elems(30) == 0
