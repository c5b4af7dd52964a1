"""Sizes past 2^31 elements: every tensor-core kernel addresses its operands with 64-bit offsets (3-D tensor maps
over units, 64-bit row and entry offsets), so a batch whose Q / K / V / O hold more than 2^31 elements, and a
database whose feature matrix does, must give the same results as a small one.  Checked against the oracle on
sampled units on both sides of the 2^31-element boundary."""
import numpy as np
import pytest
import torch

import oracle
from tests._util import check_close, check_search, storage

pytestmark = pytest.mark.gpu
DEV = "cuda"
B, L, H, S, d = 140, 32, 32, 128, 128  # 140 * 32 * 32 * 128 * 128 = 2.35e9 elements (4.7 GB) per tensor
UNIT = S * d


@pytest.fixture(scope="module")
def ac():
    import paper_2510_25979_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(ac):
    return ac.Context(0)


@pytest.fixture(scope="module")
def big():
    assert B * L * H * UNIT > 2 ** 31
    g = torch.Generator(device=DEV).manual_seed(31)
    t = {k: torch.empty(B, L, H, S, d, dtype=torch.bfloat16, device=DEV).normal_(generator=g) for k in "QKV"}
    yield t
    del t
    torch.cuda.empty_cache()


def _sample_units():
    """(b, l, h) units: the first, the first whose elements start past 2^31, and the last."""
    u = -(-2 ** 31 // UNIT)
    cut = (u // (L * H), (u // H) % L, u % H)
    return [(0, 0, 0), cut, (B - 1, L - 1, H - 1)]


def _unit_np(t, units):
    return storage(torch.stack([t[b, l, h] for b, l, h in units]))


def test_attend_past_2g_elements(ac, ctx, big):
    O = ac.attncache_attend_full(ctx, big["Q"], big["K"], big["V"])
    torch.cuda.synchronize()
    units = _sample_units()
    off = [i * UNIT for i in range(len(units))]
    ref = oracle.attend(_unit_np(big["Q"], units), _unit_np(big["K"], units), _unit_np(big["V"], units), "bf16", off,
                        S, d)
    check_close(torch.stack([O[b, l, h] for b, l, h in units]), ref, torch.bfloat16, "attend > 2^31 elements")
    del O


def test_apply_past_2g_elements(ac, ctx, big):
    N = 3
    g = torch.Generator(device=DEV).manual_seed(5)
    Qm, Km = (torch.randn(N, L, H, S, d, device=DEV, generator=g).to(torch.bfloat16) for _ in range(2))
    maps = ac.attncache_capture_maps(ctx, Qm, Km, packed=True)
    x = torch.randn(N, 128, device=DEV, generator=g)
    db = ac.Database(ctx, (x / x.norm(dim=1, keepdim=True)).to(torch.bfloat16), maps, packed=True, seq_len=S)
    idx = torch.arange(B, device=DEV) % N
    O = ac.attncache_apply_cached(db, idx, big["V"])
    torch.cuda.synchronize()
    units = _sample_units()
    dense = {e: storage(ac.attncache_fetch_maps(db, e)) for e in range(N)}  # [L][H][S][S] each
    A = np.stack([dense[int(idx[b])][l, h] for b, l, h in units])
    ref = oracle.apply(A, "bf16", [i * S * S for i in range(len(units))], _unit_np(big["V"], units), "bf16",
                       [i * UNIT for i in range(len(units))], S, d)
    check_close(torch.stack([O[b, l, h] for b, l, h in units]), ref, torch.bfloat16, "apply > 2^31 elements")
    del O, db, maps


def test_search_past_2g_elements(ac, ctx):
    N, D = 2_200_000, 1024  # 2.25e9 feature elements
    assert N * D > 2 ** 31
    g = torch.Generator(device=DEV).manual_seed(77)
    x = torch.empty(N, D, dtype=torch.bfloat16, device=DEV)
    for i in range(0, N, 1 << 18):  # normalised rows, built in slices
        r = torch.randn(min(1 << 18, N - i), D, device=DEV, generator=g)
        x[i:i + r.shape[0]] = (r / r.norm(dim=1, keepdim=True)).to(torch.bfloat16)
    db = ac.Database(ctx, x)
    q = torch.stack([x[N - 1], x[2_100_001], x[7]])
    r = torch.randn(1, D, device=DEV, generator=g)
    q = torch.cat([q, (r / r.norm()).to(torch.bfloat16)])
    idx, score, hit = ac.attncache_search(db, q, 0.9)
    torch.cuda.synchronize()
    assert idx[:3].tolist() == [N - 1, 2_100_001, 7] and hit.tolist() == [1, 1, 1, 0]
    check_search(q, x, idx, score, hit, 0.9)
    del db, x
    torch.cuda.empty_cache()


def test_capture_past_2g_elements(ac, ctx, big):
    """DENSE maps of the whole batch: 140 * 32 * 32 * 128 * 128 = 2.35e9 map elements written."""
    M = ac.attncache_capture_maps(ctx, big["Q"], big["K"], packed=False)
    torch.cuda.synchronize()
    assert M.numel() > 2 ** 31
    units = _sample_units()
    P = oracle.attention_map(_unit_np(big["Q"], units), _unit_np(big["K"], units), "bf16",
                             [i * UNIT for i in range(len(units))], S, d)
    got = torch.stack([M[b, l, h].reshape(S, S) for b, l, h in units])
    check_close(got, P, torch.bfloat16, "capture > 2^31 map elements")
    del M
