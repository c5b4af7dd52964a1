"""Seeded randomized parity: random shapes across the ranges the C ABI accepts -- sequence lengths
with and without a partial last 128-row block, head dims on the tensor-core (64, 128) and CUDA-core paths, bf16
and fp16, grouped-query heads, PACKED and DENSE maps -- for the miss attention (Alg. 2 l.376-381), the capture
(Fig. 4 step 1) and A.V with the captured maps as the database (Alg. 2 l.373-375), each against the fp64 oracle on
sampled units within the stated tolerances; the search (Alg. 1 l.255-257) under the A5 exactness
rule; the f4 projections, RoPE and the f2 feature projector."""
import numpy as np
import pytest
import torch

import oracle
from tests._util import DT_NAME, check_close, storage

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def ac():
    import paper_2510_25979_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(ac):
    return ac.Context(0)


def _expand(t, H):
    """[B][L][Hkv][S][d] -> [B][L][H][S][d] (query head h reads K/V head h // (H // Hkv))."""
    return t.repeat_interleave(H // t.shape[2], dim=2).contiguous()


@pytest.mark.parametrize("seed", range(48))
def test_random_shapes_attend_capture_apply(ac, ctx, seed):
    rng = np.random.default_rng(7000 + seed)
    S = int(rng.choice([1, 5, 8, 40, 64, 96, 127, 128, 136, 200, 256, 264, 384, 520]))
    d = int(rng.choice([64, 128, 64, 128, 32, 80]))
    dt = torch.bfloat16 if rng.random() < 0.7 else torch.float16
    name = DT_NAME[dt]
    L, H = int(rng.integers(1, 3)), int(rng.choice([1, 2, 4]))
    Hkv = int(rng.choice([h for h in (1, 2, 4) if H % h == 0]))
    B, N = int(rng.integers(1, 4)), int(rng.integers(1, 4))
    packed = bool(rng.random() < 0.5)
    g = torch.Generator(device=DEV).manual_seed(seed)
    rnd = lambda *shape: torch.randn(*shape, device=DEV, generator=g).to(dt)  # noqa: E731
    what = f"S={S} d={d} {name} L={L} H={H} Hkv={Hkv} B={B} packed={packed}"
    units = [(b, l, h) for b in range(B) for l in range(L) for h in range(H)]
    pick = [units[i] for i in sorted(rng.choice(len(units), min(len(units), 6), replace=False))]
    off = [(((b * L + l) * H + h) * S * d) for b, l, h in pick]

    # miss attention (GQA through the expanded K/V on the oracle side)
    Q, K, V = rnd(B, L, H, S, d), rnd(B, L, Hkv, S, d), rnd(B, L, Hkv, S, d)
    O = ac.attncache_attend_full(ctx, Q, K, V)
    torch.cuda.synchronize()
    ref = oracle.attend(storage(Q), storage(_expand(K, H)), storage(_expand(V, H)), name, off, S, d)
    check_close(torch.stack([O[b, l, h] for b, l, h in pick]), ref, dt, "attend " + what)

    if S % 8:  # capture / 16-byte map rows need S % 8 == 0 (include/attncache.h: ERR_SHAPE)
        with pytest.raises(ac.AttnCacheError):
            ac.attncache_capture_maps(ctx, Q, K, map_dtype=dt, packed=packed)
        return
    # capture N entries, then A.V with them as the database
    Qm, Km = rnd(N, L, H, S, d), rnd(N, L, Hkv, S, d)
    maps = ac.attncache_capture_maps(ctx, Qm, Km, map_dtype=dt, packed=packed)
    x = torch.randn(N, 1024, device=DEV, generator=g)
    x = (x / x.norm(dim=1, keepdim=True)).to(torch.bfloat16)
    db = ac.Database(ctx, x, maps, packed=packed, seq_len=S)
    dense = torch.stack([ac.attncache_fetch_maps(db, e) for e in range(N)])  # [N][L][H][S][S]
    m_units = [(e, l, h) for e in range(N) for l in range(L) for h in range(H)]
    m_pick = [m_units[i] for i in sorted(rng.choice(len(m_units), min(len(m_units), 6), replace=False))]
    m_off = [(((e * L + l) * H + h) * S * d) for e, l, h in m_pick]
    P = oracle.attention_map(storage(Qm), storage(_expand(Km, H)), name, m_off, S, d)
    got = torch.stack([dense[e, l, h] for e, l, h in m_pick]).double().cpu().numpy()
    iu = np.triu_indices(S, 1)
    assert np.all(got[:, iu[0], iu[1]] == 0.0), "capture: non-zero above the diagonal " + what
    assert np.max(np.abs(got - P)) <= 4e-3, f"capture {what}: max-abs {np.max(np.abs(got - P))}"
    idx = torch.as_tensor(rng.integers(0, N, B), device=DEV)
    Vh = rnd(B, L, Hkv, S, d)
    Oa = ac.attncache_apply_cached(db, idx, Vh)
    torch.cuda.synchronize()
    ents = idx.cpu().numpy()
    a_off = [(((int(ents[b]) * L + l) * H + h) * S * S) for b, l, h in pick]
    v_off = [(((b * L + l) * Hkv + h // (H // Hkv)) * S * d) for b, l, h in pick]
    ref = oracle.apply(storage(dense), name, a_off, storage(Vh), name, v_off, S, d)
    check_close(torch.stack([Oa[b, l, h] for b, l, h in pick]), ref, dt, "apply " + what)


@pytest.mark.parametrize("seed", range(24))
def test_random_shapes_search(ac, ctx, seed):
    """Alg. 1 l.255-257 over random DB sizes, batch sizes, feature dims (multiples of 64: tcgen05; others and fp32:
    CUDA cores) and thresholds, with planted exact matches and near-duplicates: the A5 exactness rule against the
    brute-force oracle (tests/_util.check_search)."""
    from tests._util import check_search
    rng = np.random.default_rng(9000 + seed)
    N = int(rng.choice([1, 2, 63, 64, 65, 200, 257, 1000, 3000]))
    B = int(rng.choice([1, 3, 64, 127, 128, 129, 300]))
    D = int(rng.choice([64, 128, 192, 1024, 96, 104, 40, 100, 30]))
    dt = torch.bfloat16 if rng.random() < 0.7 else torch.float32
    tau = float(rng.choice([0.0, 0.5, 0.9, 0.99, 1.0]))
    g = torch.Generator(device=DEV).manual_seed(seed)
    x = torch.randn(N, D, device=DEV, generator=g)
    x = (x / x.norm(dim=1, keepdim=True)).to(dt)
    q = torch.randn(B, D, device=DEV, generator=g)
    q = (q / q.norm(dim=1, keepdim=True)).to(dt)
    planted = rng.choice(B, min(B, max(1, B // 3)), replace=False)
    q[torch.as_tensor(planted, device=DEV)] = x[torch.as_tensor(rng.integers(0, N, len(planted)), device=DEV)]
    if N > 1:  # an exact duplicate entry: the tie must go to the lower index
        x[N - 1] = x[0]
    if (D * x.element_size()) % 16:  # feature rows must be 16-byte multiples (include/attncache.h: ERR_ALIGNMENT)
        with pytest.raises(ac.AttnCacheError):
            ac.Database(ctx, x)
        return
    db = ac.Database(ctx, x)
    idx, score, hit = ac.attncache_search(db, q, tau)
    torch.cuda.synchronize()
    check_search(q, x, idx, score, hit, tau)


@pytest.mark.parametrize("seed", range(16))
def test_random_shapes_linear_rope_project(ac, ctx, seed):
    """f4 projections (attncache_linear, head-major output), RoPE and the f2 feature projector over random
    shapes on both the tcgen05 and the CUDA-core paths, against oracle.linear / oracle.rope / oracle.project."""
    import math
    rng = np.random.default_rng(11000 + seed)
    dt = torch.bfloat16 if rng.random() < 0.7 else torch.float16
    name = DT_NAME[dt]
    g = torch.Generator(device=DEV).manual_seed(seed)
    # linear: X [B][S][K] x W [N][K] -> [B][1][H][S][d]
    S = int(rng.choice([8, 40, 96, 128, 200, 256]))
    B = int(rng.integers(1, 4))
    K = int(rng.choice([64, 128, 256, 200, 72]))
    d = int(rng.choice([32, 64, 128, 48]))
    H = int(rng.choice([1, 2, 3]))
    X = torch.randn(B, S, K, device=DEV, generator=g).to(dt)
    W = (torch.randn(H * d, K, device=DEV, generator=g) / math.sqrt(K)).to(dt)
    Y = ac.attncache_linear(ctx, X, W, H)
    torch.cuda.synchronize()
    ref = oracle.linear(storage(X.view(B * S, K)), storage(W), name).reshape(B, S, H, d).transpose(0, 2, 1, 3)
    check_close(Y.view(B, H, S, d).reshape(-1, S, d), ref.reshape(-1, S, d), dt, f"linear B={B} S={S} K={K} H={H} d={d}")
    # RoPE on the projected heads (in place), in the 16-bit dtype: angles p * theta in fp32 (reading R29)
    de = d - d % 2
    R = torch.randn(B, H, S, de, device=DEV, generator=g).to(dt)
    ref_r = oracle.rope(storage(R), name, S, de, base=10000.0)
    got = ac.attncache_rope(R.clone(), 10000.0)
    torch.cuda.synchronize()
    assert np.abs(got.double().cpu().numpy().reshape(ref_r.shape) - ref_r).max() <= (2e-2 if dt == torch.bfloat16 else 4e-3)
    # feature projector: f = normalize(W2 relu(W1 h + b1) + b2)
    n, E, Hd, D = int(rng.choice([1, 5, 128, 130])), int(rng.choice([64, 256, 96])), int(rng.choice([64, 128, 192])), \
        int(rng.choice([64, 128, 1024]))
    h = torch.randn(n, E, device=DEV, generator=g).to(torch.bfloat16)
    W1 = (torch.randn(Hd, E, device=DEV, generator=g) / math.sqrt(E)).to(torch.bfloat16)
    W2 = (torch.randn(D, Hd, device=DEV, generator=g) / math.sqrt(Hd)).to(torch.bfloat16)
    b1 = torch.randn(Hd, device=DEV, generator=g) * 0.1
    b2 = torch.randn(D, device=DEV, generator=g) * 0.1
    f = ac.attncache_project_features(ctx, h, W1, b1, W2, b2)
    torch.cuda.synchronize()
    ref_f = oracle.project(storage(h), "bf16", storage(W1), b1.cpu().numpy(), storage(W2), b2.cpu().numpy())
    # one "unit" per row: max-abs over all elements and rel-L2 per row (the north_star bf16 bounds)
    check_close(f.unsqueeze(1), ref_f[:, None, :], f.dtype, f"project n={n} E={E} Hd={Hd} D={D}")
