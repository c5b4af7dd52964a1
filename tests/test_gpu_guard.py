"""Out-of-bounds write detection without a sanitizer (compute-sanitizer is closed on this pool): every output a
kernel writes is placed inside a larger buffer whose guard bands hold a sentinel pattern; after the call the
bands must be intact (a write past either end of any output shows up here), over seeded shapes with partial
last blocks, grouped-query heads, odd batch sizes and both map layouts.  Inputs get guard bands too, which
also catches a kernel that writes into its inputs."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = "cuda"
GUARD = 8192  # elements on each side (keeps 16-byte alignment for every dtype here)


@pytest.fixture(scope="module")
def ac():
    import paper_2510_25979_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(ac):
    return ac.Context(0)


class Guarded:
    """A tensor of `shape` at offset GUARD inside a sentinel-filled buffer."""

    def __init__(self, shape, dtype, fill=None):
        n = int(np.prod(shape))
        self.buf = torch.empty(GUARD + n + GUARD, dtype=dtype, device=DEV)
        if dtype.is_floating_point:
            self.buf.fill_(-12345.0)
        else:
            self.buf.fill_(-77 if dtype != torch.uint8 else 0xA5)
        self.sentinel = self.buf[:1].clone()
        self.t = self.buf[GUARD:GUARD + n].view(shape)
        if fill is not None:
            self.t.copy_(fill)

    def intact(self):
        torch.cuda.synchronize()
        return bool(torch.all(self.buf[:GUARD] == self.sentinel)) and bool(torch.all(self.buf[-GUARD:] == self.sentinel))


@pytest.mark.parametrize("seed", range(12))
def test_guard_bands_attend_capture_apply_search(ac, ctx, seed):
    rng = np.random.default_rng(500 + seed)
    S = int(rng.choice([8, 40, 128, 136, 200, 264, 384]))
    d = int(rng.choice([64, 128, 32]))
    dt = torch.bfloat16 if rng.random() < 0.7 else torch.float16
    L, H = int(rng.integers(1, 3)), int(rng.choice([1, 2, 4]))
    Hkv = int(rng.choice([h for h in (1, 2, 4) if H % h == 0]))
    B, N = int(rng.integers(1, 4)), int(rng.integers(1, 4))
    packed = bool(rng.random() < 0.5)
    g = torch.Generator(device=DEV).manual_seed(seed)
    rnd = lambda *shape: torch.randn(*shape, device=DEV, generator=g).to(dt)  # noqa: E731
    Q = Guarded((B, L, H, S, d), dt, rnd(B, L, H, S, d))
    K = Guarded((B, L, Hkv, S, d), dt, rnd(B, L, Hkv, S, d))
    V = Guarded((B, L, Hkv, S, d), dt, rnd(B, L, Hkv, S, d))
    O = Guarded((B, L, H, S, d), dt)
    ac.attncache_attend_full(ctx, Q.t, K.t, V.t, O.t)
    assert all(x.intact() for x in (Q, K, V, O)), "attend"
    # capture into a guarded DB block, then A.V from it
    Qm, Km = Guarded((N, L, H, S, d), dt, rnd(N, L, H, S, d)), Guarded((N, L, Hkv, S, d), dt, rnd(N, L, Hkv, S, d))
    mshape = (N, L, H, ac.attncache_packed_map_elems(S)) if packed else (N, L, H, S, S)
    M = Guarded(mshape, dt)
    ac.attncache_capture_maps(ctx, Qm.t, Km.t, map_dtype=dt, packed=packed, out=M.t)
    assert Qm.intact() and Km.intact() and M.intact(), "capture"
    x = torch.randn(N, 1024, device=DEV, generator=g)
    X = Guarded((N, 1024), torch.bfloat16, (x / x.norm(dim=1, keepdim=True)).to(torch.bfloat16))
    db = ac.Database(ctx, X.t, M.t, packed=packed, seq_len=S)
    idx = torch.as_tensor(rng.integers(0, N, B), device=DEV)
    Oa = Guarded((B, L, H, S, d), dt)
    ac.attncache_apply_cached(db, idx, V.t, O=Oa.t)
    assert V.intact() and Oa.intact() and M.intact(), "apply"
    # search outputs
    q = Guarded((B, 1024), torch.bfloat16, X.t[idx])
    gi, gs, gh = Guarded((B,), torch.int64), Guarded((B,), torch.float32), Guarded((B,), torch.uint8)
    ac.attncache_search(db, q.t, 0.5, gi.t, gs.t, gh.t)
    assert all(t.intact() for t in (q, gi, gs, gh, X)), "search"
    assert torch.equal(gi.t, idx) or torch.all(gs.t >= 0.999)  # planted exact matches (duplicates may tie)


@pytest.mark.parametrize("seed", range(6))
def test_guard_bands_support_kernels(ac, ctx, seed):
    """The f4 projection (head-major epilogue), RoPE (in place), the feature projector and the row gather of the
    relocation (world 1), each with guarded inputs and outputs."""
    import math
    rng = np.random.default_rng(900 + seed)
    g = torch.Generator(device=DEV).manual_seed(seed)
    S, B, K = int(rng.choice([8, 40, 128, 200])), int(rng.integers(1, 4)), int(rng.choice([64, 128, 200]))
    d, H = int(rng.choice([32, 64, 128])), int(rng.choice([1, 2, 3]))
    X = Guarded((B, S, K), torch.bfloat16, torch.randn(B, S, K, device=DEV, generator=g))
    W = Guarded((H * d, K), torch.bfloat16, torch.randn(H * d, K, device=DEV, generator=g) / math.sqrt(K))
    Y = Guarded((B, 1, H, S, d), torch.bfloat16)
    ac.attncache_linear(ctx, X.t, W.t, H, out=Y.t)
    assert X.intact() and W.intact() and Y.intact(), "linear"
    ac.attncache_rope(Y.t.view(B, H, S, d), 10000.0)
    assert Y.intact(), "rope"
    n, E, Hd, D = int(rng.choice([1, 5, 130])), int(rng.choice([64, 96])), int(rng.choice([64, 192])), \
        int(rng.choice([64, 1024]))
    h = Guarded((n, E), torch.bfloat16, torch.randn(n, E, device=DEV, generator=g))
    W1 = Guarded((Hd, E), torch.bfloat16, torch.randn(Hd, E, device=DEV, generator=g) / math.sqrt(E))
    W2 = Guarded((D, Hd), torch.bfloat16, torch.randn(D, Hd, device=DEV, generator=g) / math.sqrt(Hd))
    b1 = Guarded((Hd,), torch.float32, torch.zeros(Hd, device=DEV))
    b2 = Guarded((D,), torch.float32, torch.zeros(D, device=DEV))
    f = Guarded((n, D), torch.bfloat16)
    ac.attncache_project_features(ctx, h.t, W1.t, b1.t, W2.t, b2.t, out=f.t)
    assert all(t.intact() for t in (h, W1, W2, b1, b2, f)), "project"
    rows = Guarded((7, 3, 40), torch.bfloat16, torch.randn(7, 3, 40, device=DEV, generator=g))
    perm = torch.as_tensor(rng.permutation(7), device=DEV)
    counts = torch.tensor([7, 7, 7], dtype=torch.int32)
    got = ac.attncache_relocate_rows(ctx, rows.t, perm, counts.tolist())
    assert rows.intact() and torch.equal(got, rows.t[perm]), "relocate"
