"""The C ABI's documented error behaviour (include/attncache.h "Errors:" lines), called through the raw
library (not the binding's own checks): each case passes one bad argument to an otherwise valid call and must
get the documented status, leave the context usable, and write nothing."""
import ctypes
import math

import pytest
import torch

pytestmark = pytest.mark.gpu
DEV = "cuda"
OK, INV, SHAPE, DTYPE, ALIGN, NOT_FOUND, EMPTY, STATE = 0, 1, 2, 3, 4, 5, 6, 9
F32, F16, BF16 = 0, 1, 2  # attncache_dtype
DENSE, PACKED = 0, 1      # attncache_map_layout


@pytest.fixture(scope="module")
def ac():
    import paper_2510_25979_b200 as m
    return m


@pytest.fixture(scope="module")
def L(ac):
    return ac.load_library()


@pytest.fixture(scope="module")
def ctx(ac):
    return ac.Context(0)


def p(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _normed(n, D, dtype):
    x = torch.randn(n, D, device=DEV)
    return (x / x.norm(dim=1, keepdim=True)).to(dtype)


@pytest.fixture(scope="module")
def setup(ac, ctx):
    N, L_, H, S, d = 4, 2, 2, 128, 64
    x = _normed(N, 128, torch.bfloat16)
    maps = ac.attncache_capture_maps(ctx, torch.randn(N, L_, H, S, d, device=DEV).to(torch.bfloat16),
                                     torch.randn(N, L_, H, S, d, device=DEV).to(torch.bfloat16))
    db = ac.Database(ctx, x, maps, packed=True, seq_len=S)
    search_only = ac.Database(ctx, x)
    return dict(N=N, L=L_, H=H, S=S, d=d, x=x, maps=maps, db=db, search_only=search_only)


def test_status_strings_and_version(L):
    for code in range(12):
        assert L.attncache_status_string(code)
    assert L.attncache_version() > 0


def test_ctx_create_errors(L):
    h = ctypes.c_void_p()
    assert L.attncache_ctx_create(0, 1, 1, None, ctypes.byref(h)) == INV        # rank outside [0, world)
    assert L.attncache_ctx_create(0, 0, 2, None, ctypes.byref(h)) == INV        # world > 1 without uid
    assert L.attncache_ctx_create(0, 0, 1, None, None) == INV                   # out NULL
    assert L.attncache_ctx_set_sm_budget(None, 8, 8) == INV


def test_db_load_errors(ac, L, ctx, setup):
    x, maps, S = setup["x"], setup["maps"], setup["S"]
    N = x.shape[0]

    def load(**over):
        f = dict(n_global=N, shard_begin=0, shard_count=N, feat_dim=x.shape[1], feat_dtype=BF16, feats=x.data_ptr(),
                 n_layers=setup["L"], n_heads=setup["H"], seq_len=S, map_dtype=BF16, maps=maps.data_ptr(),
                 map_layout=PACKED, maps_noncausal=0)
        f.update(over)
        h = ctypes.c_void_p()
        st = L.attncache_db_load(ctx.handle, ctypes.byref(ac._DbDesc(**f)), ctypes.byref(h))
        if st == OK:
            L.attncache_db_free(h)
        return st

    assert load() == OK
    assert load(shard_count=N + 1) == INV                        # shard past n_global
    assert load(feats=0) == INV                                  # null feats with shard_count > 0
    assert load(feat_dtype=F16) == DTYPE                         # feats must be F32 or BF16
    assert load(feats=x.data_ptr() + 2) == ALIGN                 # base not 16-byte aligned
    assert load(map_dtype=F32) == DTYPE                          # maps must be F16 / BF16
    assert load(maps_noncausal=1) == INV                         # PACKED maps are causal only


def test_search_errors(ac, L, ctx, setup):
    db, x = setup["db"], setup["x"]
    q = x[:3].contiguous()
    idx = torch.full((3,), -7, dtype=torch.int64, device=DEV)
    score = torch.zeros(3, device=DEV)
    hit = torch.zeros(3, dtype=torch.uint8, device=DEV)
    args = lambda tau, i=idx: (db.handle, p(q), 3, ctypes.c_float(tau), p(i), p(score), p(hit), None)  # noqa: E731
    assert L.attncache_search(*args(math.nan)) == INV            # NaN tau
    assert L.attncache_search(db.handle, p(q), 3, ctypes.c_float(0.5), None, p(score), p(hit), None) == INV
    assert torch.all(idx == -7)                                  # nothing written on an error
    assert L.attncache_search(*args(0.5)) == OK
    torch.cuda.synchronize()
    assert idx.tolist() == [0, 1, 2]
    empty = ac.Database(ctx, x[:0].contiguous(), n_global=0)
    assert L.attncache_search(empty.handle, p(q), 3, ctypes.c_float(0.5), p(idx), p(score), p(hit), None) == EMPTY


def test_apply_errors(ac, L, ctx, setup):
    db, S, d, L_, H = setup["db"], setup["S"], setup["d"], setup["L"], setup["H"]
    idx = torch.tensor([0, 3], device=DEV)
    V = torch.randn(2, L_, H, S, d, device=DEV).to(torch.bfloat16)
    O = torch.full_like(V, 7.0)

    def apply(lb=0, le=L_, hd=d, dt=BF16, v=None, o=None, dbh=None):
        return L.attncache_apply_cached(dbh or db.handle, p(idx), None, 2, lb, le, hd, dt, v or p(V), o or p(O), None)

    assert apply(le=L_ + 1) == SHAPE                             # layer range outside [0, n_layers)
    assert apply(lb=1, le=1) in (OK, SHAPE)                      # an empty range is allowed or refused, never runs
    assert apply(hd=0) == SHAPE                                  # head_dim <= 0
    assert apply(dt=F16) == DTYPE                                # bf16 maps with fp16 activations
    assert apply(v=ctypes.c_void_p(V.data_ptr() + 2)) == ALIGN   # V base not 16-byte aligned
    assert apply(dbh=setup["search_only"].handle) == STATE       # a database without maps
    torch.cuda.synchronize()
    assert torch.all(O == 7.0)                                   # nothing written by a refused call
    bad = torch.tensor([0, 99], device=DEV)                      # an entry outside the shard: deferred NOT_FOUND
    assert L.attncache_apply_cached(db.handle, p(bad), None, 2, 0, L_, d, BF16, p(V), p(O), None) == OK
    assert L.attncache_ctx_sync(ctx.handle) == NOT_FOUND
    assert L.attncache_ctx_sync(ctx.handle) == OK                # reported once, then cleared


def test_attend_capture_errors(L, ctx, setup):
    S, d, L_, H = setup["S"], setup["d"], setup["L"], setup["H"]
    Q = torch.randn(1, L_, H, S, d, device=DEV).to(torch.bfloat16)
    O = torch.empty_like(Q)
    assert L.attncache_attend_full(ctx.handle, 1, L_, H, S, d, F16 + 7, p(Q), p(Q), p(Q), ctypes.c_float(0.0),
                                   None, p(O), None) == DTYPE
    assert L.attncache_attend_full_gqa(ctx.handle, 1, L_, H, 3, S, d, BF16, p(Q), p(Q), p(Q), ctypes.c_float(0.0),
                                       None, p(O), None) == SHAPE  # n_kv_heads does not divide n_heads
    out = torch.empty(1, L_, H, S * S, dtype=torch.bfloat16, device=DEV)
    assert L.attncache_capture_maps(ctx.handle, 1, L_, H, S - 4, d, BF16, p(Q), p(Q), ctypes.c_float(0.0), None,
                                    BF16, DENSE, p(out), None) == SHAPE  # S % 8 != 0
    assert L.attncache_capture_maps(ctx.handle, 1, L_, H, S, d, BF16, p(Q), p(Q), ctypes.c_float(0.0), None,
                                    F32, DENSE, p(out), None) == DTYPE   # map dtype F32


def test_support_call_errors(L, ctx, setup):
    X = torch.randn(2, 8, 64, device=DEV).to(torch.bfloat16)
    W = torch.randn(96, 64, device=DEV).to(torch.bfloat16)
    Y = torch.empty(2 * 8 * 96, dtype=torch.bfloat16, device=DEV)
    # N = 96 is not whole heads of head_dim 64
    assert L.attncache_linear(ctx.handle, p(X), 16, 64, p(W), 96, BF16, None, 8, 64, p(Y), None) == SHAPE
    R = torch.randn(4, 8, 7, device=DEV).to(torch.bfloat16)
    assert L.attncache_rope(p(R), 4, 8, 7, BF16, ctypes.c_float(10000.0), None) == SHAPE  # odd head dim
    counts = (ctypes.c_int32 * 3)(2, 2, 2)  # world 1: send 2 rows to rank 0, but n_home = 3
    src = torch.zeros(3, 8, device=DEV)
    so = torch.arange(3, device=DEV)
    dst = torch.zeros(2, 8, device=DEV)
    assert L.attncache_relocate_rows(ctx.handle, p(src), 3, 32, p(so), counts, p(dst), None) == INV


def test_prefill_host_errors(L, setup):
    db, S, d, L_, H = setup["db"], setup["S"], setup["d"], setup["L"], setup["H"]
    q = setup["x"][:2].contiguous()  # device memory: the call takes page-locked host buffers only
    Qd = torch.zeros(2, L_, H, S, d, dtype=torch.bfloat16, device=DEV)
    i64 = torch.zeros(2, dtype=torch.int64, device=DEV)
    f32 = torch.zeros(2, device=DEV)
    u8 = torch.zeros(2, dtype=torch.uint8, device=DEV)
    assert L.attncache_prefill_host(db.handle, p(q), 2, ctypes.c_float(0.5), p(Qd), p(Qd), p(Qd), d, BF16, p(Qd),
                                    p(i64), p(f32), p(u8), 16, 4) == INV
    qh = q.cpu().pin_memory()
    Qh = Qd.cpu().pin_memory()
    i64h, f32h, u8h = i64.cpu().pin_memory(), f32.cpu().pin_memory(), u8.cpu().pin_memory()
    assert L.attncache_prefill_host(db.handle, p(qh), 2, ctypes.c_float(0.5), p(Qh), p(Qh), p(Qh), d, BF16, p(Qh),
                                    p(i64h), p(f32h), p(u8h), 16, 1) == INV  # depth outside [2, 8]
    assert L.attncache_prefill_host(db.handle, p(qh), 2, ctypes.c_float(math.nan), p(Qh), p(Qh), p(Qh), d, BF16,
                                    p(Qh), p(i64h), p(f32h), p(u8h), 16, 4) == INV  # NaN tau
