"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the same seeded bytes.

Tolerances and the search exactness rule are in tests/_util.py (BASELINE.json north_star).
Sizes: every config's per-entry shape (L, H, S, d, D) is exercised; small-N databases keep the
oracle fast, and test_full_step_llama32 runs BASELINE.json configs[1] at full size in the launch
configuration bench.py times, checking every search decision and sampled output units.
"""
import math

import numpy as np
import pytest
import torch

import oracle
import synth
from tests._util import DT_NAME, check_close, check_search, storage

pytestmark = pytest.mark.gpu
DEV = "cuda"


@pytest.fixture(scope="module")
def ac():
    from paper_2510_25979_b200 import build
    build.build()
    import paper_2510_25979_b200 as m
    return m


@pytest.fixture(scope="module")
def ctx(ac):
    return ac.Context(0)


def _normed(n, D, dtype, seed):
    g = torch.Generator(device=DEV).manual_seed(seed)
    x = torch.randn(n, D, device=DEV, generator=g)
    return (x / x.norm(dim=1, keepdim=True)).to(dtype)


def _units(rows, n_lay, H):
    """All (row, layer, head) units of the given batch rows."""
    return [(b, l, h) for b in rows for l in range(n_lay) for h in range(H)]


def _apply_ref(maps_np, map_dt, ents, V_np, v_dt, units, L, H, S, d, layer_begin=0, n_lay=None):
    n_lay = L if n_lay is None else n_lay
    a_off = [(((ents[b] * L + layer_begin + l) * H + h) * S * S) for b, l, h in units]
    v_off = [(((b * n_lay + l) * H + h) * S * d) for b, l, h in units]
    return oracle.apply(maps_np, map_dt, a_off, V_np, v_dt, v_off, S, d)


def _gather_units(O, units):
    return torch.stack([O[b, l, h] for b, l, h in units])


# ------------------------------------------------------------------------------------------------
# search (Alg. 1 l.255-257)
# ------------------------------------------------------------------------------------------------

def test_search_tiny_config(ac, ctx):
    cfg = synth.CONFIGS["tiny"]
    x = synth.features(cfg, 0, cfg.N, DEV)
    db = ac.Database(ctx, x)
    q, pos, tgt = synth.queries(cfg, DEV)
    idx, score, hit = ac.attncache_search(db, q, cfg.tau)
    torch.cuda.synchronize()
    check_search(q, x, idx, score, hit, cfg.tau)
    assert hit.sum().item() == cfg.n_hit
    assert idx[pos].cpu().tolist() == tgt.tolist()


@pytest.mark.parametrize("cfg_name", ["llama32_1b", "llama3_8b"])
def test_search_full_feature_db(ac, ctx, cfg_name):
    cfg = synth.CONFIGS[cfg_name]
    x = synth.features(cfg, 0, cfg.N, DEV)
    db = ac.Database(ctx, x)
    q, pos, tgt = synth.queries(cfg, DEV)
    idx, score, hit = ac.attncache_search(db, q, cfg.tau)
    check_search(q, x, idx, score, hit, cfg.tau)
    assert idx[pos].cpu().tolist() == tgt.tolist() and hit.sum().item() == cfg.n_hit
    idx2, score2, hit2 = ac.attncache_search(db, q, cfg.tau)  # deterministic
    assert torch.equal(idx, idx2) and torch.equal(score, score2) and torch.equal(hit, hit2)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("N,B,D", [(1000, 130, 1024), (1, 3, 384), (4097, 257, 4096)])
def test_search_ragged_with_planted_ties(ac, ctx, dtype, N, B, D):
    x = _normed(N, D, dtype, 11)
    q = _normed(B, D, dtype, 12)
    if N > 700:
        x[700] = x[3]           # exact duplicates inside and across tiles: the lowest index wins
        x[N - 1] = x[3]
        q[0] = x[3]
        q[1] = x[N - 1]
    db = ac.Database(ctx, x)
    idx, score, hit = ac.attncache_search(db, q, 0.9)
    check_search(q, x, idx, score, hit, 0.9)
    if N > 700:
        assert idx[0].item() == 3 and idx[1].item() == 3


def test_search_basis_ties_and_exact_threshold(ac, ctx):
    D = 1024
    for dtype in (torch.float32, torch.bfloat16):
        x = torch.eye(D, device=DEV, dtype=dtype)
        pairs = [(3, 11), (900, 2), (1023, 0), (500, 501)]
        q = torch.zeros(len(pairs) + 1, D, device=DEV)
        for r, (i, j) in enumerate(pairs):
            q[r, i] = q[r, j] = 1 / math.sqrt(2)
        q[-1, 77] = 1.0
        db = ac.Database(ctx, x)
        idx, score, hit = ac.attncache_search(db, q.to(dtype), 0.5)
        assert idx.cpu().tolist() == [min(p) for p in pairs] + [77]
        assert score[-1].item() == 1.0 and hit.all()
        # inclusive gate at an exactly representable score (tests/golden/search_threshold.json)
        xt = torch.zeros(2, D, device=DEV)
        xt[1, 0], xt[1, 1] = 0.90625, math.sqrt(1 - 0.90625 ** 2)
        xt[0, 5] = 1.0
        db = ac.Database(ctx, xt.to(dtype))
        e0 = torch.zeros(1, D, device=DEV, dtype=dtype)
        e0[0, 0] = 1
        idx, score, hit = ac.attncache_search(db, e0, 0.90625)
        assert idx.item() == 1 and score.item() == 0.90625 and hit.item() == 1
        _, _, hit = ac.attncache_search(db, e0, float(np.nextafter(np.float32(0.90625), np.float32(1))))
        assert hit.item() == 0


def test_search_errors_and_degenerate(ac, ctx):
    x = _normed(64, 384, torch.float32, 1)
    db = ac.Database(ctx, x)
    q = _normed(4, 384, torch.float32, 2)
    with pytest.raises(ac.AttnCacheError) as e:
        ac.attncache_search(db, q, float("nan"))
    assert e.value.name == "ATTNCACHE_ERR_INVALID_ARGUMENT"
    _, _, hit = ac.attncache_search(db, q, 2.0)
    assert hit.sum().item() == 0                          # tau > 1: every query misses
    empty = ac.Database(ctx, torch.zeros(0, 384, device=DEV))
    with pytest.raises(ac.AttnCacheError) as e:
        ac.attncache_search(empty, q, 0.5)
    assert e.value.name == "ATTNCACHE_ERR_EMPTY"
    ac.attncache_search(db, q[:0], 0.5)                   # B = 0 is a no-op
    with pytest.raises(ac.AttnCacheError) as e:
        ac.Database(ctx, x.to(torch.float16))
    assert e.value.name == "ATTNCACHE_ERR_DTYPE"


def test_search_sharded_keys_equal_single_rank(ac, ctx):
    cfg = synth.CONFIGS["llama32_1b"]
    x = synth.features(cfg, 0, cfg.N, DEV)
    x[3000] = x[17]                                       # a cross-shard duplicate
    q, _, _ = synth.queries(cfg, DEV)
    q[5] = x[3000]
    ref = ac.attncache_search(ac.Database(ctx, x), q, cfg.tau)
    bounds = [0, 1000, 1001, 2500, cfg.N]                 # includes a 1-entry shard
    keys = torch.stack([ac.attncache_search_keys(ac.Database(ctx, x[a:b], n_global=cfg.N, shard_begin=a), q)
                        for a, b in zip(bounds, bounds[1:])])
    got = ac.attncache_keys_decode(keys, cfg.tau)
    for r, g in zip(ref, got):
        assert torch.equal(r, g)
    assert got[0][5].item() == 17


@pytest.fixture(scope="module")
def sweep_db(ac, ctx):
    """BASELINE.json configs[4]: 1M x 1024 bf16 features (2.05 GB), built once for the module."""
    cfg = synth.CONFIGS["search_sweep"]
    x = synth.features(cfg, 0, cfg.N, DEV)
    return cfg, x, ac.Database(ctx, x)


@pytest.mark.parametrize("B", [1, 64, 1024, 8192])
def test_search_sweep_1m_sampled(ac, ctx, sweep_db, B):
    """configs[4] at every batch the bench times (the full batch is searched in the bench's launch
    configuration); min(B, 128) sampled queries, half planted hits and half misses, are checked against the
    brute-force oracle over all 1M entries (>= 128 queries)."""
    cfg, x, db = sweep_db
    q, pos, tgt = synth.queries(cfg, DEV, B=B)
    idx, score, hit = ac.attncache_search(db, q, cfg.tau)
    assert ac.attncache_variant("search", q.dtype, 0, cfg.D) == "tc"
    assert idx[pos].cpu().tolist() == tgt.tolist()        # planted hits find their entry
    assert hit[pos].all() and hit.sum().item() == len(pos)
    n = min(B, 128)
    misses = torch.nonzero(hit == 0).flatten().cpu()
    sample = torch.cat([pos[:n - min(n // 2, len(misses))], misses[:n // 2]])
    assert len(sample) == n
    s = sample.to(DEV)
    check_search(q[s], x, idx[s], score[s], hit[s], cfg.tau)


def test_search_mid_tile_and_simt_bf16(ac, ctx):
    """The 128-entry tile of search_tc_kernel (N = 50,000 with B = 128: fewer than 2 work items per SM with
    256-entry tiles, enough with 128), the bf16 CUDA-core search (D = 200 is not a multiple of the 64-element
    tensor-core chunk) and the two-query-tile kernel with a ragged batch (B = 300: a pair and a lone tile; a
    partial entry tile), each against the oracle with planted cross-tile duplicates."""
    for N, B, D in ((50_000, 128, 1024), (777, 33, 200), (100_003, 300, 1024)):
        x = _normed(N, D, torch.bfloat16, 31)
        q = _normed(B, D, torch.bfloat16, 32)
        x[N - 5] = x[130]
        x[257] = x[130]
        q[0] = x[N - 5]
        db = ac.Database(ctx, x)
        idx, score, hit = ac.attncache_search(db, q, 0.9)
        check_search(q, x, idx, score, hit, 0.9)
        assert idx[0].item() == 130 and hit[0].item() == 1
        want = "tc" if D % 64 == 0 else "ffma"
        assert ac.attncache_variant("search", torch.bfloat16, 0, D) == want


# ------------------------------------------------------------------------------------------------
# apply (Alg. 2 l.373-375)
# ------------------------------------------------------------------------------------------------

def test_apply_tiny_config_all_units(ac, ctx):
    cfg = synth.CONFIGS["tiny"]
    x = synth.features(cfg, 0, cfg.N, DEV)
    maps = synth.maps(cfg, 0, cfg.N, DEV)
    db = ac.Database(ctx, x, maps)
    q, pos, tgt = synth.queries(cfg, DEV)
    idx, score, hit = ac.attncache_search(db, q, cfg.tau)
    V = synth.activations(cfg, "v", 0, cfg.B, device=DEV)
    O = torch.full_like(V, 7.0)
    ac.attncache_apply_cached(db, idx, V, O, hit=hit)
    ctx.sync()
    rows = torch.nonzero(hit).flatten().tolist()
    miss = [b for b in range(cfg.B) if b not in rows]
    assert torch.all(O[miss] == 7.0)                      # rows that missed are untouched
    units = _units(rows, cfg.L, cfg.H)
    ref = _apply_ref(storage(maps), "f16", idx.cpu().numpy(), storage(V), "f32", units, cfg.L, cfg.H, cfg.S, cfg.d)
    check_close(_gather_units(O, units), ref, V.dtype, "apply tiny")


@pytest.mark.parametrize("cfg_name,N,B,n_sample", [("llama32_1b", 48, 8, None), ("llama3_8b", 8, 4, 48),
                                                    ("long_prefill", 4, 3, 12)])
def test_apply_config_shapes(ac, ctx, cfg_name, N, B, n_sample):
    cfg = synth.CONFIGS[cfg_name].with_(N=N)
    x = synth.features(cfg, 0, N, DEV)
    maps = synth.maps(cfg, 0, N, DEV)
    db = ac.Database(ctx, x, maps)
    idx = torch.tensor([(5 * b + 1) % N for b in range(B)], device=DEV)
    hit = torch.tensor([1 if b % 4 != 2 else 0 for b in range(B)], device=DEV, dtype=torch.uint8)
    V = synth.activations(cfg, "v", 0, B, device=DEV)
    O = torch.full_like(V, 3.0)
    ac.attncache_apply_cached(db, idx, V, O, hit=hit)
    ctx.sync()
    rows = torch.nonzero(hit).flatten().tolist()
    assert torch.all(O[hit == 0] == 3.0)
    units = _units(rows, cfg.L, cfg.H)
    if n_sample:
        rng = np.random.default_rng(0)
        units = [units[i] for i in sorted(rng.choice(len(units), n_sample, replace=False))]
        units += [(rows[-1], cfg.L - 1, cfg.H - 1)]
    ref = _apply_ref(storage(maps), "bf16", idx.cpu().numpy(), storage(V), "bf16", units, cfg.L, cfg.H, cfg.S, cfg.d)
    check_close(_gather_units(O, units), ref, V.dtype, f"apply {cfg_name}")
    O2 = torch.full_like(V, 3.0)
    ac.attncache_apply_cached(db, idx, V, O2, hit=hit)
    assert torch.equal(O, O2)                             # bitwise deterministic


@pytest.mark.parametrize("S,d", [(128, 64), (256, 128), (32, 64)])
def test_apply_identity_and_one_hot_are_exact(ac, ctx, S, d):
    L, H, N = 2, 3, 2
    maps = torch.zeros(N, L, H, S, S, device=DEV, dtype=torch.bfloat16)
    maps[0] = torch.eye(S, device=DEV, dtype=torch.bfloat16)
    maps[1, ..., 0] = 1.0
    db = ac.Database(ctx, _normed(N, 1024, torch.bfloat16, 3), maps)
    V = torch.randn(2, L, H, S, d, device=DEV).to(torch.bfloat16)
    O = ac.attncache_apply_cached(db, torch.tensor([0, 1], device=DEV), V)
    torch.cuda.synchronize()
    assert torch.equal(O[0], V[0])                        # A = I gives O = V bitwise
    assert torch.equal(O[1], V[1, :, :, :1, :].expand(L, H, S, d))


def test_apply_layer_slices_equal_all_layers(ac, ctx):
    # Alg. 2 runs layer by layer; a per-layer call must equal the all-layer call bitwise (reading R13)
    cfg = synth.CONFIGS["llama32_1b"].with_(N=6, L=4)
    db = ac.Database(ctx, synth.features(cfg, 0, 6, DEV), synth.maps(cfg, 0, 6, DEV))
    idx = torch.tensor([5, 0, 3], device=DEV)
    V = synth.activations(cfg, "v", 0, 3, device=DEV)
    O_all = ac.attncache_apply_cached(db, idx, V)
    for l in range(cfg.L):
        Vl = V[:, l:l + 1].contiguous()
        Ol = ac.attncache_apply_cached(db, idx, Vl, layer_begin=l, layer_end=l + 1)
        assert torch.equal(Ol[:, 0], O_all[:, l])


def test_apply_out_of_shard_index_is_deferred_not_found(ac, ctx):
    cfg = synth.CONFIGS["llama32_1b"].with_(N=4, L=1)
    db = ac.Database(ctx, synth.features(cfg, 0, 4, DEV), synth.maps(cfg, 0, 4, DEV))
    V = synth.activations(cfg, "v", 0, 2, device=DEV)
    O = torch.zeros_like(V)
    ac.attncache_apply_cached(db, torch.tensor([1, 4], device=DEV), V, O)
    with pytest.raises(ac.AttnCacheError) as e:
        ctx.sync()
    assert e.value.name == "ATTNCACHE_ERR_NOT_FOUND"
    assert torch.all(O[1] == 0) and not torch.all(O[0] == 0)
    ctx.sync()  # cleared
    with pytest.raises(ac.AttnCacheError) as e:
        ac.attncache_apply_cached(db, torch.tensor([1, 2], device=DEV), V[:, :, :, :64].contiguous())
    assert e.value.name == "ATTNCACHE_ERR_SHAPE"


@pytest.mark.parametrize("cfg_name,N,B", [("tiny", 6, 4), ("llama32_1b", 6, 3), ("llama3_8b", 3, 2),
                                          ("long_prefill", 2, 2)])
def test_apply_packed_layout_equals_dense(ac, ctx, cfg_name, N, B):
    """The PACKED DB layout holds exactly the bytes A.V reads: results are bitwise identical."""
    cfg = synth.CONFIGS[cfg_name].with_(N=N)
    x = synth.features(cfg, 0, N, DEV)
    dense = synth.maps(cfg, 0, N, DEV)
    packed = ac.attncache_pack_maps(dense)
    assert packed.shape[-1] == ac.attncache_packed_map_elems(cfg.S)
    db_d = ac.Database(ctx, x, dense)
    db_p = ac.Database(ctx, x, packed, packed=True, seq_len=cfg.S)
    idx = torch.tensor([(3 * b + 1) % N for b in range(B)], device=DEV)
    V = synth.activations(cfg, "v", 0, B, device=DEV)
    O_d = ac.attncache_apply_cached(db_d, idx, V)
    O_p = ac.attncache_apply_cached(db_p, idx, V)
    assert torch.equal(O_d, O_p)
    for e in (0, N - 1):                                   # fetch expands PACKED back to DENSE
        assert torch.equal(ac.attncache_fetch_maps(db_p, e), dense[e])
        assert torch.equal(ac.attncache_fetch_maps(db_d, e, 1, 2), dense[e, 1:2])


# ------------------------------------------------------------------------------------------------
# attend (Alg. 2 l.376-381, Eq. 5)
# ------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("cfg_name,B,n_sample", [("tiny", 3, None), ("llama32_1b", 3, 24), ("llama3_8b", 2, 12),
                                                 ("long_prefill", 2, 6)])
def test_attend_config_shapes(ac, ctx, cfg_name, B, n_sample):
    cfg = synth.CONFIGS[cfg_name]
    Q, K, V = (synth.activations(cfg, k, 0, B, device=DEV) for k in "qkv")
    skip = torch.zeros(B, dtype=torch.uint8, device=DEV)
    skip[1] = 1
    O = torch.full_like(V, 5.0)
    ac.attncache_attend_full(ctx, Q, K, V, O, skip=skip)
    torch.cuda.synchronize()
    assert torch.all(O[1] == 5.0)
    rows = [b for b in range(B) if b != 1]
    units = _units(rows, cfg.L, cfg.H)
    if n_sample:
        rng = np.random.default_rng(1)
        units = [units[i] for i in sorted(rng.choice(len(units), n_sample, replace=False))]
    off = [(((b * cfg.L + l) * cfg.H + h) * cfg.S * cfg.d) for b, l, h in units]
    ref = oracle.attend(storage(Q), storage(K), storage(V), DT_NAME[Q.dtype], off, cfg.S, cfg.d)
    check_close(_gather_units(O, units), ref, V.dtype, f"attend {cfg_name}")


@pytest.mark.parametrize("S,d", [(1, 64), (5, 64), (128, 64), (200, 128), (373, 64), (373, 128), (1019, 128)])
def test_attend_odd_lengths(ac, ctx, S, d):
    """Any S on the tensor-core kernels (a last, partial 128-row block): the paper's context lengths (Table 3,
    PAPER.md:617-622: 373 and 1019 tokens) and tiny ones."""
    assert ac.attncache_variant("attend", torch.bfloat16, S, d) == "tc"
    Q, K, V = (torch.randn(2, 2, 2, S, d, device=DEV).to(torch.bfloat16) for _ in range(3))
    O = ac.attncache_attend_full(ctx, Q, K, V)
    torch.cuda.synchronize()
    units = _units([0, 1], 2, 2)
    off = [(((b * 2 + l) * 2 + h) * S * d) for b, l, h in units]
    ref = oracle.attend(storage(Q), storage(K), storage(V), "bf16", off, S, d)
    check_close(_gather_units(O, units), ref, torch.bfloat16, "attend odd")
    if S == 1:
        assert torch.equal(O, V)


@pytest.mark.parametrize("S,d", [(200, 64), (376, 128), (1016, 128), (40, 64)])
def test_partial_blocks_apply_capture_attend(ac, ctx, S, d):
    """S % 128 != 0 on the tensor-core A.V and capture kernels (maps need S % 8 == 0: 16-byte map rows):
    A.V against the oracle with PACKED and DENSE maps, the captured maps against the oracle's causal softmax
    (DENSE zeros above the diagonal, PACKED row lengths), and capture -> reuse equal to attention."""
    assert ac.attncache_variant("apply", torch.bfloat16, S, d) == "tc"
    assert ac.attncache_variant("capture", torch.bfloat16, S, d) == "tc"
    g = torch.Generator(device=DEV).manual_seed(S + d)
    B, L, H, N = 3, 2, 2, 4
    Qm, Km = (torch.randn(N, L, H, S, d, device=DEV, generator=g).to(torch.bfloat16) for _ in range(2))
    dense = ac.attncache_capture_maps(ctx, Qm, Km, packed=False)
    packed = ac.attncache_capture_maps(ctx, Qm, Km, packed=True)
    units = _units(list(range(N)), L, H)
    off = [(((b * L + l) * H + h) * S * d) for b, l, h in units]
    P = oracle.attention_map(storage(Qm), storage(Km), "bf16", off, S, d)
    got = torch.stack([dense[b, l, h] for b, l, h in units]).double().cpu().numpy()
    iu = np.triu_indices(S, 1)
    assert np.all(got[:, iu[0], iu[1]] == 0.0)
    assert np.max(np.abs(got - P)) <= 3e-3
    x = _normed(N, 1024, torch.bfloat16, 5)
    db_p = ac.Database(ctx, x, packed, packed=True, seq_len=S)
    db_d = ac.Database(ctx, x, dense)
    assert torch.equal(torch.stack([ac.attncache_fetch_maps(db_p, e) for e in range(N)]), dense)
    V = torch.randn(B, L, H, S, d, device=DEV, generator=g).to(torch.bfloat16)
    idx = torch.tensor([2, 0, 3], device=DEV)
    O_p = ac.attncache_apply_cached(db_p, idx, V)
    O_d = ac.attncache_apply_cached(db_d, idx, V)
    torch.cuda.synchronize()
    assert torch.equal(O_p, O_d)
    u = _units(list(range(B)), L, H)
    ref = _apply_ref(storage(dense), "bf16", idx.cpu().numpy(), storage(V), "bf16", u, L, H, S, d)
    check_close(_gather_units(O_p, u), ref, torch.bfloat16, f"apply S={S}")
    # capture -> reuse: A.V with the captured maps of (Q, K) is attention on (Q, K, V) up to map rounding
    Qa, Ka = Qm[[2, 0, 3]].contiguous(), Km[[2, 0, 3]].contiguous()
    O_att = ac.attncache_attend_full(ctx, Qa, Ka, V)
    torch.cuda.synchronize()
    d_max = (O_att.double() - O_p.double()).abs().max().item()
    assert d_max < 3e-2, d_max


@pytest.mark.parametrize("S,d", [(128, 64), (256, 128), (200, 64)])
def test_fp16_tensor_core_paths(ac, ctx, S, d):
    """The fp16 variants of the tensor-core kernels (the configs are bf16): capture of fp16 maps from fp16
    Q, K, A.V with those maps (single-row-block and paired kernels), attention, each against the oracle."""
    assert ac.attncache_variant("apply", torch.float16, S, d) == "tc"
    g = torch.Generator(device=DEV).manual_seed(S * 7 + d)
    N, B, L, H = 3, 2, 2, 2
    Qm, Km = (torch.randn(N, L, H, S, d, device=DEV, generator=g).to(torch.float16) for _ in range(2))
    maps = ac.attncache_capture_maps(ctx, Qm, Km, map_dtype=torch.float16, packed=True)
    db = ac.Database(ctx, _normed(N, 1024, torch.bfloat16, 9), maps, packed=True, seq_len=S)
    dense = torch.stack([ac.attncache_fetch_maps(db, e) for e in range(N)])
    units_m = _units(list(range(N)), L, H)
    off_m = [(((b * L + l) * H + h) * S * d) for b, l, h in units_m]
    P = oracle.attention_map(storage(Qm), storage(Km), "f16", off_m, S, d)
    assert np.max(np.abs(torch.stack([dense[b, l, h] for b, l, h in units_m]).double().cpu().numpy() - P)) <= 2e-3
    Q, K, V = (torch.randn(B, L, H, S, d, device=DEV, generator=g).to(torch.float16) for _ in range(3))
    idx = torch.tensor([2, 0], device=DEV)
    O = ac.attncache_apply_cached(db, idx, V)
    A = ac.attncache_attend_full(ctx, Q, K, V)
    torch.cuda.synchronize()
    u = _units(list(range(B)), L, H)
    ref = _apply_ref(storage(dense), "f16", idx.cpu().numpy(), storage(V), "f16", u, L, H, S, d)
    check_close(_gather_units(O, u), ref, torch.float16, f"fp16 apply S={S}")
    off = [(((b * L + l) * H + h) * S * d) for b, l, h in u]
    ref = oracle.attend(storage(Q), storage(K), storage(V), "f16", off, S, d)
    check_close(_gather_units(A, u), ref, torch.float16, f"fp16 attend S={S}")


def test_capture_then_reuse_matches_full_attention(ac, ctx):
    """maps captured from an input, stored as a DB entry, reproduce full attention."""
    cfg = synth.CONFIGS["llama32_1b"].with_(N=2, L=2, H=4)
    Q, K, V = (synth.activations(cfg, k, 0, 1, device=DEV) for k in "qkv")
    units = _units([0], cfg.L, cfg.H)
    off = [((l * cfg.H + h) * cfg.S * cfg.d) for _, l, h in units]
    P = oracle.attention_map(storage(Q), storage(K), "bf16", off, cfg.S, cfg.d)  # fp64 capture
    maps = torch.zeros(2, cfg.L, cfg.H, cfg.S, cfg.S, dtype=torch.bfloat16)
    maps[1] = torch.from_numpy(P.reshape(cfg.L, cfg.H, cfg.S, cfg.S)).to(torch.bfloat16)
    db = ac.Database(ctx, synth.features(cfg, 0, 2, DEV), maps.to(DEV))
    O_reuse = ac.attncache_apply_cached(db, torch.tensor([1], device=DEV), V)
    O_full = ac.attncache_attend_full(ctx, Q, K, V)
    torch.cuda.synchronize()
    ref = oracle.attend(storage(Q), storage(K), storage(V), "bf16", off, cfg.S, cfg.d)
    check_close(O_reuse[0].reshape(-1, cfg.S, cfg.d), ref, torch.bfloat16, "reuse")
    check_close(O_full[0].reshape(-1, cfg.S, cfg.d), ref, torch.bfloat16, "full")


# ------------------------------------------------------------------------------------------------
# the whole step at BASELINE.json configs[1] full size, as bench.py runs it
# ------------------------------------------------------------------------------------------------

@pytest.mark.slow
@pytest.mark.parametrize("cfg_name", ["llama32_1b", "llama3_8b", "long_prefill"])
def test_full_step(ac, ctx, cfg_name):
    """BASELINE.json configs[1-3] at full size in the launch configuration bench.py times (the bench's PACKED
    DB, the whole batch in one step): every search decision checked, sampled A.V and attention units vs the
    oracle."""
    from paper_2510_25979_b200.pipeline import PrefillStep
    cfg = synth.CONFIGS[cfg_name]
    x = synth.features(cfg, 0, cfg.N, DEV)
    # the bench's DB: PACKED maps built by the library from the generator's dense maps
    maps = ac.pack_db_maps(lambda b, out: synth.fill_maps(cfg, out, b), cfg.N, cfg.L, cfg.H, cfg.S,
                           torch.bfloat16, DEV, chunk=max(1, (1 << 30) // cfg.map_bytes_per_entry))
    db = ac.Database(ctx, x, maps, packed=True, seq_len=cfg.S)
    q, pos, tgt = synth.queries(cfg, DEV)
    Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=DEV) for k in "qkv")
    O = torch.empty_like(V)
    step = PrefillStep(ctx, db, cfg.tau)
    idx, score, hit = step(q, Q, K, V, O)
    ctx.sync()
    check_search(q, x, idx, score, hit, cfg.tau)
    assert hit.sum().item() == cfg.n_hit and idx[pos].cpu().tolist() == tgt.tolist()
    rng = np.random.default_rng(2)
    hits = torch.nonzero(hit).flatten().tolist()
    misses = torch.nonzero(hit == 0).flatten().tolist()
    hu = [(hits[i], int(rng.integers(cfg.L)), int(rng.integers(cfg.H))) for i in rng.choice(len(hits), 24)]
    hu.append((hits[-1], cfg.L - 1, cfg.H - 1))
    ents = idx.cpu().numpy()
    dense = {e: synth.maps(cfg, int(e), 1, DEV)[0] for e in set(int(ents[b]) for b, _, _ in hu)}
    A_np = np.stack([storage(dense[int(ents[b])][l, h]) for b, l, h in hu]).reshape(-1)
    v_off = [(((b * cfg.L + l) * cfg.H + h) * cfg.S * cfg.d) for b, l, h in hu]
    Vs = storage(V)
    ref = oracle.apply(A_np, "bf16", [u * cfg.S * cfg.S for u in range(len(hu))], Vs, "bf16", v_off, cfg.S, cfg.d)
    check_close(_gather_units(O, hu), ref, torch.bfloat16, "step apply")
    mu = [(misses[i], int(rng.integers(cfg.L)), int(rng.integers(cfg.H))) for i in rng.choice(len(misses), 12)]
    off = [(((b * cfg.L + l) * cfg.H + h) * cfg.S * cfg.d) for b, l, h in mu]
    ref = oracle.attend(storage(Q), storage(K), Vs, "bf16", off, cfg.S, cfg.d)
    check_close(_gather_units(O, mu), ref, torch.bfloat16, "step attend")
    del db, maps, Q, K, V, O
    torch.cuda.empty_cache()


@pytest.mark.parametrize("layout", [False, True])
def test_collective_ctx_world1_matches_single_gpu_step(ac, ctx, monkeypatch, layout):
    """The library's collective calls over its own NCCL communicator (a world-1 ctx made from a unique id;
    ATTNCACHE_FORCE_ROUTE makes apply_cached take the routed path - route plan, count exchange, V and idx
    sent to the owner, A.V, O returned and scattered - even at world 1) reproduce the local single-GPU step
    bitwise, with and without a declared batch layout (the counts all-gather + host sync vs none); the
    owner-affinity calls (search_all, device plan, relocate_rows, local apply) likewise.  The multi-rank
    protocol is covered by tests/test_dist_gloo.py and test_torchrun_world (>= 2 GPUs)."""
    from paper_2510_25979_b200.dist import AffinityPrefill, ShardedPrefill
    from paper_2510_25979_b200.pipeline import PrefillStep
    monkeypatch.setenv("ATTNCACHE_FORCE_ROUTE", "1")
    cctx = ac.Context(0, rank=0, world=1, uid=ac.attncache_get_unique_id())
    assert ac.attncache_ctx_info(cctx) == (0, 1)
    cfg = synth.CONFIGS["llama32_1b"].with_(N=64, B=16, L=2)
    x = synth.features(cfg, 0, cfg.N, DEV)
    maps = ac.attncache_pack_maps(synth.maps(cfg, 0, cfg.N, DEV))
    db = ac.Database(ctx, x, maps, packed=True, seq_len=cfg.S)
    cdb = ac.Database(cctx, x, maps, packed=True, seq_len=cfg.S)          # collective load (world 1)
    q, pos, tgt = synth.queries(cfg, DEV)
    Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=DEV) for k in "qkv")
    O1, O2 = torch.empty_like(V), torch.empty_like(V)
    r1 = PrefillStep(ctx, db, cfg.tau)(q, Q, K, V, O1)
    r2 = ShardedPrefill(cctx, cdb, cfg.tau, sizes=[cfg.B] if layout else None)(q, Q, K, V, O2)
    cctx.sync()
    for a, b in zip(r1, r2):
        assert torch.equal(a, b)
    assert torch.equal(O1, O2)
    # owner-affinity placement: at world size 1 every query is local and the result is the same
    aff = AffinityPrefill(cctx, cdb, cfg.tau, sizes=[cfg.B], hit_cost=1.0, miss_cost=1.3)
    plan = aff.plan(q)
    loc = aff.local_queries(plan)
    assert loc.tolist() == list(range(cfg.B))
    assert torch.equal(plan["idx"], r1[0]) and torch.equal(plan["hit"], r1[2])
    X = torch.randn(cfg.B, cfg.S, 64, device=DEV, dtype=torch.bfloat16)
    assert torch.equal(aff.relocate(X, plan), X)
    O3 = torch.empty_like(V)
    aff.apply_local(plan, loc, V, O3, Q, K)
    cctx.sync()
    assert torch.equal(O1, O3)
    # a layout that disagrees with the call is an error, not a hang
    cctx.set_batch_layout([cfg.B + 1])
    with pytest.raises(ac.AttnCacheError) as e:
        ac.attncache_search(cdb, q, cfg.tau)
    assert e.value.name == "ATTNCACHE_ERR_STATE"
    cctx.set_batch_layout(None)
    del cdb
    cctx.close()


def test_host_prefill_pipeline_matches_device_step(ac, ctx):
    """pipeline.HostPrefill (pinned host buffers, chunked copies overlapping the kernels, ragged last
    chunk) returns exactly what the device-resident step computes."""
    from paper_2510_25979_b200.pipeline import HostPrefill, PrefillStep
    cfg = synth.CONFIGS["llama32_1b"].with_(N=48, B=37, L=2)
    x = synth.features(cfg, 0, cfg.N, DEV)
    maps = ac.attncache_pack_maps(synth.maps(cfg, 0, cfg.N, DEV))
    db = ac.Database(ctx, x, maps, packed=True, seq_len=cfg.S)
    q, _, _ = synth.queries(cfg, DEV)
    Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=DEV) for k in "qkv")
    step = PrefillStep(ctx, db, cfg.tau)
    O_dev = torch.empty_like(V)
    ref = step(q, Q, K, V, O_dev)
    Oh = torch.empty(V.shape, dtype=V.dtype).pin_memory()
    got = HostPrefill(step, chunk=8, depth=2)(q.cpu().pin_memory(), Q.cpu().pin_memory(), K.cpu().pin_memory(),
                                               V.cpu().pin_memory(), Oh)
    torch.cuda.synchronize()
    for r, g in zip(ref, got):
        assert torch.equal(r.cpu(), g)
    assert torch.equal(O_dev.cpu(), Oh)


def test_repeat_runs_are_bitwise_identical(ac, ctx):
    """racecheck does not see the async proxy (TMA/tcgen05), so every tensor-core
    kernel is re-run on identical inputs and must reproduce its output bit for bit."""
    for name, over in (("llama32_1b", dict(N=24, B=10, L=2)), ("llama3_8b", dict(N=24, B=10, L=2)),
                       ("long_prefill", dict(N=4, B=3, L=1))):
        cfg = synth.CONFIGS[name].with_(**over)
        x = synth.features(cfg, 0, cfg.N, DEV)
        maps = ac.attncache_pack_maps(synth.maps(cfg, 0, cfg.N, DEV))
        db = ac.Database(ctx, x, maps, packed=True, seq_len=cfg.S)
        q, _, _ = synth.queries(cfg, DEV)
        Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=DEV) for k in "qkv")
        idx0 = torch.arange(cfg.B, device=DEV) % cfg.N
        ref = None
        for _ in range(20):
            s = ac.attncache_search(db, q, cfg.tau)
            Oa = ac.attncache_apply_cached(db, idx0, V)
            Of = ac.attncache_attend_full(ctx, Q, K, V)
            cur = (*s, Oa, Of)
            if ref is None:
                ref = tuple(t.clone() for t in cur)
            else:
                assert all(torch.equal(a, b) for a, b in zip(ref, cur)), name


def test_sm_budget_does_not_change_results(ac):
    """attncache_ctx_set_sm_budget: every kernel's output is independent of its CTA count, so a
    small budget (odd CTA counts, fewer CTAs than work items) must reproduce the default run bit for bit; the
    setter rejects values outside [1, SM count]."""
    c = ac.Context(0)
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    for name, over in (("llama32_1b", dict(N=24, B=10, L=2)), ("llama3_8b", dict(N=24, B=10, L=2)),
                       ("long_prefill", dict(N=4, B=3, L=1))):
        cfg = synth.CONFIGS[name].with_(**over)
        x = synth.features(cfg, 0, cfg.N, DEV)
        maps = ac.attncache_pack_maps(synth.maps(cfg, 0, cfg.N, DEV))
        db = ac.Database(c, x, maps, packed=True, seq_len=cfg.S)
        q, _, _ = synth.queries(cfg, DEV)
        Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=DEV) for k in "qkv")
        idx0 = torch.arange(cfg.B, device=DEV) % cfg.N
        out = []
        for budget in (None, (7, 3), (1, 1)):
            if budget is not None:
                c.set_sm_budget(*budget)
            s = ac.attncache_search(db, q, cfg.tau)
            Oa = ac.attncache_apply_cached(db, idx0, V)
            Of = ac.attncache_attend_full(c, Q, K, V)
            cap = ac.attncache_capture_maps(c, Q[:1], K[:1])
            out.append(tuple(t.clone() for t in (*s, Oa, Of, cap)))
        c.set_sm_budget(sms, sms)
        for o in out[1:]:
            assert all(torch.equal(a, b) for a, b in zip(out[0], o)), name
        del db
    for bad in ((0, 10), (10, 0), (sms + 1, 10), (10, sms + 1)):
        with pytest.raises(ac.AttnCacheError):
            c.set_sm_budget(*bad)


@pytest.mark.parametrize("cfg_name,B,n_sample", [("tiny", 2, None), ("llama32_1b", 2, 24), ("llama3_8b", 1, 12),
                                                 ("long_prefill", 1, 4)])
@pytest.mark.parametrize("packed", [False, True])
def test_capture_maps_match_oracle_attention_map(ac, ctx, cfg_name, B, n_sample, packed):
    """§8(f) f1: captured maps = the oracle's fp64 causal softmax (Eq. 5) rounded to the map dtype;
    exact zeros above the diagonal, rows sum to 1 within the map dtype's rounding."""
    cfg = synth.CONFIGS[cfg_name].with_(L=min(2, synth.CONFIGS[cfg_name].L))
    Q, K = (synth.activations(cfg, k, 0, B, device=DEV) for k in "qk")
    mdt = synth.torch_dtype(cfg.map_dtype)
    maps = ac.attncache_capture_maps(ctx, Q, K, map_dtype=mdt, packed=packed)
    dense = maps
    torch.cuda.synchronize()
    if packed:  # expand through a DB for comparison (fetch returns DENSE maps)
        db = ac.Database(ctx, synth.features(cfg.with_(N=B), 0, B, DEV), maps, packed=True, seq_len=cfg.S)
        dense = torch.stack([ac.attncache_fetch_maps(db, b) for b in range(B)])
    units = _units(list(range(B)), cfg.L, cfg.H)
    if n_sample:
        rng = np.random.default_rng(3)
        units = [units[i] for i in sorted(rng.choice(len(units), n_sample, replace=False))]
    off = [(((b * cfg.L + l) * cfg.H + h) * cfg.S * cfg.d) for b, l, h in units]
    P = oracle.attention_map(storage(Q), storage(K), DT_NAME[Q.dtype], off, cfg.S, cfg.d)
    got = torch.stack([dense[b, l, h] for b, l, h in units]).double().cpu().numpy()
    iu = np.triu_indices(cfg.S, 1)
    assert np.all(got[:, iu[0], iu[1]] == 0.0)
    assert np.max(np.abs(got - P)) <= 3e-3
    assert np.max(np.abs(got.sum(-1) - 1.0)) <= 2.5e-3


def test_capture_then_reuse_through_the_gpu_path(ac, ctx):
    """Capture maps with the GPU (DB building), store them as PACKED DB entries, then the hit branch
    A.V reproduces the miss branch's attention (at configs[1] shapes)."""
    cfg = synth.CONFIGS["llama32_1b"].with_(L=2, N=3)
    Q, K, V = (synth.activations(cfg, k, 0, 3, device=DEV) for k in "qkv")
    maps = ac.attncache_capture_maps(ctx, Q, K, map_dtype=torch.bfloat16, packed=True)
    db = ac.Database(ctx, synth.features(cfg, 0, 3, DEV), maps, packed=True, seq_len=cfg.S)
    O_reuse = ac.attncache_apply_cached(db, torch.tensor([0, 1, 2], device=DEV), V)
    O_full = ac.attncache_attend_full(ctx, Q, K, V)
    torch.cuda.synchronize()
    units = _units([0, 1, 2], cfg.L, cfg.H)
    off = [(((b * cfg.L + l) * cfg.H + h) * cfg.S * cfg.d) for b, l, h in units]
    ref = oracle.attend(storage(Q), storage(K), storage(V), "bf16", off, cfg.S, cfg.d)
    check_close(_gather_units(O_reuse, units), ref, torch.bfloat16, "captured reuse")
    check_close(_gather_units(O_full, units), ref, torch.bfloat16, "full")


def test_rope_kernel_matches_oracle(ac, ctx):
    """f4 support kernel: RoPE (rotate-half, reading R29) against the oracle.  fp32 angles p*theta
    carry ~3 ulp relative error, i.e. up to S*3*2^-24 ~ 2e-4 rad at S = 1024, times |x| <~ 5.  Covers the
    16-byte 16-bit path (d % 16 == 0), the scalar path (fp32; d = 40) and long sequences."""
    cases = ((torch.float32, 256, 128, 3e-4), (torch.bfloat16, 256, 128, 2e-2), (torch.float16, 1024, 64, 4e-3),
             (torch.bfloat16, 1024, 128, 2e-2), (torch.bfloat16, 48, 40, 2e-2))
    for dtype, S, d, tol in cases:
        X = torch.randn(3, 2, S, d, device=DEV).to(dtype)
        ref = oracle.rope(storage(X), DT_NAME[dtype], S, d, base=500000.0)
        Y = ac.attncache_rope(X.clone(), 500000.0)
        torch.cuda.synchronize()
        err = np.abs(Y.double().cpu().numpy().reshape(ref.shape) - ref).max()
        assert err <= tol, (dtype, S, d, err)


def test_eq5_block_cached_equals_full_with_captured_maps(ac, ctx):
    """f4: with maps captured from the block's own Q, K (RoPE applied) the cached block (V projection
    + A.V) reproduces the full block (projections + RoPE + attention) — Alg. 2's two branches agree."""
    from paper_2510_25979_b200.block import AttentionBlock
    cfg = synth.CONFIGS["llama32_1b"].with_(B=3, N=3, L=1, H=4)
    X, (Wq, Wk, Wv) = synth.block_inputs(cfg, DEV)
    db0 = ac.Database(ctx, synth.features(cfg, 0, 3, DEV),
                      torch.zeros(3, 1, cfg.H, ac.attncache_packed_map_elems(cfg.S), dtype=torch.bfloat16, device=DEV),
                      packed=True, seq_len=cfg.S)
    blk = AttentionBlock(ctx, db0, Wq, Wk, Wv, cfg.H, cfg.d)
    Q, K = blk._proj(X, blk.Wq), blk._proj(X, blk.Wk)
    ac.attncache_rope(Q, blk.rope_base)
    ac.attncache_rope(K, blk.rope_base)
    maps = ac.attncache_capture_maps(ctx, Q, K, packed=True)
    blk.db = ac.Database(ctx, synth.features(cfg, 0, 3, DEV), maps, packed=True, seq_len=cfg.S)
    idx = torch.arange(3, device=DEV)
    O_full = blk.full(X)
    O_cached = blk.cached(X, idx, torch.ones(3, dtype=torch.uint8, device=DEV), idx[:0])
    O_mixed = blk.cached(X, idx, torch.tensor([1, 0, 1], dtype=torch.uint8, device=DEV), idx[1:2])
    torch.cuda.synchronize()
    d = (O_full.double() - O_cached.double()).abs().max().item()
    assert d < 3e-2, d
    assert torch.equal(O_mixed[1], O_full[1])


def _round_bf16(a: np.ndarray) -> torch.Tensor:
    """fp64 oracle values rounded once (RN-even) to bf16: the storage dtype of the block's activations."""
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16)


@pytest.mark.parametrize("M,K,N,S,d", [(256, 256, 256, 128, 64), (3 * 96, 192, 128, 96, 32), (2 * 40, 200, 96, 40, 48)])
def test_linear_head_major_matches_oracle(ac, ctx, M, K, N, S, d):
    """f4 projections (attncache_linear): Y = X W^T stored head-major [B][H][S][d], against oracle.linear; the
    tcgen05 path (K, N multiples of 64, d % 32 == 0, ragged M) and the CUDA-core path (K = 200)."""
    g = torch.Generator(device=DEV).manual_seed(41)
    X = torch.randn(M // S, S, K, device=DEV, generator=g).to(torch.bfloat16)
    W = (torch.randn(N, K, device=DEV, generator=g) / math.sqrt(K)).to(torch.bfloat16)
    Y = ac.attncache_linear(ctx, X, W, N // d)
    ref = oracle.linear(storage(X.view(M, K)), storage(W), "bf16")            # [M][N] = [(b, s)][(h, c)]
    ref = ref.reshape(M // S, S, N // d, d).transpose(0, 2, 1, 3)              # -> [b][h][s][c]
    check_close(Y.view(M // S, N // d, S, d).reshape(-1, S, d), ref.reshape(-1, S, d), torch.bfloat16, "linear")


@pytest.mark.parametrize("n_kv", [None, 2, 1])
def test_eq5_block_matches_oracle(ac, ctx, n_kv):
    """f4 (Eq. 5; Alg. 2 l.372-381) against the oracle composed step by step: q, k, v =
    oracle.linear (rounded to the bf16 activation dtype), RoPE (oracle.rope, rounded), causal softmax attention
    (oracle.attend) for the full block; v then A.V with the DB's maps (oracle.apply) for the cached block.
    n_kv: grouped-query K / V projections (query head h reads K / V head h // (H / n_kv)); the oracle gets the
    K / V heads repeated, the multi-head definition of the same block."""
    from paper_2510_25979_b200.block import AttentionBlock
    cfg = synth.CONFIGS["llama32_1b"].with_(B=3, N=3, L=1, H=4)
    X, (Wq, Wk, Wv) = synth.block_inputs(cfg, DEV, n_kv_heads=n_kv)
    E, S, H, d = X.shape[2], cfg.S, cfg.H, cfg.d
    Hkv = H if n_kv is None else n_kv
    maps = ac.attncache_pack_maps(synth.maps(cfg, 0, 3, DEV))
    db = ac.Database(ctx, synth.features(cfg, 0, 3, DEV), maps, packed=True, seq_len=S)
    blk = AttentionBlock(ctx, db, Wq, Wk, Wv, H, d)
    assert blk.Hkv == Hkv
    O_full = blk.full(X)
    idx = torch.tensor([2, 0, 1], device=DEV)
    O_cached = blk.cached(X, idx, torch.ones(3, dtype=torch.uint8, device=DEV), idx[:0])
    O_mixed = blk.cached(X, idx, torch.tensor([0, 1, 0], dtype=torch.uint8, device=DEV), torch.tensor([0, 2], device=DEV))
    torch.cuda.synchronize()
    Xs = storage(X.view(-1, E))

    def heads(W, nh):  # oracle projection -> bf16 [B][nh][S][d], then K / V heads repeated up to H
        y = oracle.linear(Xs, storage(W), "bf16").reshape(cfg.B, S, nh, d).transpose(0, 2, 1, 3)
        return _round_bf16(y.copy()).repeat_interleave(H // nh, dim=1).contiguous()

    Qo, Ko, Vo = heads(Wq, H), heads(Wk, Hkv), heads(Wv, Hkv)
    Qr = _round_bf16(oracle.rope(storage(Qo), "bf16", S, d, base=blk.rope_base))
    Kr = _round_bf16(oracle.rope(storage(Ko), "bf16", S, d, base=blk.rope_base))
    units = [(b, h) for b in range(cfg.B) for h in range(H)]
    off = [((b * H + h) * S * d) for b, h in units]
    ref = oracle.attend(storage(Qr), storage(Kr), storage(Vo), "bf16", off, S, d)
    check_close(torch.stack([O_full[b, 0, h] for b, h in units]), ref, torch.bfloat16, "eq5 full block")
    check_close(torch.stack([O_mixed[b, 0, h] for b, h in units if b != 1]),
                ref[[i for i, (b, h) in enumerate(units) if b != 1]], torch.bfloat16, "eq5 mixed block (misses)")
    dense = storage(synth.maps(cfg, 0, 3, DEV))
    a_off = [((int(idx[b]) * H + h) * S * S) for b, h in units]
    ref = oracle.apply(dense, "bf16", a_off, storage(Vo), "bf16", off, S, d)
    check_close(torch.stack([O_cached[b, 0, h] for b, h in units]), ref, torch.bfloat16, "eq5 cached block")
    check_close(torch.stack([O_mixed[1, 0, h] for h in range(H)]), ref[H:2 * H], torch.bfloat16,
                "eq5 mixed block (hit)")


@pytest.mark.parametrize("cfg_name,N,B", [("tiny", 5, 3), ("llama32_1b", 4, 3), ("llama3_8b", 2, 2)])
def test_apply_noncausal_encoder_maps(ac, ctx, cfg_name, N, B):
    """f3: bidirectional (encoder) maps — A.V over every column."""
    cfg = synth.CONFIGS[cfg_name].with_(N=N, L=min(2, synth.CONFIGS[cfg_name].L))
    maps = synth.maps(cfg, 0, N, DEV, causal=False)
    db = ac.Database(ctx, synth.features(cfg, 0, N, DEV), maps, causal=False)
    idx = torch.tensor([(2 * b + 1) % N for b in range(B)], device=DEV)
    V = synth.activations(cfg, "v", 0, B, device=DEV)
    O = ac.attncache_apply_cached(db, idx, V)
    torch.cuda.synchronize()
    units = _units(list(range(B)), cfg.L, cfg.H)
    ref = _apply_ref(storage(maps), cfg.map_dtype, idx.cpu().numpy(), storage(V), cfg.act_dtype, units, cfg.L, cfg.H,
                     cfg.S, cfg.d)
    check_close(_gather_units(O, units), ref, V.dtype, f"non-causal {cfg_name}")
    with pytest.raises(ac.AttnCacheError):
        ac.Database(ctx, synth.features(cfg, 0, N, DEV), ac.attncache_pack_maps(maps), packed=True, seq_len=cfg.S,
                    causal=False)


def test_per_layer_search_attncache_f(ac, ctx):
    """f3 AttnCache-f: one feature DB per layer sharing the map DB's index; each layer applies the
    maps of its own top-1 entry (or runs full attention on its misses)."""
    from paper_2510_25979_b200.pipeline import PerLayerPrefill
    base = synth.CONFIGS["llama32_1b"].with_(N=32, B=6, L=2)
    maps = synth.maps(base, 0, base.N, DEV)
    map_db = ac.Database(ctx, synth.features(base, 0, base.N, DEV), maps)
    cfgs = [base.with_(seed=100 + l) for l in range(base.L)]  # each layer: its own embeddings
    fdbs = [ac.Database(ctx, synth.features(c, 0, c.N, DEV)) for c in cfgs]
    step = PerLayerPrefill(ctx, map_db, fdbs, base.tau)
    for l, c in enumerate(cfgs):
        q, pos, tgt = synth.queries(c, DEV)
        Q, K, V = (synth.activations(base, k, 0, base.B, layer_begin=l, layer_end=l + 1, device=DEV) for k in "qkv")
        O = torch.empty_like(V)
        idx, score, hit = step.layer(l, q, Q, K, V, O)
        torch.cuda.synchronize()
        assert idx[pos].cpu().tolist() == tgt.tolist()
        for b in range(base.B):
            units = [(b, 0, h) for h in range(base.H)]
            v_off = [(((b * 1 + 0) * base.H + h) * base.S * base.d) for _, _, h in units]
            if hit[b]:
                a_off = [((int(idx[b]) * base.L + l) * base.H + h) * base.S * base.S for _, _, h in units]
                ref = oracle.apply(storage(maps), "bf16", a_off, storage(V), "bf16", v_off, base.S, base.d)
            else:
                ref = oracle.attend(storage(Q), storage(K), storage(V), "bf16", v_off, base.S, base.d)
            check_close(_gather_units(O, units), ref, torch.bfloat16, f"layer {l} row {b}")


# ------------------------------------------------------------------------------------------------
# feature projector (f2; Alg. 1 l.254; readings R30-R32)
# ------------------------------------------------------------------------------------------------

def _project_check(ac, ctx, cfg, B, E, Hd, feat_dtype=None, tc=True):
    h, W1, b1, W2, b2 = synth.projector_inputs(cfg, B=B, device=DEV, E=E, hidden=Hd)
    f = ac.attncache_project_features(ctx, h, W1, b1, W2, b2, feat_dtype=feat_dtype)
    torch.cuda.synchronize()
    assert ac.attncache_variant("project", h.dtype, E, Hd) == ("tc" if tc else "ffma")
    dt = DT_NAME[h.dtype]
    ref = oracle.project(storage(h), dt, storage(W1), b1.cpu().numpy(), storage(W2), b2.cpu().numpy())
    # one "unit" per row: max-abs over all elements, rel-L2 per row (north_star bf16 bounds; fp32: _util)
    check_close(f.unsqueeze(1), ref[:, None, :], f.dtype, f"project {cfg.name} B={B} E={E} Hd={Hd}")
    return f, (h, W1, b1, W2, b2)


@pytest.mark.parametrize("name,B", [("llama32_1b", 256), ("llama32_1b", 1), ("llama32_1b", 130),
                                    ("llama3_8b", 37), ("search_sweep", 257)])
def test_project_parity_tc(ac, ctx, name, B):
    cfg = synth.CONFIGS[name]
    f, _ = _project_check(ac, ctx, cfg, B, synth.EMBED_DIM[name], cfg.D)
    n = f.double().norm(dim=1)
    assert torch.all((n - 1).abs() < 1e-2)                 # unit rows (bf16 rounding of each element)


def test_project_parity_ffma_paths(ac, ctx):
    """fp32 (configs[0], FFMA) and a bf16 shape the tensor-core path does not take (dims not multiples of 64)."""
    _project_check(ac, ctx, synth.CONFIGS["tiny"], 8, 256, 384, tc=False)
    cfg = synth.CONFIGS["llama32_1b"].with_(D=40)
    _project_check(ac, ctx, cfg, 19, 200, 72, tc=False)


def test_project_deterministic_and_zero_output(ac, ctx):
    cfg = synth.CONFIGS["llama32_1b"]
    h, W1, b1, W2, b2 = synth.projector_inputs(cfg, B=300, device=DEV)
    f1 = ac.attncache_project_features(ctx, h, W1, b1, W2, b2)
    f2 = ac.attncache_project_features(ctx, h, W1, b1, W2, b2)
    assert torch.equal(f1, f2)
    z = ac.attncache_project_features(ctx, h, W1, b1, torch.zeros_like(W2), torch.zeros_like(b2))
    assert torch.equal(z, torch.zeros_like(z))             # y = 0 gives f = 0 (reading R32)


def test_project_then_search(ac, ctx):
    """Alg. 1 l.254-257 end to end: DB rows and queries both embedded by the projector (Fig. 4 step 2),
    queries are noisy copies of DB embeddings; the search decisions on the projected features follow the
    exactness rule and the planted rows are found."""
    cfg = synth.CONFIGS["llama32_1b"]
    E = synth.EMBED_DIM[cfg.name]
    h_db, W1, b1, W2, b2 = synth.projector_inputs(cfg, B=500, device=DEV)
    feats = ac.attncache_project_features(ctx, h_db, W1, b1, W2, b2)
    g = torch.Generator(device=DEV).manual_seed(3)
    rows = torch.tensor([3, 77, 499, 250], device=DEV)
    hq = h_db[rows].float() + 0.01 * torch.randn(len(rows), E, device=DEV, generator=g)
    hq = torch.cat([hq, torch.randn(4, E, device=DEV, generator=g)]).to(h_db.dtype)
    q = ac.attncache_project_features(ctx, hq, W1, b1, W2, b2)
    db = ac.Database(ctx, feats)
    idx, score, hit = ac.attncache_search(db, q, 0.9)
    torch.cuda.synchronize()
    check_search(q, feats, idx, score, hit, 0.9)
    assert idx[:4].tolist() == rows.tolist() and hit[:4].tolist() == [1] * 4


def test_project_errors(ac, ctx):
    cfg = synth.CONFIGS["llama32_1b"]
    h, W1, b1, W2, b2 = synth.projector_inputs(cfg, B=4, device=DEV)
    L = ac.load_library()
    args = (W1.data_ptr(), b1.data_ptr(), W1.shape[0], W2.data_ptr(), b2.data_ptr(), W2.shape[0], 2)
    assert L.attncache_project_features(ctx.handle, None, 4, h.shape[1], 2, *args, None, None) == 1  # NULL h
    f = torch.empty(4, cfg.D, dtype=torch.bfloat16, device=DEV)
    assert L.attncache_project_features(ctx.handle, h.data_ptr(), 4, 0, 2, *args, f.data_ptr(), None) == 2  # SHAPE
    assert L.attncache_project_features(ctx.handle, h.data_ptr(), 4, 196, 2, *args, f.data_ptr(), None) == 4  # pitch
    out = ac.attncache_project_features(ctx, h[:0], W1, b1, W2, b2)
    assert out.shape == (0, cfg.D)


# ------------------------------------------------------------------------------------------------
# grouped-query attention (SURVEY.md §8(f) f3 "optional GQA n_kv_heads"): a query head h reads K/V
# head h // (H // Hkv).  The expected values repeat the K/V heads on the host (GQA is MHA with shared
# K/V heads) and use the MHA oracle; the library reads the un-repeated tensors.
# ------------------------------------------------------------------------------------------------

def _repeat_heads(X, H):
    """[B][L][Hkv][S][d] -> [B][L][H][S][d] (host-side reference construction)."""
    return X.repeat_interleave(H // X.shape[2], dim=2).contiguous()


@pytest.mark.parametrize("cfg_name,N,B,Hkv,n_sample", [("llama32_1b", 12, 3, 2, 48), ("llama32_1b", 12, 3, 1, 48),
                                                       ("llama3_8b", 4, 2, 4, 24), ("tiny", 6, 3, 2, None)])
def test_gqa_apply_attend_capture(ac, ctx, cfg_name, N, B, Hkv, n_sample):
    base = synth.CONFIGS[cfg_name]
    cfg = base.with_(N=N, B=B, L=2, H=8 if base.H > 4 else 4)
    H = cfg.H
    x = synth.features(cfg, 0, cfg.N, DEV)
    maps = synth.maps(cfg, 0, cfg.N, DEV)
    db = ac.Database(ctx, x, maps)
    g = torch.Generator(device=DEV).manual_seed(11)
    adt = synth.torch_dtype(cfg.act_dtype)
    Q = torch.randn(B, cfg.L, H, cfg.S, cfg.d, device=DEV, generator=g).to(adt)
    K, V = (torch.randn(B, cfg.L, Hkv, cfg.S, cfg.d, device=DEV, generator=g).to(adt) for _ in range(2))
    idx = torch.randperm(cfg.N, generator=torch.Generator().manual_seed(1))[:B].to(DEV)
    O_apply = ac.attncache_apply_cached(db, idx, V)
    O_att = ac.attncache_attend_full(ctx, Q, K, V)
    torch.cuda.synchronize()
    assert O_apply.shape == Q.shape and O_att.shape == Q.shape
    Vr, Kr = _repeat_heads(V, H), _repeat_heads(K, H)
    units = _units(list(range(B)), cfg.L, H)
    if n_sample:
        rng = np.random.default_rng(5)
        units = [units[i] for i in sorted(rng.choice(len(units), n_sample, replace=False))]
    ents = idx.cpu().numpy()
    ref = _apply_ref(storage(maps), cfg.map_dtype, ents, storage(Vr), cfg.act_dtype, units, cfg.L, H, cfg.S, cfg.d)
    check_close(_gather_units(O_apply, units), ref, adt, f"gqa apply {cfg_name} Hkv={Hkv}")
    off = [(((b * cfg.L + l) * H + h) * cfg.S * cfg.d) for b, l, h in units]
    ref = oracle.attend(storage(Q), storage(Kr), storage(Vr), cfg.act_dtype, off, cfg.S, cfg.d)
    check_close(_gather_units(O_att, units), ref, adt, f"gqa attend {cfg_name} Hkv={Hkv}")
    # the repeated-head MHA call gives the same bits (the kernels only index differently)
    assert torch.equal(O_apply, ac.attncache_apply_cached(db, idx, Vr))
    assert torch.equal(O_att, ac.attncache_attend_full(ctx, Q, Kr, Vr))
    if cfg.S % 8 == 0 and cfg.map_dtype in ("f16", "bf16"):
        m1 = ac.attncache_capture_maps(ctx, Q, K, map_dtype=synth.torch_dtype(cfg.map_dtype), packed=False)
        m2 = ac.attncache_capture_maps(ctx, Q, Kr, map_dtype=synth.torch_dtype(cfg.map_dtype), packed=False)
        assert torch.equal(m1, m2)


def test_gqa_errors(ac, ctx):
    cfg = synth.CONFIGS["llama32_1b"].with_(N=4, B=2, L=1, H=8)
    db = ac.Database(ctx, synth.features(cfg, 0, cfg.N, DEV), synth.maps(cfg, 0, cfg.N, DEV))
    V = torch.zeros(2, 1, 3, cfg.S, cfg.d, device=DEV, dtype=torch.bfloat16)  # 3 does not divide 8
    with pytest.raises(ac.AttnCacheError) as e:
        ac.attncache_apply_cached(db, torch.arange(2, device=DEV), V)
    assert e.value.status == 2
    Q = torch.zeros(2, 1, 8, cfg.S, cfg.d, device=DEV, dtype=torch.bfloat16)
    with pytest.raises(ac.AttnCacheError):
        ac.attncache_attend_full(ctx, Q, V, V)


# ------------------------------------------------------------------------------------------------
# multi-GPU path on one GPU: g virtual shards (one Database per contiguous entry range, SURVEY.md §4
# "fake multi-shard"), the real per-rank kernels of the routed and the owner-affinity placements, with
# local copies standing in for the NCCL exchanges; the result must equal the single-shard step bitwise
# (reading R19).  Ownership is skewed on purpose: all hits on one shard, no hits, hits only off shard 0.
# ------------------------------------------------------------------------------------------------

@pytest.mark.parametrize("pattern", ["spread", "one_shard", "no_hits", "remote_only"])
def test_virtual_shards_routed_and_affinity_equal_single_gpu(ac, ctx, pattern):
    from paper_2510_25979_b200.dist import shard_range
    from paper_2510_25979_b200.pipeline import PrefillStep
    cfg = synth.CONFIGS["llama32_1b"].with_(N=40, B=12, L=2)
    world = 3
    x = synth.features(cfg, 0, cfg.N, DEV)
    maps = ac.attncache_pack_maps(synth.maps(cfg, 0, cfg.N, DEV))
    g = torch.Generator(device=DEV).manual_seed(2)
    tg = torch.Generator().manual_seed(4)
    if pattern == "spread":
        tgt = torch.randperm(cfg.N, generator=tg)[:9]
    elif pattern == "one_shard":
        tgt = torch.randperm(shard_range(cfg.N, world, 1)[1], generator=tg)[:9] + shard_range(cfg.N, world, 1)[0]
    elif pattern == "remote_only":
        tgt = torch.randperm(cfg.N - shard_range(cfg.N, world, 0)[1], generator=tg)[:9] + shard_range(cfg.N, world, 1)[0]
    else:
        tgt = torch.tensor([], dtype=torch.int64)
    q = torch.randn(cfg.B, cfg.D, device=DEV, generator=g)
    q[:len(tgt)] = x[tgt.to(DEV)].float() + 0.001 * torch.randn(len(tgt), cfg.D, device=DEV, generator=g)
    q = (q / q.norm(dim=1, keepdim=True)).to(x.dtype)
    Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=DEV) for k in "qkv")
    O_ref = torch.empty_like(V)
    ref = PrefillStep(ctx, ac.Database(ctx, x, maps, packed=True, seq_len=cfg.S), cfg.tau)(q, Q, K, V, O_ref)
    torch.cuda.synchronize()
    dbs, begins = [], []
    for r in range(world):
        b0, c0 = shard_range(cfg.N, world, r)
        begins.append(b0)
        dbs.append(ac.Database(ctx, x[b0:b0 + c0], maps[b0:b0 + c0], n_global=cfg.N, shard_begin=b0, packed=True,
                               seq_len=cfg.S))
    # sharded search: every shard's keys over all queries ("all-gather"), decode
    keys = torch.stack([ac.attncache_search_keys(db, q) for db in dbs])
    idx, score, hit = ac.attncache_keys_decode(keys, cfg.tau)
    for a, b in zip(ref, (idx, score, hit)):
        assert torch.equal(a, b)
    sb = torch.tensor(begins + [cfg.N], dtype=torch.int64, device=DEV)
    # routed: bucket the hits by owner, ship V rows, A.V on the owner's shard, scatter O back
    owner, counts, order = ac.attncache_route_plan(idx, hit, sb)
    O_routed = torch.empty_like(V)
    off = 0
    for r, n in enumerate(counts.tolist()):
        if n:
            rows = order[off:off + n].contiguous()
            V_r = ac.attncache_gather_rows(V, rows)
            O_r = ac.attncache_apply_cached(dbs[r], ac.attncache_gather_rows(idx, rows), V_r)
            ac.attncache_scatter_rows(O_r, rows, O_routed)
        off += n
    ac.attncache_attend_full(ctx, Q, K, V, O_routed, skip=hit)
    # owner-affinity: the plan places every query once; each "rank" processes its queries locally
    assign, load = ac.attncache_affinity_plan(idx, hit, sb, 1.0, 1.3)
    O_aff = torch.empty_like(V)
    for r in range(world):
        loc = torch.nonzero(assign == r).flatten().to(DEV)
        if not loc.numel():
            continue
        V_l, Q_l, K_l = (t.index_select(0, loc).contiguous() for t in (V, Q, K))
        idx_l, hit_l = idx.index_select(0, loc).contiguous(), hit.index_select(0, loc).contiguous()
        O_l = torch.empty_like(V_l)
        ac.attncache_apply_cached(dbs[r], idx_l, V_l, O_l, hit=hit_l)
        ac.attncache_attend_full(ctx, Q_l, K_l, V_l, O_l, skip=hit_l)
        O_aff.index_copy_(0, loc, O_l)
    ctx.sync()
    assert torch.equal(O_routed, O_ref)
    assert torch.equal(O_aff, O_ref)
    # ... and against the oracle: the sharded decisions, every hit unit (A.V with the owner's maps) and every
    # miss unit (causal attention) of the routed result
    check_search(q, x, idx, score, hit, cfg.tau)
    dense = storage(synth.maps(cfg, 0, cfg.N, DEV))
    ents = idx.cpu().numpy()
    hits = torch.nonzero(hit).flatten().tolist()
    misses = torch.nonzero(hit == 0).flatten().tolist()
    if hits:
        u = _units(hits, cfg.L, cfg.H)
        ref_a = _apply_ref(dense, DT_NAME[maps.dtype], ents, storage(V), DT_NAME[V.dtype], u, cfg.L, cfg.H, cfg.S, cfg.d)
        check_close(_gather_units(O_routed, u), ref_a, V.dtype, f"virtual shards apply {pattern}")
    if misses:
        u = _units(misses, cfg.L, cfg.H)
        off = [(((b * cfg.L + l) * cfg.H + h) * cfg.S * cfg.d) for b, l, h in u]
        ref_m = oracle.attend(storage(Q), storage(K), storage(V), DT_NAME[V.dtype], off, cfg.S, cfg.d)
        check_close(_gather_units(O_routed, u), ref_m, V.dtype, f"virtual shards attend {pattern}")
    if pattern == "no_hits":
        assert int(hit.sum()) == 0
    if pattern == "one_shard":
        assert set(owner[hit.bool()].tolist()) == {1}


def test_graphed_prefill_step_equals_eager(ac, ctx):
    """pipeline.GraphedPrefillStep: the captured step replays to the eager step's bits, and a replay after
    new inputs are written into its static buffers gives the eager result for those inputs."""
    from paper_2510_25979_b200.pipeline import GraphedPrefillStep, PrefillStep
    cfg = synth.CONFIGS["llama32_1b"].with_(N=64, B=8, L=2)
    x = synth.features(cfg, 0, cfg.N, DEV)
    db = ac.Database(ctx, x, ac.attncache_pack_maps(synth.maps(cfg, 0, cfg.N, DEV)), packed=True, seq_len=cfg.S)
    step = PrefillStep(ctx, db, cfg.tau)
    q, _, _ = synth.queries(cfg, DEV)
    Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=DEV) for k in "qkv")
    gstep = GraphedPrefillStep(step, q, Q, K, V)
    O_e = torch.empty_like(V)
    ref = tuple(t.clone() for t in step(q, Q, K, V, O_e))
    out = gstep.replay()
    torch.cuda.synchronize()
    for a, b in zip((*ref, O_e), out):
        assert torch.equal(a, b)
    # new inputs: a different query batch (other hit pattern) and other activations
    q2, _, _ = synth.queries(cfg.with_(seed=5), DEV)
    Q2, K2, V2 = (synth.activations(cfg.with_(seed=5), k, 0, cfg.B, device=DEV) for k in "qkv")
    for dst, src in zip(gstep.inputs, (q2, Q2, K2, V2)):
        dst.copy_(src)
    out = tuple(t.clone() for t in gstep.replay())
    O_e2 = torch.empty_like(V)
    ref2 = step(q2, Q2, K2, V2, O_e2)
    torch.cuda.synchronize()
    for a, b in zip((*ref2, O_e2), out):
        assert torch.equal(a, b)
    # an eager call with a LARGER batch on the same ctx and stream grows (stream-ordered: frees and
    # reallocates) that stream's scratch; the graph captured its own scratch, so later replays are unaffected
    big = cfg.with_(B=48)
    qb, _, _ = synth.queries(big, DEV)
    Qb, Kb, Vb = (synth.activations(big, k, 0, big.B, device=DEV) for k in "qkv")
    step(qb, Qb, Kb, Vb, torch.empty_like(Vb))
    junk = torch.full((1 << 22,), 7, dtype=torch.int64, device=DEV)  # reuse freed memory with other bytes
    out3 = tuple(t.clone() for t in gstep.replay())
    torch.cuda.synchronize()
    for a, b in zip(out, out3):
        assert torch.equal(a, b)
    del junk


def test_binding_rejects_mismatched_buffers(ac, ctx):
    """the binding checks what the C ABI cannot see (shapes, dtypes, lengths, devices) before any
    pointer reaches the library: a wrong-width or wrong-dtype query matrix, an O of another dtype or shape, a
    hit mask of the wrong length or dtype, an int32 idx, pageable host buffers for the host-buffer call."""
    cfg = synth.CONFIGS["llama32_1b"].with_(N=8, B=3, L=2)
    x = synth.features(cfg, 0, cfg.N, DEV)
    db = ac.Database(ctx, x, ac.attncache_pack_maps(synth.maps(cfg, 0, cfg.N, DEV)), packed=True, seq_len=cfg.S)
    q, _, _ = synth.queries(cfg, DEV)
    V = synth.activations(cfg, "v", 0, cfg.B, device=DEV)
    idx = torch.zeros(cfg.B, dtype=torch.int64, device=DEV)
    bad = [lambda: ac.attncache_search(db, q[:, :512].contiguous(), 0.9),
           lambda: ac.attncache_search(db, q.float(), 0.9),
           lambda: ac.attncache_search(db, q, 0.9, idx=torch.empty(2, dtype=torch.int64, device=DEV)),
           lambda: ac.attncache_apply_cached(db, idx, V, torch.empty_like(V, dtype=torch.float32)),
           lambda: ac.attncache_apply_cached(db, idx, V, V[:2].clone()),
           lambda: ac.attncache_apply_cached(db, idx, V, hit=torch.ones(2, dtype=torch.uint8, device=DEV)),
           lambda: ac.attncache_apply_cached(db, idx, V, hit=torch.ones(cfg.B, dtype=torch.int32, device=DEV)),
           lambda: ac.attncache_apply_cached(db, idx.int(), V),
           lambda: ac.attncache_attend_full(ctx, V, V, V, torch.empty(1, device=DEV)),
           lambda: ac.attncache_attend_full(ctx, V, V, V, skip=torch.zeros(cfg.B + 1, dtype=torch.uint8, device=DEV)),
           lambda: ac.attncache_prefill_host(db, q.cpu(), V.cpu(), V.cpu(), V.cpu(), 0.9)]
    for f in bad:
        with pytest.raises(ValueError):
            f()


def test_edge_cases_empty_skipped_and_extreme_shapes(ac, ctx):
    """Empty batches are no-ops; fully skipped rows leave O (and capture outputs) untouched; the longest
    sequence the attention accepts (S = 8192) matches the oracle on sampled rows and S = 8193 is refused;
    head dims the tensor-core kernels do not take (d = 32) run on the CUDA-core kernels."""
    cfg = synth.CONFIGS["llama32_1b"].with_(N=8, B=4, L=1, H=2)
    db = ac.Database(ctx, synth.features(cfg, 0, cfg.N, DEV), synth.maps(cfg, 0, cfg.N, DEV))
    V = synth.activations(cfg, "v", 0, cfg.B, device=DEV)
    Q, K = (synth.activations(cfg, k, 0, cfg.B, device=DEV) for k in "qk")
    idx = torch.arange(cfg.B, device=DEV)
    # empty batches
    assert ac.attncache_apply_cached(db, idx[:0], V[:0]).shape[0] == 0
    assert ac.attncache_attend_full(ctx, Q[:0], K[:0], V[:0]).shape[0] == 0
    # everything skipped: outputs untouched
    O = torch.full_like(V, 7.0)
    ac.attncache_apply_cached(db, idx, V, O, hit=torch.zeros(cfg.B, dtype=torch.uint8, device=DEV))
    ac.attncache_attend_full(ctx, Q, K, V, O, skip=torch.ones(cfg.B, dtype=torch.uint8, device=DEV))
    maps = torch.full((cfg.B, cfg.L, cfg.H, ac.attncache_packed_map_elems(cfg.S)), 5.0, dtype=torch.bfloat16, device=DEV)
    ac.attncache_capture_maps(ctx, Q, K, out=maps, skip=torch.ones(cfg.B, dtype=torch.uint8, device=DEV))
    torch.cuda.synchronize()
    assert torch.all(O == 7.0) and torch.all(maps == 5.0)
    # S = 8192 (the attention's limit): sampled rows of one unit vs the oracle
    g = torch.Generator(device=DEV).manual_seed(9)
    Ql, Kl, Vl = (torch.randn(1, 1, 1, 8192, 128, device=DEV, generator=g).to(torch.bfloat16) for _ in range(3))
    Ol = ac.attncache_attend_full(ctx, Ql, Kl, Vl)
    torch.cuda.synchronize()
    ref = oracle.attend(storage(Ql), storage(Kl), storage(Vl), "bf16", [0], 8192, 128)[0]
    rows = [0, 1, 127, 128, 4095, 8191]
    check_close(Ol[0, 0, 0, rows].unsqueeze(0), ref[rows][None], torch.bfloat16, "attend S=8192")
    with pytest.raises(ac.AttnCacheError) as e:
        z = torch.zeros(1, 1, 1, 8193, 64, device=DEV, dtype=torch.bfloat16)
        ac.attncache_attend_full(ctx, z, z, z)
    assert e.value.name == "ATTNCACHE_ERR_SHAPE"
    # d = 32: CUDA-core kernels for A.V and attention
    c32 = cfg.with_(d=32)
    V32, Q32, K32 = (synth.activations(c32, k, 0, cfg.B, device=DEV) for k in "vqk")
    assert ac.attncache_variant("apply", V32.dtype, c32.S, 32) == "ffma"
    O32 = ac.attncache_apply_cached(db, idx, V32)
    A32 = ac.attncache_attend_full(ctx, Q32, K32, V32)
    torch.cuda.synchronize()
    units = _units(list(range(cfg.B)), cfg.L, cfg.H)
    ref = _apply_ref(storage(db.maps), cfg.map_dtype, idx.cpu().numpy(), storage(V32), cfg.act_dtype, units, cfg.L,
                     cfg.H, cfg.S, 32)
    check_close(_gather_units(O32, units), ref, torch.bfloat16, "apply d=32")
    off = [(((b * cfg.L + l) * cfg.H + h) * cfg.S * 32) for b, l, h in units]
    ref = oracle.attend(storage(Q32), storage(K32), storage(V32), cfg.act_dtype, off, cfg.S, 32)
    check_close(_gather_units(A32, units), ref, torch.bfloat16, "attend d=32")


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 8, 32])
def test_affinity_plan_device_matches_host(ac, ctx, world):
    """attncache_affinity_plan_device: assign and load bitwise equal to the host plan (exact ties, zero costs,
    empty shards and empty home blocks included), and every rank's lists equal to the ones derived from the
    host plan the way dist.AffinityPrefill does on the host path."""
    g = np.random.default_rng(100 + world)
    costs = [(1.0, 1.0), (2.0, 1.5), (0.0, 1.0), (1.0, 0.0), (0.0, 0.0), (3.3e6, 1.7e7)]
    for trial in range(12):
        n = int(g.choice([0, 1, 7, 300, 2048, 5000]))
        N = int(g.integers(world, 20000))
        cuts = np.sort(g.integers(0, N, world - 1)).tolist() if world > 1 else []
        sb = [0] + cuts + [N]
        hcuts = np.sort(g.integers(0, n + 1, world - 1)).tolist() if world > 1 else []
        hb = [0] + hcuts + [n]
        idx = g.integers(0, N, n).astype(np.int64)
        hit = (g.random(n) < float(g.choice([0.0, 0.5, 0.8, 1.0]))).astype(np.uint8)
        hc, mc = costs[trial % len(costs)]
        assign_h, load_h = ac.attncache_affinity_plan(idx, hit, sb, hc, mc)
        idx_d, hit_d = torch.from_numpy(idx).to(DEV), torch.from_numpy(hit).to(DEV)
        for rank in sorted({0, world - 1, int(g.integers(0, world))}):
            out = ac.attncache_affinity_plan_device(ctx, idx_d, hit_d, sb, hb, rank, hc, mc)
            torch.cuda.synchronize()
            assert np.array_equal(out["assign"].cpu().numpy(), assign_h), (world, trial, rank)
            assert np.array_equal(out["load"][:world].cpu().numpy(), load_h), (world, trial, rank)
            counts = out["counts"].cpu().tolist()
            loc = np.nonzero(assign_h == rank)[0]
            mine = assign_h[hb[rank]:hb[rank + 1]].astype(np.int64)
            assert counts[:world] == np.bincount(mine, minlength=world).tolist()
            assert counts[world:2 * world] == [int((assign_h[hb[s]:hb[s + 1]] == rank).sum()) for s in range(world)]
            assert counts[2 * world] == loc.shape[0]
            assert np.array_equal(out["loc"][:loc.shape[0]].cpu().numpy(), loc)
            assert np.array_equal(out["idx_loc"][:loc.shape[0]].cpu().numpy(), np.where(hit[loc] == 1, idx[loc], 0))
            assert np.array_equal(out["hit_loc"][:loc.shape[0]].cpu().numpy(), hit[loc])
            assert np.array_equal(out["send_order"].cpu().numpy(), np.argsort(mine, kind="stable"))
    with pytest.raises(ac.AttnCacheError):
        ac.attncache_affinity_plan_device(ctx, idx_d[:0], hit_d[:0], list(range(34)), [0] * 34, 0)  # world 33
