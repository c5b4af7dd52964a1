"""Pins for the CPU oracle (oracle/) against what the paper and mathematics fix.

Each test cites the passage it pins.  None of these re-types the oracle's
formula as its expectation: expectations come from exact rational arithmetic
(brute force with fractions.Fraction on tiny inputs), closed forms, special
cases that reduce to a textbook value, a different library routine
(torch SDPA in fp64), invariants, or hand-computed golden fixtures under
tests/golden/.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def _bf16_bits(a):
    return torch.tensor(np.asarray(a, np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def _exact(a, dtype):
    """Exact rational value of stored elements (numpy's own float decoding, not the oracle's)."""
    if dtype == "bf16":
        f = (a.astype(np.uint32) << 16).view(np.float32)
    else:
        f = a
    return [Fraction(float(v)) for v in np.asarray(f, np.float64).reshape(-1)]


# ----------------------------------------------------------------------------------------------
# decoders (exactness of fp16/bf16 -> fp64 is what every other pin relies on)
# ----------------------------------------------------------------------------------------------

def test_decode_matches_numpy_and_torch():
    rng = np.random.default_rng(1)
    h = rng.integers(0, 1 << 16, 4096, dtype=np.uint16)
    h = h[(h & 0x7C00) != 0x7C00]  # finite only
    ref16 = h.view(np.float16).astype(np.float64)
    assert np.array_equal(oracle.decode(h.view(np.float16), "f16"), ref16)
    refbf = torch.from_numpy(h.view(np.int16)).view(torch.bfloat16).double().numpy()
    assert np.array_equal(oracle.decode(h, "bf16"), refbf)
    f = rng.standard_normal(64).astype(np.float32)
    assert np.array_equal(oracle.decode(f, "f32"), f.astype(np.float64))


# ----------------------------------------------------------------------------------------------
# search — Alg. 1 l.255-257, north_star: exact top-1, lowest-index tie-break
# ----------------------------------------------------------------------------------------------

@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_search_equals_exact_rational_brute_force(dtype):
    rng = np.random.default_rng(2)
    B, N, D = 6, 40, 7
    xf = rng.standard_normal((N, D)).astype(np.float32)
    qf = rng.standard_normal((B, D)).astype(np.float32)
    xf[17] = xf[5]          # planted duplicate: tie must go to index 5
    qf[0] = xf[17]
    x = xf if dtype == "f32" else _bf16_bits(xf)
    q = qf if dtype == "f32" else _bf16_bits(qf)
    X = np.array(_exact(x, dtype), dtype=object).reshape(N, D)
    Q = np.array(_exact(q, dtype), dtype=object).reshape(B, D)
    idx, s1, s2, hit = oracle.search(q, x, dtype, tau=0.5)
    for b in range(B):
        s = [sum(Q[b, k] * X[i, k] for k in range(D)) for i in range(N)]
        best = max(s)
        arg = s.index(best)  # first (lowest) index attaining the max
        runner = sorted(s, reverse=True)[1]
        assert idx[b] == arg
        assert abs(s1[b] - float(best)) <= 1e-12 * max(1.0, abs(float(best)))
        assert abs(s2[b] - float(runner)) <= 1e-12 * max(1.0, abs(float(runner)))
        assert hit[b] == (s1[b] >= np.float64(np.float32(0.5)))
    assert idx[0] == 5 and s1[0] == s2[0]


def test_search_basis_vectors_and_exact_ties():
    D = 16
    x = _bf16_bits(np.eye(D, dtype=np.float32))
    q = _bf16_bits(np.eye(D, dtype=np.float32)[::-1].copy())
    idx, s1, _, hit = oracle.search(q, x, "bf16", tau=1.0)
    assert list(idx) == list(range(D))[::-1]
    assert np.all(s1 == 1.0) and np.all(hit == 1)
    # (e_i + e_j)/sqrt(2): both coordinates have identical bits -> an exact tie -> min(i, j)
    pairs = [(3, 11), (9, 2), (15, 0)]
    qq = np.zeros((len(pairs), D), np.float32)
    for r, (i, j) in enumerate(pairs):
        qq[r, i] = qq[r, j] = 1 / math.sqrt(2)
    idx, s1, s2, _ = oracle.search(_bf16_bits(qq), x, "bf16", tau=0.0)
    assert list(idx) == [min(p) for p in pairs]
    assert np.all(s1 == s2)


def test_search_threshold_is_inclusive():
    g = _gold("search_threshold.json")
    D = 8
    x = np.zeros((3, D), np.float32)
    x[1, 0] = g["x0"]
    x[1, 1] = math.sqrt(1 - g["x0"] ** 2)
    x[0, 2] = x[2, 3] = 1.0
    q = np.zeros((1, D), np.float32)
    q[0, 0] = 1.0
    for dtype, xs, qs in (("f32", x, q), ("bf16", _bf16_bits(x), _bf16_bits(q))):
        idx, s1, _, hit = oracle.search(qs, xs, dtype, tau=g["tau_hit"])
        assert idx[0] == 1 and s1[0] == g["x0"] and hit[0] == 1
        _, _, _, hit = oracle.search(qs, xs, dtype, tau=g["tau_miss"])
        assert hit[0] == 0


def test_search_self_query_and_orthogonal():
    rng = np.random.default_rng(3)
    N, D = 64, 384
    x = rng.standard_normal((N, D))
    x = (x / np.linalg.norm(x, axis=1, keepdims=True)).astype(np.float32)
    q = x[[7, 40]].copy()
    idx, s1, _, hit = oracle.search(q, x, "f32", tau=0.9)
    assert list(idx) == [7, 40] and np.all(hit == 1)
    for b, i in enumerate([7, 40]):
        exact = sum(Fraction(float(v)) ** 2 for v in x[i])
        assert abs(s1[b] - float(exact)) < 1e-12
        assert abs(s1[b] - 1.0) < 1e-6   # unit norm within fp32 rounding (reading R2)
    # orthogonal: exact zero
    xo = np.zeros((2, 4), np.float32)
    xo[0, 0] = xo[1, 1] = 1
    qo = np.zeros((1, 4), np.float32)
    qo[0, 2] = 1
    idx, s1, _, hit = oracle.search(qo, xo, "f32", tau=0.0)
    assert s1[0] == 0.0 and idx[0] == 0 and hit[0] == 1  # 0 >= 0 is a hit; lowest index on the 0-0 tie


def test_search_empty_db_and_tau_above_one():
    q = np.ones((2, 4), np.float32) / 2
    idx, s1, _, hit = oracle.search(q, np.zeros((0, 4), np.float32), "f32", tau=0.0)
    assert list(idx) == [-1, -1] and np.all(np.isneginf(s1)) and np.all(hit == 0)
    x = np.eye(4, dtype=np.float32)
    _, _, _, hit = oracle.search(x, x, "f32", tau=2.0)
    assert np.all(hit == 0)


def test_search_hit_rate_monotone_in_tau():
    # SPEC.md:492 / PAPER.md:883 (Fig. 6): lowering theta can only raise the hit rate
    rng = np.random.default_rng(4)
    x = rng.standard_normal((200, 32)).astype(np.float32)
    x /= np.linalg.norm(x, axis=1, keepdims=True)
    q = x[rng.integers(0, 200, 50)] + 0.3 * rng.standard_normal((50, 32)).astype(np.float32)
    q = (q / np.linalg.norm(q, axis=1, keepdims=True)).astype(np.float32)
    rates = [oracle.search(q, x, "f32", tau=t)[3].mean() for t in (0.995, 0.99, 0.95, 0.9, 0.85, 0.5)]
    assert all(a <= b for a, b in zip(rates, rates[1:]))


def test_search_sharded_reduction_equals_unsharded():
    # north_star: each GPU does a local top-1 and the (score, index) pairs are reduced.
    rng = np.random.default_rng(5)
    N, D = 301, 24
    x = rng.standard_normal((N, D)).astype(np.float32)
    x[250] = x[20]                     # duplicate across shards: global tie -> 20
    q = np.concatenate([x[[20]], rng.standard_normal((9, D)).astype(np.float32)])
    ref = oracle.search(q, x, "f32", tau=0.0)
    for g in (2, 3, 8):
        bounds = np.linspace(0, N, g + 1).astype(int)
        best = [(-math.inf, None)] * len(q)
        for r in range(g):
            lo, hi = bounds[r], bounds[r + 1]
            li, ls, _, _ = oracle.search(q, x[lo:hi], "f32", tau=0.0)
            for b in range(len(q)):
                if li[b] < 0:
                    continue
                cand = (ls[b], -(lo + li[b]))
                if best[b][1] is None or cand > (best[b][0], -best[b][1]):
                    best[b] = (ls[b], lo + li[b])
        assert [b[1] for b in best] == list(ref[0])
    assert ref[0][0] == 20


# ----------------------------------------------------------------------------------------------
# apply — Alg. 2 l.373-375: O = attn_map . v
# ----------------------------------------------------------------------------------------------

def test_apply_golden_3x3():
    g = _gold("apply_3x3.json")
    A = np.array(g["A"], np.float32)
    V = np.array(g["V"], np.float32)
    for adt in ("f32", "f16", "bf16"):
        As = A.astype(np.float16) if adt == "f16" else (_bf16_bits(A) if adt == "bf16" else A)
        O = oracle.apply(As, adt, [0], V, "f32", [0], g["S"], g["d"])
        assert np.array_equal(O[0], np.array(g["O"]))


@pytest.mark.parametrize("S,d", [(32, 64), (128, 64)])
def test_apply_identity_and_one_hot(S, d):
    rng = np.random.default_rng(6)
    V = rng.standard_normal((S, d)).astype(np.float32)
    Vb = _bf16_bits(V)
    I = np.eye(S, dtype=np.float32)
    O = oracle.apply(_bf16_bits(I), "bf16", [0], Vb, "bf16", [0], S, d)
    assert np.array_equal(O[0], oracle.decode(Vb, "bf16").reshape(S, d))
    E0 = np.zeros((S, S), np.float32)
    E0[:, 0] = 1.0
    O = oracle.apply(E0.astype(np.float16), "f16", [0], V, "f32", [0], S, d)
    assert np.array_equal(O[0], np.repeat(V[:1].astype(np.float64), S, axis=0))


def test_apply_uniform_causal_gives_prefix_mean():
    S, d = 64, 16
    rng = np.random.default_rng(7)
    V = rng.standard_normal((S, d)).astype(np.float32)
    A = np.tril(np.ones((S, S))) / np.arange(1, S + 1)[:, None]
    O = oracle.apply(A.astype(np.float32), "f32", [0], V, "f32", [0], S, d)[0]
    prefix_mean = np.cumsum(V.astype(np.float64), axis=0) / np.arange(1, S + 1)[:, None]
    assert np.max(np.abs(O - prefix_mean)) < 1e-6


def test_apply_constant_v_and_linearity():
    S, d = 32, 8
    rng = np.random.default_rng(8)
    z = rng.standard_normal((S, S))
    z[np.triu_indices(S, 1)] = -np.inf
    A = np.exp(z - z.max(1, keepdims=True))
    A = (A / A.sum(1, keepdims=True)).astype(np.float16)
    rowsum = A.astype(np.float64).sum(1)
    O = oracle.apply(A, "f16", [0], np.full((S, d), 3.0, np.float32), "f32", [0], S, d)[0]
    assert np.allclose(O, 3.0 * rowsum[:, None], rtol=0, atol=1e-12)
    V1 = rng.integers(-8, 8, (S, d)).astype(np.float32)
    V2 = rng.integers(-8, 8, (S, d)).astype(np.float32)
    O12 = oracle.apply(A, "f16", [0, 0], np.stack([V1 + V2, V1 - V2]), "f32", [0, S * d], S, d)
    O1 = oracle.apply(A, "f16", [0], V1, "f32", [0], S, d)[0]
    O2 = oracle.apply(A, "f16", [0], V2, "f32", [0], S, d)[0]
    assert np.allclose(O12[0], O1 + O2, atol=1e-9) and np.allclose(O12[1], O1 - O2, atol=1e-9)


def test_apply_exact_rational_brute_force_and_offsets():
    rng = np.random.default_rng(9)
    S, d, U = 5, 3, 3
    A = rng.standard_normal((U, S, S)).astype(np.float32)   # deliberately not symmetric
    V = rng.standard_normal((U, S, d)).astype(np.float32)
    a_off = [2 * S * S, 0, S * S]                            # units in a permuted order
    v_off = [0, 2 * S * d, S * d]
    O = oracle.apply(A, "f32", a_off, V, "f32", v_off, S, d)
    for u in range(U):
        Au = A.reshape(-1)[a_off[u]:a_off[u] + S * S].reshape(S, S)
        Vu = V.reshape(-1)[v_off[u]:v_off[u] + S * d].reshape(S, d)
        for i in range(S):
            for c in range(d):
                ex = sum(Fraction(float(Au[i, j])) * Fraction(float(Vu[j, c])) for j in range(S))
                assert abs(O[u, i, c] - float(ex)) < 1e-12


# ----------------------------------------------------------------------------------------------
# attend — Alg. 2 l.376-381, Eq. 5: softmax(QK^T/sqrt(d_k)) . V, causal
# ----------------------------------------------------------------------------------------------

def test_attend_golden_ln2():
    g = _gold("softmax_ln2.json")
    Q, K, V = (np.array(g[k], np.float32) for k in "QKV")
    O = oracle.attend(Q, K, V, "f32", [0], g["S"], g["d"])[0]
    P = oracle.attention_map(Q, K, "f32", [0], g["S"], g["d"])[0]
    assert np.max(np.abs(O - np.array(g["O"]))) < g["tol"]
    assert np.max(np.abs(P - np.array(g["P"]))) < g["tol"]


def test_attend_single_token_and_zero_query():
    rng = np.random.default_rng(10)
    d = 64
    Q1, K1, V1 = (rng.standard_normal((1, d)).astype(np.float32) for _ in range(3))
    assert np.array_equal(oracle.attend(Q1, K1, V1, "f32", [0], 1, d)[0], V1.astype(np.float64))
    S = 48
    K = rng.standard_normal((S, d)).astype(np.float32)
    V = rng.standard_normal((S, d)).astype(np.float32)
    O = oracle.attend(np.zeros((S, d), np.float32), K, V, "f32", [0], S, d)[0]
    prefix_mean = np.cumsum(V.astype(np.float64), 0) / np.arange(1, S + 1)[:, None]
    assert np.max(np.abs(O - prefix_mean)) < 1e-12


def test_attend_dominant_diagonal_gives_v():
    S = d = 32
    rng = np.random.default_rng(11)
    E = 40.0 * np.eye(S, dtype=np.float32)
    V = rng.standard_normal((S, d)).astype(np.float32)
    O = oracle.attend(E, E, V, "f32", [0], S, d)[0]   # z_ii = 1600/sqrt(32) ~ 283, others 0
    assert np.max(np.abs(O - V)) < 1e-100 + 1e-9


@pytest.mark.parametrize("S,d,dtype", [(32, 64, "f32"), (128, 64, "bf16"), (70, 16, "f16")])
def test_attend_matches_torch_sdpa_fp64(S, d, dtype):
    # independent library routine: torch.nn.functional.scaled_dot_product_attention(is_causal=True)
    rng = np.random.default_rng(12)
    U = 3
    raw = [rng.standard_normal((U, S, d)).astype(np.float32) for _ in range(3)]
    if dtype == "bf16":
        st = [_bf16_bits(r) for r in raw]
    elif dtype == "f16":
        st = [r.astype(np.float16) for r in raw]
    else:
        st = raw
    O = oracle.attend(*st, dtype, [u * S * d for u in range(U)], S, d)
    dec = [torch.from_numpy(oracle.decode(s, dtype).reshape(U, S, d)) for s in st]
    ref = torch.nn.functional.scaled_dot_product_attention(*dec, is_causal=True).numpy()
    assert np.max(np.abs(O - ref)) < 1e-12


def test_capture_then_reuse_equals_full_attention():
    # SPEC.md:144/158 and Alg. 2: reusing the map captured from the same input reproduces full attention.
    rng = np.random.default_rng(13)
    S, d = 40, 16
    Q, K, V = (rng.standard_normal((S, d)).astype(np.float32) for _ in range(3))
    P = oracle.attention_map(Q, K, "f32", [0], S, d)[0]
    assert np.all(P[np.triu_indices(S, 1)] == 0.0)
    assert np.allclose(P.sum(1), 1.0, atol=1e-13)
    O_full = oracle.attend(Q, K, V, "f32", [0], S, d)[0]
    O_reuse = oracle.apply(P.astype(np.float32), "f32", [0], V, "f32", [0], S, d)[0]
    assert np.max(np.abs(O_full - O_reuse)) < 1e-5     # only the fp32 storage of P differs


# ----------------------------------------------------------------------------------------------
# generated inputs — the invariants north_star states for the DB (row-stochastic, lower-triangular)
# ----------------------------------------------------------------------------------------------

def test_generated_tiny_inputs_invariants():
    import synth
    cfg = synth.CONFIGS["tiny"]
    M = synth.maps(cfg, 0, 3)
    Md = M.double().numpy()
    S = cfg.S
    iu = np.triu_indices(S, 1)
    assert np.all(M.view(torch.int16).numpy()[..., iu[0], iu[1]] == 0)      # exact +0.0 above diagonal
    assert np.all(np.abs(Md.sum(-1) - 1.0) <= 6e-4)                           # fp16 rounding (R12)
    assert np.all(Md[..., 0, 0] == 1.0)
    x = synth.features(cfg, 0, cfg.N)
    assert torch.allclose(x.double().norm(dim=1), torch.ones(cfg.N, dtype=torch.float64), atol=1e-6)
    q, pos, tgt = synth.queries(cfg)
    idx, s1, s2, hit = oracle.search(q.numpy(), x.numpy(), "f32", cfg.tau)
    assert sorted(np.nonzero(hit)[0].tolist()) == sorted(pos.tolist())       # planted hits hit
    assert [idx[p] for p in pos.tolist()] == tgt.tolist()                    # ... their own target
    assert np.all(s1[~hit.astype(bool)] < 0.5)                               # random misses are far below tau
    # the generator is deterministic and shard-independent
    assert torch.equal(synth.features(cfg, 100, 50), x[100:150])
    assert torch.equal(synth.maps(cfg, 2, 1)[0], M[2])


# ----------------------------------------------------------------------------------------------
# RoPE — Alg. 2 l.379 (rotate-half convention, reading R29); SPEC.md:55-58 examples
# ----------------------------------------------------------------------------------------------

def test_rope_pins():
    rng = np.random.default_rng(14)
    S, d = 40, 16
    X = rng.standard_normal((2, S, d)).astype(np.float32)
    Y = oracle.rope(X, "f32", S, d)
    assert np.array_equal(Y[:, 0], X[:, 0].astype(np.float64))                 # position 0: identity
    n_x = X.astype(np.float64)[..., : d // 2] ** 2 + X.astype(np.float64)[..., d // 2:] ** 2
    n_y = Y[..., : d // 2] ** 2 + Y[..., d // 2:] ** 2
    assert np.allclose(n_x, n_y, atol=1e-12)                                   # pairwise isometry
    # d = 2: pair (x0, x1) at position p rotated by exactly p radians (theta_0 = base^0 = 1)
    X2 = np.tile(np.array([[1.0, 0.0]], np.float32), (5, 1))[None]
    Y2 = oracle.rope(X2, "f32", 5, 2)[0]
    assert np.allclose(Y2, np.stack([np.cos(np.arange(5)), np.sin(np.arange(5))], 1), atol=1e-15)
    # relative-position property: <R_p q, R_p' k> depends only on p - p'
    q = rng.standard_normal(d).astype(np.float32)
    k = rng.standard_normal(d).astype(np.float32)
    Q = oracle.rope(np.tile(q, (S, 1))[None], "f32", S, d)[0]
    K = oracle.rope(np.tile(k, (S, 1))[None], "f32", S, d)[0]
    assert abs(Q[10] @ K[7] - Q[30] @ K[27]) < 1e-9 and abs(Q[5] @ K[5] - q.astype(np.float64) @ k) < 1e-9


def test_rope_frequency_schedule_golden():
    """The frequencies theta_i = base^(-2i/d) for i >= 1 (a wrong exponent such as base^(-i/d) passes every
    invariant above): hand-computed angles of tests/golden/rope_theta.json."""
    g = _gold("rope_theta.json")
    for c in g["cases"]:
        d, p, i = c["d"], c["p"], c["i"]
        X = np.zeros((1, p + 1, d), np.float32)
        X[0, :, i] = 1.0                                                        # e_i at every position
        Y = oracle.rope(X, "f32", p + 1, d, base=c["base"])[0, p]
        want = np.zeros(d)
        want[i], want[i + d // 2] = c["cos"], c["sin"]
        assert np.allclose(Y, want, atol=1e-12), (c, Y)


# ----------------------------------------------------------------------------------------------
# oracle_scores — the checker behind every near-tie search decision (tests/_util.py check_search)
# ----------------------------------------------------------------------------------------------

@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_scores_equal_exact_rational_pairs(dtype):
    """s[p] = q[qb[p]] . x[xi[p]]: exact rational inner products on pairs whose q and x row counts differ
    (B = 5, N = 23), so swapping the roles of qb and xi, or of q and x, changes the value or the range."""
    rng = np.random.default_rng(21)
    B, N, D = 5, 23, 9
    xf = rng.standard_normal((N, D)).astype(np.float32)
    qf = (3.0 * rng.standard_normal((B, D))).astype(np.float32)   # a different scale than x
    x = xf if dtype == "f32" else _bf16_bits(xf)
    q = qf if dtype == "f32" else _bf16_bits(qf)
    X = np.array(_exact(x, dtype), dtype=object).reshape(N, D)
    Q = np.array(_exact(q, dtype), dtype=object).reshape(B, D)
    qb = np.array([0, 4, 2, 2, 1, 3, 4], np.int64)
    xi = np.array([22, 0, 7, 8, 19, 3, 11], np.int64)
    s = oracle.scores(q, x, dtype, qb, xi)
    for p in range(len(qb)):
        want = sum(Q[qb[p], k] * X[xi[p], k] for k in range(D))
        assert abs(s[p] - float(want)) <= 1e-12 * max(1.0, abs(float(want))), (p, s[p], float(want))
    # consistency with the search: the score at the oracle's own top-1 / runner-up is s1 / s2
    idx, s1, s2, _ = oracle.search(q, x, dtype, tau=0.0)
    assert np.array_equal(oracle.scores(q, x, dtype, np.arange(B), idx), s1)
    second = []
    for b in range(B):
        row = oracle.scores(q, x, dtype, np.full(N, b), np.arange(N))
        order = np.argsort(-row, kind="stable")
        second.append(row[order[1]])
        assert order[0] == idx[b]
    assert np.array_equal(np.array(second), s2)
    with pytest.raises(IndexError):
        oracle.scores(q, x, dtype, np.array([B]), np.array([0]))             # qb indexes q, not x


# ----------------------------------------------------------------------------------------------
# feature projector — Alg. 1 l.254, PAPER.md:278 two-layer MLP; readings R30-R32
# ----------------------------------------------------------------------------------------------

def _proj_inputs(rng, B, E, Hd, D, dtype):
    h = rng.standard_normal((B, E)).astype(np.float32)
    W1 = (rng.standard_normal((Hd, E)) / math.sqrt(E)).astype(np.float32)
    W2 = (rng.standard_normal((D, Hd)) / math.sqrt(Hd)).astype(np.float32)
    b1 = (0.1 * rng.standard_normal(Hd)).astype(np.float32)
    b2 = (0.1 * rng.standard_normal(D)).astype(np.float32)
    if dtype == "bf16":
        h, W1, W2 = _bf16_bits(h), _bf16_bits(W1), _bf16_bits(W2)
    return h, W1, b1, W2, b2


@pytest.mark.parametrize("dtype", ["bf16", "f32"])
def test_project_golden_hand_computed(dtype):
    g = _gold("project_mlp.json")
    conv = _bf16_bits if dtype == "bf16" else (lambda a: np.asarray(a, np.float32))
    f = oracle.project(conv(g["h"]), dtype, conv(g["W1"]), np.float32(g["b1"]), conv(g["W2"]), np.float32(g["b2"]))
    assert np.allclose(f, np.array(g["f"]), rtol=0, atol=1e-15)


def test_project_identity_weights_is_normalisation():
    """W1 = I, b1 = 0, W2 = I, b2 = 0: f = relu(h) / ||relu(h)|| (closed form; ReLU zeroes negatives)."""
    rng = np.random.default_rng(5)
    E = 16
    h = rng.standard_normal((6, E)).astype(np.float32)
    h[0] = np.abs(h[0])                                     # all positive: f = h / ||h||
    I = np.eye(E, dtype=np.float32)
    z = np.zeros(E, np.float32)
    f = oracle.project(h, "f32", I, z, I, z)
    r = np.maximum(h.astype(np.float64), 0.0)
    for b in range(6):
        n = math.sqrt(sum(float(v) ** 2 for v in r[b]))
        assert np.allclose(f[b], r[b] / n, rtol=0, atol=1e-15)
    assert np.allclose(f[0], h[0] / np.linalg.norm(h[0].astype(np.float64)), rtol=0, atol=1e-15)


def test_project_exact_rational_brute_force():
    """Tiny bf16 instance: hidden layer and pre-normalisation output in exact rationals; f^2 * ||y||^2 = y^2
    and the signs agree (the oracle's sqrt is the only inexact step)."""
    rng = np.random.default_rng(9)
    B, E, Hd, D = 3, 5, 4, 3
    h, W1, b1, W2, b2 = _proj_inputs(rng, B, E, Hd, D, "bf16")
    f = oracle.project(h, "bf16", W1, b1, W2, b2)
    hq, W1q, W2q = _exact(h, "bf16"), _exact(W1, "bf16"), _exact(W2, "bf16")
    for b in range(B):
        z = [max(Fraction(0), sum(W1q[j * E + k] * hq[b * E + k] for k in range(E)) + Fraction(float(b1[j])))
             for j in range(Hd)]
        y = [sum(W2q[c * Hd + j] * z[j] for j in range(Hd)) + Fraction(float(b2[c])) for c in range(D)]
        nn = sum(v * v for v in y)
        for c in range(D):
            assert abs(float(f[b, c]) ** 2 * float(nn) - float(y[c] * y[c])) <= 1e-12 * float(nn)
            assert (f[b, c] > 0) == (y[c] > 0)


def test_project_invariants():
    """Unit norm; positive scaling of (W2, b2) leaves f unchanged (bitwise: x4 is exact); permuting the
    output units permutes f; permuting the hidden units (rows of W1/b1, columns of W2) leaves f unchanged."""
    rng = np.random.default_rng(11)
    B, E, Hd, D = 7, 24, 16, 12
    h, W1, b1, W2, b2 = _proj_inputs(rng, B, E, Hd, D, "f32")
    f = oracle.project(h, "f32", W1, b1, W2, b2)
    assert np.allclose(np.linalg.norm(f, axis=1), 1.0, rtol=0, atol=1e-14)
    f4 = oracle.project(h, "f32", W1, b1, (4 * W2).astype(np.float32), (4 * b2).astype(np.float32))
    assert np.array_equal(f4, f)
    perm = rng.permutation(D)
    fp = oracle.project(h, "f32", W1, b1, np.ascontiguousarray(W2[perm]), np.ascontiguousarray(b2[perm]))
    assert np.allclose(fp, f[:, perm], rtol=0, atol=1e-14)
    hp = rng.permutation(Hd)
    fh = oracle.project(h, "f32", np.ascontiguousarray(W1[hp]), np.ascontiguousarray(b1[hp]),
                        np.ascontiguousarray(W2[:, hp]), b2)
    assert np.allclose(fh, f, rtol=0, atol=1e-14)


def test_project_matches_library_mlp():
    """Independent library special case: torch.nn.functional.linear + relu + normalize in fp64."""
    rng = np.random.default_rng(13)
    B, E, Hd, D = 9, 64, 32, 48
    h, W1, b1, W2, b2 = _proj_inputs(rng, B, E, Hd, D, "bf16")
    f = oracle.project(h, "bf16", W1, b1, W2, b2)
    t = lambda a: torch.from_numpy(a.view(np.int16)).view(torch.bfloat16).double()  # noqa: E731
    z = torch.relu(torch.nn.functional.linear(t(h), t(W1), torch.from_numpy(b1).double()))
    y = torch.nn.functional.linear(z, t(W2), torch.from_numpy(b2).double())
    ref = torch.nn.functional.normalize(y, dim=1).numpy()
    assert np.allclose(f, ref, rtol=0, atol=1e-13)


# ----------------------------------------------------------------------------------------------
# projections — Alg. 2 l.372, l.377-378 (f4 block comparison; reading R34: W in the nn.Linear layout)
# ----------------------------------------------------------------------------------------------

@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_linear_exact_rational_and_layout(dtype):
    """Y = X W^T against exact rationals on a non-square W (N = 5 != K = 7, so W [K][N] would not even fit),
    identity weights give X back exactly, and a golden 2 x 2 case computed by hand."""
    rng = np.random.default_rng(31)
    M, K, N = 4, 7, 5
    Xf = rng.standard_normal((M, K)).astype(np.float32)
    Wf = rng.standard_normal((N, K)).astype(np.float32)
    X = Xf if dtype == "f32" else _bf16_bits(Xf)
    W = Wf if dtype == "f32" else _bf16_bits(Wf)
    XE = np.array(_exact(X, dtype), dtype=object).reshape(M, K)
    WE = np.array(_exact(W, dtype), dtype=object).reshape(N, K)
    Y = oracle.linear(X, W, dtype)
    for m in range(M):
        for n in range(N):
            want = float(sum(XE[m, k] * WE[n, k] for k in range(K)))
            assert abs(Y[m, n] - want) <= 1e-12 * max(1.0, abs(want))
    I = np.eye(K, dtype=np.float32)
    assert np.array_equal(oracle.linear(X, I if dtype == "f32" else _bf16_bits(I), dtype),
                          np.asarray(_exact(X, dtype), dtype=np.float64).reshape(M, K))
    # [[1, 2], [3, 4]] . [[5, 6], [7, 8]]^T = [[17, 23], [39, 53]]
    A = np.array([[1, 2], [3, 4]], np.float32)
    B = np.array([[5, 6], [7, 8]], np.float32)
    assert np.array_equal(oracle.linear(A, B, "f32"), np.array([[17.0, 23.0], [39.0, 53.0]]))
