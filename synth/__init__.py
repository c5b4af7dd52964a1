"""Seeded synthetic inputs for the AttnCache hot path — shared by tests, bench and smoke.

This module holds NONE of the method's arithmetic (no search, no A.V, no
attention): it only draws the workload recipe of BASELINE.json's configs
 with torch random generators, on any device.
Both the CUDA path and the CPU oracle consume the bytes it produces; neither
side's code lives here.

Determinism: every tensor kind x global index has its own generator seeded
with ``seed_for(seed, kind, index)``, so an entry's bytes do not depend on
which GPU (shard) or which batch slice generates it.
"""
from __future__ import annotations

import dataclasses
import math

import torch

__all__ = ["Config", "CONFIGS", "seed_for", "features", "fill_maps", "maps", "query_plan", "queries",
           "activations", "torch_dtype", "FEAT_CHUNK", "EMBED_DIM", "projector_inputs"]

_TD = {"f32": torch.float32, "f16": torch.float16, "bf16": torch.bfloat16}
_KINDS = {"feat": 1, "map": 2, "qnoise": 3, "qmiss": 4, "targets": 5, "positions": 6,
          "q": 7, "k": 8, "v": 9, "misc": 10, "x": 11, "wq": 12, "wk": 13, "wv": 14, "proj": 15}
FEAT_CHUNK = 4096  # feature rows are drawn in fixed chunks of this many entries


def torch_dtype(name: str) -> torch.dtype:
    return _TD[name]


@dataclasses.dataclass(frozen=True)
class Config:
    """One BASELINE.json config (index in BASELINE.json "configs" given by ``bj_index``)."""
    name: str
    bj_index: int
    N: int            # DB entries
    D: int            # feature dim
    feat_dtype: str   # storage dtype of features and queries
    L: int            # layers
    H: int            # heads
    S: int            # sequence length (paper's L in Eq. 5)
    d: int            # head dim (paper's d_k)
    map_dtype: str
    act_dtype: str    # Q, K, V, O dtype
    B: int            # query batch
    hit_rate: float
    sigma: float      # hit-query noise norm (reading R6)
    tau: float = 0.9
    seed: int = 0

    @property
    def n_hit(self) -> int:
        # DESIGN.md reading R8: n_hit = floor(h*B + 0.5)
        return int(math.floor(self.hit_rate * self.B + 0.5))

    def with_(self, **kw) -> "Config":
        return dataclasses.replace(self, **kw)

    @property
    def map_bytes_per_entry(self) -> int:
        return self.L * self.H * self.S * self.S * _TD[self.map_dtype].itemsize


CONFIGS = {
    # configs[0] — "Tiny CPU-scale" (2 misses of 8: hit_rate 0.75)
    "tiny": Config("tiny", 0, N=256, D=384, feat_dtype="f32", L=4, H=4, S=32, d=64, map_dtype="f16",
                   act_dtype="f32", B=8, hit_rate=0.75, sigma=0.05),
    # configs[1] — Llama-3.2-1B-shaped
    "llama32_1b": Config("llama32_1b", 1, N=4096, D=1024, feat_dtype="bf16", L=16, H=32, S=128, d=64,
                         map_dtype="bf16", act_dtype="bf16", B=256, hit_rate=0.8, sigma=0.05),
    # configs[2] — Llama-3-8B-shaped
    "llama3_8b": Config("llama3_8b", 2, N=1024, D=4096, feat_dtype="bf16", L=32, H=32, S=256, d=128,
                        map_dtype="bf16", act_dtype="bf16", B=128, hit_rate=0.9, sigma=0.05),
    # configs[3] — Long-prefill
    "long_prefill": Config("long_prefill", 3, N=256, D=4096, feat_dtype="bf16", L=8, H=32, S=1024, d=128,
                           map_dtype="bf16", act_dtype="bf16", B=32, hit_rate=0.5, sigma=0.05),
    # configs[4] — Search-bound sweep (no maps); B in {1, 64, 1024, 8192}
    "search_sweep": Config("search_sweep", 4, N=1_000_000, D=1024, feat_dtype="bf16", L=0, H=0, S=0, d=0,
                           map_dtype="bf16", act_dtype="bf16", B=1024, hit_rate=0.5, sigma=0.02),
}


def seed_for(seed: int, kind: str, index: int) -> int:
    """splitmix64 of (seed, kind, index) -> a 63-bit generator seed."""
    x = (seed * 0x9E3779B97F4A7C15 + _KINDS[kind] * 0xBF58476D1CE4E5B9 + index * 0x94D049BB133111EB)
    x &= (1 << 64) - 1
    for _ in range(2):
        x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9 & ((1 << 64) - 1)
        x = (x ^ (x >> 27)) * 0x94D049BB133111EB & ((1 << 64) - 1)
        x ^= x >> 31
    return x & ((1 << 63) - 1)


def _gen(device, seed: int, kind: str, index: int) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(seed_for(seed, kind, index))
    return g


def _normalize_rows(x: torch.Tensor) -> torch.Tensor:
    return x / x.norm(dim=-1, keepdim=True)


def features(cfg: Config, begin: int, count: int, device="cpu") -> torch.Tensor:
    """DB feature rows [begin, begin+count): normalize(N(0, I_D)) in fp32, then cast (RN)."""
    out = torch.empty(count, cfg.D, dtype=_TD[cfg.feat_dtype], device=device)
    c0, c1 = begin // FEAT_CHUNK, (begin + count + FEAT_CHUNK - 1) // FEAT_CHUNK
    for c in range(c0, c1):
        rows = min(FEAT_CHUNK, cfg.N - c * FEAT_CHUNK)
        z = torch.randn(rows, cfg.D, generator=_gen(device, cfg.seed, "feat", c), device=device)
        lo, hi = max(begin, c * FEAT_CHUNK), min(begin + count, c * FEAT_CHUNK + rows)
        out[lo - begin:hi - begin] = _normalize_rows(z[lo - c * FEAT_CHUNK:hi - c * FEAT_CHUNK]).to(out.dtype)
    return out


def _feature_rows(cfg: Config, rows: torch.Tensor, device) -> torch.Tensor:
    """Stored feature rows at arbitrary global indices, decoded to fp32."""
    rows = rows.to("cpu")
    out = torch.empty(rows.numel(), cfg.D, dtype=torch.float32, device=device)
    chunks = rows // FEAT_CHUNK
    for c in torch.unique(chunks).tolist():
        sel = (chunks == c).nonzero().flatten()
        base = c * FEAT_CHUNK
        blk = features(cfg, base, min(FEAT_CHUNK, cfg.N - base), device).float()
        out[sel.to(device)] = blk[(rows[sel] - base).to(device)]
    return out


def fill_maps(cfg: Config, out: torch.Tensor, begin: int, causal: bool = True) -> torch.Tensor:
    """Write the maps of entries [begin, begin+len(out)) into out [n][L][H][S][S].

    Per (entry, layer, head): logits ~ N(0,1), causal mask (j > i -> -inf), softmax over j in
    fp32, cast round-to-nearest to the map dtype (BASELINE.json configs; readings R11, R12).
    causal=False draws the bidirectional maps of an encoder (f3: PAPER.md:774-775), no mask.
    This is the DB producer's capture recipe, not part of the hot path.
    """
    n, S = out.shape[0], cfg.S
    dev = out.device
    upper = torch.triu(torch.ones(S, S, dtype=torch.bool, device=dev), diagonal=1)
    # logits are drawn per entry (its own generator); mask, softmax and the cast run on groups of entries
    # (row-wise operations: the bytes do not depend on the grouping), bounded to ~256 MB of fp32 logits
    per = cfg.L * cfg.H * S * S
    group = max(1, min(n, (64 << 20) // max(per, 1)))
    for e0 in range(0, n, group):
        g = min(group, n - e0)
        z = torch.empty(g, cfg.L * cfg.H, S, S, device=dev)
        for e in range(g):
            torch.randn(cfg.L * cfg.H, S, S, generator=_gen(dev, cfg.seed, "map", begin + e0 + e), device=dev,
                        out=z[e])
        if causal:
            z.masked_fill_(upper, float("-inf"))
        out[e0:e0 + g].view(g, cfg.L * cfg.H, S, S).copy_(torch.softmax(z, dim=-1))
    return out


def maps(cfg: Config, begin: int, count: int, device="cpu", causal: bool = True) -> torch.Tensor:
    out = torch.empty(count, cfg.L, cfg.H, cfg.S, cfg.S, dtype=_TD[cfg.map_dtype], device=device)
    return fill_maps(cfg, out, begin, causal)


def query_plan(cfg: Config, B: int | None = None):
    """Which batch positions are planted hits and their DB targets (readings R8, R9).

    Returns (hit_pos int64[n_hit], targets int64[n_hit]); targets are drawn without replacement.
    """
    B = cfg.B if B is None else B
    n_hit = int(math.floor(cfg.hit_rate * B + 0.5))
    pos = torch.randperm(B, generator=_gen("cpu", cfg.seed, "positions", B))[:n_hit]
    tgt = torch.randperm(cfg.N, generator=_gen("cpu", cfg.seed, "targets", B))[:n_hit]
    return pos, tgt


def queries(cfg: Config, device="cpu", B: int | None = None):
    """Query batch [B][D] in the feature dtype.

    Planted hit at position p with target t: normalize(x_t + (sigma/sqrt(D)) z), z ~ N(0, I)
    (reading R6: the noise vector has norm ~sigma).  Miss: normalize(N(0, I)) (reading R7).
    Returns (q, hit_pos, targets).
    """
    B = cfg.B if B is None else B
    pos, tgt = query_plan(cfg, B)
    q = torch.empty(B, cfg.D, dtype=torch.float32, device=device)
    is_hit = torch.zeros(B, dtype=torch.bool)
    is_hit[pos] = True
    x_t = _feature_rows(cfg, tgt, device) if len(tgt) else None
    for k, p in enumerate(pos.tolist()):
        z = torch.randn(cfg.D, generator=_gen(device, cfg.seed, "qnoise", p), device=device)
        q[p] = x_t[k] + (cfg.sigma / math.sqrt(cfg.D)) * z
    for p in (~is_hit).nonzero().flatten().tolist():
        q[p] = torch.randn(cfg.D, generator=_gen(device, cfg.seed, "qmiss", p), device=device)
    return _normalize_rows(q).to(_TD[cfg.feat_dtype]), pos, tgt


def activations(cfg: Config, kind: str, b_begin: int, count: int, layer_begin: int = 0,
                layer_end: int | None = None, device="cpu", out: torch.Tensor | None = None) -> torch.Tensor:
    """Q, K or V rows for queries [b_begin, b_begin+count) and layers [layer_begin, layer_end):
    [count][L'][H][S][d], N(0,1) cast to the activation dtype; one generator per (query, layer)."""
    assert kind in ("q", "k", "v")
    layer_end = cfg.L if layer_end is None else layer_end
    Lp = layer_end - layer_begin
    if out is None:
        out = torch.empty(count, Lp, cfg.H, cfg.S, cfg.d, dtype=_TD[cfg.act_dtype], device=device)
    dev = out.device
    for i in range(count):
        for l in range(Lp):
            g = _gen(dev, cfg.seed, kind, (b_begin + i) * 65536 + layer_begin + l)
            out[i, l].copy_(torch.randn(cfg.H, cfg.S, cfg.d, generator=g, device=dev))
    return out


def block_inputs(cfg: Config, device="cpu", B: int | None = None, n_kv_heads: int | None = None):
    """Eq. 5 block-level comparison inputs (f4): hidden states X [B][S][E] ~ N(0,1) and projection
    weights W_Q [E][E], W_K, W_V [Hkv*d][E] ~ N(0, 1/E) (nn.Linear layout), E = H * d, Hkv = n_kv_heads (default
    H: multi-head), in the activation dtype (synthetic: no trained weights are available)."""
    B = cfg.B if B is None else B
    E = cfg.H * cfg.d
    Ekv = (cfg.H if n_kv_heads is None else n_kv_heads) * cfg.d
    dt = _TD[cfg.act_dtype]
    X = torch.randn(B, cfg.S, E, generator=_gen(device, cfg.seed, "x", 0), device=device).to(dt)
    W = [(torch.randn(n, E, generator=_gen(device, cfg.seed, k, 0), device=device) / math.sqrt(E)).to(dt)
         for k, n in (("wq", E), ("wk", Ekv), ("wv", Ekv))]
    return X, W


# Model hidden size E of the sentence embedding that the feature projector maps to the D-dim feature
# (reading R30: Llama-3.2-1B 2048, Llama-3-8B 4096; tiny / sweep configs use small stand-ins).
EMBED_DIM = {"tiny": 256, "llama32_1b": 2048, "llama3_8b": 4096, "long_prefill": 4096, "search_sweep": 1024}


def projector_inputs(cfg: Config, B: int | None = None, device="cpu", E: int | None = None,
                     hidden: int | None = None):
    """Feature-projector inputs (f2; readings R30-R31): sentence embeddings h [B][E] ~ N(0,1) and synthetic
    weights W1 [Hd][E] ~ N(0, 1/E), W2 [D][Hd] ~ N(0, 1/Hd) in the activation dtype (fp32 for fp32 features),
    biases b1 [Hd], b2 [D] ~ N(0, 0.01) fp32.  Hd = D unless given.  No trained projector is available."""
    B = cfg.B if B is None else B
    E = EMBED_DIM[cfg.name] if E is None else E
    Hd = cfg.D if hidden is None else hidden
    dt = _TD[cfg.act_dtype] if cfg.feat_dtype != "f32" else torch.float32
    h = torch.randn(B, E, generator=_gen(device, cfg.seed, "proj", 0), device=device).to(dt)
    W1 = (torch.randn(Hd, E, generator=_gen(device, cfg.seed, "proj", 1), device=device) / math.sqrt(E)).to(dt)
    W2 = (torch.randn(cfg.D, Hd, generator=_gen(device, cfg.seed, "proj", 2), device=device) / math.sqrt(Hd)).to(dt)
    b1 = 0.1 * torch.randn(Hd, generator=_gen(device, cfg.seed, "proj", 3), device=device)
    b2 = 0.1 * torch.randn(cfg.D, generator=_gen(device, cfg.seed, "proj", 4), device=device)
    return h, W1, b1, W2, b2
