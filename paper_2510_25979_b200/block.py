"""Eq. 5 block-level comparison (Table 4).

One attention block of one layer over a query batch, the two ways Alg. 2 runs it:

  full   (miss, Alg. 2 l.376-381):  Q = X W_Q, K = X W_K, V = X W_V, RoPE(Q, K), softmax(QK^T/sqrt(d)) V
  cached (hit,  Alg. 2 l.373-375):  V = X W_V, O = A_cached . V        ("Q and K are neither computed
                                                                        nor stored")

Every step runs in this library: the projections are attncache_linear (a tcgen05 GEMM X W^T, W in the
nn.Linear layout [H*d][E], whose epilogue stores the head-major [B][H][S][d] layout the attention and A.V
kernels read, so no permute pass follows), then attncache_rope, attncache_attend_full /
attncache_apply_cached.  Weights are synthetic (no trained model is available); timing does not depend on
their values.  Grouped-query attention: W_K, W_V with n_kv_heads * d rows (n_kv_heads dividing n_heads), K and V
then have n_kv_heads heads and query head h reads K / V head h // (n_heads // n_kv_heads) (the `_gqa` calls).
"""
from __future__ import annotations

import torch

from . import Context, Database, attncache_apply_cached, attncache_attend_full, attncache_linear, attncache_rope


class AttentionBlock:
    """One layer's attention block; projection weights in the nn.Linear layout: W_Q [H*d][E], W_K and W_V
    [Hkv*d][E] (Hkv = H: multi-head; Hkv < H: grouped-query)."""

    def __init__(self, ctx: Context, db: Database, W_Q: torch.Tensor, W_K: torch.Tensor, W_V: torch.Tensor,
                 n_heads: int, head_dim: int, layer: int = 0, rope_base: float = 500000.0):
        self.Wq, self.Wk, self.Wv = W_Q, W_K, W_V
        self.H, self.d = n_heads, head_dim
        if W_Q.shape[0] != n_heads * head_dim or W_K.shape != W_V.shape or W_K.shape[0] % head_dim or \
                n_heads % (W_K.shape[0] // head_dim):
            raise ValueError("AttentionBlock: W_Q [H*d][E], W_K = W_V [Hkv*d][E] with Hkv dividing H")
        self.Hkv = W_K.shape[0] // head_dim
        self.ctx, self.db, self.layer, self.rope_base = ctx, db, layer, rope_base

    def _proj(self, X, W):
        # [B][S][E] x [heads*d][E]^T -> head-major [B][1][heads][S][d] (one layer), in the GEMM's epilogue
        return attncache_linear(self.ctx, X, W, W.shape[0] // self.d)

    def full(self, X: torch.Tensor) -> torch.Tensor:
        Q, K, V = self._proj(X, self.Wq), self._proj(X, self.Wk), self._proj(X, self.Wv)
        attncache_rope(Q, self.rope_base)
        attncache_rope(K, self.rope_base)
        return attncache_attend_full(self.ctx, Q, K, V)

    def cached(self, X: torch.Tensor, idx: torch.Tensor, hit: torch.Tensor, miss_rows: torch.Tensor) -> torch.Tensor:
        """Hits: V projection + A.V with the cached maps of `layer`; misses: the full block."""
        V = self._proj(X, self.Wv)
        O = attncache_apply_cached(self.db, idx, V, hit=hit, layer_begin=self.layer, layer_end=self.layer + 1)
        if miss_rows.numel():
            Xm = X.index_select(0, miss_rows)
            Q, K = self._proj(Xm, self.Wq), self._proj(Xm, self.Wk)
            attncache_rope(Q, self.rope_base)
            attncache_rope(K, self.rope_base)
            O.index_copy_(0, miss_rows, attncache_attend_full(self.ctx, Q, K, V.index_select(0, miss_rows)))
        return O
