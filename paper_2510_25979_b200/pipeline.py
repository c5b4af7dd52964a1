"""One AttnCache prefill attention step on one GPU: the whole hot path (SURVEY.md §8(a) a1-a8, N=1).

    search (Alg. 1 l.255-257) -> hit branch O = A.V (Alg. 2 l.373-375) for hits
                              -> miss branch softmax(QK^T/sqrt(d)).V (Alg. 2 l.376-381) for misses

Pure orchestration over the C ABI: no arithmetic here.  At N = 1 the routing
rows of §8(a) (a5, a7) are the identity, so hits are served in place.
"""
from __future__ import annotations

from typing import Optional

import torch

from . import (Context, Database, attncache_apply_cached, attncache_attend_full, attncache_prefill_host,
               attncache_project_features, attncache_search)


class PrefillStep:
    """Runs search -> apply_cached(hits) -> attend_full(misses) for one query batch.

    Buffers for idx/score/hit are allocated once per batch size; all calls are enqueued on one stream.
    """

    def __init__(self, ctx: Context, db: Database, tau: float, layer_begin: int = 0, layer_end: Optional[int] = None):
        self.ctx, self.db, self.tau = ctx, db, float(tau)
        self.layer_begin = layer_begin
        self.layer_end = db.maps.shape[1] if layer_end is None else layer_end
        self._bufs = {}

    def _outputs(self, B: int, device):
        if B not in self._bufs:
            self._bufs[B] = (torch.empty(B, dtype=torch.int64, device=device),
                             torch.empty(B, dtype=torch.float32, device=device),
                             torch.empty(B, dtype=torch.uint8, device=device))
        return self._bufs[B]

    def search(self, queries: torch.Tensor, stream=None):
        idx, score, hit = self._outputs(queries.shape[0], queries.device)
        return attncache_search(self.db, queries, self.tau, idx, score, hit, stream=stream)

    def attend(self, idx, hit, Q, K, V, O, stream=None):
        attncache_apply_cached(self.db, idx, V, O, hit=hit, layer_begin=self.layer_begin,
                               layer_end=self.layer_end, stream=stream)
        attncache_attend_full(self.ctx, Q, K, V, O, skip=hit, stream=stream)
        return O

    def __call__(self, queries, Q, K, V, O, stream=None):
        idx, score, hit = self.search(queries, stream=stream)
        self.attend(idx, hit, Q, K, V, O, stream=stream)
        return idx, score, hit


class GraphedPrefillStep:
    """A PrefillStep captured once as a CUDA graph for fixed shapes: search -> apply_cached -> attend_full
    replay as one graph launch (the library's launches, the memset of the search keys and the device-side
    row selection need no host round trip, so the whole step is capturable).  For small, latency-bound
    batches this removes the per-call host overhead of the six launches.

    The graph reads and writes its own static buffers: fill ``inputs`` (q, Q, K, V) in place, call
    ``replay()``, read ``outputs`` (idx, score, hit, O)."""

    def __init__(self, step: PrefillStep, q, Q, K, V, stream=None):
        self.step = step
        self.inputs = tuple(t.clone() for t in (q, Q, K, V))
        self.O = torch.empty_like(V)
        step(*self.inputs, self.O)  # warm-up: grows the library's scratch before capture (no cudaMalloc inside)
        torch.cuda.synchronize()
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(self.graph, stream=stream, capture_error_mode="thread_local"):
            res = step(*self.inputs, self.O)
        self.outputs = (*res, self.O)

    def replay(self):
        self.graph.replay()
        return self.outputs


class FeatureProjector:
    """Alg. 1 l.254 `f <- feature_projector(h)`: the two-layer MLP that maps
    sentence embeddings h [B][E] to L2-normalised feature vectors [B][D] in the DB's feature dtype, which
    `PrefillStep.search` then takes (Alg. 1 l.255).  Weights in the nn.Linear layout (readings R30-R32)."""

    def __init__(self, ctx: Context, W1, b1, W2, b2, feat_dtype=None):
        self.ctx, self.W1, self.b1, self.W2, self.b2 = ctx, W1, b1, W2, b2
        self.feat_dtype = W1.dtype if feat_dtype is None else feat_dtype
        self._out = {}

    def __call__(self, h, stream=None):
        B = h.shape[0]
        if B not in self._out:
            self._out[B] = torch.empty(B, self.W2.shape[0], dtype=self.feat_dtype, device=h.device)
        return attncache_project_features(self.ctx, h, self.W1, self.b1, self.W2, self.b2, out=self._out[B],
                                          stream=stream)


class PerLayerPrefill:
    """AttnCache-f (Table 4): a search per layer.

    Each layer l has its own feature DB (embeddings of that layer's hidden states) sharing the index
    space of one map DB; layer l's hits apply that layer's maps of their own top-1 entry, its misses
    run full attention.  Tensors are per layer (as a model produces them): q_l [B][D], Q_l/K_l/V_l/O_l
    [B][1][H][S][d].
    """

    def __init__(self, ctx: Context, map_db: Database, feature_dbs, tau: float):
        self.ctx, self.map_db, self.feature_dbs, self.tau = ctx, map_db, list(feature_dbs), float(tau)

    def layer(self, l: int, q_l, Q_l, K_l, V_l, O_l, stream=None):
        idx, score, hit = attncache_search(self.feature_dbs[l], q_l, self.tau, stream=stream)
        attncache_apply_cached(self.map_db, idx, V_l, O_l, hit=hit, layer_begin=l, layer_end=l + 1, stream=stream)
        attncache_attend_full(self.ctx, Q_l, K_l, V_l, O_l, skip=hit, stream=stream)
        return idx, score, hit


class HostPrefill:
    """The same step end to end from pinned host buffers: one C-ABI call (attncache_prefill_host) that does
    every copy inside the library - H2D of the queries, search, D2H of the decisions, then chunk-pipelined
    H2D of V (every row) and Q, K (miss rows only: Alg. 2 computes q, k only on a miss), the kernels, and D2H
    of O over a ring of `depth` device slots on three library streams.  Synchronous: when the call returns,
    O_h and the returned idx/score/hit (pinned host tensors) hold the results."""

    def __init__(self, step: PrefillStep, chunk: Optional[int] = None, depth: int = 4):
        # chunk None: ~192 MB of V per pipeline chunk (attncache_prefill_host's default)
        self.step, self.chunk, self.depth = step, None if chunk is None else int(chunk), int(depth)
        self._out = {}

    def __call__(self, q_h, Q_h, K_h, V_h, O_h):
        B = q_h.shape[0]
        if B not in self._out:
            self._out[B] = tuple(torch.empty(B, dtype=dt).pin_memory() for dt in (torch.int64, torch.float32,
                                                                                  torch.uint8))
        idx, score, hit = self._out[B]
        attncache_prefill_host(self.step.db, q_h, Q_h, K_h, V_h, self.step.tau, O=O_h, idx=idx, score=score, hit=hit,
                               chunk=self.chunk, depth=self.depth)
        return idx, score, hit
