"""One AttnCache prefill attention step on one GPU: the whole hot path (SURVEY.md §8(a) a1-a8, N=1).

    search (Alg. 1 l.255-257) -> hit branch O = A.V (Alg. 2 l.373-375) for hits
                              -> miss branch softmax(QK^T/sqrt(d)).V (Alg. 2 l.376-381) for misses

Pure orchestration over the C ABI: no arithmetic here.  At N = 1 the routing
rows of §8(a) (a5, a7) are the identity, so hits are served in place.
"""
from __future__ import annotations

from typing import Optional

import torch

from . import (Context, Database, attncache_apply_cached, attncache_attend_full, attncache_search)


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
