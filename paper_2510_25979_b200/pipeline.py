"""One AttnCache prefill attention step on one GPU: the whole hot path (SURVEY.md §8(a) a1-a8, N=1).

    search (Alg. 1 l.255-257) -> hit branch O = A.V (Alg. 2 l.373-375) for hits
                              -> miss branch softmax(QK^T/sqrt(d)).V (Alg. 2 l.376-381) for misses

Pure orchestration over the C ABI: no arithmetic here.  At N = 1 the routing
rows of §8(a) (a5, a7) are the identity, so hits are served in place.
"""
from __future__ import annotations

from typing import Optional

import torch

from . import (Context, Database, attncache_apply_cached, attncache_attend_full, attncache_project_features,
               attncache_search)


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
    """The same step end to end from (pinned) host buffers, pipelined over chunks of the batch.

    search on all queries (H2D of the queries, D2H of the hit mask: the host must know the misses,
    whose Q and K exist only on a miss — Alg. 2 l.376-378), then per chunk of `chunk` rows: H2D of
    V (every row) and of Q, K (miss rows only) on a copy-in stream, apply_cached + attend_full on the
    compute stream, D2H of O on a copy-out stream.  A ring of `depth` device chunk buffers lets the
    copies of chunk k+1 and k-1 overlap the kernels of chunk k (PCIe is full duplex).
    """

    def __init__(self, step: PrefillStep, chunk: int = 32, depth: int = 3):
        self.step, self.chunk, self.depth = step, int(chunk), int(depth)
        self._dev = None

    def _buffers(self, row_shape, dtype, device):
        key = (tuple(row_shape), dtype, device)
        if self._dev is None or self._dev[0] != key:
            c, R = self.chunk, self.depth
            mk = lambda: [torch.empty((c, *row_shape), dtype=dtype, device=device) for _ in range(R)]
            self._dev = (key, mk(), mk(), mk(), mk())  # V, Q, K, O rings
        return self._dev[1:]

    def __call__(self, q_h, Q_h, K_h, V_h, O_h, device=None):
        device = device or self.step.db.device
        comp = torch.cuda.current_stream(device)
        cin, cout = torch.cuda.Stream(device), torch.cuda.Stream(device)
        B = q_h.shape[0]
        qd = q_h.to(device, non_blocking=True)
        idx, score, hit = self.step.search(qd)
        hit_h = hit.cpu()  # one host sync: which rows need Q and K
        Vr, Qr, Kr, Or = self._buffers(V_h.shape[1:], V_h.dtype, device)
        R, c = self.depth, self.chunk
        ev_in = [torch.cuda.Event() for _ in range(R)]
        ev_comp = [torch.cuda.Event() for _ in range(R)]
        ev_out = [torch.cuda.Event() for _ in range(R)]
        used = [False] * R
        n_chunks = (B + c - 1) // c
        miss = (hit_h == 0).tolist()
        for k in range(n_chunks):
            r = k % R
            b0, b1 = k * c, min(B, (k + 1) * c)
            n = b1 - b0
            with torch.cuda.stream(cin):
                if used[r]:
                    cin.wait_event(ev_comp[r])
                Vr[r][:n].copy_(V_h[b0:b1], non_blocking=True)
                for b in range(b0, b1):
                    if miss[b]:
                        Qr[r][b - b0].copy_(Q_h[b], non_blocking=True)
                        Kr[r][b - b0].copy_(K_h[b], non_blocking=True)
                ev_in[r].record(cin)
            comp.wait_event(ev_in[r])
            if used[r]:
                comp.wait_event(ev_out[r])  # O slot drained to the host
            self.step.attend(idx[b0:b1], hit[b0:b1], Qr[r][:n], Kr[r][:n], Vr[r][:n], Or[r][:n], stream=comp)
            ev_comp[r].record(comp)
            with torch.cuda.stream(cout):
                cout.wait_event(ev_comp[r])
                O_h[b0:b1].copy_(Or[r][:n], non_blocking=True)
                ev_out[r].record(cout)
            used[r] = True
        comp.wait_stream(cout)
        res = tuple(t.to("cpu", non_blocking=True) for t in (idx, score, hit))
        return res
