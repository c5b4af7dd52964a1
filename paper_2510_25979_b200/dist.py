"""Multi-GPU data-parallel AttnCache step (BASELINE.json north_star) over the library's
own NCCL communicator.

The memoization database shards by contiguous entry ranges across ranks (one process per GPU); each query
has a home rank.  Every exchange runs INSIDE libattncache (include/attncache.h, COLLECTIVE calls); torch is
used for device memory, streams and, once, to broadcast the NCCL unique id (``Context.from_process_group``).

  a2-a4  attncache_search          C1 query all-gather, K1 local top-1, C2 u64 max-all-reduce of the keys, K2
  a5-a7  attncache_apply_cached    K3 bucket hits by owner, C3 counts, C4 V -> owner, K4 A.V, C5 O -> home
  a8     attncache_attend_full     misses: local causal attention

Owner-affinity variant (``AffinityPrefill``): ``attncache_search_all`` gives every rank the whole batch's
decisions, ``attncache_affinity_plan_device`` places each query ONCE (hits on the owner of their entry,
misses on the least-loaded ranks), ``attncache_relocate_rows`` moves each request's state there, and every
layer then runs locally (``attncache_apply_cached_local``): no V or O crosses NVLink per layer.

tests/dist_model.py keeps the same protocol written with torch.distributed (gloo) for the CPU tests.
"""
from __future__ import annotations

from typing import List, Optional

import numpy as np
import torch

from . import (Context, Database, attncache_affinity_plan_device, attncache_apply_cached,
               attncache_apply_cached_local, attncache_attend_full, attncache_relocate_rows, attncache_search,
               attncache_search_all)


def shard_range(n: int, world: int, rank: int):
    """Contiguous entry range [begin, begin + count) of `rank` (the first n % world ranks get one more)."""
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, base + (1 if rank < extra else 0)


class ShardedPrefill:
    """One rank's view of the sharded step (north_star's routing).  All ranks call the same methods in the
    same order (NCCL semantics); home batch sizes may differ per rank and may be 0.  `sizes` (every rank's
    home batch size) may be declared once: the collective search then needs no host round trip."""

    def __init__(self, ctx: Context, db: Database, tau: float, sizes: Optional[List[int]] = None):
        self.ctx, self.db, self.tau = ctx, db, float(tau)
        self.rank, self.world = ctx.rank, ctx.world
        self.sizes = None if sizes is None else [int(s) for s in sizes]
        if self.sizes is not None:
            ctx.set_batch_layout(self.sizes)

    def search(self, q_home: torch.Tensor, stream=None):
        """(idx, score, hit) of this rank's home queries: the global top-1 over every rank's shard."""
        return attncache_search(self.db, q_home, self.tau, stream=stream)

    def apply_routed(self, idx_home, hit_home, V_home, O_home, layer_begin=0, layer_end=None, stream=None):
        return attncache_apply_cached(self.db, idx_home, V_home, O_home, hit=hit_home, layer_begin=layer_begin,
                                      layer_end=layer_end, stream=stream)

    def __call__(self, q_home, Q_home, K_home, V_home, O_home, stream=None):
        idx, score, hit = self.search(q_home, stream=stream)
        self.apply_routed(idx, hit, V_home, O_home, stream=stream)
        if q_home.shape[0]:
            attncache_attend_full(self.ctx, Q_home, K_home, V_home, O_home, skip=hit, stream=stream)
        return idx, score, hit


class AffinityPrefill(ShardedPrefill):
    """Owner-affinity placement: the sharded search, then one placement of every query on
    the rank that processes all of its layers locally.  hit_cost / miss_cost weight the greedy miss
    placement; callers pass the algorithmic HBM bytes of one query's A.V and of one query's attention."""

    def __init__(self, ctx: Context, db: Database, tau: float, sizes: List[int], hit_cost: float = 1.0,
                 miss_cost: float = 1.0):
        super().__init__(ctx, db, tau, sizes)
        self.hit_cost, self.miss_cost = float(hit_cost), float(miss_cost)
        n = db.n_global
        self._sb = [shard_range(n, self.world, r)[0] for r in range(self.world)] + [n]
        self._hb = np.cumsum([0] + self.sizes).tolist()
        self.total = int(self._hb[-1])

    def plan(self, q_home: torch.Tensor, stream=None):
        """Search + placement.  Returns a dict with the whole batch's idx/score/hit and plan arrays (device),
        the host counts (send_n | recv_n | n_loc: one small D2H) and this rank's local queries."""
        st = stream if stream is not None else torch.cuda.current_stream(q_home.device)
        with torch.cuda.stream(st):  # every output is allocated (caching allocator) and written on `st`
            idx, score, hit = attncache_search_all(self.db, q_home, self.tau, total=self.total, stream=st)
            out = attncache_affinity_plan_device(self.ctx, idx, hit, self._sb, self._hb, self.rank, self.hit_cost,
                                                 self.miss_cost, stream=st)
            counts = out["counts"].tolist()                     # one small D2H: waits for this stream only
        w = self.world
        n_loc = counts[2 * w]
        return {"idx": idx, "score": score, "hit": hit, "assign": out["assign"], "sizes": self.sizes,
                "load": out["load"], "loc": out["loc"][:n_loc], "send_order": out["send_order"], "counts": counts,
                "send_n": counts[:w], "recv_n": counts[w:2 * w], "idx_loc": out["idx_loc"][:n_loc],
                "hit_loc": out["hit_loc"][:n_loc]}

    def local_queries(self, plan) -> torch.Tensor:
        """Global batch positions this rank processes, ascending (int64, CPU)."""
        return plan["loc"].cpu()

    def relocate(self, rows_home: torch.Tensor, plan, stream=None) -> torch.Tensor:
        """Moves each home row (one query's request state, e.g. its hidden states [S][E]) to the rank the plan
        assigns it to (COLLECTIVE, inside the library).  Returns the rows of `local_queries(plan)` in order."""
        return attncache_relocate_rows(self.ctx, rows_home, plan["send_order"], plan["counts"], stream=stream)

    def apply_local(self, plan, loc, V_loc, O_loc, Q_loc=None, K_loc=None, layer_begin=0, layer_end=None,
                    stream=None):
        """All the layers of this rank's queries, locally: O = A.V for hits (the maps are in this shard),
        causal attention for misses.  V_loc/O_loc (and Q_loc/K_loc) are [len(loc)][L'][H][S][d]."""
        if not loc.numel():
            return O_loc
        idx_loc, hit_loc = plan["idx_loc"], plan["hit_loc"]
        attncache_apply_cached_local(self.db, idx_loc, V_loc, O_loc, hit=hit_loc, layer_begin=layer_begin,
                                     layer_end=layer_end, stream=stream)                         # K4
        if Q_loc is not None:
            attncache_attend_full(self.ctx, Q_loc, K_loc, V_loc, O_loc, skip=hit_loc, stream=stream)  # K5
        return O_loc
