"""Multi-GPU data-parallel AttnCache step (BASELINE.json north_star).

The memoization database shards by contiguous entry ranges across ranks (one process per GPU).
Each query has a home rank.  One step:

  a2  C1  all-gather the query batch                               (torch.distributed, NCCL)
  a3  K1  local exact top-1 over this shard -> packed keys          (attncache_search_keys)
  a4  C2  all-gather the keys; K2 max over shards + tau gate        (attncache_keys_decode)
  a5  K3  bucket the home hits by owner rank                        (attncache_route_plan)
      C3  exchange per-peer row counts (host sync: sizes the buffers)
  a6  C4  V rows -> owner (all_to_all);  K4  O = A.V on the owner  (attncache_apply_cached)
  a7  C5  O rows -> home  (all_to_all);  K3  scatter into O          (attncache_scatter_rows)
  a8  K5  misses: local causal attention                            (attncache_attend_full)

Owner-affinity variant (`AffinityPrefill`): after the search, which every rank
runs for the whole batch, each query is placed ONCE, before the layer loop, on the rank that will
process all its layers: a hit on the owner of its entry, misses on the least-loaded ranks
(attncache_affinity_plan, a host function of the C ABI).  The request's hidden state moves once
(one all_to_all of [S][E] rows) instead of V and O for every layer, so NVLink carries
B*S*E*2 bytes per batch rather than 2*B*L*H*S*d*2, and every A.V reads local maps.

Collectives are torch.distributed (NCCL over NVLink/NVSwitch on the GPU box, gloo in the CPU
tests); every per-rank computation goes through `ops`, which in the product is `CudaOps` (the C
ABI).  The CPU tests inject their own reference ops to check this host logic with world size 2-3.
"""
from __future__ import annotations

from typing import List, Optional

import numpy as np
import torch
import torch.distributed as dist

from . import (Context, Database, attncache_affinity_plan, attncache_affinity_plan_device, attncache_apply_cached, attncache_attend_full,
               attncache_gather_rows, attncache_keys_decode, attncache_route_plan, attncache_scatter_rows,
               attncache_search_keys)


def shard_range(n: int, world: int, rank: int):
    """Contiguous entry range [begin, begin + count) of `rank` (the first n % world ranks get one more)."""
    base, extra = divmod(n, world)
    begin = rank * base + min(rank, extra)
    return begin, base + (1 if rank < extra else 0)


class CudaOps:
    """The product's per-rank kernels (C ABI) for one shard."""

    def __init__(self, ctx: Context, db: Database):
        self.ctx, self.db = ctx, db

    def search_keys(self, q):
        return attncache_search_keys(self.db, q)

    def keys_decode(self, keys_all, tau):
        return attncache_keys_decode(keys_all, tau)

    def route_plan(self, idx, hit, shard_begins):
        return attncache_route_plan(idx, hit, shard_begins)

    def gather_rows(self, src, rows):
        return attncache_gather_rows(src, rows)

    def scatter_rows(self, src, rows, dst):
        return attncache_scatter_rows(src, rows, dst)

    def apply_cached(self, idx, V, layer_begin=0, layer_end=None):
        return attncache_apply_cached(self.db, idx, V, layer_begin=layer_begin, layer_end=layer_end)

    def apply_cached_masked(self, idx, hit, V, O, layer_begin=0, layer_end=None):
        return attncache_apply_cached(self.db, idx, V, O, hit=hit, layer_begin=layer_begin, layer_end=layer_end)

    def affinity_plan_device(self, idx, hit, shard_begins, home_begins, rank, hit_cost, miss_cost):
        return attncache_affinity_plan_device(self.ctx, idx, hit, shard_begins, home_begins, rank, hit_cost, miss_cost)

    def attend_full(self, Q, K, V, O, skip):
        return attncache_attend_full(self.ctx, Q, K, V, O, skip=skip)


class ShardedPrefill:
    """One rank's view of the sharded step.  All ranks must call the same methods in the same order
    (NCCL semantics); home batch sizes may differ per rank and may be 0."""

    def __init__(self, ops, n_global: int, tau: float, group=None, device="cuda"):
        self.ops, self.n_global, self.tau, self.group = ops, int(n_global), float(tau), group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.device = torch.device(device)
        begins = [shard_range(self.n_global, self.world, r)[0] for r in range(self.world)] + [self.n_global]
        self.shard_begins = torch.tensor(begins, dtype=torch.int64, device=self.device)

    # ---- a2-a4: sharded search -------------------------------------------------------------------
    def _home_sizes(self, b_home: int) -> List[int]:
        t = torch.tensor([b_home], dtype=torch.int64, device=self.device)
        out = torch.empty(self.world, dtype=torch.int64, device=self.device)
        dist.all_gather_into_tensor(out, t, group=self.group)
        return out.cpu().tolist()

    def search(self, q_home: torch.Tensor):
        """Returns this rank's (idx, score, hit) for its home queries: the global top-1 over all shards."""
        idx, score, hit, sizes = self.search_all(q_home)
        lo = sum(sizes[:self.rank])
        hi = lo + sizes[self.rank]
        return idx[lo:hi].contiguous(), score[lo:hi].contiguous(), hit[lo:hi].contiguous()

    def search_all(self, q_home: torch.Tensor, sizes: Optional[List[int]] = None):
        """The global top-1 of EVERY query of the batch (each rank decodes all keys after C2), in the
        order of the home blocks (rank 0's queries first); returns (idx, score, hit, home sizes).
        `sizes` (the home batch size of every rank) may be passed when known, saving one exchange."""
        sizes = self._home_sizes(q_home.shape[0]) if sizes is None else list(sizes)
        bmax = max(max(sizes), 1)
        D = q_home.shape[1]
        if min(sizes) == bmax:  # equal home blocks: gather in place, no padding
            q_all = torch.empty(self.world * bmax, D, dtype=q_home.dtype, device=self.device)
            dist.all_gather_into_tensor(q_all, q_home.contiguous(), group=self.group)          # C1
        else:
            pad = torch.zeros(bmax, D, dtype=q_home.dtype, device=self.device)
            pad[:q_home.shape[0]] = q_home
            q_all = torch.empty(self.world * bmax, D, dtype=q_home.dtype, device=self.device)
            dist.all_gather_into_tensor(q_all, pad, group=self.group)                          # C1
            q_all = q_all.view(self.world, bmax, D)
            q_all = torch.cat([q_all[r, :sizes[r]] for r in range(self.world)]) if sum(sizes) else q_all[0, :0]
        keys = self.ops.search_keys(q_all.contiguous())                                         # K1
        keys_all = torch.empty(self.world * keys.shape[0], dtype=keys.dtype, device=self.device)
        dist.all_gather_into_tensor(keys_all, keys, group=self.group)                           # C2
        idx, score, hit = self.ops.keys_decode(keys_all.view(self.world, -1), self.tau)         # K2
        return idx, score, hit, sizes

    # ---- a5-a7: route hits to the owner, compute A.V there, return O ---------------------------------
    def apply_routed(self, idx_home, hit_home, V_home, O_home, layer_begin=0, layer_end=None):
        b_home = idx_home.shape[0]
        owner, counts, order = self.ops.route_plan(idx_home, hit_home, self.shard_begins)       # K3
        send_counts = counts.to(torch.int64)
        recv_counts = torch.empty_like(send_counts)
        dist.all_to_all_single(recv_counts, send_counts, group=self.group)                       # C3
        send_n = send_counts.cpu().tolist()
        recv_n = recv_counts.cpu().tolist()
        rows = order[:sum(send_n)].contiguous()
        row_shape = V_home.shape[1:]
        V_send = self.ops.gather_rows(V_home, rows) if sum(send_n) else V_home[:0]
        idx_send = self.ops.gather_rows(idx_home, rows) if sum(send_n) else idx_home[:0]
        V_recv = torch.empty((sum(recv_n), *row_shape), dtype=V_home.dtype, device=self.device)
        idx_recv = torch.empty(sum(recv_n), dtype=idx_home.dtype, device=self.device)
        dist.all_to_all_single(V_recv, V_send, recv_n, send_n, group=self.group)                 # C4
        dist.all_to_all_single(idx_recv, idx_send, recv_n, send_n, group=self.group)
        if sum(recv_n):
            O_recv = self.ops.apply_cached(idx_recv, V_recv, layer_begin, layer_end)            # K4
        else:
            O_recv = V_recv
        O_back = torch.empty((sum(send_n), *row_shape), dtype=V_home.dtype, device=self.device)
        dist.all_to_all_single(O_back, O_recv, send_n, recv_n, group=self.group)                 # C5
        if sum(send_n):
            self.ops.scatter_rows(O_back, rows, O_home)                                          # K3
        return O_home

    # ---- the whole step ----------------------------------------------------------------------------
    def __call__(self, q_home, Q_home, K_home, V_home, O_home):
        idx, score, hit = self.search(q_home)
        self.apply_routed(idx, hit, V_home, O_home)
        if q_home.shape[0]:
            self.ops.attend_full(Q_home, K_home, V_home, O_home, hit)                           # K5
        return idx, score, hit


class AffinityPrefill(ShardedPrefill):
    """Owner-affinity placement: the sharded search, then one placement of every
    query on the rank that processes all of its layers locally.

    hit_cost / miss_cost weight the greedy miss placement (attncache_affinity_plan); callers pass the
    algorithmic HBM bytes of one query's A.V and of one query's attention.

    With the product's ops (CudaOps, world <= 32) the placement runs on the device
    (attncache_affinity_plan_device, bitwise the host plan) and only the all_to_all counts come back
    (one small D2H).  Otherwise (the gloo reference ops): one small D2H of the decoded top-1 of every
    query, the C host placement, and one small H2D of this rank's relocation order and local idx/hit."""

    def __init__(self, ops, n_global: int, tau: float, hit_cost: float = 1.0, miss_cost: float = 1.0,
                 group=None, device="cuda"):
        super().__init__(ops, n_global, tau, group=group, device=device)
        self.hit_cost, self.miss_cost = float(hit_cost), float(miss_cost)
        self._sb_host = np.asarray([shard_range(self.n_global, self.world, r)[0] for r in range(self.world)]
                                   + [self.n_global], dtype=np.int64)

    def plan(self, q_home: torch.Tensor, sizes: Optional[List[int]] = None):
        """Search + placement.  Returns a dict with the whole batch's idx/score/hit (device), `assign`
        (numpy int32[B], the processing rank of every query), the home sizes, the per-rank loads, and
        this rank's local queries with their idx/hit on the device."""
        idx, score, hit, sizes = self.search_all(q_home, sizes)
        if hasattr(self.ops, "affinity_plan_device") and self.world <= 32:
            # the plan on the device (bitwise the host plan); only the all_to_all counts come back
            home_begins = np.cumsum([0] + list(sizes)).tolist()
            out = self.ops.affinity_plan_device(idx, hit, self._sb_host.tolist(), home_begins, self.rank,
                                                self.hit_cost, self.miss_cost)
            counts = out["counts"].tolist()                                                      # one small D2H
            w = self.world
            n_loc = counts[2 * w]
            return {"idx": idx, "score": score, "hit": hit, "assign": out["assign"], "sizes": sizes,
                    "load": out["load"], "loc": out["loc"][:n_loc], "send_order": out["send_order"],
                    "send_n": counts[:w], "recv_n": counts[w:2 * w], "idx_loc": out["idx_loc"][:n_loc],
                    "hit_loc": out["hit_loc"][:n_loc]}
        code = torch.where(hit.bool(), idx, torch.full_like(idx, -1)).cpu().numpy()            # one D2H
        hit_h = (code >= 0).astype(np.uint8)
        assign, load = attncache_affinity_plan(np.maximum(code, 0), hit_h, self._sb_host, self.hit_cost,
                                               self.miss_cost)
        loc = np.nonzero(assign == self.rank)[0]
        lo = sum(sizes[:self.rank])
        mine = assign[lo:lo + sizes[self.rank]].astype(np.int64)
        send_order = np.argsort(mine, kind="stable")                                            # by destination, then b
        send_n = np.bincount(mine, minlength=self.world).tolist()
        bounds = np.cumsum([0] + list(sizes))
        recv_n = [int((assign[bounds[r]:bounds[r + 1]] == self.rank).sum()) for r in range(self.world)]
        # one H2D: [send_order | idx_loc | hit_loc] as int64
        n_loc = loc.shape[0]
        host = np.concatenate([send_order, code[loc].clip(min=0), hit_h[loc].astype(np.int64)])
        dev = torch.from_numpy(host).to(self.device, non_blocking=False)
        return {"idx": idx, "score": score, "hit": hit, "assign": assign, "sizes": sizes, "load": load,
                "loc": torch.from_numpy(loc), "send_order": dev[:send_order.shape[0]], "send_n": send_n,
                "recv_n": recv_n, "idx_loc": dev[send_order.shape[0]:send_order.shape[0] + n_loc],
                "hit_loc": dev[send_order.shape[0] + n_loc:].to(torch.uint8)}

    def local_queries(self, plan) -> torch.Tensor:
        """Global batch positions this rank processes, ascending (int64, CPU)."""
        return plan["loc"].cpu()

    def relocate(self, rows_home: torch.Tensor, plan) -> torch.Tensor:
        """Moves each home row (one query's request state, e.g. its hidden states [S][E]) to the rank
        the plan assigns it to: one all_to_all.  Returns the rows of `local_queries(plan)` in that order
        (home blocks are contiguous and ascending in rank, so sources arrive in global order)."""
        send_n, recv_n = plan["send_n"], plan["recv_n"]
        row_shape = rows_home.shape[1:]
        send = self.ops.gather_rows(rows_home, plan["send_order"]) if rows_home.shape[0] else rows_home[:0]
        recv = torch.empty((sum(recv_n), *row_shape), dtype=rows_home.dtype, device=self.device)
        dist.all_to_all_single(recv, send.contiguous(), recv_n, send_n, group=self.group)
        return recv

    def apply_local(self, plan, loc, V_loc, O_loc, Q_loc=None, K_loc=None, layer_begin=0, layer_end=None):
        """All the layers of this rank's queries, locally: O = A.V for hits (the maps are in this shard),
        causal attention for misses.  V_loc/O_loc (and Q_loc/K_loc) are [len(loc)][L'][H][S][d]."""
        if not loc.numel():
            return O_loc
        idx_loc, hit_loc = plan["idx_loc"], plan["hit_loc"]
        self.ops.apply_cached_masked(idx_loc, hit_loc, V_loc, O_loc, layer_begin, layer_end)     # K4
        if Q_loc is not None:
            self.ops.attend_full(Q_loc, K_loc, V_loc, O_loc, hit_loc)                           # K5
        return O_loc
