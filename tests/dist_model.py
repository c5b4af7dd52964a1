"""Protocol model of the library's collective calls, written with torch.distributed — TEST INFRASTRUCTURE.

The product's multi-GPU step (paper_2510_25979_b200/dist.py) runs every exchange inside libattncache over
its own NCCL communicator (include/attncache.h COLLECTIVE calls).  Those calls cannot run on a GPU-less
host, so tests/test_dist_gloo.py checks the same protocol here, step for step, with gloo at world size 2-3
and reference per-rank ops built on the oracle:

  a2  C1  all-gather the query batch
  a3  K1  local exact top-1 over this shard -> packed keys
  a4  C2  max over shards of the keys (the library: one NCCL u64 max-all-reduce); K2 decode + tau gate
  a5  K3  bucket the home hits by owner rank; C3 exchange per-peer row counts (host round trip)
  a6  C4  V rows -> owner;  K4  O = A.V on the owner
  a7  C5  O rows -> home;   K3  scatter into O
  a8  K5  misses: local causal attention

and the owner-affinity placement (attncache_affinity_plan, the C ABI's host function, then one relocation
of every query's request state).
"""
from __future__ import annotations

from typing import List, Optional

import numpy as np
import torch
import torch.distributed as dist

from paper_2510_25979_b200 import attncache_affinity_plan
from paper_2510_25979_b200.dist import shard_range


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

    The product runs the same placement on the device (attncache_affinity_plan_device, bitwise the host
    plan; GPU-tested against it); this model uses the host function: one D2H of the decoded top-1 of every
    query, the C host placement, and one H2D of this rank's relocation order and local idx/hit."""

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
