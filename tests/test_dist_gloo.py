"""N>1 host logic on CPU: the collective protocol (tests/dist_model.py, the model of the library's COLLECTIVE calls) under
torch.distributed/gloo with world size 2 and 3, with the per-rank kernels replaced by reference ops built on the oracle.

Checks (north_star): the sharded search (query all-gather, local top-1 as packed
keys, key all-gather + max) equals the single-process oracle search bit-for-bit (idx, hit), routed
hits return A.V computed on the owner, misses get local full attention, for uneven shards, uneven
home batches (including an empty one) and a duplicate entry planted across shards.
"""
import os
import socket
import struct

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from tests._util import storage

TAU = 0.9


def _key(score64, gidx):
    """Packed key (include/attncache.h, reading R3), re-derived here: ord(f32 score) << 32 | ~idx."""
    s = np.float32(score64) + np.float32(0.0)
    b = struct.unpack("<I", struct.pack("<f", s))[0]
    o = (~b & 0xFFFFFFFF) if b & 0x80000000 else (b | 0x80000000)
    return (o << 32) | (0xFFFFFFFF - int(gidx))


def _unkey(k):
    o = k >> 32
    b = (o & 0x7FFFFFFF) if o & 0x80000000 else (~o & 0xFFFFFFFF)
    return struct.unpack("<f", struct.pack("<I", b))[0], 0xFFFFFFFF - (k & 0xFFFFFFFF)


class RefOps:
    """Reference per-rank ops on CPU tensors (test infrastructure, not the product)."""

    def __init__(self, cfg, x_shard, maps_shard, begin):
        self.cfg, self.x, self.maps, self.begin = cfg, x_shard, maps_shard, begin

    def search_keys(self, q):
        keys = np.zeros(q.shape[0], dtype=np.uint64)
        if self.x.shape[0] and q.shape[0]:
            idx, s1, _, _ = oracle.search(storage(q), storage(self.x), "f32", TAU)
            keys[:] = [_key(s, self.begin + i) for s, i in zip(s1, idx)]
        return torch.from_numpy(keys.view(np.int64).copy())

    def keys_decode(self, keys_all, tau):
        u = keys_all.numpy().view(np.uint64).max(axis=0)
        out = [(-1, float("-inf"), 0) if k == 0 else (lambda s, i: (i, s, int(s >= np.float32(tau))))(*_unkey(int(k)))
               for k in u]
        return (torch.tensor([o[0] for o in out], dtype=torch.int64),
                torch.tensor([o[1] for o in out], dtype=torch.float32),
                torch.tensor([o[2] for o in out], dtype=torch.uint8))

    def route_plan(self, idx, hit, shard_begins):
        sb = shard_begins.tolist()
        owner = [-1 if not h else max(r for r in range(len(sb) - 1) if sb[r] <= i) for i, h in zip(idx.tolist(), hit.tolist())]
        counts = [owner.count(r) for r in range(len(sb) - 1)]
        order = [b for r in range(len(sb) - 1) for b in range(len(owner)) if owner[b] == r]
        return (torch.tensor(owner, dtype=torch.int32), torch.tensor(counts, dtype=torch.int32),
                torch.tensor(order + [0], dtype=torch.int64))

    def gather_rows(self, src, rows):
        return src[rows].contiguous()

    def scatter_rows(self, src, rows, dst):
        dst[rows] = src
        return dst

    def apply_cached(self, idx, V, layer_begin=0, layer_end=None):
        c = self.cfg
        units = [(b, l, h) for b in range(V.shape[0]) for l in range(c.L) for h in range(c.H)]
        ents = (idx - self.begin).tolist()
        assert all(0 <= e < self.maps.shape[0] for e in ents), "a routed row is not owned by this rank"
        a_off = [((ents[b] * c.L + l) * c.H + h) * c.S * c.S for b, l, h in units]
        v_off = [((b * c.L + l) * c.H + h) * c.S * c.d for b, l, h in units]
        O = oracle.apply(storage(self.maps), "f16", a_off, storage(V), "f32", v_off, c.S, c.d)
        return torch.from_numpy(O.astype(np.float32)).view(V.shape)

    def apply_cached_masked(self, idx, hit, V, O, layer_begin=0, layer_end=None):
        sel = torch.nonzero(hit).flatten()
        if sel.numel():
            O[sel] = self.apply_cached(idx[sel], V[sel].contiguous(), layer_begin, layer_end)
        return O

    def attend_full(self, Q, K, V, O, skip):
        c = self.cfg
        for b in range(Q.shape[0]):
            if skip[b]:
                continue
            off = [((b * c.L + l) * c.H + h) * c.S * c.d for l in range(c.L) for h in range(c.H)]
            res = oracle.attend(storage(Q), storage(K), storage(V), "f32", off, c.S, c.d)
            O[b] = torch.from_numpy(res.astype(np.float32)).view(O[b].shape)
        return O


def _worker(rank, world, port, homes):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.dist_model import ShardedPrefill, shard_range
        cfg = synth.CONFIGS["tiny"]
        x = synth.features(cfg, 0, cfg.N)
        x[200] = x[3]                                     # duplicate across shards: global top-1 is 3
        maps = synth.maps(cfg, 0, cfg.N)
        q, _, _ = synth.queries(cfg)
        q[1] = x[200]
        Q, K, V = (synth.activations(cfg, k, 0, cfg.B) for k in "qkv")
        begin, count = shard_range(cfg.N, world, rank)
        ops = RefOps(cfg, x[begin:begin + count], maps[begin:begin + count], begin)
        step = ShardedPrefill(ops, cfg.N, TAU, device="cpu")
        lo = sum(homes[:rank])
        hi = lo + homes[rank]
        O = torch.full_like(V[lo:hi], float("nan"))
        idx, score, hit = step(q[lo:hi].contiguous(), Q[lo:hi].contiguous(), K[lo:hi].contiguous(),
                               V[lo:hi].contiguous(), O)
        # single-process oracle over the whole DB
        i_o, s1, _, h_o = oracle.search(storage(q), storage(x), "f32", TAU)
        assert idx.tolist() == i_o[lo:hi].tolist(), (rank, idx.tolist(), i_o[lo:hi].tolist())
        assert hit.tolist() == h_o[lo:hi].tolist()
        assert np.allclose(score.numpy(), s1[lo:hi], atol=1e-6)
        if lo <= 1 < hi:
            assert idx[1 - lo].item() == 3
        c = cfg
        for bl in range(hi - lo):
            b = lo + bl
            off = [((b * c.L + l) * c.H + h) * c.S * c.d for l in range(c.L) for h in range(c.H)]
            if h_o[b]:
                a_off = [((i_o[b] * c.L + l) * c.H + h) * c.S * c.S for l in range(c.L) for h in range(c.H)]
                ref = oracle.apply(storage(maps), "f16", a_off, storage(V), "f32", off, c.S, c.d)
            else:
                ref = oracle.attend(storage(Q), storage(K), storage(V), "f32", off, c.S, c.d)
            got = O[bl].double().numpy().reshape(ref.shape)
            assert np.max(np.abs(got - ref)) < 1e-5, (rank, b)
    finally:
        dist.destroy_process_group()


def _affinity_worker(rank, world, port, homes):
    """Owner-affinity placement: the plan is identical on every rank, each hit is
    processed on the owner of its entry, relocated request rows arrive intact, and every query's
    output computed on its assigned rank equals the single-process oracle."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from tests.dist_model import AffinityPrefill, shard_range
        cfg = synth.CONFIGS["tiny"]
        x = synth.features(cfg, 0, cfg.N)
        x[200] = x[3]
        maps = synth.maps(cfg, 0, cfg.N)
        q, _, _ = synth.queries(cfg)
        q[1] = x[200]
        Q, K, V = (synth.activations(cfg, k, 0, cfg.B) for k in "qkv")
        Xh = torch.randn(cfg.B, cfg.S, 24, generator=torch.Generator().manual_seed(7))  # request state rows
        begin, count = shard_range(cfg.N, world, rank)
        ops = RefOps(cfg, x[begin:begin + count], maps[begin:begin + count], begin)
        step = AffinityPrefill(ops, cfg.N, TAU, hit_cost=1.0, miss_cost=1.5, device="cpu")
        lo = sum(homes[:rank])
        hi = lo + homes[rank]
        plan = step.plan(q[lo:hi].contiguous())
        i_o, s1, _, h_o = oracle.search(storage(q), storage(x), "f32", TAU)
        assert plan["idx"].tolist() == i_o.tolist() and plan["hit"].tolist() == h_o.tolist()
        assign = plan["assign"]
        every = [torch.empty(len(assign), dtype=torch.int32) for _ in range(world)]
        dist.all_gather(every, torch.from_numpy(assign))
        assert all(a.tolist() == assign.tolist() for a in every), "plans differ across ranks"
        for b in range(cfg.B):
            if h_o[b]:
                r = assign[b].item()
                b0, c0 = shard_range(cfg.N, world, r)
                assert b0 <= i_o[b] < b0 + c0, (b, r)       # processed where its maps live
        loc = step.local_queries(plan)
        got_rows = step.relocate(Xh[lo:hi].contiguous(), plan)
        assert torch.equal(got_rows, Xh[loc]), rank
        O = torch.full_like(V[loc], float("nan"))
        step.apply_local(plan, loc, V[loc].contiguous(), O, Q[loc].contiguous(), K[loc].contiguous())
        c = cfg
        for k, b in enumerate(loc.tolist()):
            off = [((b * c.L + l) * c.H + h) * c.S * c.d for l in range(c.L) for h in range(c.H)]
            if h_o[b]:
                a_off = [((i_o[b] * c.L + l) * c.H + h) * c.S * c.S for l in range(c.L) for h in range(c.H)]
                ref = oracle.apply(storage(maps), "f16", a_off, storage(V), "f32", off, c.S, c.d)
            else:
                ref = oracle.attend(storage(Q), storage(K), storage(V), "f32", off, c.S, c.d)
            assert np.max(np.abs(O[k].double().numpy().reshape(ref.shape) - ref)) < 1e-5, (rank, b)
        total = torch.tensor([loc.numel()])
        dist.all_reduce(total)
        assert total.item() == cfg.B                        # every query placed exactly once
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,homes", [(2, [5, 3]), (3, [4, 0, 4])])
def test_affinity_prefill_gloo(world, homes):
    mp.spawn(_affinity_worker, args=(world, _free_port(), homes), nprocs=world, join=True)


def test_affinity_plan_minimises_max_load():
    """attncache_affinity_plan (the C ABI's host function) against brute force: hits on their owner,
    and the greedy miss placement reaches the minimum possible maximum load on small instances."""
    import itertools
    from paper_2510_25979_b200 import attncache_affinity_plan
    g = np.random.default_rng(3)
    for trial in range(300):
        world = int(g.integers(1, 4))
        n = int(g.integers(0, 8))
        cuts = np.sort(g.integers(0, 20, world - 1)) if world > 1 else np.array([], dtype=np.int64)
        sb = [0] + cuts.tolist() + [20]                     # may contain empty shards
        idx = g.integers(0, 20, n)
        hit = (g.random(n) < 0.5).astype(np.uint8)
        hc, mc = float(g.choice([1.0, 2.0])), float(g.choice([1.0, 1.5, 3.0]))
        assign, load = attncache_affinity_plan(torch.from_numpy(idx), torch.from_numpy(hit), sb, hc, mc)
        assign = assign.tolist()
        owner = [max(r for r in range(world) if sb[r] <= e and e < sb[r + 1]) for e in idx]
        for b in range(n):
            if hit[b]:
                assert assign[b] == owner[b]
        base = [0.0] * world
        for b in range(n):
            if hit[b]:
                base[owner[b]] += hc
        misses = [b for b in range(n) if not hit[b]]
        best = min((max(base[r] + mc * sum(1 for a in combo if a == r) for r in range(world))
                    for combo in itertools.product(range(world), repeat=len(misses))), default=max(base))
        assert max(load.tolist()) == pytest.approx(best), (trial, sb, idx, hit)
        assert load.tolist() == pytest.approx([hc * sum(1 for b in range(n) if hit[b] and assign[b] == r)
                                               + mc * sum(1 for b in misses if assign[b] == r) for r in range(world)])


def test_affinity_plan_errors():
    from paper_2510_25979_b200 import AttnCacheError, attncache_affinity_plan
    idx = torch.tensor([3, 25], dtype=torch.int64)
    hit = torch.tensor([1, 1], dtype=torch.uint8)
    with pytest.raises(AttnCacheError):                     # a hit outside the DB
        attncache_affinity_plan(idx, hit, [0, 10, 20])
    with pytest.raises(AttnCacheError):                     # negative cost
        attncache_affinity_plan(idx[:1], hit[:1], [0, 10, 20], -1.0, 1.0)
    with pytest.raises(AttnCacheError):                     # decreasing shard_begins
        attncache_affinity_plan(idx[:1], hit[:1], [0, 12, 10])
    a, l = attncache_affinity_plan(idx[:0], hit[:0], [0, 10, 20])
    assert a.numel() == 0 and l.tolist() == [0.0, 0.0]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("world,homes", [(2, [5, 3]), (3, [4, 0, 4])])
def test_sharded_prefill_gloo(world, homes):
    assert sum(homes) == synth.CONFIGS["tiny"].B
    mp.spawn(_worker, args=(world, _free_port(), homes), nprocs=world, join=True)


def test_shard_range_partitions():
    from paper_2510_25979_b200.dist import shard_range
    for n in (0, 1, 7, 256, 1000):
        for w in (1, 2, 3, 8):
            parts = [shard_range(n, w, r) for r in range(w)]
            assert parts[0][0] == 0 and sum(c for _, c in parts) == n
            assert all(parts[r][0] + parts[r][1] == parts[r + 1][0] for r in range(w - 1))
