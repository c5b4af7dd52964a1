"""One rank of the multi-GPU check (launched by tests/test_gpu_multi.py under torch.distributed.run, one
process per GPU): the library's collective step over its own NCCL communicator must equal, bitwise, the
single-GPU step on the whole DB (reading R19: outputs do not depend on the shard count), for the routed and
the owner-affinity placements, under skewed ownership.  Exits non-zero on a mismatch."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import synth  # noqa: E402
import paper_2510_25979_b200 as ac  # noqa: E402
from paper_2510_25979_b200.dist import AffinityPrefill, ShardedPrefill, shard_range  # noqa: E402
from paper_2510_25979_b200.pipeline import PrefillStep  # noqa: E402


def main():
    rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    # ATTNCACHE_TEST_SINGLE_DEVICE=1 (tests/test_gpu_fake_nccl.py): every rank on GPU 0, the library's collectives
    # over tests/native/fake_nccl.cpp (ATTNCACHE_NCCL_LIB), torch.distributed over gloo (uid broadcast only)
    single = os.environ.get("ATTNCACHE_TEST_SINGLE_DEVICE") == "1"
    if single:
        local = 0
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    if single:
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=dev)
    cctx = ac.Context.from_process_group(local)
    lctx = ac.Context(local)
    cfg = synth.CONFIGS["llama32_1b"].with_(N=8 * world + 3, B=4 * world + 1, L=2)
    x = synth.features(cfg, 0, cfg.N, dev)
    maps = ac.attncache_pack_maps(synth.maps(cfg, 0, cfg.N, dev))
    full_db = ac.Database(lctx, x, maps, packed=True, seq_len=cfg.S)
    b0, c0 = shard_range(cfg.N, world, rank)
    db = ac.Database(cctx, x[b0:b0 + c0].contiguous(), maps[b0:b0 + c0].contiguous(), n_global=cfg.N, shard_begin=b0,
                     packed=True, seq_len=cfg.S)
    for pattern in ("spread", "one_shard", "remote_only", "no_hits"):
        g = torch.Generator(device=dev).manual_seed(5)
        if pattern == "spread":
            tgt = torch.randperm(cfg.N, generator=torch.Generator().manual_seed(1))[:cfg.B - 2]
        elif pattern == "one_shard":  # every hit owned by the last rank
            lb, lc = shard_range(cfg.N, world, world - 1)
            tgt = lb + torch.randperm(lc, generator=torch.Generator().manual_seed(2))[:min(lc, cfg.B - 2)]
        elif pattern == "remote_only":  # no hit owned by rank 0
            s1 = shard_range(cfg.N, world, 1)[0]
            tgt = s1 + torch.randperm(cfg.N - s1, generator=torch.Generator().manual_seed(3))[:cfg.B - 2]
        else:
            tgt = torch.tensor([], dtype=torch.int64)
        q = torch.randn(cfg.B, cfg.D, device=dev, generator=g)
        q[:len(tgt)] = x[tgt.to(dev)].float() + 0.001 * torch.randn(len(tgt), cfg.D, device=dev, generator=g)
        q = (q / q.norm(dim=1, keepdim=True)).to(x.dtype)
        Q, K, V = (synth.activations(cfg, k, 0, cfg.B, device=dev) for k in "qkv")
        O_ref = torch.empty_like(V)
        ref = PrefillStep(lctx, full_db, cfg.tau)(q, Q, K, V, O_ref)
        sizes = [shard_range(cfg.B, world, r)[1] for r in range(world)]
        hb, hc = shard_range(cfg.B, world, rank)
        sl = slice(hb, hb + hc)
        for layout in (None, sizes):
            cctx.set_batch_layout(None)
            O = torch.empty_like(V[sl])
            got = ShardedPrefill(cctx, db, cfg.tau, layout)(q[sl].contiguous(), Q[sl].contiguous(), K[sl].contiguous(),
                                                            V[sl].contiguous(), O)
            cctx.sync()
            for a, b in zip(ref, got):
                assert torch.equal(a[sl], b), (rank, pattern, "search")
            assert torch.equal(O_ref[sl], O), (rank, pattern, "routed O")
        aff = AffinityPrefill(cctx, db, cfg.tau, sizes, hit_cost=1.0, miss_cost=1.3)
        plan = aff.plan(q[sl].contiguous())
        assert torch.equal(plan["idx"], ref[0]) and torch.equal(plan["hit"], ref[2]), (rank, pattern, "search_all")
        loc = aff.local_queries(plan)
        moved = aff.relocate(V[sl].contiguous(), plan)
        assert torch.equal(moved, V[loc.to(dev)]), (rank, pattern, "relocate")
        O_loc = torch.empty_like(moved)
        aff.apply_local(plan, loc, moved, O_loc, Q[loc.to(dev)].contiguous(), K[loc.to(dev)].contiguous())
        cctx.sync()
        assert torch.equal(O_loc, O_ref[loc.to(dev)]), (rank, pattern, "affinity O")
        n = torch.tensor([loc.numel()], device="cpu" if single else dev)
        dist.all_reduce(n)
        assert n.item() == cfg.B, "every query placed exactly once"
    del db, full_db
    cctx.close()
    dist.destroy_process_group()
    if rank == 0:
        print(f"multi_gpu_step: world {world} ok")


if __name__ == "__main__":
    main()
