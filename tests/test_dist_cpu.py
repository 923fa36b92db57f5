"""Multi-process host-side checks of the multi-GPU path (gloo, world_size 2,
CPU only): the NCCL unique id travels through torch.distributed exactly as
bench.py does it, and the cyclic tile shards of every rank are disjoint and
cover all target tiles (the partition dist.cu / sparse_tc.cu use)."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1602_06097_b200 import tile_shard


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, ntiles_list, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        uid = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)          # how bench.py ships the ncclUniqueId
        ok_uid = uid[0] == bytes(range(128))
        shards = {n: tile_shard(n, rank, world) for n in ntiles_list}
        gathered = [None] * world
        dist.all_gather_object(gathered, shards)
        t = torch.tensor([float(rank + 1)])
        dist.all_reduce(t, op=dist.ReduceOp.MAX)          # max-over-ranks timing, as in bench.py
        q.put((rank, ok_uid, gathered, float(t.item())))
    finally:
        dist.destroy_process_group()


def test_two_rank_partition_and_uid_exchange():
    world = 2
    ntiles_list = [0, 1, 2, 3, 55, 313, 1172]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, ntiles_list, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, ok_uid, gathered, mx in res:
        assert ok_uid and mx == float(world)
        for n in ntiles_list:
            all_tiles = sorted(t for g in range(world) for t in gathered[g][n])
            assert all_tiles == list(range(n))                     # disjoint and complete
            sizes = [len(gathered[g][n]) for g in range(world)]
            assert max(sizes) - min(sizes) <= 1                    # balanced


@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_tile_shard_mirror(world):
    for n in (0, 1, 7, 55, 1172):
        tiles = sorted(t for g in range(world) for t in tile_shard(n, g, world))
        assert tiles == list(range(n))


def _gather_worker(rank, world, port, mN, ld, q):
    """C7 (dist.cu: dist_gather_dnew) over gloo: each rank updates only the rows of its cyclic target
    tiles (slots of the lead order), packs them into the slot-ordered buffer, runs one in-place
    all-gather per round of G tiles, and unpacks the other ranks' rows into D's row order."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = torch.Generator().manual_seed(7)
        order = torch.randperm(mN, generator=g)                    # slot -> D row (targets by lead)
        D0 = torch.randint(0, 65521, (mN, ld), generator=g, dtype=torch.int32)   # spliced D
        Dnew = torch.randint(0, 65521, (mN, ld), generator=g, dtype=torch.int32)  # what the sweep writes
        D = D0.clone()
        ntile = (mN + 127) // 128
        for slot in range(mN):                                     # this rank's sparse phase
            if (slot // 128) % world == rank:
                D[order[slot]] = Dnew[order[slot]]
        rounds = (ntile + world - 1) // world
        Dp = torch.zeros(rounds * world * 128, ld, dtype=torch.int32)
        own = ((ntile - rank + world - 1) // world) * 128          # k_pack_own's grid
        for l in range(own):
            slot = (rank + world * (l // 128)) * 128 + l % 128
            if slot < mN:
                Dp[slot] = D[order[slot]]
        for k in range(rounds):                                    # grouped in-place all-gathers
            rnd = Dp[k * world * 128:(k + 1) * world * 128]
            parts = list(rnd.split(128))
            dist.all_gather(parts, parts[rank].clone())
            for i, p in enumerate(parts):
                rnd[i * 128:(i + 1) * 128] = p
        for slot in range(mN):                                     # k_unpack_others
            if (slot // 128) % world != rank:
                D[order[slot]] = Dp[slot]
        q.put((rank, bool(torch.equal(D, Dnew))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mN", [(2, 300), (3, 1000), (2, 128), (3, 100)])
def test_dnew_gather_protocol(world, mN):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, mN, 16, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok in res), res
