"""Multi-process (gloo, world_size 2, CPU) coverage of the user-sharded
serving plumbing: stable routing, result gather to rank 0, stat all-reduce,
and order-preserving reassembly."""

import os
import socket
import zlib

import numpy as np
import torch.multiprocessing as mp

from paper_2602_22732_b200 import sharding as sh


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _fake_results(uid, T=3, width=5):
    rng = np.random.default_rng(zlib.crc32(uid.encode()))
    n = int(rng.integers(0, width + 1))
    return [(tuple(int(x) for x in rng.integers(0, 16, size=T)), float(-rng.random() * 10))
            for _ in range(n)]


def _worker(rank, world, port, uids, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    parts = sh.partition(uids, world)
    local = [_fake_results(uids[i]) for i in parts[rank]]
    n_max = max(len(p) for p in parts)
    gathered = sh.gather_results(local, 3, 5, n_max)
    stats = sh.all_reduce_stats({"requests": len(parts[rank]),
                                 "results": sum(len(r) for r in local)})
    if rank == 0:
        q.put((sh.merge_in_order(uids, gathered, world), stats))
    dist.barrier()
    dist.destroy_process_group()


def test_shard_routing_is_stable_and_balanced():
    uids = [f"user{i:06d}" for i in range(4000)]
    for world in (1, 2, 4, 8):
        parts = sh.partition(uids, world)
        assert sorted(i for p in parts for i in p) == list(range(4000))
        sizes = [len(p) for p in parts]
        assert max(sizes) - min(sizes) < 0.1 * 4000 / world + 20
    assert sh.shard_of("user000042", 8) == sh.shard_of("user000042", 8)
    assert [sh.shard_of(u, 2) for u in uids[:8]] == [sh.shard_of(u, 2) for u in uids[:8]]


def test_pack_roundtrip():
    res = [_fake_results(f"u{i}") for i in range(7)]
    assert sh.unpack_results(*sh.pack_results(res, 3, 5)) == res


def test_gather_and_stats_world2_gloo():
    uids = [f"user{i:06d}" for i in range(37)]
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, uids, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, stats = q.get()
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert merged == [_fake_results(u) for u in uids]
    assert stats["requests"] == 37
    assert stats["results"] == sum(len(_fake_results(u)) for u in uids)
