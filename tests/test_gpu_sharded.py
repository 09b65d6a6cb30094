"""User-sharded serving on the GPU: real decode outputs routed
by user, decoded per rank, gathered to rank 0 -- compared with one process
decoding every user; and bench.py's multi-rank arm (routing, point-to-point
result gather, stat all-reduce).  The box has one GPU, so the ranks share
cuda:0 and talk over gloo (NCCL needs one GPU per rank); the code paths are
the ones the NCCL run takes."""

import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
N_USERS = 29
WIDTHS = (8, 16, 24)


def _need_gpu():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _features(i):
    return np.random.default_rng(1000 + i).normal(size=(40 + 7 * (i % 5), 16))


def _decode(users_idx):
    """One BeamDecoder over the given users (C1 model): device result tensors."""
    from paper_2602_22732_b200.decode import BeamDecoder
    from paper_2602_22732_b200.model import DecoderConfig, DecoderModel
    model = DecoderModel(DecoderConfig(16, 16, 32, 2, 1, (256, 256, 256), 4, seed=2))
    feats = [_features(i) for i in users_idx]
    dec = BeamDecoder(model, [f.shape[0] for f in feats], [WIDTHS] * len(feats),
                      device=torch.device("cuda", 0))
    f = torch.from_numpy(np.concatenate(feats, 0).astype(np.float32)).cuda() if feats else None
    if feats:
        dec.run(features=f)
    torch.cuda.synchronize()
    return dec


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2602_22732_b200 import sharding as sh
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    users = [f"user{i:06d}" for i in range(N_USERS)]
    mine = sh.partition(users, world)[rank]
    dec = _decode(mine)
    got = sh.gather_decoded(dec.count, dec.tokens, dec.score, len(mine))
    stats = sh.all_reduce_stats({"requests": len(mine),
                                 "results": int(dec.count[:len(mine)].sum().item())})
    if rank == 0:
        per_rank = [sh.decoded_to_lists(c, t, s, 3) for c, t, s in got]
        q.put((sh.merge_in_order(users, per_rank, world), stats))
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_decode_matches_one_process():
    _need_gpu()
    import torch.multiprocessing as mp
    from paper_2602_22732_b200 import sharding as sh
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    merged, stats = q.get()
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    dec = _decode(list(range(N_USERS)))
    want = sh.decoded_to_lists(dec.count[:N_USERS], dec.tokens, dec.score, 3)
    # the fused per-request kernel: every request's decode is independent of
    # the batch it rides in, so the sharded results are bit-identical
    assert merged == want
    assert stats["requests"] == N_USERS
    assert stats["results"] == sum(len(r) for r in want)


def test_bench_two_ranks():
    """bench.py under torchrun with 2 ranks: user routing, ragged per-rank
    batches, point-to-point result gather to rank 0, stat all-reduce."""
    _need_gpu()
    env = dict(os.environ, GR4AD_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--config", "c1", "--steps", "3", "--warmup", "3",
           "--no-cpu-baseline"]
    out = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1, out.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    sh = d["sharding"]
    assert sum(sh["per_rank"]) == sh["users"] == 2 * 64
    assert sh["gathered_results"] == d["results_per_step"] == 2 * 64 * 32
