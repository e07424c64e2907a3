"""Multi-rank path on CPU: world-size 2, 4 and 8 gloo process groups.  Each rank computes its
shard's integer partials with the oracle (no GPU here), packs them into the product's single
int64 buffer and all-reduces; the result must equal the single-process oracle bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2508_09229_b200.shard import Packed, shard_range

L, E, K, N, C, SEED = 5, 32, 4, 3001, 7, 13


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import evaluate as oe
        from oracle import gen as og
        from oracle import stats as ost
        a, b = shard_range(N, rank, world)
        sel, bounds = og.generate(L, E, K, 1.2, N, C, SEED, tok_range=(a, b))
        rng = np.random.default_rng(0)
        p = rng.integers(0, 9, (L, 8))
        assigns = [rng.integers(0, 8, (L, E)) for _ in range(4)]
        pk = Packed(L, E, 4, C)
        pk.counts.copy_(torch.as_tensor(ost.counts(sel, E)))
        for i, asg in enumerate(assigns):
            pk.sums[i].copy_(torch.as_tensor(oe.chunk_sums(sel, oe.pe_table(p, asg), bounds, a)))
        pk.allreduce()
        q.put((rank, pk.counts.numpy().copy(), pk.sums.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4, 8])
def test_gloo_sharded_partials_equal_single(world):
    from oracle import evaluate as oe
    from oracle import gen as og
    from oracle import stats as ost
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    sel, bounds = og.generate(L, E, K, 1.2, N, C, SEED)
    rng = np.random.default_rng(0)
    p = rng.integers(0, 9, (L, 8))
    assigns = [rng.integers(0, 8, (L, E)) for _ in range(4)]
    want_c = ost.counts(sel, E)
    want_s = np.stack([oe.chunk_sums(sel, oe.pe_table(p, a), bounds) for a in assigns])
    for rank, c, s in res:
        assert np.array_equal(c, want_c), rank
        assert np.array_equal(s, want_s), rank


def test_shard_ranges_partition():
    for n in (0, 1, 7, 1000, 10_000_001):
        for g in (1, 2, 3, 4, 8):
            rs = [shard_range(n, r, g) for r in range(g)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(g - 1))
