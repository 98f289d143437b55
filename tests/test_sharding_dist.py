"""Multi-process (gloo, world_size 2, CPU) checks of the batch x head sharding path:
shard ranges, counter-based input generation per shard, the MAX-over-ranks timing
reduction and the check-only gather."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import mbci_inputs as gen
from paper_2506_22169_b200 import sharding


def test_shard_range_partitions():
    for batch in (0, 1, 7, 96, 512):
        for world in (1, 2, 3, 4, 8):
            spans = [sharding.shard_range(batch, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == batch
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        sharding.shard_range(8, 2, 2)


def test_shard_inputs_bit_identical_to_full():
    full = gen.make_chain_inputs(7, "bf16", 6, 40, 56, 64, 32, 1, valid_len_range=(10, 56))
    for r in range(3):
        lo, hi = sharding.shard_range(6, r, 3)
        part = gen.make_chain_inputs(7, "bf16", hi - lo, 40, 56, 64, 32, 1, batch_start=lo,
                                     valid_len_range=(10, 56))
        assert np.array_equal(part.A, full.A[lo:hi])
        assert np.array_equal(part.B, full.B[lo:hi])
        assert np.array_equal(part.D, full.D[lo:hi])
        assert np.array_equal(part.valid_len, full.valid_len[lo:hi])


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
        lo, hi = sharding.shard_range(5, rank, world)
        t = sharding.max_over_ranks(1.5 + rank)
        tot = sharding.sum_over_ranks(hi - lo)
        local = torch.arange(lo * 3, lo * 3 + 6, dtype=torch.float32).reshape(2, 3) if hi - lo == 2 else \
            torch.full((2, 3), -1.0)
        g = sharding.gather_rows(local)
        q.put((rank, t, tot, g.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, t, tot, g in res:
        assert t == 2.5            # max over ranks
        assert tot == 5            # every β owned once
        assert len(g) == 4


def test_key_range_and_split_grid():
    for N in (0, 1, 8, 21, 512, 1000, 4096):
        for parts in (1, 2, 3, 4, 8):
            spans = [sharding.key_range(N, p, parts) for p in range(parts)]
            assert spans[0][0] == 0 and spans[-1][1] == N
            for (a, b), (c, d) in zip(spans, spans[1:]):
                assert b == c and (b % 8 == 0 or b == N)
    assert [sharding.split_grid(r, 8, 2) for r in range(8)] == [(r // 2, r % 2) for r in range(8)]
    assert sharding.key_groups(8, 4) == [[0, 1, 2, 3], [4, 5, 6, 7]]
    with pytest.raises(ValueError):
        sharding.split_grid(0, 6, 4)


def _split_worker(rank, world, port, q):
    """World-2 split-N over gloo: each rank computes its key range's partial (E_r, lse_r) with the
    oracle (CPU stand-in for mbci_chain_run_partial), the group all-gathers them
    (sharding.gather_partials, the exchange step) and combines them."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    import oracle
    from split_util import local_valid, lse_combine, slice_keys
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        inp = gen.make_chain_inputs(5, "bf16", 3, 12, 40, 16, 8, 1, valid_len_range=(0, 40))
        g, part = sharding.split_grid(rank, world, world)
        n0, n1 = sharding.key_range(inp.N, part, world)
        sub = slice_keys(inp, n0, n1)
        v = local_valid(inp.valid_len, n0, n1)
        E_r = torch.from_numpy(oracle.chain(sub, "softmax", 0.3, v))
        lse_r = torch.from_numpy(oracle.row_lse(sub, 0.3, v))
        E_all, lse_all = sharding.gather_partials(E_r, lse_r)
        merged = lse_combine(E_all.numpy(), lse_all.numpy())
        full = oracle.chain(inp, "softmax", 0.3, inp.valid_len)
        q.put((rank, (n0, n1), float(np.max(np.abs(merged - full)))))
    finally:
        dist.destroy_process_group()


def test_gloo_split_n_two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_split_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=180) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert [r[1] for r in res] == [(0, 24), (24, 40)]
    for _, _, err in res:
        assert err < 1e-12
