"""World-size-2 CPU test (gloo) of the multi-GPU protocol that dflop_search_plans runs over
NCCL: shard the candidate family, pack (T, id) into one u64, MIN all-reduce, and let the
owner broadcast the winner's assignment.  The per-rank compute is the CPU oracle.
-m "not gpu".
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, k, K, out_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle import oracle as O
    from paper_2603_25120_b200 import sharding, synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = synth.presets()[k]
    _, q, _, _ = O.predict(p.model, p.plan, *p.features(0))
    b, e = sharding.shard_range(K, rank, world)
    r = O.balance(q, p.plan, K, p.R, p.G, p.seed(0), b, e, per_candidate=False)
    key = torch.tensor([sharding.pack_key(r["T"], r["c"])], dtype=torch.int64)
    dist.all_reduce(key, op=dist.ReduceOp.MIN)
    T, c = sharding.unpack_key(int(key.item()))
    owner = sharding.owner_of(K, c, world)
    assign = torch.from_numpy(r["assign"].astype(np.int64)) if rank == owner else torch.zeros(p.n, dtype=torch.int64)
    dist.broadcast(assign, src=owner)
    out_q.put((rank, T, c, owner, assign.numpy().tolist()))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("k,K", [(1, 96), (2, 40)])
def test_two_rank_protocol_matches_single_process(O, presets, k, K):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, k, K, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=300) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = presets[k]
    _, qq, _, _ = O.predict(p.model, p.plan, *p.features(0))
    whole = O.balance(qq, p.plan, K, p.R, p.G, p.seed(0), per_candidate=False)
    for rank, T, c, owner, assign in results:
        assert (T, c) == (whole["T"], whole["c"])
        assert assign == whole["assign"].tolist()


def test_shard_arithmetic():
    from paper_2603_25120_b200 import sharding
    for K in (1, 7, 1000, 1_000_000):
        for G in (1, 2, 3, 8):
            ranges = [sharding.shard_range(K, g, G) for g in range(G)]
            assert ranges[0][0] == 0 and ranges[-1][1] == K
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            for c in (0, K // 2, K - 1):
                b, e = ranges[sharding.owner_of(K, c, G)]
                assert b <= c < e
    assert sharding.unpack_key(sharding.pack_key(123456789, 4242)) == (123456789, 4242)
