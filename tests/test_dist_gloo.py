"""World-size-2 CPU test (gloo) of the multi-GPU protocol that dflop_search_plans /
dflop_search_plans_batches run around their NCCL collectives (P:796
the communicator, P:738 the argmin over candidates, Eq. (1) over batches).  The
protocol steps are the PRODUCT's host code, called through the C ABI of libdflop.so on CPU
(csrc/protocol.cpp: dflop_shard_range, dflop_pack_key, dflop_select_plan, dflop_owner_of --
the same functions api.cpp calls); only the per-rank candidate evaluation is the CPU oracle
(the GPU kernels need a GPU) and the collectives are gloo instead of NCCL.  -m "not gpu".
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


def _plans(p):
    """two Stage-B plans over the preset's pipeline (different N_mb), p = 'Stage-A rank'"""
    a = dict(p.plan)
    b = dict(p.plan, n_mb=max(1, p.plan["n_mb"] // 2))
    return [a, b]


def _worker(rank, world, port, k, K, D, out_q):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    from oracle import oracle as O
    from paper_2603_25120_b200 import dflop, synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    p = synth.presets()[k]
    plans = _plans(p)
    b0, e0 = dflop.shard_range(K, rank, world)                      # product: rank's candidate range
    keys = np.full(len(plans) * D, np.iinfo(np.uint64).max, np.uint64)
    local = {}
    for pi, pl in enumerate(plans):
        for b in range(D):
            _, q, _, _ = O.predict(p.model, pl, *p.features(b))
            seed = (p.seed(0)[0], p.seed(0)[1] + b)                  # batch b's family (R33)
            if e0 > b0:
                r = O.balance(q, pl, K, p.R, p.G, seed, b0, e0, per_candidate=False)
                keys[pi * D + b] = dflop.pack_key(r["T"], pi * K + r["c"])   # product: packed key
                local[(pi, b)] = r
    t = torch.from_numpy(keys.view(np.int64).copy())
    dist.all_reduce(t, op=dist.ReduceOp.MIN)                          # NCCL min all-reduce -> gloo
    red = t.numpy().view(np.uint64)
    win_p, obj = dflop.select_plan(red, len(plans), D)                # product: Eq. (1) plan choice
    out = []
    for b in range(D):
        key = int(red[win_p * D + b])
        c = (key & 0xFFFFFF) - win_p * K
        owner = dflop.owner_of(K, c, world)                           # product: who broadcasts
        n = p.n
        if rank == owner:
            r = local[(win_p, b)]
            assert r["c"] == c
            assign = torch.from_numpy(r["assign"].astype(np.int64))
        else:
            assign = torch.zeros(n, dtype=torch.int64)
        dist.broadcast(assign, src=owner)
        out.append((key >> 24, c, owner, assign.numpy().tolist()))
    out_q.put((rank, win_p, [int(v) for v in obj], out))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("k,K,D", [(1, 96, 1), (2, 40, 2), (1, 3, 2)])
def test_two_rank_protocol_matches_single_process(O, presets, k, K, D):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, k, K, D, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    results = [q.get(timeout=300) for _ in range(2)]
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    # single process, oracle only: per (plan, batch) the whole family, then Eq. (1)'s
    # lexicographic minimum of (sum_b T_B, plan) and each batch's winner
    p = presets[k]
    plans = _plans(p)
    whole = {}
    for pi, pl in enumerate(plans):
        for b in range(D):
            _, qq, _, _ = O.predict(p.model, pl, *p.features(b))
            whole[(pi, b)] = O.balance(qq, pl, K, p.R, p.G, (p.seed(0)[0], p.seed(0)[1] + b), per_candidate=False)
    objs = [sum(whole[(pi, b)]["T"] for b in range(D)) for pi in range(len(plans))]
    wp = min(range(len(plans)), key=lambda pi: (objs[pi], pi))
    for rank, win_p, obj, out in results:
        assert win_p == wp and obj == objs
        for b, (T, c, owner, assign) in enumerate(out):
            w = whole[(wp, b)]
            assert (T, c) == (w["T"], w["c"])
            assert assign == w["assign"].tolist()


def test_shard_arithmetic_through_libdflop():
    from paper_2603_25120_b200 import dflop
    for K in (1, 7, 1000, 1_000_000, 1 << 24):
        for G in (1, 2, 3, 8):
            ranges = [dflop.shard_range(K, g, G) for g in range(G)]
            assert ranges[0][0] == 0 and ranges[-1][1] == K
            assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
            for c in (0, K // 2, K - 1):
                b, e = ranges[dflop.owner_of(K, c, G)]
                assert b <= c < e
            assert dflop.owner_of(K, K, G) == 0xFFFFFFFF
    key = dflop.pack_key(123456789, 4242)
    assert (key >> 24, key & 0xFFFFFF) == (123456789, 4242)
    assert dflop.pack_key(1 << 41, 5) >> 24 == (1 << 40) - 1          # saturated T (overflow bit set by kernels)
    # lexicographic (T, id) order == integer key order
    assert dflop.pack_key(7, 3) < dflop.pack_key(7, 4) < dflop.pack_key(8, 0)
    with pytest.raises(dflop.DflopError):
        dflop.shard_range(10, 2, 2)


def test_select_plan_rules():
    from paper_2603_25120_b200 import dflop
    M = np.iinfo(np.uint64).max
    k = lambda T, i: dflop.pack_key(T, i)
    # P = 3 plans x D = 2 batches: objective = sum of T over batches; ties -> lower p
    keys = [k(5, 0), k(7, 1), k(6, 2), k(6, 3), k(9, 4), k(2, 5)]
    win, obj = dflop.select_plan(keys, 3, 2)
    assert list(obj) == [12, 12, 11] and win == 2
    keys[5] = M                                                       # plan 2 misses a batch
    win, obj = dflop.select_plan(keys, 3, 2)
    assert win == 0 and obj[2] == M
    win, obj = dflop.select_plan(keys, 3, 2, batch_n=[4, 0])          # an empty batch contributes 0
    assert list(obj) == [5, 6, 9] and win == 0
    with pytest.raises(dflop.DflopError):
        dflop.select_plan([M, M], 2, 1)
