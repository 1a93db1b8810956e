"""Multi-GPU check of dflop_search_plans (run under torchrun, one rank per GPU).

Every rank evaluates its shard of the candidate family; one NCCL min all-reduce picks the
winner and its owner broadcasts the assignment.  Rank 0 also runs the whole family on its
own GPU (comm = NULL) and the two results must be identical (the winner does not depend
on the number of GPUs).

    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 tools/dist_check.py --config 3 --K 8192
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch
import torch.distributed as dist

from paper_2603_25120_b200 import dflop as D
from paper_2603_25120_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--K", type=int, default=8192)
ap.add_argument("--batches", type=int, default=0, help="N2: Eq. (1) over this many batches (0 = one batch)")
a = ap.parse_args()
rank, world, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
torch.cuda.set_device(local)
dist.init_process_group("nccl", device_id=torch.device("cuda", local))
p = synth.presets()[a.config]
comm = D.Comm(rank, world, local)
search_kw = dict(plan=p.plan) if p.plan is not None else dict(cluster=p.cluster, mem=p.mem(), gbs=p.gbs, top_p=16)
if a.batches:
    feats = [p.features(b) for b in range(a.batches)]
    offs = np.concatenate([[0], np.cumsum([len(fb[0]) for fb in feats])])
    t, f, x = (torch.from_numpy(np.concatenate([fb[i] for fb in feats]).astype(np.uint32).view(np.int32)).cuda()
               for i in range(3))
    run = lambda cm: D.search_plans_batches(p.model, t, f, x, offs, K=a.K, R=p.R, G=p.G, seed=p.seed(0),
                                            comm=cm, **search_kw)
else:
    t, f, x = (torch.from_numpy(v.astype(np.uint32).view(np.int32)).cuda() for v in p.features(0))
    run = lambda cm: D.search_plans(p.model, t, f, x, K=a.K, R=p.R, G=p.G, seed=p.seed(0), comm=cm, **search_kw)
res = run(comm)
assign = res["assign"].cpu().numpy()
ok = True
if rank == 0:
    ref = run(None)
    ok = (res["makespan"], res["cand"], res["cmax"]) == (ref["makespan"], ref["cand"], ref["cmax"])
    ok = ok and bool((assign == ref["assign"].cpu().numpy()).all())
    ok = ok and res["owner_rank"] == D.owner_of(a.K, res["cand"], world)
    ok = ok and res["plan"] == ref["plan"] and res["stage_a_rank"] == ref["stage_a_rank"]
    if a.batches:
        ok = ok and [b["makespan"] for b in res["batches"]] == [b["makespan"] for b in ref["batches"]]
# every rank must hold the same winner and assignment
h = torch.tensor([res["makespan"], res["cand"], int(assign.astype(np.int64).sum())], dtype=torch.int64).cuda()
hmax, hmin = h.clone(), h.clone()
dist.all_reduce(hmax, op=dist.ReduceOp.MAX)
dist.all_reduce(hmin, op=dist.ReduceOp.MIN)
ok = ok and bool((hmax == hmin).all().item())
flag = torch.tensor([1 if ok else 0], dtype=torch.int32).cuda()
dist.all_reduce(flag, op=dist.ReduceOp.MIN)
if rank == 0:
    print(json.dumps({"world": world, "config": a.config, "K": a.K, "batches": a.batches, "T": res["makespan"],
                      "cand": res["cand"],
                      "owner": res["owner_rank"], "ok": bool(flag.item())}), flush=True)
comm.close()
dist.destroy_process_group()
sys.exit(0 if flag.item() else 1)
