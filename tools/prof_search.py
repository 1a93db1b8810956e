"""Times dflop_search_plans in Algorithm-1 mode (config 4: 64-GPU plan space, GBS 2048,
top-P plans balanced with K candidates each) -- the a6 row of SURVEY 8(a).

    python tools/prof_search.py [--P 64] [--K 4096] [--reps 3]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2603_25120_b200 import dflop as D
from paper_2603_25120_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--P", type=int, default=64)
ap.add_argument("--K", type=int, default=4096)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--batches", type=int, default=0, help="N2: Eq. (1) over this many batches")
a = ap.parse_args()
p = synth.presets()[4]
if a.batches:
    feats = [p.features(b) for b in range(a.batches)]
    offs = np.concatenate([[0], np.cumsum([len(fb[0]) for fb in feats])])
    t, f, x = (torch.from_numpy(np.concatenate([fb[i] for fb in feats]).astype(np.uint32).view(np.int32)).cuda()
               for i in range(3))
else:
    t, f, x = (torch.from_numpy(v.astype(np.uint32).view(np.int32)).cuda() for v in p.features(0))
D.profile_read(reset=True)
for rep in range(a.reps):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if a.batches:
        r = D.search_plans_batches(p.model, t, f, x, offs, K=a.K, R=p.R, G=p.G, seed=p.seed(0), cluster=p.cluster,
                                   mem=p.mem(), gbs=p.gbs, top_p=a.P)
        r["stage_a_makespan"] = r["stage_a_makespan"]
    else:
        r = D.search_plans(p.model, t, f, x, K=a.K, R=p.R, G=p.G, seed=p.seed(0), cluster=p.cluster, mem=p.mem(),
                           gbs=p.gbs, top_p=a.P)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) * 1e3
    print(json.dumps({"rep": rep, "ms": round(dt, 2), "P": a.P, "K": a.K, "batches": a.batches, "plan": r["plan"],
                      "T_B": r["makespan"],
                      "T_A": r["stage_a_makespan"], "alg1_plan": r["alg1_plan"], "alg1_T_A": r["alg1_makespan"],
                      "stage_a_rank": r["stage_a_rank"], "cand": r["cand"], "n_feasible": r["n_feasible"],
                      "n_pairs": r["n_pairs"], "n_candidates": r["n_candidates"]}), flush=True)
