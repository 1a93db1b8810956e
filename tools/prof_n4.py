"""N4 timings on a preset's search winner: (a) microbatch-order search, (b) routing plan.

    python tools/prof_n4.py --config 5 --rounds 64 --e-dp 4
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2603_25120_b200 import dflop as D
from paper_2603_25120_b200 import synth

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--K", type=int, default=65536)
ap.add_argument("--rounds", type=int, default=64)
ap.add_argument("--e-dp", type=int, default=4)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
p = synth.presets()[a.config]
t, f, x = (torch.from_numpy(v.astype(np.uint32).view(np.int32)).cuda() for v in p.features(0))
res = D.search_plans(p.model, t, f, x, K=a.K, R=p.R, G=p.G, seed=p.seed(0), plan=p.plan)
_, ticks = D.predict_costs(p.model, p.plan, t, f, x, want_f32=False)


def timed(fn):
    out, best = None, 1e30
    for _ in range(a.reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        out = fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return out, best


o, ms_o = timed(lambda: D.order_search(ticks, p.plan, res["assign"], rounds=a.rounds))
rp = dict(p.plan, e_dp=a.e_dp)
r, ms_r = timed(lambda: D.route_plan(ticks, rp, res["assign"]))
load = r["enc_load"].cpu().numpy().view(np.uint64).astype(np.float64)
print(json.dumps({"config": a.config, "K": a.K, "winner_T": res["makespan"], "ordered_T": o["makespan"],
                  "gain": 1 - o["makespan"] / res["makespan"], "order_ms": round(ms_o, 3), "rounds": a.rounds,
                  "route_ms": round(ms_r, 3), "e_dp": a.e_dp,
                  "encoder_range_imbalance": float((load.max(1) / np.maximum(load.mean(1), 1)).max())}))
