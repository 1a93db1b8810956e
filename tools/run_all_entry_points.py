"""Small end-to-end run of every entry point of libdflop.so (a crash/regression check; the
GPU pool does not allow compute-sanitizer):

    python tools/run_all_entry_points.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np
import torch

from paper_2603_25120_b200 import dflop as D
from paper_2603_25120_b200 import synth


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a).astype(np.uint32).view(np.int32)).cuda()


P = synth.presets()
for k in (1, 2, 3, 5):
    p = P[k]
    t, f, x = (dev(a) for a in p.features(0))
    _, ticks = D.predict_costs(p.model, p.plan, t, f, x)
    r = D.balance_microbatches(ticks, p.plan, 512, p.R, p.G, p.seed(0), want_groups=True, per_candidate=True)
    r4 = D.balance_microbatches(ticks, p.plan, 256, p.R, p.G, p.seed(0), mode=D.MODE_ORDER4)
    res = D.search_plans(p.model, t, f, x, K=512, R=p.R, G=p.G, seed=p.seed(0), plan=p.plan)
    D.order_search(ticks, p.plan, res["assign"], rounds=4)
    D.route_plan(ticks, dict(p.plan, e_dp=3), res["assign"])
    if p.n <= 256:
        D.exact_cmax(ticks, p.plan, node_budget=10 ** 6, init_assign=res["assign"])
p = P[4]
t, f, x = (dev(a) for a in p.features(0))
D.search_plans(p.model, t, f, x, K=64, R=p.R, G=p.G, seed=p.seed(0), cluster=p.cluster, mem=p.mem(), gbs=p.gbs,
               top_p=4)
p = P[2]
feats = [p.features(b) for b in range(3)]
offs = np.concatenate([[0], np.cumsum([len(fb[0]) for fb in feats])])
cat = [dev(np.concatenate([fb[i] for fb in feats])) for i in range(3)]
rho = np.ones((3, 32), np.float32)
rho[1, 8] = 0.5
D.search_plans_batches(dict(p.model, correction={"active": True, "rho": rho}), *cat, offs, K=256, R=p.R, G=p.G,
                       seed=p.seed(0), plan=p.plan)
fwd, bwd = synth.random_durations(8, 4, 6, seed=1, hi=100)
D.simulate_1f1b(torch.from_numpy(fwd.view(np.int64)).cuda(), torch.from_numpy(bwd.view(np.int64)).cuda())
torch.cuda.synchronize()
print("all entry points ok")
