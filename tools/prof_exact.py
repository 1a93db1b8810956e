"""N3 exact C_max: node throughput and certificates on a preset batch.

    python tools/prof_exact.py --config 1 --budgets 1e8 1e9 1e10 [--batch 0]
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
ap.add_argument("--config", type=int, default=1)
ap.add_argument("--batch", type=int, default=0)
ap.add_argument("--budgets", type=float, nargs="+", default=[1e8, 1e9])
a = ap.parse_args()
p = synth.presets()[a.config]
t, f, x = (torch.from_numpy(v.astype(np.uint32).view(np.int32)).cuda() for v in p.features(a.batch))
_, ticks = D.predict_costs(p.model, p.plan, t, f, x, want_f32=False)
D.exact_cmax(ticks, p.plan, node_budget=1000)  # warm-up
for b in a.budgets:
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = D.exact_cmax(ticks, p.plan, node_budget=int(b))
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1)
    print(json.dumps({"config": a.config, "batch": a.batch, "budget": int(b), "ms": round(ms, 2),
                      "nodes": r["nodes"], "nodes_per_s": r["nodes"] / ms * 1e3, "proven": r["proven"],
                      "cmax": r["cmax"], "lb": r["lower_bound"], "gap": r["cmax"] / max(1, r["lower_bound"]) - 1,
                      "makespan": r["makespan"]}), flush=True)
