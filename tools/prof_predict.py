"""a1 (k_predict) at large n: the HBM-bound regime of SURVEY 8(d).  Algorithmic bytes per
sample and plan: 12 in (three u32 features) + 32 out (f32 and u32 [4] rows) = 44 B.

    python tools/prof_predict.py [--log2n 26] [--reps 10] [--no-f32]
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
ap.add_argument("--log2n", type=int, default=26)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--no-f32", action="store_true")
ap.add_argument("--correction", action="store_true", help="active N1 correction table (random ratios)")
a = ap.parse_args()
p = synth.presets()[a.config]
model = dict(p.model)
if a.correction:
    rho = np.clip(np.random.default_rng(0).lognormal(0.0, 0.4, (3, 32)), 0.3, 3.0).astype(np.float32)
    model["correction"] = {"active": True, "rho": rho}
n = 1 << a.log2n
base = [torch.from_numpy(v.astype(np.uint32).view(np.int32)).cuda() for v in p.features(0)]
reps = (n + base[0].numel() - 1) // base[0].numel()
t, f, x = (b.repeat(reps)[:n].contiguous() for b in base)  # the batch's feature mix, tiled
want = not a.no_f32
D.predict_costs(model, p.plan, t, f, x, want_f32=want)
torch.cuda.synchronize()
ms = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    D.predict_costs(model, p.plan, t, f, x, want_f32=want)
    e1.record()
    e1.synchronize()
    ms.append(e0.elapsed_time(e1))
best = min(ms)
byt = n * (12 + (32 if want else 16))
peak = None
try:
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                       "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass
gbs = byt / best / 1e6
print(json.dumps({"kernel": "k_predict", "correction": a.correction, "n": n, "ms_best": round(best, 4), "ms_median": round(sorted(ms)[len(ms) // 2], 4),
                  "bytes": byt, "GB_s": round(gbs, 1), "peak_GB_s": peak,
                  "frac": round(gbs / peak, 3) if peak else None, "samples_per_s": n / best * 1e3}))
