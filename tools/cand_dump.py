"""Dumps the per-candidate makespans of one preset (for A/B comparisons of two library
builds, selected with DFLOP_LIB):  python tools/cand_dump.py --config 5 --K 1000000 --out x.npy"""
import argparse
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
ap.add_argument("--out", required=True)
a = ap.parse_args()
p = synth.presets()[a.config]
t, f, x = (torch.from_numpy(v.astype(np.uint32).view(np.int32)).cuda() for v in p.features(0))
_, ticks = D.predict_costs(p.model, p.plan, t, f, x, want_f32=False)
r = D.balance_microbatches(ticks, p.plan, a.K, p.R, p.G, p.seed(0), per_candidate=True)
np.save(a.out, np.stack([r["cand_T"].cpu().numpy(), r["cand_cmax"].cpu().numpy()]))
print(a.out, D.cand_result(r["best"]))
