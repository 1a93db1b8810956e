"""Times dflop_balance_microbatches on one preset (no oracle): the command ncu profiles.

    python tools/prof_balance.py --config 5 --K 8192 [--reps 2]
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
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--K", type=int, default=8192)
ap.add_argument("--R", type=int, default=-1)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--mode", type=int, default=0, help="16 = DFLOP_MODE_ORDER4")
ap.add_argument("--plan", default="", help='JSON plan (e.g. a config-4 Stage-B plan), else the preset\'s')
a = ap.parse_args()
p = synth.presets()[a.config]
plan = json.loads(a.plan) if a.plan else p.plan
R = p.R if a.R < 0 else a.R
t, f, x = (torch.from_numpy(v.astype(np.uint32).view(np.int32)).cuda() for v in p.features(0))
_, ticks = D.predict_costs(p.model, plan, t, f, x, want_f32=False)
for rep in range(a.reps):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = D.balance_microbatches(ticks, plan, a.K, R, p.G, p.seed(0), mode=a.mode)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    best = D.cand_result(r["best"])
    print(f"rep {rep}: K={a.K} R={R} {ms:.2f} ms  {a.K / ms * 1e3:.0f} cand/s  best c={best['cand']} T={best['makespan']}",
          flush=True)
    if "timing" in D.LIB_PATH:  # diagnostic build: per-phase cycles of the candidate kernel
        import ctypes
        out = (ctypes.c_ulonglong * 8)()
        D.lib().dflop_debug_phase_cycles(out, 1)
        tot = sum(out) or 1
        names = ["lpt", "ref_jstar", "ref_lists", "ref_pairs", "ref_apply", "score", "other", "-"]
        print("   phases: " + "  ".join(f"{nm}={v / tot * 100:.1f}%" for nm, v in zip(names, out) if v), flush=True)
