"""Seeded synthetic inputs for the DFLOP plan-candidate path (arXiv 2603.25120).

This module holds INPUTS only -- none of the method's arithmetic.  It is the one
module that both the CUDA path's tests/bench and the CPU oracle consume, so that
both sides see byte-identical inputs ("input recipe").

What it generates, per preset (BASELINE.json configs):

* per-sample features: image tiles, video frames, text tokens (u32 SoA), drawn
  with numpy ``PCG64(1000*k + b)`` from mixtures shaped like the paper's mixed
  dataset (tab:dataset_composition): single image / multi-image /
  video / text-only, with heavy-tailed tile, frame and text-length laws;
* model shapes (public model-card values: layers, hidden size, tokens per
  encoder instance, LLM tokens per tile/frame) for the MLLMs of
  tab:mllm_configs;
* a synthetic Model-Profiler output standing in for the measured grids of
  P:440-446: throughput sampled at powers-of-two knots from a saturating law
  (shape of fig:input_shape) and linear memory grids at two layer
  counts;
* the plan theta, candidate-family sizes K/R/G and Philox seeds.

The throughput law is only used to *fill the knots*; what the method does with
the grid (interpolation, FLOP accounting, durations) lives in the kernels and,
independently, in ``oracle/``.
"""
from __future__ import annotations

import dataclasses
import math
from typing import Dict, List, Optional

import numpy as np

GIB = float(1 << 30)


# --------------------------------------------------------------------------
# Model shapes (public model cards).  tau_* = LLM tokens per tile / frame after
# the connector; e_seq = tokens per encoder instance ("E_seq_len remains fixed").
# --------------------------------------------------------------------------
ENCODERS = {
    "siglip-so400m": dict(e_layers=27, e_hidden=1152, e_seq=729, tau_tile=729, tau_frame=196),
    "clip-vit-l14-336": dict(e_layers=24, e_hidden=1024, e_seq=577, tau_tile=576, tau_frame=144),
    "internvit-6b": dict(e_layers=45, e_hidden=3200, e_seq=1025, tau_tile=256, tau_frame=256),
    "qwen2-vl-vit": dict(e_layers=32, e_hidden=1280, e_seq=1024, tau_tile=256, tau_frame=128),
}
LLMS = {
    "qwen2.5-7b": dict(l_layers=28, l_hidden=3584),
    "qwen2.5-32b": dict(l_layers=64, l_hidden=5120),
    "qwen2.5-72b": dict(l_layers=80, l_hidden=8192),
    "qwen2-72b": dict(l_layers=80, l_hidden=8192),
}

# Synthetic profile constants (A100-class, the paper's hardware P:876).
P_E, P_LIN, P_ATT = 1.6e14, 2.0e14, 1.2e14
HALF_E, HALF_LIN, HALF_ATT = 4.0, 1024.0, 4096.0
BETA = 0.15
TP_KNOTS = [1.0, 2.0, 4.0, 8.0]
E_KNOTS = [float(2 ** k) for k in range(0, 11)]          # 1 .. 1024
L_KNOTS = [float(2 ** k) for k in range(7, 18)]          # 128 .. 131072


def _thr_law(peak: float, half: float, x: float, tp: float) -> float:
    """Saturating per-GPU throughput with TP degradation (fig:input_shape shape)."""
    sat = x / (x + half)
    return peak * sat / (1.0 + BETA * math.log2(tp) * half / (x + half))


def thr_grid(peak: float, half: float, knots: List[float]) -> Dict:
    return dict(
        x=list(knots),
        tp=list(TP_KNOTS),
        v=[[_thr_law(peak, half, x, tp) for x in knots] for tp in TP_KNOTS],
    )


def mem_grids(enc: Dict, llm: Dict) -> Dict:
    """Linear memory grids at layer counts {1, 2}, Korthikanti-style estimates.

    model state: 16 B per parameter (bf16 weights + grads + fp32 Adam) / tp,
    12*h^2 parameters per layer; activations: 34 B * tokens * h per layer / tp.
    """
    def ms(h):
        return dict(l=[1.0, 2.0], tp=list(TP_KNOTS), x=[0.0],
                    v=[[[16.0 * 12.0 * h * h * l / tp] for tp in TP_KNOTS] for l in (1.0, 2.0)])

    e_x = [0.0] + [float(2 ** k) for k in range(0, 21)]      # encoder effective batch
    l_x = [0.0] + [float(2 ** k) for k in range(7, 27)]      # packed LLM tokens
    he, es, hl = enc["e_hidden"], enc["e_seq"], llm["l_hidden"]
    as_e = dict(l=[1.0, 2.0], tp=list(TP_KNOTS), x=e_x,
                v=[[[34.0 * l * b * es * he / tp for b in e_x] for tp in TP_KNOTS] for l in (1.0, 2.0)])
    as_l = dict(l=[1.0, 2.0], tp=list(TP_KNOTS), x=l_x,
                v=[[[34.0 * l * s * hl / tp for s in l_x] for tp in TP_KNOTS] for l in (1.0, 2.0)])
    return dict(ms_e=ms(he), as_e=as_e, ms_l=ms(hl), as_l=as_l)


def cost_model(encoder: str, llm: str, tick_ns: float = 1.0, bwd_ratio: float = 2.0, e_attn: int = 0) -> Dict:
    enc, lm = ENCODERS[encoder], LLMS[llm]
    m = dict(enc)
    m.update(lm)
    m.update(
        e_attn=e_attn,
        bwd_ratio=bwd_ratio,
        tick_ns=tick_ns,
        thr_e=thr_grid(P_E, HALF_E, E_KNOTS),
        thr_att=thr_grid(P_ATT, HALF_ATT, L_KNOTS),
        thr_lin=thr_grid(P_LIN, HALF_LIN, L_KNOTS),
    )
    return m


# --------------------------------------------------------------------------
# Feature mixtures (tab:dataset_composition P:812-832; fig:patch-triple P:984-1004).
# --------------------------------------------------------------------------
def _lognormal_int(rng, median, sigma, lo, hi, size):
    x = np.exp(rng.normal(math.log(median), sigma, size))
    return np.clip(np.round(x), lo, hi).astype(np.int64)


def _features(kind: int, n: int, rng: np.random.Generator):
    tiles = np.zeros(n, np.int64)
    frames = np.zeros(n, np.int64)
    text = np.zeros(n, np.int64)
    if kind in (1, 2, 3, 4):
        if kind == 1:
            probs = [0.50, 0.25, 0.0, 0.25]          # single / multi / video / text-only
        elif kind == 2:
            probs = [0.52, 0.48, 0.0, 0.0]           # 65k : 60k
        else:
            probs = [0.35, 0.32, 0.33, 0.0]
        cat = rng.choice(4, size=n, p=probs)
        single_tiles = np.array([2, 3, 4, 5, 7, 10])   # AnyRes base + grid
        t_single = single_tiles[rng.integers(0, len(single_tiles), n)]
        multi_hi = {1: 6, 2: 12, 3: 12, 4: 12}[kind]
        t_multi = rng.integers(2, multi_hi + 1, n)
        if kind == 3:
            tail = rng.random(n) < 0.15
            f_body = rng.integers(8, 33, n)
            u = 1.0 - rng.random(n)                    # (0, 1]
            f_tail = np.minimum(np.floor(32.0 * u ** (-1.0 / 1.2)), 512).astype(np.int64)
            f_video = np.where(tail, f_tail, f_body)
        else:
            f_video = rng.integers(8, 33, n)
        if kind == 2:
            txt = _lognormal_int(rng, 200, 1.0, 8, 4096, n)
        else:
            txt = _lognormal_int(rng, 256, 0.9, 8, 4096, n)
        txt_only = _lognormal_int(rng, 1024, 0.8, 32, 8192, n)
        tiles = np.where(cat == 0, t_single, np.where(cat == 1, t_multi, 0))
        frames = np.where(cat == 2, f_video, 0)
        text = np.where(cat == 3, txt_only, txt)
    elif kind == 5:
        cat = rng.choice(4, size=n, p=[0.30, 0.20, 0.30, 0.20])
        t_img = np.clip(np.ceil(np.exp(rng.normal(math.log(4.0), 1.0, n))), 1, 64).astype(np.int64)
        n_img = rng.integers(2, 9, n)
        per_img = np.clip(np.round(np.exp(rng.normal(math.log(2.0), 0.7, n))), 1, 16).astype(np.int64)
        u = 1.0 - rng.random(n)
        f_video = np.minimum(np.floor(16.0 * u ** (-1.0 / 1.1)), 768).astype(np.int64)
        txt = _lognormal_int(rng, 256, 0.9, 8, 4096, n)
        txt_only = _lognormal_int(rng, 1024, 1.0, 32, 32768, n)
        tiles = np.where(cat == 0, t_img, np.where(cat == 1, n_img * per_img, 0))
        frames = np.where(cat == 2, f_video, 0)
        text = np.where(cat == 3, txt_only, txt)
    else:
        raise ValueError(kind)
    return (tiles.astype(np.uint32), frames.astype(np.uint32), text.astype(np.uint32))


@dataclasses.dataclass
class Preset:
    """One BASELINE.json configuration."""
    k: int
    name: str
    n: int
    plan: Optional[Dict]            # fixed theta, or None for the searched config 4
    model: Dict
    K: int
    R: int
    G: int
    cluster: Optional[Dict] = None  # config 4: n_gpus, gpus_per_node, mem_per_gpu
    gbs: int = 0
    top_p: int = 0
    K_scaling: str = "strong"       # "weak": K per GPU; "strong": K total

    def features(self, batch: int = 0):
        """(tiles, frames, text) u32 arrays for global batch ``batch`` (seed 1000*k + b)."""
        rng = np.random.Generator(np.random.PCG64(1000 * self.k + batch))
        return _features(self.k, self.n, rng)

    def seed(self, batch: int = 0):
        """Philox key (0xDF100000 + k, b)."""
        return (0xDF100000 + self.k, batch)

    def mem(self) -> Dict:
        enc = {key: self.model[key] for key in ("e_hidden", "e_seq")}
        llm = {"l_hidden": self.model["l_hidden"]}
        g = mem_grids(enc, llm)
        g["mem_per_gpu"] = (self.cluster or {}).get("mem_per_gpu", 80.0 * GIB)
        return g


def plan(e_tp, e_pp, e_dp, l_tp, l_pp, l_dp, n_mb) -> Dict:
    return dict(e_tp=e_tp, e_pp=e_pp, e_dp=e_dp, l_tp=l_tp, l_pp=l_pp, l_dp=l_dp, n_mb=n_mb)


def presets() -> Dict[int, Preset]:
    return {
        1: Preset(1, "cfg1-n32-m4-s2", 32, plan(1, 1, 1, 1, 1, 1, 4),
                  cost_model("siglip-so400m", "qwen2.5-7b", tick_ns=1000.0), K=65536, R=16, G=8),
        2: Preset(2, "cfg2-n256-m16-s4", 256, plan(1, 1, 1, 2, 3, 1, 16),
                  cost_model("clip-vit-l14-336", "qwen2.5-7b", tick_ns=1000.0), K=65536, R=16, G=8),
        3: Preset(3, "cfg3-n1024-m32-s8", 1024, plan(1, 1, 1, 4, 7, 1, 32),
                  cost_model("siglip-so400m", "qwen2.5-32b", tick_ns=1000.0), K=65536, R=16, G=8, K_scaling="weak"),
        4: Preset(4, "cfg4-search-64gpu-gbs2048", 2048, None,
                  cost_model("internvit-6b", "qwen2.5-72b", tick_ns=1000.0), K=4096, R=16, G=8,
                  cluster=dict(n_gpus=64, gpus_per_node=8, mem_per_gpu=80.0 * GIB), gbs=2048, top_p=64),
        5: Preset(5, "cfg5-n4096-m64-s16", 4096, plan(1, 2, 1, 8, 14, 1, 64),
                  cost_model("qwen2-vl-vit", "qwen2-72b", tick_ns=1000.0), K=1_000_000, R=16, G=8),
    }


def random_costs(n: int, seed: int, lo: int = 0, hi: int = 1000, heavy: bool = False) -> np.ndarray:
    """Random integer cost matrix [4][n] (ef, eb, lf, lb) for balance/simulator tests."""
    rng = np.random.Generator(np.random.PCG64(seed))
    if heavy:
        x = np.floor(hi * (1.0 - rng.random((2, n))) ** (-1.0 / 1.3)).astype(np.int64)
        x = np.minimum(x, 50 * hi)
    else:
        x = rng.integers(lo, hi + 1, (2, n))
    f = x.astype(np.uint32)
    b = (2 * x).astype(np.uint32)
    return np.stack([f[0], b[0], f[1], b[1]]).astype(np.uint32)


def random_durations(C: int, S: int, M: int, seed: int, hi: int = 100) -> tuple:
    rng = np.random.Generator(np.random.PCG64(seed))
    fwd = rng.integers(0, hi + 1, (C, S, M)).astype(np.uint64)
    bwd = rng.integers(0, 2 * hi + 1, (C, S, M)).astype(np.uint64)
    return fwd, bwd
