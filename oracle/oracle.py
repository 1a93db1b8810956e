"""ctypes binding of the CPU ORACLE (oracle/dflop_oracle.c).  TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
leg may import this module.  It marshals the seeded inputs of
``paper_2603_25120_b200.synth`` (plain dicts / numpy arrays) into the oracle's
own C structs; nothing here is shared with the CUDA path's binding.

ctypes releases the GIL during foreign calls, so ``balance_threaded`` runs the
single-threaded oracle over candidate ranges on all host cores.
"""
from __future__ import annotations

import concurrent.futures as cf
import ctypes as C
import os
import subprocess
from typing import Dict, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
SRC = os.path.join(HERE, "dflop_oracle.c")

MAX_X, MAX_TP = 32, 4


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C11, no FMA contraction)."""
    if force or not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < max(
            os.path.getmtime(SRC), os.path.getmtime(os.path.join(HERE, "dflop_oracle.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared",
                               "-o", LIB_PATH, SRC, "-lm"])
    return LIB_PATH


class OrcGrid(C.Structure):
    _fields_ = [("n_x", C.c_uint32), ("n_tp", C.c_uint32), ("x", C.c_double * MAX_X),
                ("tp", C.c_double * MAX_TP), ("v", (C.c_double * MAX_X) * MAX_TP)]


class OrcMGrid(C.Structure):
    _fields_ = [("n_x", C.c_uint32), ("n_tp", C.c_uint32), ("l", C.c_double * 2),
                ("tp", C.c_double * MAX_TP), ("x", C.c_double * MAX_X),
                ("v", ((C.c_double * MAX_X) * MAX_TP) * 2)]


class OrcModel(C.Structure):
    _fields_ = [("e_layers", C.c_uint32), ("e_hidden", C.c_uint32), ("e_seq", C.c_uint32),
                ("e_attn", C.c_uint32), ("l_layers", C.c_uint32), ("l_hidden", C.c_uint32),
                ("tau_tile", C.c_uint32), ("tau_frame", C.c_uint32), ("bwd_ratio", C.c_double),
                ("tick_ns", C.c_double), ("thr_e", OrcGrid), ("thr_att", OrcGrid), ("thr_lin", OrcGrid)]


class OrcMem(C.Structure):
    _fields_ = [("ms_e", OrcMGrid), ("as_e", OrcMGrid), ("ms_l", OrcMGrid), ("as_l", OrcMGrid),
                ("mem_per_gpu", C.c_double)]


CORR_BINS, TRACK_WIN = 32, 4096


class OrcTracker(C.Structure):
    _fields_ = [("alpha", C.c_double), ("cost", C.c_double), ("window", C.c_uint32), ("active", C.c_uint32),
                ("observed", (C.c_double * CORR_BINS) * 3), ("predicted", (C.c_double * CORR_BINS) * 3),
                ("seen", (C.c_uint8 * CORR_BINS) * 3), ("n_benefits", C.c_uint64),
                ("last", C.c_double * TRACK_WIN)]


class OrcPlan(C.Structure):
    _fields_ = [(k, C.c_uint32) for k in ("e_tp", "e_pp", "e_dp", "l_tp", "l_pp", "l_dp", "n_mb")]


class OrcBParams(C.Structure):
    _fields_ = [("mode", C.c_uint32), ("K", C.c_uint32), ("R", C.c_uint32), ("G", C.c_uint32),
                ("seed", C.c_uint32 * 2)]


_lib = None


def build_variant(src_text: str, tag: str) -> str:
    """Compile a MODIFIED copy of the oracle source (mutation tests of the pins,
    tests/test_oracle_worked.py) into /tmp; returns the .so path.  Never used by lib()."""
    import tempfile
    d = tempfile.mkdtemp(prefix=f"orc_{tag}_")
    src = os.path.join(d, "dflop_oracle.c")
    with open(src, "w") as f:
        f.write(src_text)
    so = os.path.join(d, "liboracle.so")
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fPIC", "-shared", "-I" + HERE,
                           "-o", so, src, "-lm"])
    return so


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = load(LIB_PATH)
    return _lib


def load(path: str):
    """ctypes handle of an oracle build with every signature declared."""
    if True:
        L = C.CDLL(path)
        P = C.POINTER
        u32p, u64p, f64p = P(C.c_uint32), P(C.c_uint64), P(C.c_double)
        L.orc_philox4x32_10.argtypes = [u32p, u32p, u32p]
        L.orc_mulhi32.argtypes = [C.c_uint32, C.c_uint32]
        L.orc_mulhi32.restype = C.c_uint32
        L.orc_interp_thr.argtypes = [P(OrcGrid), C.c_double, C.c_double]
        L.orc_interp_thr.restype = C.c_double
        L.orc_interp_mem.argtypes = [P(OrcMGrid), C.c_double, C.c_double, C.c_double]
        L.orc_interp_mem.restype = C.c_double
        L.orc_predict.argtypes = [P(OrcModel), P(OrcPlan), u32p, u32p, u32p, C.c_uint32, f64p, u32p, u32p]
        L.orc_predict_corrected.argtypes = [P(OrcModel), P(OrcPlan), u32p, u32p, u32p, C.c_uint32, f64p, f64p,
                                            u32p, u32p]
        L.orc_exact_cmax.argtypes = [u32p, C.c_uint32, C.c_uint32, C.c_uint64, u32p, u32p, u64p, u64p, u32p, u64p]
        L.orc_order_search.argtypes = [u32p, C.c_uint32, P(OrcPlan), u32p, C.c_uint32, u32p, u64p]
        L.orc_route_plan.argtypes = [u32p, C.c_uint32, P(OrcPlan), u32p, u32p, u32p, u32p, u32p, u64p]
        L.orc_shape_bin.argtypes = [C.c_uint64]
        L.orc_shape_bin.restype = C.c_uint32
        L.orc_base_order.argtypes = [u32p, C.c_uint32, u32p]
        L.orc_simulate_1f1b.argtypes = [u64p, u64p, C.c_uint32, C.c_uint32, u64p, u64p]
        L.orc_run_candidate.argtypes = [u32p, C.c_uint32, P(OrcPlan), P(OrcBParams), u32p, C.c_uint32,
                                        u32p, u64p, u64p]
        L.orc_balance.argtypes = [u32p, C.c_uint32, P(OrcPlan), P(OrcBParams), C.c_uint32, C.c_uint32,
                                  u64p, u64p, u64p, u32p, u64p, u32p]
        L.orc_groups.argtypes = [u32p, C.c_uint32, C.c_uint32, u32p, u32p]
        L.orc_find_combs.argtypes = [C.c_uint32, C.c_uint32, u32p, C.c_uint32]
        L.orc_find_combs.restype = C.c_uint32
        L.orc_enumerate_configs.argtypes = [C.c_uint32, C.c_uint32, u32p, C.c_uint64]
        L.orc_enumerate_configs.restype = C.c_uint64
        L.orc_batch_means.argtypes = [P(OrcModel), u32p, u32p, u32p, C.c_uint32, f64p, f64p]
        L.orc_stage_a_pair.argtypes = [P(OrcModel), P(OrcMem), u32p, C.c_uint32, C.c_uint32, C.c_double,
                                       C.c_double, u64p, f64p, f64p, u64p, u64p]
        L.orc_stage_a_pair.restype = C.c_int
        L.orc_stage_a_all.argtypes = [P(OrcModel), P(OrcMem), C.c_uint32, C.c_uint32, C.c_uint32, C.c_double,
                                      C.c_double, u64p, C.c_uint64]
        L.orc_stage_a_all.restype = C.c_uint64
        L.orc_stage_a_top.argtypes = [u64p, C.c_uint64, C.c_uint32, u64p]
        L.orc_stage_a_top.restype = C.c_uint32
    L.orc_exact_pairs.argtypes = [u32p, C.c_uint32, C.c_uint32, u32p, u32p, u64p, u64p, u64p]
    L.orc_tracker_init.argtypes = [P(OrcTracker), C.c_double, C.c_uint32, C.c_double]
    L.orc_tracker_record.argtypes = [P(OrcTracker), C.c_uint32, C.c_uint64, C.c_double, C.c_double]
    L.orc_tracker_record.restype = C.c_double
    L.orc_tracker_rho.argtypes = [P(OrcTracker), f64p]
    L.orc_tracker_cost_benefit.argtypes = [P(OrcTracker), f64p, C.c_uint32]
    L.orc_tracker_cost_benefit.restype = C.c_uint32
    return L


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(C.POINTER(t))


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


# ---------------------------------------------------------------- marshalling
def grid_struct(g: Dict) -> OrcGrid:
    s = OrcGrid()
    s.n_x, s.n_tp = len(g["x"]), len(g["tp"])
    for k, x in enumerate(g["x"]):
        s.x[k] = x
    for a, t in enumerate(g["tp"]):
        s.tp[a] = t
        for k, v in enumerate(g["v"][a]):
            s.v[a][k] = v
    return s


def mgrid_struct(g: Dict) -> OrcMGrid:
    s = OrcMGrid()
    s.n_x, s.n_tp = len(g["x"]), len(g["tp"])
    s.l[0], s.l[1] = g["l"]
    for k, x in enumerate(g["x"]):
        s.x[k] = x
    for a, t in enumerate(g["tp"]):
        s.tp[a] = t
    for q in range(2):
        for a in range(len(g["tp"])):
            for k in range(len(g["x"])):
                s.v[q][a][k] = g["v"][q][a][k]
    return s


def model_struct(m: Dict) -> OrcModel:
    s = OrcModel()
    for k in ("e_layers", "e_hidden", "e_seq", "e_attn", "l_layers", "l_hidden", "tau_tile", "tau_frame"):
        setattr(s, k, int(m[k]))
    s.bwd_ratio, s.tick_ns = float(m["bwd_ratio"]), float(m["tick_ns"])
    s.thr_e, s.thr_att, s.thr_lin = grid_struct(m["thr_e"]), grid_struct(m["thr_att"]), grid_struct(m["thr_lin"])
    return s


def mem_struct(g: Dict) -> OrcMem:
    s = OrcMem()
    for k in ("ms_e", "as_e", "ms_l", "as_l"):
        setattr(s, k, mgrid_struct(g[k]))
    s.mem_per_gpu = float(g["mem_per_gpu"])
    return s


def plan_struct(p: Dict) -> OrcPlan:
    return OrcPlan(*[int(p[k]) for k in ("e_tp", "e_pp", "e_dp", "l_tp", "l_pp", "l_dp", "n_mb")])


def bparams_struct(K: int, R: int, G: int, seed: Sequence[int], mode: int = 0) -> OrcBParams:
    b = OrcBParams()
    b.mode, b.K, b.R, b.G = mode, K, R, G
    b.seed[0], b.seed[1] = int(seed[0]) & 0xFFFFFFFF, int(seed[1]) & 0xFFFFFFFF
    return b


# ---------------------------------------------------------------- wrappers
def philox(ctr, key):
    c, k, o = _u32(ctr), _u32(key), np.zeros(4, np.uint32)
    lib().orc_philox4x32_10(_p(c, C.c_uint32), _p(k, C.c_uint32), _p(o, C.c_uint32))
    return o


def mulhi32(u, n):
    return lib().orc_mulhi32(u, n)


def interp_thr(g: Dict, x: float, tp: float) -> float:
    s = grid_struct(g)
    return lib().orc_interp_thr(C.byref(s), x, tp)


def interp_mem(g: Dict, l: float, tp: float, x: float) -> float:
    s = mgrid_struct(g)
    return lib().orc_interp_mem(C.byref(s), l, tp, x)


def predict(model: Dict, plan: Dict, tiles, frames, text):
    """Returns (cost_f64[4][n] ns, cost_q[4][n] ticks, status, first_bad_index)."""
    t, f, x = _u32(tiles), _u32(frames), _u32(text)
    n = len(t)
    cf64 = np.zeros((4, n), np.float64)
    cq = np.zeros((4, n), np.uint32)
    bad = np.zeros(1, np.uint32)
    ms, ps = model_struct(model), plan_struct(plan)
    st = lib().orc_predict(C.byref(ms), C.byref(ps), _p(t, C.c_uint32), _p(f, C.c_uint32), _p(x, C.c_uint32),
                           n, _p(cf64, C.c_double), _p(cq, C.c_uint32), _p(bad, C.c_uint32))
    return cf64, cq, st, int(bad[0])


CORR_BINS = 32


class Tracker:
    """The oracle's N1 tracker (orc_tracker_*)."""

    def __init__(self, alpha=0.25, window=10, cost=0.0):
        self.s = OrcTracker()
        assert lib().orc_tracker_init(C.byref(self.s), alpha, window, cost) == 0

    def record(self, grid: int, x: int, th_actual: float, th_pred: float) -> float:
        return lib().orc_tracker_record(C.byref(self.s), grid, int(x), th_actual, th_pred)

    def rho(self):
        r = np.zeros((3, CORR_BINS))
        lib().orc_tracker_rho(C.byref(self.s), _p(r, C.c_double))
        return r

    def cost_benefit(self, benefits) -> bool:
        b = np.ascontiguousarray(np.asarray(list(benefits), dtype=np.float64))
        return bool(lib().orc_tracker_cost_benefit(C.byref(self.s), _p(b, C.c_double) if b.size else None, b.size))


def shape_bin(x: int) -> int:
    return int(lib().orc_shape_bin(C.c_uint64(int(x))))


def predict_corrected(model: Dict, plan: Dict, tiles, frames, text, rho):
    """a1 with Adaptive Correction ratios rho[3][32] (N1); rho=None is predict()."""
    t, f, x = _u32(tiles), _u32(frames), _u32(text)
    n = len(t)
    cf64 = np.zeros((4, n), np.float64)
    cq = np.zeros((4, n), np.uint32)
    bad = np.zeros(1, np.uint32)
    ms, ps = model_struct(model), plan_struct(plan)
    r = None if rho is None else np.ascontiguousarray(np.asarray(rho, np.float64).reshape(3, CORR_BINS))
    st = lib().orc_predict_corrected(C.byref(ms), C.byref(ps), _p(t, C.c_uint32), _p(f, C.c_uint32),
                                     _p(x, C.c_uint32), n, None if r is None else _p(r, C.c_double),
                                     _p(cf64, C.c_double), _p(cq, C.c_uint32), _p(bad, C.c_uint32))
    return cf64, cq, st, int(bad[0])


def base_order(cost_q):
    q = _u32(cost_q)
    n = q.shape[1]
    o = np.zeros(n, np.uint32)
    lib().orc_base_order(_p(q, C.c_uint32), n, _p(o, C.c_uint32))
    return o


def simulate_1f1b(fwd, bwd):
    """fwd, bwd: [S][M] -> (makespan, stage_busy[S])."""
    f, b = _u64(fwd), _u64(bwd)
    S, M = f.shape
    T = np.zeros(1, np.uint64)
    busy = np.zeros(S, np.uint64)
    st = lib().orc_simulate_1f1b(_p(f, C.c_uint64), _p(b, C.c_uint64), S, M, _p(T, C.c_uint64),
                                 _p(busy, C.c_uint64))
    assert st == 0, st
    return int(T[0]), busy


def run_candidate(cost_q, plan: Dict, K, R, G, seed, c, mode=0, order=None):
    q = _u32(cost_q)
    n = q.shape[1]
    pi = base_order(q) if order is None else _u32(order)
    a = np.zeros(n, np.uint32)
    T, cm = np.zeros(1, np.uint64), np.zeros(1, np.uint64)
    ps, bs = plan_struct(plan), bparams_struct(K, R, G, seed, mode)
    st = lib().orc_run_candidate(_p(q, C.c_uint32), n, C.byref(ps), C.byref(bs), _p(pi, C.c_uint32), c,
                                 _p(a, C.c_uint32), _p(T, C.c_uint64), _p(cm, C.c_uint64))
    assert st == 0, st
    return a, int(T[0]), int(cm[0])


def balance(cost_q, plan: Dict, K, R, G, seed, c0=0, c1=None, mode=0, per_candidate=True):
    """Runs candidates [c0, c1) single-threaded.  Returns dict(T, c, cmax, assign, cand_T, cand_cmax)."""
    q = _u32(cost_q)
    n = q.shape[1]
    c1 = K if c1 is None else c1
    nc = c1 - c0
    cT = np.zeros(max(nc, 1), np.uint64) if per_candidate else None
    cC = np.zeros(max(nc, 1), np.uint64) if per_candidate else None
    bT, bC, bc = np.zeros(1, np.uint64), np.zeros(1, np.uint64), np.zeros(1, np.uint32)
    a = np.zeros(max(n, 1), np.uint32)
    ps, bs = plan_struct(plan), bparams_struct(K, R, G, seed, mode)
    st = lib().orc_balance(_p(q, C.c_uint32), n, C.byref(ps), C.byref(bs), c0, c1,
                           _p(cT, C.c_uint64) if per_candidate else None,
                           _p(cC, C.c_uint64) if per_candidate else None,
                           _p(bT, C.c_uint64), _p(bc, C.c_uint32), _p(bC, C.c_uint64), _p(a, C.c_uint32))
    assert st == 0, st
    out = dict(T=int(bT[0]), c=int(bc[0]), cmax=int(bC[0]), assign=a[:n].copy())
    if per_candidate:
        out["cand_T"], out["cand_cmax"] = cT[:nc], cC[:nc]
    return out


def balance_threaded(cost_q, plan: Dict, K, R, G, seed, c0=0, c1=None, mode=0, threads: Optional[int] = None,
                     per_candidate=True):
    """Same result as ``balance``; candidate ranges run concurrently on host threads."""
    c1 = K if c1 is None else c1
    threads = threads or os.cpu_count() or 1
    nc = c1 - c0
    chunks = max(1, min(threads * 4, nc))
    bounds = [c0 + (nc * k) // chunks for k in range(chunks + 1)]
    with cf.ThreadPoolExecutor(threads) as ex:
        parts = list(ex.map(lambda k: balance(cost_q, plan, K, R, G, seed, bounds[k], bounds[k + 1], mode,
                                              per_candidate), range(chunks)))
    best = min(parts, key=lambda r: (r["T"], r["c"]))
    out = dict(T=best["T"], c=best["c"], cmax=best["cmax"], assign=best["assign"])
    if per_candidate:
        out["cand_T"] = np.concatenate([p["cand_T"] for p in parts])
        out["cand_cmax"] = np.concatenate([p["cand_cmax"] for p in parts])
    return out


def groups(assign, m):
    a = _u32(assign)
    n = len(a)
    off = np.zeros(m + 1, np.uint32)
    items = np.zeros(max(n, 1), np.uint32)
    lib().orc_groups(_p(a, C.c_uint32), n, m, _p(off, C.c_uint32), _p(items, C.c_uint32))
    return off, items[:n]


def find_combs(gpus, node):
    n = lib().orc_find_combs(gpus, node, None, 0)
    out = np.zeros((max(n, 1), 3), np.uint32)
    lib().orc_find_combs(gpus, node, _p(out, C.c_uint32), n)
    return out[:n]


def enumerate_configs(n_gpus, node):
    n = lib().orc_enumerate_configs(n_gpus, node, None, 0)
    out = np.zeros((max(n, 1), 6), np.uint32)
    lib().orc_enumerate_configs(n_gpus, node, _p(out, C.c_uint32), n)
    return out[:n]


def batch_means(model: Dict, tiles, frames, text):
    t, f, x = _u32(tiles), _u32(frames), _u32(text)
    mb, ms = np.zeros(1), np.zeros(1)
    m = model_struct(model)
    lib().orc_batch_means(C.byref(m), _p(t, C.c_uint32), _p(f, C.c_uint32), _p(x, C.c_uint32), len(t),
                          _p(mb, C.c_double), _p(ms, C.c_double))
    return float(mb[0]), float(ms[0])


def stage_a_pair(model: Dict, mem: Dict, cfg6, i, gbs, mean_b, mean_s):
    c = _u32(cfg6)
    T = np.zeros(1, np.uint64)
    me, ml = np.zeros(1), np.zeros(1)
    ed, ld = np.zeros(1, np.uint64), np.zeros(1, np.uint64)
    ms, mm = model_struct(model), mem_struct(mem)
    ok = lib().orc_stage_a_pair(C.byref(ms), C.byref(mm), _p(c, C.c_uint32), i, gbs, mean_b, mean_s,
                                _p(T, C.c_uint64), _p(me, C.c_double), _p(ml, C.c_double),
                                _p(ed, C.c_uint64), _p(ld, C.c_uint64))
    return dict(feasible=bool(ok), T_A=int(T[0]), mem_e=float(me[0]), mem_l=float(ml[0]),
                e_dur=int(ed[0]), l_dur=int(ld[0]))


def stage_a_all(model: Dict, mem: Dict, n_gpus, node, gbs, mean_b, mean_s):
    cfgs = enumerate_configs(n_gpus, node)
    n_pairs = int(sum(gbs // int(c[5]) for c in cfgs))
    T = np.zeros(max(n_pairs, 1), np.uint64)
    ms, mm = model_struct(model), mem_struct(mem)
    k = lib().orc_stage_a_all(C.byref(ms), C.byref(mm), n_gpus, node, gbs, mean_b, mean_s, _p(T, C.c_uint64),
                              n_pairs)
    assert k == n_pairs
    return T[:n_pairs], cfgs


def stage_a_top(T_A, P):
    t = _u64(T_A)
    top = np.zeros(max(P, 1), np.uint64)
    k = lib().orc_stage_a_top(_p(t, C.c_uint64), len(t), P, _p(top, C.c_uint64))
    return top[:k]


def pair_to_config(cfgs, gbs, pair_index):
    """Map an enumeration-order pair index to (eps, i)."""
    k = int(pair_index)
    for e, c in enumerate(cfgs):
        nm = gbs // int(c[5])
        if k < nm:
            return e, k + 1
        k -= nm
    raise IndexError(pair_index)


def search(model: Dict, mem: Dict, cluster: Dict, tiles, frames, text, gbs, top_p, K, R, G, seed,
           top_pairs=None, threads=None):
    """Algorithm 1 Stage A + the balanced Stage B.  ``top_pairs`` may pin the
    Stage-A selection (two-level parity: the GPU's selection fed to the oracle)."""
    mb, msq = batch_means(model, tiles, frames, text)
    T_A, cfgs = stage_a_all(model, mem, cluster["n_gpus"], cluster["gpus_per_node"], gbs, mb, msq)
    if top_pairs is None:
        top_pairs = stage_a_top(T_A, top_p)
    best = None
    for rank, pidx in enumerate(top_pairs):
        e, i = pair_to_config(cfgs, gbs, pidx)
        c = cfgs[e]
        plan = dict(e_tp=int(c[0]), e_pp=int(c[1]), e_dp=int(c[2]), l_tp=int(c[3]), l_pp=int(c[4]),
                    l_dp=int(c[5]), n_mb=i)
        _, q, st, _ = predict(model, plan, tiles, frames, text)
        if st != 0:
            raise RuntimeError("oracle predict overflow")
        r = balance_threaded(q, plan, K, R, G, seed, threads=threads, per_candidate=False)
        key = (r["T"], rank, r["c"])
        if best is None or key < best[0]:
            best = (key, dict(plan=plan, T_B=r["T"], T_A=int(T_A[pidx]), rank=rank, c=r["c"], cmax=r["cmax"],
                              assign=r["assign"], pair=int(pidx)))
    out = best[1]
    out["n_configs"] = len(cfgs)
    out["n_pairs"] = len(T_A)
    out["n_feasible"] = int(np.count_nonzero(T_A != np.uint64(2 ** 64 - 1)))
    out["top_pairs"] = np.asarray(top_pairs, np.uint64)
    out["T_A_all"] = T_A
    return out


def expected_makespan_choice(plans, batch_costs, K, R, G, seed, threads=None):
    """N2, Eq. (1): for each plan (in Stage-A rank order) the sum over the sample's
    batches of T_B(b) -- the batch's best candidate makespan, batch b's family keyed
    (seed[0], seed[1] + b) (R33) -- and theta* = argmin (sum, rank).  batch_costs[p][b] is
    the [4][n_b] tick array of plan p on batch b.  Returns (winner rank, sums, per-batch
    results of every plan)."""
    sums, per = [], []
    for p, plan in enumerate(plans):
        tot, rows = 0, []
        for b, q in enumerate(batch_costs[p]):
            r = balance_threaded(q, plan, K, R, G, (seed[0], seed[1] + b), threads=threads, per_candidate=False)
            tot += int(r["T"])
            rows.append(r)
        sums.append(tot)
        per.append(rows)
    win = min(range(len(plans)), key=lambda p: (sums[p], p))
    return win, sums, per


def exact_cmax(cost_q, m, node_budget=10 ** 7, init_assign=None):
    """N3 branch and bound: dict(cmax, lb, proven, nodes, assign)."""
    q = _u32(cost_q)
    n = q.shape[1]
    a = np.zeros(max(n, 1), np.uint32)
    ia = None if init_assign is None else np.ascontiguousarray(np.asarray(init_assign, np.uint32))
    cm, lb, nodes = np.zeros(1, np.uint64), np.zeros(1, np.uint64), np.zeros(1, np.uint64)
    pr = np.zeros(1, np.uint32)
    st = lib().orc_exact_cmax(_p(q, C.c_uint32), n, m, int(node_budget), None if ia is None else _p(ia, C.c_uint32),
                              _p(a, C.c_uint32), _p(cm, C.c_uint64), _p(lb, C.c_uint64), _p(pr, C.c_uint32),
                              _p(nodes, C.c_uint64))
    if st != 0:
        raise ValueError(f"orc_exact_cmax status {st}")
    return dict(cmax=int(cm[0]), lb=int(lb[0]), proven=bool(pr[0]), nodes=int(nodes[0]), assign=a[:n])


def exact_pairs(cost_q, m, init_assign=None):
    """N3 certificate by pair decomposition (m = 2 or 4, n <= 40): the optimum C_max."""
    q = _u32(cost_q)
    n = q.shape[1]
    a = np.zeros(max(n, 1), np.uint32)
    cm, lb, vis = np.zeros(1, np.uint64), np.zeros(1, np.uint64), np.zeros(1, np.uint64)
    ia = None if init_assign is None else _u32(init_assign)
    st = lib().orc_exact_pairs(_p(q, C.c_uint32), n, m, _p(ia, C.c_uint32) if ia is not None else None,
                               _p(a, C.c_uint32), _p(cm, C.c_uint64), _p(lb, C.c_uint64), _p(vis, C.c_uint64))
    assert st == 0, st
    return dict(cmax=int(cm[0]), lb=int(lb[0]), visited=int(vis[0]), assign=a[:n])


def order_search(cost_q, plan: Dict, assign, rounds=64):
    """N4(a): per replica the slot order (bucket per slot) and its 1F1B makespan."""
    q = _u32(cost_q)
    n = q.shape[1]
    a = np.ascontiguousarray(np.asarray(assign, np.uint32))
    M, rep = plan["n_mb"], plan["l_dp"]
    order = np.zeros(M * rep, np.uint32)
    T = np.zeros(rep, np.uint64)
    st = lib().orc_order_search(_p(q, C.c_uint32), n, C.byref(plan_struct(plan)), _p(a, C.c_uint32), rounds,
                                _p(order, C.c_uint32), _p(T, C.c_uint64))
    if st != 0:
        raise ValueError(f"orc_order_search status {st}")
    return order.reshape(rep, M), T


def route_plan(cost_q, plan: Dict, assign):
    """N4(b): dict(pos_item, slot_off, enc_off [N_mb][E_dp+1], llm_off [N_mb][L_dp+1], enc_load)."""
    q = _u32(cost_q)
    n = q.shape[1]
    a = np.ascontiguousarray(np.asarray(assign, np.uint32))
    M, R, G = plan["n_mb"], plan["l_dp"], plan["e_dp"]
    pos = np.zeros(max(n, 1), np.uint32)
    so = np.zeros(M + 1, np.uint32)
    eo = np.zeros(M * (G + 1), np.uint32)
    lo = np.zeros(M * (R + 1), np.uint32)
    el = np.zeros(M * G, np.uint64)
    st = lib().orc_route_plan(_p(q, C.c_uint32), n, C.byref(plan_struct(plan)), _p(a, C.c_uint32), _p(pos, C.c_uint32),
                              _p(so, C.c_uint32), _p(eo, C.c_uint32), _p(lo, C.c_uint32), _p(el, C.c_uint64))
    if st != 0:
        raise ValueError(f"orc_route_plan status {st}")
    return dict(pos_item=pos[:n], slot_off=so, enc_off=eo.reshape(M, G + 1), llm_off=lo.reshape(M, R + 1),
                enc_load=el.reshape(M, G))
