"""Thin ctypes binding of libdflop.so (include/dflop.h) -- argument marshalling only.

Every step of the path runs in the library's CUDA kernels; this module converts the
seeded inputs (plain dicts from ``synth``) into the C structs, allocates device buffers
and workspaces with torch (plumbing), and calls the C ABI with the same names.  There is
no CPU fallback: if the library or a CUDA device is missing, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DFLOP_LIB") or os.path.join(HERE, "libdflop.so")

MAX_X, MAX_TP = 32, 4
MODE_HEURISTIC, MODE_EXHAUSTIVE, MODE_ORDER4 = 0, 1, 16
SEARCH_FIXED, SEARCH_ALG1 = 0, 1
DEV_COST_OVERFLOW, DEV_MAKESPAN_OVERFLOW = 1, 2
STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "SHAPE", 3: "OVERFLOW", 4: "INFEASIBLE", 5: "CUDA", 6: "NCCL",
          7: "WORKSPACE_TOO_SMALL", 8: "UNSUPPORTED"}

EXPORTS = ["dflop_abi_version", "dflop_last_error", "dflop_release_caches", "dflop_predict_costs",
           "dflop_balance_microbatches", "dflop_simulate_1f1b", "dflop_index_groups", "dflop_search_plans",
           "dflop_get_unique_id", "dflop_comm_init", "dflop_comm_destroy", "dflop_profile_enable",
           "dflop_profile_read", "dflop_search_plans_batches", "dflop_exact_cmax", "dflop_order_search",
           "dflop_route_plan", "dflop_shard_range", "dflop_owner_of", "dflop_pack_key", "dflop_select_plan"]


class DflopError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"{STATUS.get(code, code)}: {msg}")
        self.code = code


# ---------------------------------------------------------------- C structs
class Grid(C.Structure):
    _fields_ = [("n_x", C.c_uint32), ("n_tp", C.c_uint32), ("x", C.c_double * MAX_X),
                ("tp", C.c_double * MAX_TP), ("v", (C.c_double * MAX_X) * MAX_TP)]


class MemGrid(C.Structure):
    _fields_ = [("n_x", C.c_uint32), ("n_tp", C.c_uint32), ("l", C.c_double * 2), ("tp", C.c_double * MAX_TP),
                ("x", C.c_double * MAX_X), ("v", ((C.c_double * MAX_X) * MAX_TP) * 2)]


CORR_BINS = 32


class ExactResult(C.Structure):
    """dflop_exact_result (N3)."""
    _fields_ = [("struct_size", C.c_uint32), ("proven", C.c_uint32), ("cmax", C.c_uint64),
                ("lower_bound", C.c_uint64), ("nodes", C.c_uint64), ("makespan", C.c_uint64),
                ("searched", C.c_uint32), ("reserved", C.c_uint32)]


class Correction(C.Structure):
    """dflop_correction (N1 Adaptive Correction): rho[3][32] = Th_actual / Th_pred."""
    _fields_ = [("struct_size", C.c_uint32), ("active", C.c_uint32), ("rho", (C.c_float * CORR_BINS) * 3)]


class CostModel(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("e_layers", C.c_uint32), ("e_hidden", C.c_uint32),
                ("e_seq", C.c_uint32), ("e_attn", C.c_uint32), ("l_layers", C.c_uint32), ("l_hidden", C.c_uint32),
                ("tau_tile", C.c_uint32), ("tau_frame", C.c_uint32), ("reserved", C.c_uint32),
                ("bwd_ratio", C.c_double), ("tick_ns", C.c_double), ("thr_e", Grid), ("thr_att", Grid),
                ("thr_lin", Grid), ("correction", C.POINTER(Correction))]


class MemModel(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("reserved", C.c_uint32), ("ms_e", MemGrid), ("as_e", MemGrid),
                ("ms_l", MemGrid), ("as_l", MemGrid), ("mem_per_gpu", C.c_double)]


class Plan(C.Structure):
    _fields_ = [(k, C.c_uint32) for k in ("e_tp", "e_pp", "e_dp", "l_tp", "l_pp", "l_dp", "n_mb")]

    def as_dict(self):
        return {k: int(getattr(self, k)) for k, _ in self._fields_}


class Cluster(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("n_gpus", C.c_uint32), ("gpus_per_node", C.c_uint32),
                ("reserved", C.c_uint32)]


class BalanceParams(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("mode", C.c_uint32), ("K", C.c_uint32), ("cand_begin", C.c_uint32),
                ("cand_end", C.c_uint32), ("R", C.c_uint32), ("G", C.c_uint32), ("seed", C.c_uint32 * 2),
                ("id_base", C.c_uint32)]


class CandResult(C.Structure):
    _fields_ = [("key", C.c_uint64), ("makespan", C.c_uint64), ("cmax", C.c_uint64), ("cand", C.c_uint32),
                ("status", C.c_uint32)]


class SearchParams(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("mode", C.c_uint32), ("fixed_plan", Plan), ("gbs", C.c_uint32),
                ("top_p", C.c_uint32), ("K", C.c_uint32), ("R", C.c_uint32), ("G", C.c_uint32),
                ("seed", C.c_uint32 * 2)]


class PlanResult(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("status_bits", C.c_uint32), ("plan", Plan), ("m", C.c_uint32),
                ("cand", C.c_uint32), ("stage_a_rank", C.c_uint32), ("owner_rank", C.c_uint32),
                ("makespan", C.c_uint64), ("cmax", C.c_uint64), ("stage_a_makespan", C.c_uint64),
                ("alg1_plan", Plan), ("reserved", C.c_uint32), ("alg1_makespan", C.c_uint64),
                ("n_configs", C.c_uint64), ("n_pairs", C.c_uint64), ("n_feasible", C.c_uint64),
                ("n_candidates", C.c_uint64)]


class Profile(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("cand_launches", C.c_uint32), ("kernel_launches", C.c_uint64),
                ("cand_ms", C.c_double), ("stage_a_launches", C.c_uint32), ("split_chunks", C.c_uint32),
                ("stage_a_ms", C.c_double)]


_lib = None


def lib():
    """Load libdflop.so; raises if it is missing (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libdflop.so not built at {LIB_PATH}; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        vp, u32, u64, sz = C.c_void_p, C.c_uint32, C.c_uint64, C.c_size_t
        P = C.POINTER
        L.dflop_abi_version.restype = u32
        L.dflop_last_error.restype = C.c_char_p
        L.dflop_predict_costs.argtypes = [P(CostModel), P(Plan), vp, vp, vp, u32, vp, vp, vp, vp]
        L.dflop_balance_microbatches.argtypes = [vp, u32, P(Plan), P(BalanceParams), vp, P(sz), vp, vp, vp, vp, vp,
                                                 vp, vp]
        L.dflop_simulate_1f1b.argtypes = [vp, vp, u32, u32, u32, vp, vp, vp]
        L.dflop_index_groups.argtypes = [vp, u32, u32, vp, vp, vp, P(sz), vp]
        L.dflop_search_plans.argtypes = [P(Cluster), P(CostModel), P(MemModel), vp, vp, vp, u32, P(SearchParams),
                                         vp, vp, P(sz), P(PlanResult), vp, vp, u64, vp]
        L.dflop_get_unique_id.argtypes = [C.c_char_p]
        L.dflop_comm_init.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_int, P(vp)]
        L.dflop_comm_destroy.argtypes = [vp]
        L.dflop_profile_enable.argtypes = [C.c_int]
        L.dflop_profile_read.argtypes = [P(Profile), C.c_int]
        L.dflop_shard_range.argtypes = [u32, u32, u32, P(u32), P(u32)]
        L.dflop_owner_of.argtypes = [u32, u32, u32]
        L.dflop_pack_key.argtypes = [u64, u32]
        L.dflop_select_plan.argtypes = [P(u64), u32, u32, P(u32), P(u32), P(u64)]
        for f in EXPORTS:
            if f not in ("dflop_abi_version", "dflop_last_error", "dflop_owner_of", "dflop_pack_key"):
                getattr(L, f).restype = C.c_int32
        L.dflop_owner_of.restype = u32
        L.dflop_pack_key.restype = u64
        _lib = L
    return _lib


def _check(code: int):
    if code != 0:
        raise DflopError(code, lib().dflop_last_error().decode())


# ---------------------------------------------------------------- marshalling
def grid_struct(g: Dict) -> Grid:
    s = Grid()
    s.n_x, s.n_tp = len(g["x"]), len(g["tp"])
    for k, x in enumerate(g["x"]):
        s.x[k] = x
    for a, t in enumerate(g["tp"]):
        s.tp[a] = t
        for k, v in enumerate(g["v"][a]):
            s.v[a][k] = v
    return s


def mem_grid_struct(g: Dict) -> MemGrid:
    s = MemGrid()
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


def cost_model_struct(m: Dict) -> CostModel:
    s = CostModel()
    s.struct_size = C.sizeof(CostModel)
    for k in ("e_layers", "e_hidden", "e_seq", "e_attn", "l_layers", "l_hidden", "tau_tile", "tau_frame"):
        setattr(s, k, int(m[k]))
    s.bwd_ratio, s.tick_ns = float(m["bwd_ratio"]), float(m["tick_ns"])
    s.thr_e, s.thr_att, s.thr_lin = grid_struct(m["thr_e"]), grid_struct(m["thr_att"]), grid_struct(m["thr_lin"])
    corr = m.get("correction")
    if corr is not None:  # {"active": bool, "rho": [3][32]} (N1), e.g. CorrectionTracker.table()
        c = Correction()
        c.struct_size = C.sizeof(Correction)
        c.active = 1 if corr.get("active", True) else 0
        rho = corr["rho"]
        for g in range(3):
            for q in range(CORR_BINS):
                c.rho[g][q] = float(rho[g][q])
        s._corr_keepalive = c          # the pointer below must outlive the call
        s.correction = C.pointer(c)
    return s


def mem_model_struct(g: Dict) -> MemModel:
    s = MemModel()
    s.struct_size = C.sizeof(MemModel)
    for k in ("ms_e", "as_e", "ms_l", "as_l"):
        setattr(s, k, mem_grid_struct(g[k]))
    s.mem_per_gpu = float(g["mem_per_gpu"])
    return s


def plan_struct(p: Dict) -> Plan:
    return Plan(*[int(p[k]) for k in ("e_tp", "e_pp", "e_dp", "l_tp", "l_pp", "l_dp", "n_mb")])


def _stream(stream) -> Optional[int]:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t) -> Optional[C.c_void_p]:
    return None if t is None else C.c_void_p(t.data_ptr())


def _u32(t):
    import torch
    assert t.dtype in (torch.int32, torch.uint32) and t.is_cuda and t.is_contiguous(), t.dtype
    return t


def _ticks(t):
    """[4][n] u32 cost ticks (int32/uint32, CUDA, contiguous: the C side reads rows n apart)."""
    _u32(t)
    assert t.dim() == 2 and t.shape[0] == 4, tuple(t.shape)
    return t


def _u64(t):
    import torch
    assert t.dtype in (torch.int64, torch.uint64) and t.is_cuda and t.is_contiguous(), t.dtype
    return t


# ---------------------------------------------------------------- API (same names as the C ABI)
# ---------------------------------------------------------------- sharding protocol (host)
def shard_range(K: int, rank: int, world: int):
    """Candidates [begin, end) of `rank` (dflop_shard_range; no GPU needed)."""
    b, e = C.c_uint32(), C.c_uint32()
    _check(lib().dflop_shard_range(K, rank, world, C.byref(b), C.byref(e)))
    return b.value, e.value


def owner_of(K: int, c: int, world: int) -> int:
    return lib().dflop_owner_of(K, c, world)


def pack_key(T: int, cand_id: int) -> int:
    return lib().dflop_pack_key(T, cand_id)


def select_plan(keys, P: int, D: int, batch_n: Optional[Sequence[int]] = None):
    """keys: P*D reduced u64 keys (plan-major).  Returns (win_p, objective[P])."""
    k = np.ascontiguousarray(np.asarray(keys, dtype=np.uint64))
    assert k.size == P * D
    obj = np.zeros(P, np.uint64)
    win = C.c_uint32()
    bn = None
    if batch_n is not None:
        bn = np.ascontiguousarray(np.asarray(batch_n, dtype=np.uint32))
    u64p, u32p = C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)
    _check(lib().dflop_select_plan(k.ctypes.data_as(u64p), P, D, bn.ctypes.data_as(u32p) if bn is not None else None,
                                   C.byref(win), obj.ctypes.data_as(u64p)))
    return win.value, obj


def abi_version() -> int:
    return int(lib().dflop_abi_version())


def profile_enable(on: bool = True):
    _check(lib().dflop_profile_enable(1 if on else 0))


def profile_read(reset: bool = True) -> Dict:
    """Synchronises the recorded candidate-kernel events; returns launches and device ms."""
    pr = Profile()
    pr.struct_size = C.sizeof(Profile)
    _check(lib().dflop_profile_read(C.byref(pr), 1 if reset else 0))
    return dict(cand_launches=pr.cand_launches, kernel_launches=pr.kernel_launches, cand_ms=pr.cand_ms,
                stage_a_launches=pr.stage_a_launches, stage_a_ms=pr.stage_a_ms,
                split_chunks=pr.split_chunks)


def predict_costs(model: Dict, plan: Dict, tiles, frames, text, want_f32: bool = True, dev_status=None, stream=None):
    """a1: returns (cost_f32 [4][n] float32 or None, cost_ticks [4][n] int32 (u32 bits))."""
    import torch
    n = tiles.numel()
    dev = tiles.device
    f32 = torch.empty((4, n), dtype=torch.float32, device=dev) if want_f32 else None
    ticks = torch.empty((4, n), dtype=torch.int32, device=dev)
    ms, ps = cost_model_struct(model), plan_struct(plan)
    _check(lib().dflop_predict_costs(C.byref(ms), C.byref(ps), _ptr(_u32(tiles)), _ptr(_u32(frames)),
                                     _ptr(_u32(text)), n, _ptr(f32), _ptr(ticks), _ptr(dev_status), _stream(stream)))
    return f32, ticks


class Workspace:
    """Grow-only device workspace (torch uint8, 256-byte aligned)."""

    def __init__(self):
        self.buf = None

    def get(self, nbytes: int, device):
        import torch
        if self.buf is None or self.buf.numel() < nbytes or self.buf.device != device:
            self.buf = torch.empty(max(nbytes, 256), dtype=torch.uint8, device=device)
        return self.buf


_default_ws = Workspace()


def balance_workspace_bytes(n: int, plan: Dict, K: int, R: int, G: int, c_begin: int = 0,
                            c_end: Optional[int] = None, mode: int = MODE_HEURISTIC) -> int:
    """The workspace dflop_balance_microbatches needs for this shape (its ws == NULL query)."""
    c_end = K if c_end is None else c_end
    bp = BalanceParams()
    bp.struct_size = C.sizeof(BalanceParams)
    bp.mode, bp.K, bp.cand_begin, bp.cand_end, bp.R, bp.G = mode, K, c_begin, c_end, R, G
    ps = plan_struct(plan)
    need = C.c_size_t(0)
    _check(lib().dflop_balance_microbatches(None, n, C.byref(ps), C.byref(bp), None, C.byref(need), None,
                                            None, None, None, None, None, None))
    return int(need.value)


def balance_microbatches(cost_ticks, plan: Dict, K: int, R: int, G: int, seed: Sequence[int], c_begin: int = 0,
                         c_end: Optional[int] = None, mode: int = MODE_HEURISTIC, id_base: int = 0,
                         want_assign: bool = True, want_groups: bool = False, per_candidate: bool = False,
                         ws: Optional[Workspace] = None, stream=None):
    """a2-a5 for one plan; returns dict with 'best' (CandResult tensor view), 'assign', 'groups', 'cand_T', ..."""
    import torch
    n = _ticks(cost_ticks).shape[1]
    dev = cost_ticks.device
    c_end = K if c_end is None else c_end
    bp = BalanceParams()
    bp.struct_size = C.sizeof(BalanceParams)
    bp.mode, bp.K, bp.cand_begin, bp.cand_end, bp.R, bp.G = mode, K, c_begin, c_end, R, G
    bp.seed[0], bp.seed[1] = int(seed[0]) & 0xFFFFFFFF, int(seed[1]) & 0xFFFFFFFF
    bp.id_base = id_base
    ps = plan_struct(plan)
    m = plan["n_mb"] * plan["l_dp"]
    need = C.c_size_t(0)
    L = lib()
    _check(L.dflop_balance_microbatches(_ptr(cost_ticks), n, C.byref(ps), C.byref(bp), None, C.byref(need), None,
                                        None, None, None, None, None, None))
    wsb = (ws or _default_ws).get(need.value, dev)
    best = torch.zeros(C.sizeof(CandResult), dtype=torch.uint8, device=dev)
    assign = torch.empty(max(n, 1), dtype=torch.int32, device=dev) if (want_assign or want_groups) else None
    offs = torch.empty(m + 1, dtype=torch.int32, device=dev) if want_groups else None
    items = torch.empty(max(n, 1), dtype=torch.int32, device=dev) if want_groups else None
    nc = c_end - c_begin
    cT = torch.empty(nc, dtype=torch.int64, device=dev) if per_candidate else None
    cC = torch.empty(nc, dtype=torch.int64, device=dev) if per_candidate else None
    have = C.c_size_t(wsb.numel())
    _check(L.dflop_balance_microbatches(_ptr(cost_ticks), n, C.byref(ps), C.byref(bp), _ptr(wsb), C.byref(have),
                                        _ptr(best), _ptr(assign), _ptr(offs), _ptr(items), _ptr(cT), _ptr(cC),
                                        _stream(stream)))
    return dict(best=best, assign=assign[:n] if assign is not None else None, offsets=offs,
                items=items[:n] if items is not None else None, cand_T=cT, cand_cmax=cC)


def cand_result(best_tensor) -> Dict:
    """Read a device CandResult (synchronises)."""
    raw = bytes(best_tensor.cpu().numpy().tobytes())
    r = CandResult.from_buffer_copy(raw)
    return dict(key=r.key, makespan=r.makespan, cmax=r.cmax, cand=r.cand, status=r.status)


def simulate_1f1b(fwd, bwd, want_busy: bool = True, stream=None):
    """fwd, bwd: int64 [C][S][M] (u64 ticks) -> (makespan [C], busy [C][S] or None)."""
    import torch
    _u64(fwd), _u64(bwd)
    assert fwd.shape == bwd.shape and fwd.dim() == 3, (tuple(fwd.shape), tuple(bwd.shape))
    Cn, S, M = fwd.shape
    out = torch.empty(Cn, dtype=torch.int64, device=fwd.device)
    busy = torch.empty((Cn, S), dtype=torch.int64, device=fwd.device) if want_busy else None
    _check(lib().dflop_simulate_1f1b(_ptr(fwd.contiguous()), _ptr(bwd.contiguous()), Cn, S, M, _ptr(out),
                                     _ptr(busy), _stream(stream)))
    return out, busy


def index_groups(assign, m: int, stream=None):
    import torch
    n = assign.numel()
    need = C.c_size_t(0)
    _check(lib().dflop_index_groups(None, n, m, None, None, None, C.byref(need), None))
    ws = torch.empty(max(need.value, 256), dtype=torch.uint8, device=assign.device)
    offs = torch.empty(m + 1, dtype=torch.int32, device=assign.device)
    items = torch.empty(max(n, 1), dtype=torch.int32, device=assign.device)
    have = C.c_size_t(ws.numel())
    _check(lib().dflop_index_groups(_ptr(assign), n, m, _ptr(offs), _ptr(items), _ptr(ws), C.byref(have),
                                    _stream(stream)))
    return offs, items[:n]


def search_plans(model: Dict, tiles, frames, text, K: int, R: int, G: int, seed: Sequence[int],
                 plan: Optional[Dict] = None, cluster: Optional[Dict] = None, mem: Optional[Dict] = None,
                 gbs: int = 0, top_p: int = 1, comm=None, want_assign: bool = True, stage_a_out=None,
                 ws: Optional[Workspace] = None, stream=None, order4: bool = False) -> Dict:
    """a1-a6 for one global batch (synchronous).  ``plan`` given -> FIXED mode; else Algorithm 1."""
    import torch
    n = tiles.numel()
    dev = tiles.device
    sp = SearchParams()
    sp.struct_size = C.sizeof(SearchParams)
    sp.mode = (SEARCH_FIXED if plan is not None else SEARCH_ALG1) | (MODE_ORDER4 if order4 else 0)
    if plan is not None:
        sp.fixed_plan = plan_struct(plan)
    sp.gbs, sp.top_p, sp.K, sp.R, sp.G = gbs, top_p, K, R, G
    sp.seed[0], sp.seed[1] = int(seed[0]) & 0xFFFFFFFF, int(seed[1]) & 0xFFFFFFFF
    ms = cost_model_struct(model)
    cl = Cluster()
    mm = MemModel()
    if cluster is not None:
        cl.struct_size = C.sizeof(Cluster)
        cl.n_gpus, cl.gpus_per_node = cluster["n_gpus"], cluster["gpus_per_node"]
    if mem is not None:
        mm = mem_model_struct(mem)
    cptr = C.c_void_p(comm.handle) if comm is not None else None
    need = C.c_size_t(0)
    L = lib()
    out = PlanResult()
    _check(L.dflop_search_plans(C.byref(cl), C.byref(ms), C.byref(mm), _ptr(tiles), _ptr(frames), _ptr(text), n,
                                C.byref(sp), cptr, None, C.byref(need), C.byref(out), None, None, 0, None))
    wsb = (ws or _default_ws).get(need.value, dev)
    assign = torch.empty(max(n, 1), dtype=torch.int32, device=dev) if want_assign else None
    have = C.c_size_t(wsb.numel())
    cap = stage_a_out.numel() if stage_a_out is not None else 0
    _check(L.dflop_search_plans(C.byref(cl), C.byref(ms), C.byref(mm), _ptr(_u32(tiles)), _ptr(_u32(frames)),
                                _ptr(_u32(text)), n, C.byref(sp), cptr, _ptr(wsb), C.byref(have), C.byref(out),
                                _ptr(assign), _ptr(stage_a_out), cap, _stream(stream)))
    r = {f: getattr(out, f) for f, _ in PlanResult._fields_ if f not in ("plan", "alg1_plan", "reserved")}
    r["plan"] = out.plan.as_dict()
    r["alg1_plan"] = out.alg1_plan.as_dict()
    r["assign"] = assign[:n] if assign is not None else None
    return r


def exact_cmax(cost_ticks, plan: Dict, node_budget: int = 10 ** 9, init_assign=None,
               ws: Optional[Workspace] = None, stream=None) -> Dict:
    """N3: exact C_max by branch and bound (synchronous).  Returns the dflop_exact_result
    fields and 'assign' (device int32 [n])."""
    import torch
    n = _ticks(cost_ticks).shape[1]
    dev = cost_ticks.device
    ps = plan_struct(plan)
    L = lib()
    need = C.c_size_t(0)
    out = ExactResult()
    _check(L.dflop_exact_cmax(_ptr(cost_ticks), n, C.byref(ps), C.c_uint64(int(node_budget)), None, None,
                              C.byref(need), C.byref(out), None, None))
    wsb = (ws or _default_ws).get(need.value, dev)
    have = C.c_size_t(wsb.numel())
    assign = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    _check(L.dflop_exact_cmax(_ptr(cost_ticks), n, C.byref(ps), C.c_uint64(int(node_budget)),
                              _ptr(_u32(init_assign)) if init_assign is not None else None, _ptr(wsb), C.byref(have),
                              C.byref(out), _ptr(assign), _stream(stream)))
    r = {f: getattr(out, f) for f, _ in ExactResult._fields_ if f not in ("struct_size", "reserved")}
    r["proven"] = bool(r["proven"])
    r["searched"] = bool(r["searched"])
    r["assign"] = assign[:n]
    return r


def order_search(cost_ticks, plan: Dict, assign, rounds: int = 64, ws: Optional[Workspace] = None,
                 stream=None) -> Dict:
    """N4(a): per replica the improved slot order (bucket per slot) and its 1F1B makespan."""
    import torch
    n = _ticks(cost_ticks).shape[1]
    dev = cost_ticks.device
    ps = plan_struct(plan)
    L = lib()
    need = C.c_size_t(0)
    _check(L.dflop_order_search(_ptr(cost_ticks), n, C.byref(ps), _ptr(_u32(assign)), rounds, None, C.byref(need), None,
                                None, None))
    wsb = (ws or _default_ws).get(need.value, dev)
    have = C.c_size_t(wsb.numel())
    M, rep = int(plan["n_mb"]), int(plan["l_dp"])
    order = torch.empty(rep * M, dtype=torch.int32, device=dev)
    T = np.zeros(rep, np.uint64)
    _check(L.dflop_order_search(_ptr(cost_ticks), n, C.byref(ps), _ptr(_u32(assign)), rounds, _ptr(wsb), C.byref(have),
                                _ptr(order), T.ctypes.data_as(C.c_void_p), _stream(stream)))
    return dict(order=order.view(rep, M), T=T, makespan=int(T.max()) if rep else 0)


def route_plan(cost_ticks, plan: Dict, assign, ws: Optional[Workspace] = None, stream=None) -> Dict:
    """N4(b): the inter-model communicator's routing plan (device tensors)."""
    import torch
    n = _ticks(cost_ticks).shape[1]
    dev = cost_ticks.device
    ps = plan_struct(plan)
    L = lib()
    need = C.c_size_t(0)
    _check(L.dflop_route_plan(_ptr(cost_ticks), n, C.byref(ps), _ptr(_u32(assign)), None, C.byref(need), None, None, None,
                              None, None, None))
    wsb = (ws or _default_ws).get(need.value, dev)
    have = C.c_size_t(wsb.numel())
    M, R, G = int(plan["n_mb"]), int(plan["l_dp"]), int(plan["e_dp"])
    pos = torch.empty(max(n, 1), dtype=torch.int32, device=dev)
    so = torch.empty(M + 1, dtype=torch.int32, device=dev)
    eo = torch.empty(M * (G + 1), dtype=torch.int32, device=dev)
    lo = torch.empty(M * (R + 1), dtype=torch.int32, device=dev)
    el = torch.empty(M * G, dtype=torch.int64, device=dev)
    _check(L.dflop_route_plan(_ptr(cost_ticks), n, C.byref(ps), _ptr(_u32(assign)), _ptr(wsb), C.byref(have), _ptr(pos),
                              _ptr(so), _ptr(eo), _ptr(lo), _ptr(el), _stream(stream)))
    return dict(pos_item=pos[:n], slot_off=so, enc_off=eo.view(M, G + 1), llm_off=lo.view(M, R + 1),
                enc_load=el.view(M, G))


def search_plans_batches(model: Dict, tiles, frames, text, batch_offsets: Sequence[int], K: int, R: int, G: int,
                         seed: Sequence[int], plan: Optional[Dict] = None, cluster: Optional[Dict] = None,
                         mem: Optional[Dict] = None, gbs: int = 0, top_p: int = 1, comm=None,
                         want_assign: bool = True, ws: Optional[Workspace] = None, stream=None,
                         order4: bool = False) -> Dict:
    """N2, Eq. (1) over a sample of D batches (synchronous): batch b = samples
    [batch_offsets[b], batch_offsets[b+1]) of the concatenated features; its family uses
    Philox key (seed[0], seed[1] + b).  Returns the dflop_plan_result fields (makespan =
    sum_b T_B(b) of theta*), 'batches' (per-batch winners), 'plan_objective' and 'assign'."""
    import torch
    offs = np.ascontiguousarray(np.asarray(batch_offsets, np.uint32))
    D = len(offs) - 1
    n = int(offs[-1] - offs[0])
    dev = tiles.device
    sp = SearchParams()
    sp.struct_size = C.sizeof(SearchParams)
    sp.mode = (SEARCH_FIXED if plan is not None else SEARCH_ALG1) | (MODE_ORDER4 if order4 else 0)
    if plan is not None:
        sp.fixed_plan = plan_struct(plan)
    sp.gbs, sp.top_p, sp.K, sp.R, sp.G = gbs, top_p, K, R, G
    sp.seed[0], sp.seed[1] = int(seed[0]) & 0xFFFFFFFF, int(seed[1]) & 0xFFFFFFFF
    ms = cost_model_struct(model)
    cl = Cluster()
    mm = MemModel()
    if cluster is not None:
        cl.struct_size = C.sizeof(Cluster)
        cl.n_gpus, cl.gpus_per_node = cluster["n_gpus"], cluster["gpus_per_node"]
    if mem is not None:
        mm = mem_model_struct(mem)
    cptr = C.c_void_p(comm.handle) if comm is not None else None
    L = lib()
    op = offs.ctypes.data_as(C.c_void_p)
    need = C.c_size_t(0)
    out = PlanResult()
    _check(L.dflop_search_plans_batches(C.byref(cl), C.byref(ms), C.byref(mm), _ptr(tiles), _ptr(frames), _ptr(text),
                                        op, D, C.byref(sp), cptr, None, C.byref(need), C.byref(out), None, None,
                                        None, None, None))
    wsb = (ws or _default_ws).get(need.value, dev)
    assign = torch.empty(max(n, 1), dtype=torch.int32, device=dev) if want_assign else None
    have = C.c_size_t(wsb.numel())
    bres = (CandResult * D)()
    P = top_p if plan is None else 1
    pobj = np.zeros(P, np.uint64)
    plans = (Plan * P)()
    _check(L.dflop_search_plans_batches(C.byref(cl), C.byref(ms), C.byref(mm), _ptr(_u32(tiles)), _ptr(_u32(frames)),
                                        _ptr(_u32(text)), op, D, C.byref(sp), cptr, _ptr(wsb), C.byref(have),
                                        C.byref(out), bres, pobj.ctypes.data_as(C.c_void_p), plans, _ptr(assign),
                                        _stream(stream)))
    r = {f: getattr(out, f) for f, _ in PlanResult._fields_ if f not in ("plan", "alg1_plan", "reserved")}
    r["plan"] = out.plan.as_dict()
    r["alg1_plan"] = out.alg1_plan.as_dict()
    r["batches"] = [dict(key=b.key, makespan=b.makespan, cmax=b.cmax, cand=b.cand, status=b.status) for b in bres]
    r["plan_objective"] = pobj
    r["plans"] = [pl.as_dict() for pl in plans]
    r["assign"] = assign[:n] if assign is not None else None
    return r


class Comm:
    """NCCL communicator owned by libdflop; the 128-byte id is broadcast with torch.distributed."""

    def __init__(self, rank: int, world: int, device: int, pg=None):
        import torch
        import torch.distributed as dist
        buf = C.create_string_buffer(128)
        if rank == 0:
            _check(lib().dflop_get_unique_id(buf))
        t = torch.tensor(list(buf.raw), dtype=torch.uint8)
        if dist.get_backend(pg) == "nccl":
            t = t.cuda(device)
        dist.broadcast(t, 0, group=pg)
        raw = bytes(t.cpu().tolist())
        h = C.c_void_p()
        _check(lib().dflop_comm_init(raw, rank, world, device, C.byref(h)))
        self.handle = h.value
        self.rank, self.world = rank, world

    def close(self):
        if self.handle:
            _check(lib().dflop_comm_destroy(C.c_void_p(self.handle)))
            self.handle = None
