"""Pure-Python brute force for tiny instances -- a third implementation, independent of
both the C oracle and the CUDA path (TEST INFRASTRUCTURE).

* ``dag_makespan``: the non-interleaved 1F1B schedule (Fig. 1) written as an
  explicit DAG (same-stage order edges + cross-stage dependency edges) and solved
  as a longest path with Kahn's algorithm -- a different algorithm from the
  oracle's worklist sweep and the GPU's precomputed slot order.
* ``all_assignments``: every one of the m^n item -> bucket maps, scored with the
  objective of P:715 (C_max) and with the 1F1B makespan of ``dag_makespan``.
* ``lpt_1d`` / ``opt_cmax_1d``: Graham's LPT and the exact optimum for
  one-dimensional loads.
"""
from __future__ import annotations

import itertools
from collections import deque
from typing import Dict, List, Sequence, Tuple


def stage_ops(s: int, S: int, M: int) -> List[Tuple[str, int]]:
    """Megatron non-interleaved 1F1B op order on stage s (R9)."""
    w = min(S - 1 - s, M)
    ops = [("F", k) for k in range(w)]
    for q in range(M - w):
        ops.append(("F", w + q))
        ops.append(("B", q))
    ops += [("B", k) for k in range(M - w, M)]
    return ops


def dag_makespan(F: Sequence[Sequence[int]], B: Sequence[Sequence[int]]) -> int:
    S, M = len(F), len(F[0])
    nodes = [(kind, s, k) for s in range(S) for kind in "FB" for k in range(M)]
    dur = {(kind, s, k): (F[s][k] if kind == "F" else B[s][k]) for (kind, s, k) in nodes}
    succ: Dict[tuple, list] = {v: [] for v in nodes}
    indeg = {v: 0 for v in nodes}

    def edge(a, b):
        succ[a].append(b)
        indeg[b] += 1

    for s in range(S):
        ops = stage_ops(s, S, M)
        for a, b in zip(ops, ops[1:]):
            edge((a[0], s, a[1]), (b[0], s, b[1]))
        for k in range(M):
            if s > 0:
                edge(("F", s - 1, k), ("F", s, k))
            if s < S - 1:
                edge(("B", s + 1, k), ("B", s, k))
            else:
                edge(("F", s, k), ("B", s, k))
    # longest path: finish(v) = dur(v) + max over predecessors finish
    start = {v: 0 for v in nodes}
    q = deque(v for v in nodes if indeg[v] == 0)
    seen = 0
    best = 0
    while q:
        v = q.popleft()
        seen += 1
        fin = start[v] + dur[v]
        best = max(best, fin)
        for w in succ[v]:
            start[w] = max(start[w], fin)
            indeg[w] -= 1
            if indeg[w] == 0:
                q.append(w)
    assert seen == len(nodes), "cycle"
    return best


def score_assignment(assign: Sequence[int], cost, plan: Dict) -> Tuple[int, int]:
    """(T, C_max) of a partition: buckets j -> replica j % L_dp, slot j // L_dp (R10)."""
    n = len(assign)
    m = plan["n_mb"] * plan["l_dp"]
    EF, EB, LF, LB = ([0] * m for _ in range(4))
    for i, j in enumerate(assign):
        EF[j] += int(cost[0][i]); EB[j] += int(cost[1][i])
        LF[j] += int(cost[2][i]); LB[j] += int(cost[3][i])
    S = plan["e_pp"] + plan["l_pp"]
    T = 0
    for rho in range(plan["l_dp"]):
        F = [[(EF if s < plan["e_pp"] else LF)[k * plan["l_dp"] + rho] for k in range(plan["n_mb"])] for s in range(S)]
        Bm = [[(EB if s < plan["e_pp"] else LB)[k * plan["l_dp"] + rho] for k in range(plan["n_mb"])] for s in range(S)]
        T = max(T, dag_makespan(F, Bm))
    cmax = max(max(EF[j] + EB[j], LF[j] + LB[j]) for j in range(m))
    return T, cmax


def all_assignments(cost, plan: Dict):
    """Yield (index, assign, T, C_max) for all m^n maps, index = sum a_i m^i."""
    n = len(cost[0])
    m = plan["n_mb"] * plan["l_dp"]
    for idx in range(m ** n):
        x, a = idx, []
        for _ in range(n):
            a.append(x % m)
            x //= m
        T, cm = score_assignment(a, cost, plan)
        yield idx, a, T, cm


def lpt_1d(loads: Sequence[int], m: int) -> Tuple[List[List[int]], int]:
    order = sorted(range(len(loads)), key=lambda i: (-loads[i], i))
    bins = [[] for _ in range(m)]
    sums = [0] * m
    for i in order:
        j = min(range(m), key=lambda j: (sums[j], j))
        bins[j].append(loads[i])
        sums[j] += loads[i]
    return bins, max(sums)


def opt_cmax_1d(loads: Sequence[int], m: int) -> int:
    best = None
    for a in itertools.product(range(m), repeat=len(loads)):
        sums = [0] * m
        for x, j in zip(loads, a):
            sums[j] += x
        v = max(sums)
        best = v if best is None else min(best, v)
    return best


def opt_cmax_2d(cost, m: int) -> int:
    """min over all m^n assignments of max_j max(E_j, L_j), E = ef + eb, L = lf + lb."""
    n = len(cost[0])
    e = [int(cost[0][i]) + int(cost[1][i]) for i in range(n)]
    l = [int(cost[2][i]) + int(cost[3][i]) for i in range(n)]
    best = None
    for a in itertools.product(range(m), repeat=n):
        E, L = [0] * m, [0] * m
        for i, j in enumerate(a):
            E[j] += e[i]
            L[j] += l[i]
        v = max(max(E), max(L))
        best = v if best is None else min(best, v)
    return best


def cmax_of(assign, cost, m: int) -> int:
    E, L = [0] * m, [0] * m
    for i, j in enumerate(assign):
        E[j] += int(cost[0][i]) + int(cost[1][i])
        L[j] += int(cost[2][i]) + int(cost[3][i])
    return max(max(E), max(L))
