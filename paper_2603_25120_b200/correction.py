"""N1 Adaptive Correction: the host-side tracker that feeds a1's correction table.

Paper: throughput of rare input shapes deviates from the interpolated profile;
the system tracks B = Th_actual - Th_pred (Eq. (6)) per input shape, feeds a penalty
function to the scheduler (here: the ratio rho = Th_actual / Th_pred that a1 multiplies into
the predicted throughput of the sample's shape bin, include/dflop.h `dflop_correction`),
and switches tracking off when the average benefit over I iterations does not exceed the
recurring cost C.  SPEC fixes the operations: record_observation
(exponential average of the observed throughput per shape bucket), cost_benefit_step
(active <- mean of the last I benefits > C, strict; deactivation is permanent).

Readings: shape bucket = (grid, floor(log2 x)) with x the encoder batch
b for thr_e and the LLM length s for thr_att / thr_lin (R30); exponential-average weight
alpha (default 0.25) is a parameter (R32).  Only host bookkeeping lives here; the lookup is
one shared-memory read per sample and grid inside k_predict.
"""
from __future__ import annotations

from typing import Dict, Iterable, List, Optional

import numpy as np

GRIDS = ("thr_e", "thr_att", "thr_lin")
BINS = 32


def shape_bin(x: int) -> int:
    """floor(log2 x) of an integer shape; x = 0 is bin 0; clamped to BINS - 1 (R30)."""
    x = int(x)
    return 0 if x <= 0 else min(BINS - 1, x.bit_length() - 1)


class CorrectionTracker:
    """Per (grid, shape bin): the exponentially averaged observed throughput, the latest
    prediction, the deviation B (Eq. (6)) and the correction ratio rho."""

    def __init__(self, alpha: float = 0.25, window: int = 10, cost: float = 0.0):
        if not 0.0 < alpha <= 1.0:
            raise ValueError("alpha must be in (0, 1]")
        if window < 1:
            raise ValueError("window I must be >= 1")
        self.alpha, self.window, self.cost = float(alpha), int(window), float(cost)
        self.observed = np.zeros((3, BINS))
        self.predicted = np.zeros((3, BINS))
        self.seen = np.zeros((3, BINS), bool)
        self.active = True
        self.benefits: List[float] = []

    @staticmethod
    def _grid(grid) -> int:
        return GRIDS.index(grid) if isinstance(grid, str) else int(grid)

    def record_observation(self, grid, x: int, th_actual: float, th_pred: float) -> float:
        """S:420 record_observation; returns the bucket's deviation B = Th_actual - Th_pred."""
        if not (th_actual > 0 and th_pred > 0):
            raise ValueError("throughputs must be > 0")
        g, q = self._grid(grid), shape_bin(x)
        if self.seen[g, q]:
            self.observed[g, q] = (1.0 - self.alpha) * self.observed[g, q] + self.alpha * th_actual
        else:
            self.observed[g, q] = th_actual
            self.seen[g, q] = True
        self.predicted[g, q] = th_pred
        return self.deviation(g, x)

    def deviation(self, grid, x: int) -> float:
        g, q = self._grid(grid), shape_bin(x)
        return float(self.observed[g, q] - self.predicted[g, q]) if self.seen[g, q] else 0.0

    def rho(self) -> np.ndarray:
        """Th_actual / Th_pred per bucket (1 where nothing was recorded)."""
        r = np.ones((3, BINS))
        r[self.seen] = self.observed[self.seen] / self.predicted[self.seen]
        return r

    def cost_benefit_step(self, realized_benefits: Iterable[float], cost: Optional[float] = None,
                          window: Optional[int] = None) -> bool:
        """S:431 cost_benefit_step: active <- mean(last I realized benefits) > C (strict);
        once off, tracking stays off for the run."""
        self.benefits.extend(float(b) for b in realized_benefits)
        I = self.window if window is None else int(window)
        C = self.cost if cost is None else float(cost)
        if self.active and len(self.benefits) >= I:
            self.active = float(np.mean(self.benefits[-I:])) > C
        return self.active

    def table(self) -> Dict:
        """The cost-model entry for include/dflop.h `dflop_correction` (model["correction"])."""
        return {"active": bool(self.active), "rho": self.rho().astype(np.float32)}
