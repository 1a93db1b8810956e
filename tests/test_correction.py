"""N1 Adaptive Correction host tracker (paper_2603_25120_b200/correction.py) against SPEC's
worked examples and the oracle's shape bins.  -m "not gpu"."""
import numpy as np
import pytest

from paper_2603_25120_b200.correction import CorrectionTracker, shape_bin


def test_shape_bin_matches_oracle(O):
    for x in list(range(0, 70)) + [1023, 1024, 4095, 4096, 65535, 1 << 33, (1 << 40) - 1]:
        assert shape_bin(x) == O.shape_bin(x), x


def test_eq6_zero_and_half():
    tr = CorrectionTracker()
    assert tr.record_observation("thr_e", 5, 100.0, 100.0) == 0.0           # S:422 actual = predicted
    assert tr.rho()[0, shape_bin(5)] == 1.0
    tr = CorrectionTracker()
    assert tr.record_observation("thr_att", 300, 50.0, 100.0) == -50.0      # S:423 B = -0.5 pred
    assert tr.rho()[1, shape_bin(300)] == 0.5
    assert (np.delete(tr.rho().ravel(), 1 * 32 + shape_bin(300)) == 1.0).all()


def test_exponential_average_converges():
    tr = CorrectionTracker(alpha=0.25)
    tr.record_observation(2, 4096, 10.0, 20.0)
    for _ in range(200):                                                  # S:424 fixed point
        tr.record_observation(2, 5000, 30.0, 20.0)                        # same bin as 4096
    assert abs(tr.observed[2, shape_bin(4096)] - 30.0) < 1e-12
    assert abs(tr.deviation(2, 4096) - 10.0) < 1e-12


@pytest.mark.parametrize("mean_b, C, active", [(3.0, 5.0, False), (5.0, 3.0, True), (4.0, 4.0, False)])
def test_cost_benefit_rule(mean_b, C, active):
    tr = CorrectionTracker(window=3, cost=C)
    assert tr.cost_benefit_step([mean_b - 1, mean_b, mean_b + 1]) is active


def test_deactivation_is_permanent_and_table():
    tr = CorrectionTracker(window=2, cost=1.0)
    assert tr.cost_benefit_step([0.5]) is True                            # fewer than I samples
    assert tr.cost_benefit_step([0.5]) is False
    assert tr.cost_benefit_step([9.0, 9.0]) is False                      # stays off
    t = tr.table()
    assert t["active"] is False and t["rho"].shape == (3, 32) and t["rho"].dtype == np.float32


# ---------------------------------------------------------------- oracle twin (oracle/orc_tracker_*)
def test_oracle_tracker_spec_examples(O):
    """The oracle's tracker, written separately from SPEC S:420-438, on the same pins."""
    t = O.Tracker()
    assert t.record(0, 5, 100.0, 100.0) == 0.0
    t = O.Tracker()
    assert t.record(1, 300, 50.0, 100.0) == -50.0
    assert t.rho()[1, O.shape_bin(300)] == 0.5
    t = O.Tracker(window=3, cost=4.0)
    assert t.cost_benefit([3.0, 4.0, 5.0]) is False                        # mean 4 > 4 is false (strict)
    t = O.Tracker(window=2, cost=1.0)
    assert t.cost_benefit([0.5]) is True and t.cost_benefit([0.5]) is False and t.cost_benefit([9, 9]) is False


def test_product_tracker_matches_oracle_twin(O):
    """Random observation and benefit sequences: the product's host tracker and the oracle's
    twin agree on every deviation B (Eq. (6)), the rho table and the active flag."""
    rng = np.random.default_rng(3)
    for trial in range(20):
        alpha = float(rng.uniform(0.05, 1.0))
        I = int(rng.integers(1, 8))
        Ccost = float(rng.uniform(0, 5))
        tr, tw = CorrectionTracker(alpha=alpha, window=I, cost=Ccost), O.Tracker(alpha, I, Ccost)
        for step in range(300):
            g = int(rng.integers(0, 3))
            x = int(rng.integers(0, 1 << int(rng.integers(1, 34))))
            a, pr = float(rng.uniform(1e12, 3e14)), float(rng.uniform(1e12, 3e14))
            assert tr.record_observation(g, x, a, pr) == pytest.approx(tw.record(g, x, a, pr), rel=1e-15, abs=1e-3)
            if step % 25 == 24:
                ben = rng.normal(Ccost, 2.0, size=int(rng.integers(0, 4))).tolist()
                assert tr.cost_benefit_step(ben) is tw.cost_benefit(ben)
        assert np.allclose(tr.rho(), tw.rho(), rtol=1e-14, atol=0)
