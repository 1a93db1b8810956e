"""N1 Adaptive Correction on the GPU: k_predict with an active correction table against the
oracle's corrected a1 (orc_predict_corrected), and end to end through dflop_search_plans.
Tolerances as for a1.  -m gpu."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2603_25120_b200.correction import CorrectionTracker, shape_bin  # noqa: E402


@pytest.fixture(scope="module")
def D():
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    from paper_2603_25120_b200 import dflop
    dflop.lib()
    return dflop


def dev_u32(a):
    return torch.from_numpy(np.ascontiguousarray(a).astype(np.uint32).view(np.int32)).cuda()


def host_u32(t):
    return t.cpu().numpy().view(np.uint32)


def random_rho(seed):
    rng = np.random.default_rng(seed)
    return np.clip(rng.lognormal(0.0, 0.4, (3, 32)), 0.3, 3.0).astype(np.float32)


@pytest.mark.parametrize("k", [1, 2, 3, 5])
def test_corrected_predict_parity(D, O, presets, k):
    p = presets[k]
    rho = random_rho(k)
    model = dict(p.model, correction={"active": True, "rho": rho})
    for b in (0, 2):
        t, f, x = p.features(b)
        cf64, cq, st, _ = O.predict_corrected(p.model, p.plan, t, f, x, rho.astype(np.float64))
        assert st == 0
        f32, ticks = D.predict_costs(model, p.plan, dev_u32(t), dev_u32(f), dev_u32(x))
        g = f32.cpu().numpy().astype(np.float64)
        ref = cf64 / p.model["tick_ns"]
        assert np.all((ref == 0) == (g == 0))
        rel = np.abs(g - ref) / np.maximum(ref, 1e-300)
        assert rel.max() <= 1e-5, rel.max()
        q = host_u32(ticks).astype(np.int64)
        assert np.all(np.abs(q - cq.astype(np.int64)) <= 1 + 1e-5 * cq)
        # the table changed something (the test is not vacuous)
        base, _, _, _ = O.predict(p.model, p.plan, t, f, x)
        assert (np.abs(cf64 - base) > 1e-6 * base).any()


def test_inactive_table_is_the_uncorrected_path(D, presets):
    p = presets[5]
    t, f, x = (dev_u32(a) for a in p.features(1))
    a32, aq = D.predict_costs(p.model, p.plan, t, f, x)
    model = dict(p.model, correction={"active": False, "rho": random_rho(9)})
    b32, bq = D.predict_costs(model, p.plan, t, f, x)
    assert torch.equal(a32, b32) and torch.equal(aq, bq)


def test_halved_encoder_throughput_doubles_duration(D, presets):
    # S:386 through the tracker: one observation at half the predicted throughput
    p = presets[3]
    t, f, x = p.features(0)
    b = t.astype(np.int64) + f
    xb = int(b.max())
    tr = CorrectionTracker()
    tr.record_observation("thr_e", xb, 0.5e12, 1e12)
    model = dict(p.model, correction=tr.table())
    a32, _ = D.predict_costs(p.model, p.plan, dev_u32(t), dev_u32(f), dev_u32(x))
    c32, _ = D.predict_costs(model, p.plan, dev_u32(t), dev_u32(f), dev_u32(x))
    a, c = a32.cpu().numpy(), c32.cpu().numpy()
    hit = np.array([bb > 0 and shape_bin(bb) == shape_bin(xb) for bb in b])
    assert hit.any() and not hit.all()
    assert (c[0, hit] == 2 * a[0, hit]).all()            # reciprocal of a halved value: exact in fp32
    assert (c[0, ~hit] == a[0, ~hit]).all() and (c[2:] == a[2:]).all()


def test_corrected_search_equals_oracle_balance(D, O, presets):
    # a1 with the correction feeds a2..a5 unchanged: the search's winner equals the oracle's
    # balance of the GPU's corrected costs (shared integer array, bit-exact)
    p = presets[2]
    model = dict(p.model, correction={"active": True, "rho": random_rho(4)})
    t, f, x = (dev_u32(a) for a in p.features(0))
    res = D.search_plans(model, t, f, x, K=2048, R=p.R, G=p.G, seed=p.seed(0), plan=p.plan)
    _, ticks = D.predict_costs(model, p.plan, t, f, x, want_f32=False)
    o = O.balance_threaded(host_u32(ticks), p.plan, 2048, p.R, p.G, p.seed(0), per_candidate=False)
    assert res["makespan"] == o["T"] and res["cand"] == o["c"] and res["cmax"] == o["cmax"]
    _, plain = D.predict_costs(p.model, p.plan, t, f, x, want_f32=False)
    assert not torch.equal(plain, ticks)


def test_invalid_correction_rejected(D, presets):
    p = presets[2]
    rho = np.ones((3, 32), np.float32)
    rho[1, 3] = 0.0
    model = dict(p.model, correction={"active": True, "rho": rho})
    t, f, x = (dev_u32(a) for a in p.features(0))
    with pytest.raises(Exception, match="rho"):
        D.predict_costs(model, p.plan, t, f, x)
