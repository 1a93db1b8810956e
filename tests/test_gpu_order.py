"""N4(a) microbatch-order search on the GPU (dflop_order_search) against
orc_order_search: bit-exact orders and makespans (same start orders, neighbourhood and
tie rules).  -m gpu."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu


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


def test_random_assignments(D, O):
    rng = np.random.default_rng(21)
    for trial in range(12):
        n_mb, l_dp = int(rng.integers(1, 12)), int(rng.integers(1, 4))
        e_pp, l_pp = int(rng.integers(1, 4)), int(rng.integers(1, 5))
        pl = dict(e_tp=1, e_pp=e_pp, e_dp=1, l_tp=1, l_pp=l_pp, l_dp=l_dp, n_mb=n_mb)
        m, n = n_mb * l_dp, int(rng.integers(1, 80))
        c = rng.integers(0, 500, (4, n)).astype(np.uint32)
        a = rng.integers(0, m, n).astype(np.uint32)
        g = D.order_search(dev_u32(c), pl, dev_u32(a), rounds=32)
        o_ord, o_T = O.order_search(c, pl, a, rounds=32)
        assert (host_u32(g["order"]).reshape(l_dp, n_mb) == o_ord).all(), trial
        assert (g["T"] == o_T).all(), trial


@pytest.mark.parametrize("k", [2, 3, 5])
def test_preset_winners(D, O, presets, k):
    # the search winner's slot order improved; equal to the oracle, never worse than identity
    p = presets[k]
    t, f, x = (dev_u32(v) for v in p.features(0))
    res = D.search_plans(p.model, t, f, x, K=512, R=p.R, G=p.G, seed=p.seed(0), plan=p.plan)
    _, ticks = D.predict_costs(p.model, p.plan, t, f, x, want_f32=False)
    rounds = 8 if k == 5 else 32
    g = D.order_search(ticks, p.plan, res["assign"], rounds=rounds)
    q = host_u32(ticks).reshape(4, -1)
    o_ord, o_T = O.order_search(q, p.plan, host_u32(res["assign"]), rounds=rounds)
    assert (host_u32(g["order"]).reshape(o_ord.shape) == o_ord).all() and (g["T"] == o_T).all()
    assert g["makespan"] <= res["makespan"]


def test_large_nmb_banded(D, O, presets):
    # N_mb > 128: the distance-16 neighbourhood
    rng = np.random.default_rng(4)
    pl = dict(e_tp=1, e_pp=1, e_dp=1, l_tp=1, l_pp=2, l_dp=1, n_mb=150)
    n = 600
    c = rng.integers(1, 1000, (4, n)).astype(np.uint32)
    a = (np.arange(n) % 150).astype(np.uint32)
    g = D.order_search(dev_u32(c), pl, dev_u32(a), rounds=4)
    o_ord, o_T = O.order_search(c, pl, a, rounds=4)
    assert (host_u32(g["order"]).reshape(o_ord.shape) == o_ord).all() and (g["T"] == o_T).all()
