"""N3 exact C_max on the GPU (dflop_exact_cmax, parallel branch and bound) against the
oracle's branch and bound and brute force: the optimum value is unique, so proven results
must agree exactly; every returned assignment must have the returned C_max; its 1F1B
makespan must equal the oracle's score of that assignment.  -m gpu."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

import bruteforce as BF  # noqa: E402


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


def plan(n_mb, l_dp=1, e_pp=1, l_pp=1):
    return dict(e_tp=1, e_pp=e_pp, e_dp=1, l_tp=1, l_pp=l_pp, l_dp=l_dp, n_mb=n_mb)


def test_random_small_vs_bruteforce_and_oracle(D, O):
    rng = np.random.default_rng(12)
    for trial in range(30):
        n, m = int(rng.integers(1, 9)), int(rng.integers(1, 4))
        c = rng.integers(0, 50, (4, n)).astype(np.uint32)
        pl = plan(m)
        g = D.exact_cmax(dev_u32(c), pl, node_budget=10 ** 8)
        o = O.exact_cmax(c, m)
        opt = BF.opt_cmax_2d(c, m)
        assert g["proven"] and o["proven"] and g["cmax"] == o["cmax"] == opt, (trial, g, o["cmax"], opt)
        a = host_u32(g["assign"])
        assert BF.cmax_of(a, c, m) == g["cmax"] and g["lower_bound"] == o["lb"]
        T, cm = BF.score_assignment(a, c, pl)
        assert g["makespan"] == T and cm == g["cmax"]


@pytest.mark.parametrize("n, m, seed", [(14, 3, 1), (18, 4, 2), (22, 2, 3), (12, 5, 4)])
def test_medium_instances_vs_oracle(D, O, n, m, seed):
    rng = np.random.default_rng(seed)
    c = rng.integers(1, 10_000, (4, n)).astype(np.uint32)
    o = O.exact_cmax(c, m, node_budget=10 ** 9)
    g = D.exact_cmax(dev_u32(c), plan(m), node_budget=10 ** 10)
    assert o["proven"] and g["proven"] and g["cmax"] == o["cmax"]
    assert BF.cmax_of(host_u32(g["assign"]), c, m) == g["cmax"]


@pytest.mark.parametrize("m", [2, 4])
def test_pair_decomposition_vs_oracle(D, O, m):
    """m = 2, 4: the GPU's exhaustive pair decomposition equals the oracle's (orc_exact_pairs)
    and brute force; proven."""
    rng = np.random.default_rng(100 + m)
    for trial in range(12):
        n = int(rng.integers(1, 9)) if trial < 8 else int(rng.integers(12, 25))
        c = rng.integers(0, 60 if trial < 8 else 50_000, (4, n)).astype(np.uint32)
        g = D.exact_cmax(dev_u32(c), plan(m), node_budget=1 << 40)
        o = O.exact_pairs(c, m)
        assert g["proven"] and g["cmax"] == o["cmax"], (trial, n, g, o["cmax"])
        if n <= 8:
            assert g["cmax"] == BF.opt_cmax_2d(c, m)
        a = host_u32(g["assign"])
        assert BF.cmax_of(a, c, m) == g["cmax"] and g["lower_bound"] == o["lb"]


def test_config1_certificate(D, O, presets):
    """N3 certificate for config 1 (n = 32, m = 4): the pair decomposition proves
    the optimum C_max of batch 0 -- the oracle's exhaustive decomposition gives the same value
    -- and the returned assignment attains it."""
    p = presets[1]
    _, ticks = D.predict_costs(p.model, p.plan, *(dev_u32(a) for a in p.features(0)), want_f32=False)
    q = host_u32(ticks).reshape(4, -1)
    g = D.exact_cmax(ticks, p.plan, node_budget=1 << 40)
    assert g["proven"] == 1
    o = O.exact_pairs(q, 4)
    assert g["cmax"] == o["cmax"] and g["lower_bound"] == o["lb"]
    a = host_u32(g["assign"])
    assert BF.cmax_of(a, q, 4) == g["cmax"]
    T, cm = BF.score_assignment(a, q, p.plan)
    assert g["makespan"] == T
    # warm start from the search winner: the same certified optimum
    t, f, x = (dev_u32(v) for v in p.features(0))
    res = D.search_plans(p.model, t, f, x, K=65536, R=p.R, G=p.G, seed=p.seed(0), plan=p.plan)
    g2 = D.exact_cmax(ticks, p.plan, node_budget=1 << 40, init_assign=res["assign"])
    assert g2["proven"] and g2["cmax"] == g["cmax"] <= res["cmax"]


def test_presets_certificate(D, O, presets):
    # tree search within a node budget: config 1 (n = 32, m = 4) below the pair decomposition's
    # 2^31 subsets is a gap certificate; config 3: LB meets the LPT
    for k in (1, 3):
        p = presets[k]
        _, ticks = D.predict_costs(p.model, p.plan, *(dev_u32(a) for a in p.features(0)), want_f32=False)
        m = p.plan["n_mb"] * p.plan["l_dp"]
        g = D.exact_cmax(ticks, p.plan, node_budget=2 * 10 ** 9)
        q = host_u32(ticks).reshape(4, -1)
        o = O.exact_cmax(q, m, node_budget=10 ** 6)
        a = host_u32(g["assign"])
        assert BF.cmax_of(a, q, m) == g["cmax"] and g["lower_bound"] == o["lb"] <= g["cmax"] <= o["cmax"]
        if o["proven"]:
            assert g["proven"] and g["cmax"] == o["cmax"]
        T, cm = BF.score_assignment(a, q, p.plan)
        assert g["makespan"] == T


def test_warm_start_from_search_winner(D, presets):
    p = presets[2]
    t, f, x = (dev_u32(a) for a in p.features(0))
    res = D.search_plans(p.model, t, f, x, K=4096, R=p.R, G=p.G, seed=p.seed(0), plan=p.plan)
    _, ticks = D.predict_costs(p.model, p.plan, t, f, x, want_f32=False)
    g = D.exact_cmax(ticks, p.plan, node_budget=10 ** 8, init_assign=res["assign"])
    assert g["cmax"] <= res["cmax"] and g["lower_bound"] <= g["cmax"]
    assert BF.cmax_of(host_u32(g["assign"]), host_u32(ticks).reshape(4, -1), 16) == g["cmax"]


def test_budget_and_errors(D):
    rng = np.random.default_rng(9)
    c = rng.integers(1, 1000, (4, 20)).astype(np.uint32)
    g = D.exact_cmax(dev_u32(c), plan(4), node_budget=1)
    assert g["cmax"] >= g["lower_bound"] and BF.cmax_of(host_u32(g["assign"]), c, 4) == g["cmax"]
    bad = torch.full((20,), 7, dtype=torch.int32, device="cuda")
    with pytest.raises(Exception, match="init_assign"):
        D.exact_cmax(dev_u32(c), plan(4), init_assign=bad)
