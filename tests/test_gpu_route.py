"""N4(b) inter-model routing plan on the GPU (dflop_route_plan) against orc_route_plan:
bit-exact (integer bookkeeping).  -m gpu."""
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


def check(D, O, c, pl, a):
    g = D.route_plan(dev_u32(c), pl, dev_u32(a))
    o = O.route_plan(c, pl, a)
    assert (host_u32(g["pos_item"]) == o["pos_item"]).all()
    assert (host_u32(g["slot_off"]) == o["slot_off"]).all()
    assert (host_u32(g["enc_off"]) == o["enc_off"]).all()
    assert (host_u32(g["llm_off"]) == o["llm_off"]).all()
    assert (g["enc_load"].cpu().numpy().view(np.uint64) == o["enc_load"]).all()


def test_random_plans(D, O):
    rng = np.random.default_rng(17)
    for trial in range(20):
        M, R, G = int(rng.integers(1, 9)), int(rng.integers(1, 5)), int(rng.integers(1, 9))
        pl = dict(e_tp=1, e_pp=1, e_dp=G, l_tp=1, l_pp=1, l_dp=R, n_mb=M)
        n = int(rng.integers(1, 3000))
        c = rng.integers(0, 5000, (4, n)).astype(np.uint32)
        a = rng.integers(0, M * R, n).astype(np.uint32)
        check(D, O, c, pl, a)


def test_search_winner_routing(D, O, presets):
    # config 5's winner routed with an encoder DP of 4 over the LLM's single data group and
    # a synthetic L_dp = 2 regrouping (the same buckets as 32 slots x 2 replicas)
    p = presets[5]
    t, f, x = (dev_u32(v) for v in p.features(0))
    res = D.search_plans(p.model, t, f, x, K=256, R=p.R, G=p.G, seed=p.seed(0), plan=p.plan)
    _, ticks = D.predict_costs(p.model, p.plan, t, f, x, want_f32=False)
    q, a = host_u32(ticks).reshape(4, -1), host_u32(res["assign"])
    for pl in (dict(p.plan, e_dp=4), dict(p.plan, e_dp=3, l_dp=2, n_mb=32)):
        check(D, O, q, pl, a)


def test_invalid_assignment(D):
    c = np.ones((4, 4), np.uint32)
    pl = dict(e_tp=1, e_pp=1, e_dp=2, l_tp=1, l_pp=1, l_dp=1, n_mb=2)
    with pytest.raises(Exception, match="bucket"):
        D.route_plan(dev_u32(c), pl, dev_u32(np.array([0, 1, 2, 0])))
