"""N2 on the GPU: dflop_search_plans_batches (Eq. (1) over a sample of batches) against the
oracle's composition (expected_makespan_choice) on the GPU's integer costs, FIXED and
Algorithm-1 modes.  -m gpu."""
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


def sample(p, batches, cut=None):
    feats = [p.features(b) for b in batches]
    if cut is not None:   # ragged batch sizes
        feats = [tuple(a[:c] for a in fb) for fb, c in zip(feats, cut)]
    offs = np.concatenate([[0], np.cumsum([len(fb[0]) for fb in feats])]).astype(np.uint32)
    cat = [np.concatenate([fb[i] for fb in feats]) for i in range(3)]
    return feats, offs, cat


@pytest.mark.parametrize("k, cut", [(2, None), (3, [1024, 300, 0, 777])])
def test_fixed_plan_over_batches(D, O, presets, k, cut):
    p = presets[k]
    batches = [0, 1, 2] if cut is None else [0, 1, 2, 3]
    feats, offs, cat = sample(p, batches, cut)
    K = 1024
    t, f, x = (dev_u32(a) for a in cat)
    res = D.search_plans_batches(p.model, t, f, x, offs, K=K, R=p.R, G=p.G, seed=p.seed(0), plan=p.plan)
    assign = host_u32(res["assign"])
    costs = []
    for b, fb in enumerate(feats):
        _, ticks = D.predict_costs(p.model, p.plan, *(dev_u32(a) for a in fb), want_f32=False)
        costs.append(host_u32(ticks))
    win, sums, per = O.expected_makespan_choice([p.plan], [costs], K, p.R, p.G, p.seed(0))
    assert res["makespan"] == sums[0] == int(res["plan_objective"][0])
    for b, r in enumerate(per[0]):
        gb = res["batches"][b]
        assert gb["makespan"] == r["T"] and gb["cand"] == r["c"] and gb["cmax"] == r["cmax"], b
        assert (assign[offs[b]:offs[b + 1]] == r["assign"]).all(), b


def test_single_batch_equals_search_plans(D, presets):
    p = presets[2]
    t, f, x = (dev_u32(a) for a in p.features(5))
    a = D.search_plans(p.model, t, f, x, K=2048, R=p.R, G=p.G, seed=p.seed(5), plan=p.plan)
    b = D.search_plans_batches(p.model, t, f, x, [0, p.n], K=2048, R=p.R, G=p.G, seed=p.seed(5), plan=p.plan)
    for key in ("makespan", "cand", "cmax", "m"):
        assert a[key] == b[key], key
    assert torch.equal(a["assign"], b["assign"])


def test_alg1_over_batches(D, O, presets):
    # Stage A on the whole sample's mean shapes (bit-identical fp64 on both sides), then the
    # Eq. (1) choice over the top-P plans x batches on the GPU's costs
    p = presets[4]
    feats, offs, cat = sample(p, [0, 1])
    K, P = 16, 4
    t, f, x = (dev_u32(a) for a in cat)
    cl = p.cluster
    res = D.search_plans_batches(p.model, t, f, x, offs, K=K, R=p.R, G=p.G, seed=p.seed(0), cluster=cl,
                                 mem=p.mem(), gbs=p.gbs, top_p=P)
    mb, ms = O.batch_means(p.model, *cat)
    T_A, cfgs = O.stage_a_all(p.model, p.mem(), cl["n_gpus"], cl["gpus_per_node"], p.gbs, mb, ms)
    plans = []
    for pidx in O.stage_a_top(T_A, P):
        e, i = O.pair_to_config(cfgs, p.gbs, pidx)
        c = cfgs[e]
        plans.append(dict(e_tp=int(c[0]), e_pp=int(c[1]), e_dp=int(c[2]), l_tp=int(c[3]), l_pp=int(c[4]),
                          l_dp=int(c[5]), n_mb=i))
    costs = [[host_u32(D.predict_costs(p.model, pl, *(dev_u32(a) for a in fb), want_f32=False)[1]) for fb in feats]
             for pl in plans]
    win, sums, per = O.expected_makespan_choice(plans, costs, K, p.R, p.G, p.seed(0))
    assert [int(v) for v in res["plan_objective"]] == sums
    assert res["plan"] == plans[win] and res["stage_a_rank"] == win and res["makespan"] == sums[win]
    for b, r in enumerate(per[win]):
        assert res["batches"][b]["makespan"] == r["T"] and res["batches"][b]["cand"] == r["c"]


def test_batch_offset_errors(D, presets):
    p = presets[2]
    t, f, x = (dev_u32(a) for a in p.features(0))
    with pytest.raises(Exception, match="offsets"):
        D.search_plans_batches(p.model, t, f, x, [0, 100, 50], K=8, R=1, G=8, seed=(1, 2), plan=p.plan)


def test_split_pipeline_over_ragged_batches(D, presets, monkeypatch):
    """Config 5's shape over three ragged batches (4,096 / 3,000 / 1,500 samples) at K = 6,000:
    the split pipeline (each batch's own workspace need within the bound computed for the
    largest; a batch whose chunks would outgrow it falls back to the merged kernel) gives the
    merged kernel's per-batch winners and assignments."""
    p = presets[5]
    feats, offs, cat = sample(p, [0, 1, 2], [4096, 3000, 1500])
    t, f, x = (dev_u32(a) for a in cat)
    K = 6000
    monkeypatch.delenv("DFLOP_SPLIT", raising=False)
    a = D.search_plans_batches(p.model, t, f, x, offs, K=K, R=p.R, G=p.G, seed=p.seed(0), plan=p.plan)
    monkeypatch.setenv("DFLOP_SPLIT", "0")
    b = D.search_plans_batches(p.model, t, f, x, offs, K=K, R=p.R, G=p.G, seed=p.seed(0), plan=p.plan)
    assert a["makespan"] == b["makespan"]
    for ga, gb in zip(a["batches"], b["batches"]):
        assert ga["makespan"] == gb["makespan"] and ga["cand"] == gb["cand"] and ga["cmax"] == gb["cmax"]
    assert (host_u32(a["assign"]) == host_u32(b["assign"])).all()
