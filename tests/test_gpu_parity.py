"""GPU parity: the CUDA path through the C-ABI (libdflop.so) against the CPU oracle on the
same seeded inputs.  Tolerances: predict fp32 vs fp64 <= 1e-5 relative
(north_star); ticks |q_gpu - q_orc| <= 1 + 1e-5 q; everything downstream of the shared
integer costs bit-exact.  -m gpu.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

from paper_2603_25120_b200 import synth  # noqa: E402


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


def host_u64(t):
    return t.cpu().numpy().view(np.uint64)


def feats(p, b=0):
    t, f, x = p.features(b)
    return (t, f, x), (dev_u32(t), dev_u32(f), dev_u32(x))


PLAN4 = dict(e_tp=8, e_pp=2, e_dp=1, l_tp=8, l_pp=6, l_dp=1, n_mb=64)


def plan_of(p):
    return p.plan if p.plan is not None else PLAN4


# ------------------------------------------------------------------ a1 predict
@pytest.mark.parametrize("e_attn", [0, 1])
@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_predict_parity(D, O, presets, k, e_attn):
    p = presets[k]
    pl = plan_of(p)
    model = dict(p.model, e_attn=e_attn)     # e_attn = 1: in-tile encoder attention 4*h_E*E_seq^2 (R1)
    for b in (0, 1):
        (t, f, x), (dt, df, dx) = feats(p, b)
        cf64, cq, st, _ = O.predict(model, pl, t, f, x)
        assert st == 0
        f32, ticks = D.predict_costs(model, pl, dt, df, dx)
        g = f32.cpu().numpy().astype(np.float64)
        ref = cf64 / p.model["tick_ns"]
        assert np.all((ref == 0) == (g == 0))
        rel = np.abs(g - ref) / np.maximum(ref, 1e-300)
        assert rel.max() <= 1e-5, rel.max()
        q = host_u32(ticks).astype(np.int64)
        assert np.all(np.abs(q - cq.astype(np.int64)) <= 1 + 1e-5 * cq)


@pytest.mark.parametrize("e_attn", [0, 1])
def test_predict_worked_example(D, O, e_attn):
    """The hand-derived worked example (tests/golden/predict_worked.txt: non-unit shapes,
    knots that are not powers of two, E_tp != L_tp) through the C-ABI: fp32 within 1e-5 of
    the exact values, ticks equal to the fixture's."""
    from test_oracle_worked import load_predict_fixture
    model, plan, items, costs = load_predict_fixture()
    model = dict(model, e_attn=e_attn)
    t, f, x = (np.array([it[j] for it in items], np.uint32) for j in (1, 2, 3))
    f32, ticks = D.predict_costs(model, plan, dev_u32(t), dev_u32(f), dev_u32(x))
    g, q = f32.cpu().numpy().astype(np.float64), host_u32(ticks)
    for i, c in enumerate(c for c in costs if c["e_attn"] == e_attn):
        for k in range(4):
            exact = float(c["ns"][k])
            assert (g[k, i] == 0) == (exact == 0) and abs(g[k, i] - exact) <= 1e-5 * exact, (c["name"], k)
        assert [int(v) for v in q[:, i]] == c["ticks"], c["name"]


@pytest.mark.parametrize("n", [0, 1, 3, 5, 4097])
def test_predict_ragged_sizes(D, O, presets, n):
    p = presets[5]
    t, f, x = (a[:n] for a in p.features(3)) if n <= 4096 else (np.tile(a, 2)[:n] for a in p.features(3))
    cf64, cq, _, _ = O.predict(p.model, p.plan, t, f, x)
    f32, ticks = D.predict_costs(p.model, p.plan, dev_u32(t), dev_u32(f), dev_u32(x))
    assert f32.shape == (4, n)
    if n:
        g = f32.cpu().numpy().astype(np.float64)
        ref = cf64 / p.model["tick_ns"]
        assert (np.abs(g - ref) <= 1e-5 * ref + 1e-30).all()


def test_predict_overflow_status(D, presets):
    p = presets[5]
    m = dict(p.model)
    m["tick_ns"] = 1e-3   # every second-scale cost overflows 2^32 ticks
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    (_, _, _), (dt, df, dx) = feats(p)
    _, ticks = D.predict_costs(m, p.plan, dt, df, dx, dev_status=st)
    assert int(st.item()) & D.DEV_COST_OVERFLOW
    assert (host_u32(ticks) == 0xFFFFFFFF).any()


# ------------------------------------------------------------------ a4 simulate
def test_simulate_parity(D, O):
    rng = np.random.default_rng(5)
    for S, M in [(1, 1), (1, 7), (2, 1), (4, 6), (8, 32), (16, 64), (32, 3), (5, 129)]:
        Cn = 24
        fwd, bwd = synth.random_durations(Cn, S, M, seed=S * 1000 + M, hi=int(rng.integers(1, 1000)))
        ms, busy = D.simulate_1f1b(torch.from_numpy(fwd.view(np.int64)).cuda(),
                                   torch.from_numpy(bwd.view(np.int64)).cuda())
        ms, busy = host_u64(ms), host_u64(busy)
        for c in range(Cn):
            T, b = O.simulate_1f1b(fwd[c], bwd[c])
            assert ms[c] == T and (busy[c] == b).all(), (S, M, c)


def test_simulate_uniform_closed_form(D):
    for S in (1, 3, 8, 16, 32):
        for M in (1, 5, 33):
            fwd = np.full((2, S, M), 3, np.uint64)
            bwd = np.full((2, S, M), 7, np.uint64)
            ms, _ = D.simulate_1f1b(torch.from_numpy(fwd.view(np.int64)).cuda(),
                                    torch.from_numpy(bwd.view(np.int64)).cuda())
            assert (host_u64(ms) == (M + S - 1) * 10).all()


def test_simulate_shape_errors(D):
    z = torch.zeros((1, 33, 2), dtype=torch.int64, device="cuda")
    with pytest.raises(D.DflopError) as e:
        D.simulate_1f1b(z, z)
    assert e.value.code == 2


# ------------------------------------------------------------------ a2-a5 balance
def gpu_balance(D, q_dev, plan, K, R, G, seed, c0, c1, mode=0):
    r = D.balance_microbatches(q_dev, plan, K, R, G, seed, c0, c1, mode=mode, want_groups=True, per_candidate=True)
    best = D.cand_result(r["best"])
    return dict(best=best, assign=host_u32(r["assign"]), offsets=host_u32(r["offsets"]),
                items=host_u32(r["items"])[: q_dev.shape[1]], cT=host_u64(r["cand_T"]), cC=host_u64(r["cand_cmax"]))


def check_balance(D, O, q_host, plan, K, R, G, seed, c0, c1, mode=0, threads=None):
    q_dev = dev_u32(q_host)
    g = gpu_balance(D, q_dev, plan, K, R, G, seed, c0, c1, mode)
    o = O.balance_threaded(q_host, plan, K, R, G, seed, c0, c1, mode=mode, threads=threads)
    assert (g["cT"] == o["cand_T"]).all(), np.nonzero(g["cT"] != o["cand_T"])[0][:10]
    assert (g["cC"] == o["cand_cmax"]).all()
    assert g["best"]["cand"] == o["c"] and g["best"]["makespan"] == o["T"] and g["best"]["cmax"] == o["cmax"]
    assert (g["assign"] == o["assign"]).all()
    m = plan["n_mb"] * plan["l_dp"]
    off, items = O.groups(o["assign"], m)
    assert (g["offsets"] == off).all() and (g["items"] == items).all()
    assert g["best"]["key"] == (o["T"] << 24) | o["c"]
    return g, o


@pytest.mark.parametrize("k,c0,c1", [(1, 0, 4096), (2, 0, 2048), (3, 0, 512), (5, 0, 48)])
def test_balance_parity_presets(D, O, presets, k, c0, c1):
    p = presets[k]
    pl = plan_of(p)
    (t, f, x), (dt, df, dx) = feats(p)
    _, ticks = D.predict_costs(p.model, pl, dt, df, dx, want_f32=False)
    q_gpu = host_u32(ticks)
    # shared integer array, direction 1: the GPU's integers fed to the oracle
    check_balance(D, O, q_gpu, pl, p.K, p.R, p.G, p.seed(0), c0, c1)
    # direction 2: the oracle's integers uploaded to the GPU
    _, q_orc, _, _ = O.predict(p.model, pl, t, f, x)
    check_balance(D, O, q_orc, pl, p.K, p.R, p.G, p.seed(0), c0, min(c1, c0 + 64))


def test_balance_shard_window_config5(D, O, presets):
    p = presets[5]
    _, q, _, _ = O.predict(p.model, p.plan, *p.features(2))
    check_balance(D, O, q, p.plan, p.K, p.R, p.G, p.seed(2), 777_000, 777_024)


@pytest.mark.parametrize("n, n_mb, l_dp, hi", [
    (4096, 64, 1, None),      # config 5's shape: k_lpt at GL = 2, 32 buckets per lane
    (2000, 50, 2, 2 ** 20),   # m = 100: GL = 2, generic bucket loop
    (1500, 64, 2, 2 ** 18),   # m = 128: GL = 4, 32 buckets per lane
    (2500, 250, 1, 5000),     # m = 250: GL = 4, generic
    (40, 64, 1, 2 ** 20),     # n < m
    (4000, 50, 1, "ldom"),    # the LLM dimension is the bottleneck: windows on l
    (4000, 50, 1, "many"),    # ~80 members per bucket: partner lists sorted in two chunks
    (3000, 48, 1, "ties"),    # three cost values: exact ties on and at the window edges
    (3000, 64, 1, "quant"),   # loads that differ below the keys' 12-bit quantisation
])
def test_split_pipeline_parity(D, O, presets, monkeypatch, n, n_mb, l_dp, hi):
    """The split pipeline (the LPT in k_lpt, then the candidate kernel from its output, chunk by
    chunk) forced on (DFLOP_SPLIT=2): every candidate equals the merged
    kernel's (DFLOP_SPLIT=0) and, on a window, the oracle's."""
    p = presets[5]
    rng = np.random.default_rng(n + n_mb)
    if hi is None:
        q = O.predict(p.model, p.plan, *p.features(1))[1]
        plan = p.plan
    elif isinstance(hi, str):
        if hi == "ldom":
            q = np.stack([rng.integers(0, 3000, n), rng.integers(0, 3000, n),
                          rng.integers(0, 60000, n), rng.integers(0, 60000, n)])
        elif hi == "many":
            q = rng.integers(0, 400, (4, n))
            q[:, rng.random(n) < 0.02] *= 300  # a few large samples
        elif hi == "ties":
            q = rng.choice(np.array([0, 1000, 3000]), size=(4, n))
        else:  # "quant": 50,000 + a few ticks: the packed loads agree above the low 12 bits
            q = 50_000 + rng.integers(0, 40, (4, n))
        q = q.astype(np.uint32)
        plan = dict(e_tp=1, e_pp=2, e_dp=1, l_tp=1, l_pp=6, l_dp=l_dp, n_mb=n_mb)
    else:
        q = rng.integers(0, hi, (4, n), dtype=np.uint64).astype(np.uint32)
        q[:, rng.random(n) < 0.2] = q[:, [0]]  # exact ties
        plan = dict(e_tp=1, e_pp=2, e_dp=1, l_tp=1, l_pp=6, l_dp=l_dp, n_mb=n_mb)
    K, seed = 5000, (3, 4)
    qd = dev_u32(q)
    monkeypatch.setenv("DFLOP_SPLIT", "0")
    merged = gpu_balance(D, qd, plan, K, p.R, p.G, seed, 0, K)
    monkeypatch.setenv("DFLOP_SPLIT", "2")
    monkeypatch.setenv("DFLOP_SPLIT_CHUNK", "1700")
    split = gpu_balance(D, qd, plan, K, p.R, p.G, seed, 0, K)
    assert (split["cT"] == merged["cT"]).all(), np.nonzero(split["cT"] != merged["cT"])[0][:10]
    assert (split["cC"] == merged["cC"]).all()
    assert split["best"] == merged["best"] and (split["assign"] == merged["assign"]).all()
    assert split["best"]["status"] == merged["best"]["status"]
    monkeypatch.setenv("DFLOP_SPLIT_CHUNK", "10")
    check_balance(D, O, q, plan, K, p.R, p.G, seed, 1690, 1714)  # across chunk boundaries


@pytest.mark.parametrize("case", [
    dict(n=0, plan=dict(e_tp=1, e_pp=1, e_dp=1, l_tp=1, l_pp=2, l_dp=1, n_mb=3)),
    dict(n=1, plan=dict(e_tp=1, e_pp=1, e_dp=1, l_tp=1, l_pp=1, l_dp=1, n_mb=1)),
    dict(n=5, plan=dict(e_tp=1, e_pp=2, e_dp=1, l_tp=1, l_pp=1, l_dp=2, n_mb=4)),        # n < m
    dict(n=37, plan=dict(e_tp=1, e_pp=3, e_dp=2, l_tp=1, l_pp=5, l_dp=3, n_mb=5)),       # replicas
    dict(n=700, plan=dict(e_tp=1, e_pp=1, e_dp=1, l_tp=1, l_pp=7, l_dp=2, n_mb=150)),    # wide apos m > 255
    dict(n=300, plan=dict(e_tp=1, e_pp=1, e_dp=1, l_tp=1, l_pp=1, l_dp=1, n_mb=2)),      # list overflow path
    dict(n=129, plan=dict(e_tp=1, e_pp=16, e_dp=1, l_tp=1, l_pp=16, l_dp=1, n_mb=9)),    # S = 32
])
def test_balance_edge_cases(D, O, case):
    n, plan = case["n"], case["plan"]
    q = synth.random_costs(n, seed=n + 17, hi=5000, heavy=True)
    for G in (1, 8, 16):
        check_balance(D, O, q, plan, K=300, R=6, G=G, seed=(n, 3), c0=0, c1=40)


def _forced_tie_costs(n_video, n_text, lt=2990):
    """Videos (e = 3000, l = 5) and text-only samples (e = 0, l = lt <= 2995): a text sample's
    bucket (E = 0, L = lt) probed by a later video gives max(0 + 3000, lt + 5) = 3000, the same
    value as an empty bucket, so the video takes the (lower) text bucket."""
    n = n_video + n_text
    q = np.zeros((4, n), np.uint32)
    for i in range(n):
        if i % 2 == 0 and i // 2 < n_video or i // 2 >= n_text:
            q[:, i] = (1000, 2000, 1, 4)          # e = 3000, l = 5
        else:
            q[:, i] = (0, 0, lt // 3, lt - lt // 3)  # e = 0, l = lt
    return q


@pytest.mark.parametrize("n_video,n_text,n_mb", [(36, 92, 64), (20, 30, 8), (100, 300, 256)])
def test_balance_lpt_empty_bucket_ties(D, O, n_video, n_text, n_mb):
    """The first-m LPT shortcut (lpt_pass) must stay off when one of the m largest samples has
    e = 0 or l = 0: a perturbed order can put a text sample before a video of the same base
    group, and the video then ties an empty bucket and takes the earlier, non-empty one."""
    q = _forced_tie_costs(n_video, n_text)
    plan = dict(e_tp=1, e_pp=1, e_dp=1, l_tp=1, l_pp=1, l_dp=1, n_mb=n_mb)
    check_balance(D, O, q, plan, K=512, R=4, G=8, seed=(5, 6), c0=0, c1=512)
    if n_video < n_mb:  # the oracle's family has candidates whose first m steps are NOT "t -> bucket t"
        order = O.base_order(q)
        top = [int(order[t]) for t in range(n_mb)]
        off = sum(sorted(int(O.run_candidate(q, plan, 512, 0, 8, (5, 6), c)[0][i]) for i in top) != list(range(n_mb))
                  for c in range(2, 40))
        assert off > 0


def test_balance_lpt_forced_prefix(D, O):
    """Every sample has e > 0 and l > 0 (config-4-like, m a third of n): the first m decisions
    are forced; per-candidate results equal the oracle's step-by-step LPT."""
    rng = np.random.default_rng(9)
    n = 600
    q = rng.integers(1, 4000, size=(4, n)).astype(np.uint32)
    for n_mb, l_dp in ((200, 1), (96, 2), (64, 1), (8, 1)):
        plan = dict(e_tp=1, e_pp=2, e_dp=1, l_tp=1, l_pp=2, l_dp=l_dp, n_mb=n_mb)
        check_balance(D, O, q, plan, K=256, R=5, G=8, seed=(11, n_mb), c0=0, c1=256)


def _packed_margin(q, m):
    """bound + C of the packed variant (k_build_items): ceil((sum e + sum l)/m) + 2 max key + max(l - e)+"""
    q = q.astype(np.int64)
    e, l = q[0] + q[1], q[2] + q[3]
    return -(-(int(e.sum()) + int(l.sum())) // m) + 2 * int(np.maximum(e, l).max()) + int(np.maximum(l - e, 0).max())


@pytest.mark.parametrize("side", [-1, 0, 1])
def test_balance_packed_offset_bound(D, O, side):
    # one LLM-heavy item (e = 0) sets C = max(l - e) and the max key; its size puts the packed
    # variant's bound + C just below / at / above 2^(32 - s): the LPT probes in the offset form
    # max(E' + e' - l' + C', L' + C') reach the top of the u32 range, or the plain u32 variant runs
    plan = dict(e_tp=1, e_pp=1, e_dp=1, l_tp=1, l_pp=3, l_dp=1, n_mb=16)
    m, s = 16, 4
    q = synth.random_costs(200, seed=5, hi=200000)
    lim = 1 << (32 - s)
    lo, hi = 0, lim
    while hi - lo > 1:  # largest LLM size X of item 0 with margin < lim
        X = (lo + hi) // 2
        q[:, 0] = (0, 0, X // 3, X - X // 3)
        lo, hi = (X, hi) if _packed_margin(q, m) < lim else (lo, X)
    X = lo + (1 if side > 0 else 0) - (5 if side < 0 else 0)
    q[:, 0] = (0, 0, X // 3, X - X // 3)
    assert (_packed_margin(q, m) < lim) == (side <= 0)
    check_balance(D, O, q, plan, K=512, R=8, G=8, seed=(9, side + 1), c0=0, c1=512)


@pytest.mark.parametrize("n_mb, l_dp", [(350, 2), (100, 1), (37, 3)])
def test_balance_lane_local_packed_lpt(D, O, n_mb, l_dp):
    # bucket sums too large for the packed variant's s = bits(m - 1) index bits but small
    # enough for the lane-local index (k = j / GL): the plain variant's LPT runs on packed
    # (v << kb | k) keys with cross-lane ties resolved by a ballot -- many identical items make
    # exact ties of (v, k) across lanes frequent
    m = n_mb * l_dp
    plan = dict(e_tp=1, e_pp=1, e_dp=1, l_tp=1, l_pp=3, l_dp=l_dp, n_mb=n_mb)
    rng = np.random.default_rng(m)
    n = 2000
    q = rng.integers(100000, 900000, (4, n)).astype(np.uint32)
    same = rng.random(n) < 0.6
    q[:, same] = np.array([300000, 600000, 250000, 500000], np.uint32)[:, None]
    s = max(1, int(np.ceil(np.log2(m))))
    assert _packed_margin(q, m) >= (1 << (32 - s))   # not the packed variant
    check_balance(D, O, q, plan, K=256, R=6, G=8, seed=(m, 5), c0=0, c1=64)
    check_balance(D, O, q, plan, K=256, R=0, G=1, seed=(m, 6), c0=0, c1=16)


def test_balance_64bit_path(D, O, presets):
    # 1 ns ticks: config 2's bucket sums exceed 2^32 -> 64-bit candidate kernel
    p = presets[2]
    m = dict(p.model)
    m["tick_ns"] = 1.0
    _, q, st, _ = O.predict(m, p.plan, *p.features(0))
    assert st == 0 and int(q[2].astype(np.int64).sum() + q[3].sum()) >= 2 ** 32
    check_balance(D, O, q, p.plan, p.K, p.R, p.G, p.seed(0), 0, 256)


def test_balance_exhaustive_vs_oracle_and_bruteforce(D, O):
    import bruteforce as BF
    rng = np.random.default_rng(21)
    for trial in range(6):
        n = int(rng.integers(2, 8))
        plan = dict(e_tp=1, e_pp=int(rng.integers(1, 3)), e_dp=1, l_tp=1, l_pp=int(rng.integers(1, 3)),
                    l_dp=int(rng.integers(1, 3)), n_mb=int(rng.integers(1, 3)))
        m = plan["n_mb"] * plan["l_dp"]
        K = m ** n
        q = rng.integers(0, 50, (4, n)).astype(np.uint32)
        g, o = check_balance(D, O, q, plan, K, 0, 1, (0, 0), 0, K, mode=1)
        bf = list(BF.all_assignments(q.tolist(), plan))
        assert g["best"]["makespan"] == min(b[2] for b in bf)


def test_balance_sharding_independent_of_g(D, O, presets):
    # the winner of the family does not depend on how [0, K) is split
    p = presets[3]
    _, q, _, _ = O.predict(p.model, p.plan, *p.features(0))
    qd = dev_u32(q)
    K = 1024
    whole = D.cand_result(D.balance_microbatches(qd, p.plan, K, p.R, p.G, p.seed(0), 0, K)["best"])
    for Gs in (2, 3, 8):
        keys = []
        for g in range(Gs):
            b, e = K * g // Gs, K * (g + 1) // Gs
            keys.append(D.cand_result(D.balance_microbatches(qd, p.plan, K, p.R, p.G, p.seed(0), b, e)["best"])["key"])
        assert min(keys) == whole["key"]


def test_balance_argument_errors(D, presets):
    p = presets[1]
    q = dev_u32(np.zeros((4, 8), np.uint32))
    with pytest.raises(D.DflopError) as e:
        D.balance_microbatches(q, p.plan, 0, 1, 1, (0, 0))
    assert e.value.code == 1
    with pytest.raises(D.DflopError):
        D.balance_microbatches(q, p.plan, 10, 1, 17, (0, 0))
    with pytest.raises(D.DflopError):
        D.balance_microbatches(q, dict(p.plan, n_mb=70000), 10, 1, 1, (0, 0))
    with pytest.raises(D.DflopError):
        D.balance_microbatches(q, p.plan, 10, 1, 1, (0, 0), mode=1)   # 4^8 > 10


# ------------------------------------------------------------------ full-size, bench launch config
def test_config5_full_family_sampled(D, O, presets):
    """K = 10^6 at N = 4096 (the bench's launch configuration): sampled candidates checked one
    by one against the oracle, the winner re-derived from the per-candidate array."""
    p = presets[5]
    (t, f, x), (dt, df, dx) = feats(p, 0)
    _, ticks = D.predict_costs(p.model, p.plan, dt, df, dx, want_f32=False)
    r = D.balance_microbatches(ticks, p.plan, p.K, p.R, p.G, p.seed(0), per_candidate=True)
    best = D.cand_result(r["best"])
    cT, cC = host_u64(r["cand_T"]), host_u64(r["cand_cmax"])
    c_star = int(np.lexsort((np.arange(p.K), cT))[0])
    assert best["cand"] == c_star and best["makespan"] == cT[c_star] and best["cmax"] == cC[c_star]
    q = host_u32(ticks)
    rng = np.random.default_rng(99)
    sample = sorted(set([0, 1, 2, p.K - 1, c_star] + rng.integers(0, p.K, 24).tolist()))
    pi = O.base_order(q)
    for c in sample:
        a, T, cm = O.run_candidate(q, p.plan, p.K, p.R, p.G, p.seed(0), c, order=pi)
        assert (T, cm) == (int(cT[c]), int(cC[c])), c
        if c == c_star:
            assert (host_u32(r["assign"]) == a).all()


# ------------------------------------------------------------------ a6 search
def test_search_fixed_equals_balance(D, O, presets):
    p = presets[2]
    (t, f, x), (dt, df, dx) = feats(p)
    res = D.search_plans(p.model, dt, df, dx, K=2048, R=p.R, G=p.G, seed=p.seed(0), plan=p.plan)
    _, q, _, _ = O.predict(p.model, p.plan, t, f, x)
    _, ticks = D.predict_costs(p.model, p.plan, dt, df, dx, want_f32=False)
    o = O.balance_threaded(host_u32(ticks), p.plan, 2048, p.R, p.G, p.seed(0), per_candidate=False)
    assert res["makespan"] == o["T"] and res["cand"] == o["c"] and res["cmax"] == o["cmax"]
    assert (host_u32(res["assign"]) == o["assign"]).all()


@pytest.mark.parametrize("e_attn", [0, 1])
def test_search_alg1_stage_a_and_b(D, O, presets, e_attn):
    p = presets[4]
    model = dict(p.model, e_attn=e_attn)
    (t, f, x), (dt, df, dx) = feats(p)
    cl = p.cluster
    n_cfg = len(O.enumerate_configs(cl["n_gpus"], cl["gpus_per_node"]))
    sa = torch.empty(6_541_832, dtype=torch.int64, device="cuda")
    K, P = 8, 4
    res = D.search_plans(model, dt, df, dx, K=K, R=p.R, G=p.G, seed=p.seed(0), cluster=cl, mem=p.mem(),
                         gbs=p.gbs, top_p=P, stage_a_out=sa)
    assert res["n_configs"] == n_cfg == 7194 and res["n_pairs"] == 6_541_832
    mb, ms = O.batch_means(model, t, f, x)
    T_orc, cfgs = O.stage_a_all(model, p.mem(), cl["n_gpus"], cl["gpus_per_node"], p.gbs, mb, ms)
    T_gpu = host_u64(sa)
    # fp64 with identical, FMA-free operation order on both sides: expected bit-identical
    assert (T_gpu == T_orc).all(), np.count_nonzero(T_gpu != T_orc)
    assert res["n_feasible"] == int(np.count_nonzero(T_orc != np.uint64(2 ** 64 - 1)))
    top = O.stage_a_top(T_orc, P)
    e, i = O.pair_to_config(cfgs, p.gbs, top[0])
    c = cfgs[e]
    assert res["alg1_plan"] == dict(e_tp=int(c[0]), e_pp=int(c[1]), e_dp=int(c[2]), l_tp=int(c[3]), l_pp=int(c[4]),
                                    l_dp=int(c[5]), n_mb=i)
    # Stage B: the oracle balances the same P plans on the GPU's integer costs
    best = None
    for rank, pidx in enumerate(top):
        e, i = O.pair_to_config(cfgs, p.gbs, pidx)
        c = cfgs[e]
        pl = dict(e_tp=int(c[0]), e_pp=int(c[1]), e_dp=int(c[2]), l_tp=int(c[3]), l_pp=int(c[4]), l_dp=int(c[5]),
                  n_mb=i)
        _, ticks = D.predict_costs(model, pl, dt, df, dx, want_f32=False)
        o = O.balance_threaded(host_u32(ticks), pl, K, p.R, p.G, p.seed(0), per_candidate=False)
        key = (o["T"], rank, o["c"])
        if best is None or key < best[0]:
            best = (key, pl, o)
    (T, rank, cstar), pl, o = best
    assert res["makespan"] == T and res["stage_a_rank"] == rank and res["cand"] == cstar
    assert res["plan"] == pl and res["cmax"] == o["cmax"]
    assert (host_u32(res["assign"]) == o["assign"]).all()


def test_search_infeasible(D, presets):
    p = presets[4]
    (_, _, _), (dt, df, dx) = feats(p)
    mem = p.mem()
    mem["mem_per_gpu"] = 1.0
    with pytest.raises(D.DflopError) as e:
        D.search_plans(p.model, dt, df, dx, K=4, R=1, G=8, seed=(1, 1), cluster=p.cluster, mem=mem, gbs=p.gbs,
                       top_p=2)
    assert e.value.code == 4


def test_config3_full_family_per_gpu_sampled(D, O, presets):
    """Config 3 at its full per-GPU family (K = 65,536, weak scaling): winner re-derived from
    the per-candidate array, sampled candidates recomputed by the oracle."""
    p = presets[3]
    (t, f, x), (dt, df, dx) = feats(p, 1)
    _, ticks = D.predict_costs(p.model, p.plan, dt, df, dx, want_f32=False)
    r = D.balance_microbatches(ticks, p.plan, p.K, p.R, p.G, p.seed(1), per_candidate=True)
    best = D.cand_result(r["best"])
    cT, cC = host_u64(r["cand_T"]), host_u64(r["cand_cmax"])
    c_star = int(np.lexsort((np.arange(p.K), cT))[0])
    assert best["cand"] == c_star and best["makespan"] == cT[c_star]
    q = host_u32(ticks)
    pi = O.base_order(q)
    rng = np.random.default_rng(5)
    for c in sorted(set([0, 1, 2, p.K - 1, c_star] + rng.integers(0, p.K, 40).tolist())):
        a, T, cm = O.run_candidate(q, p.plan, p.K, p.R, p.G, p.seed(1), c, order=pi)
        assert (T, cm) == (int(cT[c]), int(cC[c])), c
        if c == c_star:
            assert (host_u32(r["assign"]) == a).all()


def test_config4_full_search_plans_rebalanced(D, O, presets):
    """Config 4 at full size (P = 64 plans x K = 4,096): the per-plan T_B of Stage B for the
    Stage-A leader, the winner and the last plan re-derived by the oracle's balance of the
    same costs over the whole family."""
    p = presets[4]
    (t, f, x), (dt, df, dx) = feats(p, 0)
    res = D.search_plans_batches(p.model, dt, df, dx, [0, p.n], K=p.K, R=p.R, G=p.G, seed=p.seed(0),
                                 cluster=p.cluster, mem=p.mem(), gbs=p.gbs, top_p=p.top_p)
    mb, ms = O.batch_means(p.model, t, f, x)
    T_A, cfgs = O.stage_a_all(p.model, p.mem(), p.cluster["n_gpus"], p.cluster["gpus_per_node"], p.gbs, mb, ms)
    top = O.stage_a_top(T_A, p.top_p)
    obj = res["plan_objective"]
    win = res["stage_a_rank"]
    assert int(obj[win]) == res["makespan"] == min(int(v) for v in obj)
    for rank in sorted({0, win, len(top) - 1}):
        e, i = O.pair_to_config(cfgs, p.gbs, top[rank])
        c = cfgs[e]
        pl = dict(e_tp=int(c[0]), e_pp=int(c[1]), e_dp=int(c[2]), l_tp=int(c[3]), l_pp=int(c[4]), l_dp=int(c[5]),
                  n_mb=i)
        _, ticks = D.predict_costs(p.model, pl, dt, df, dx, want_f32=False)
        o = O.balance_threaded(host_u32(ticks), pl, p.K, p.R, p.G, p.seed(0), per_candidate=False)
        assert int(obj[rank]) == o["T"], rank
        if rank == win:
            assert res["cand"] == o["c"] and res["cmax"] == o["cmax"]


def test_global_item_table_path(D, O, presets):
    """n large enough that the per-CTA item table does not fit in shared memory (the kernel
    reads the records from global memory): parity on a window of candidates."""
    p = presets[5]
    t, f, x = (np.tile(a, 5)[:20000] for a in p.features(4))
    _, q, st, _ = O.predict(p.model, p.plan, t, f, x)
    assert st == 0
    check_balance(D, O, q, p.plan, 4096, 4, p.G, p.seed(4), 100, 148)


@pytest.mark.parametrize("k, over, c0, c1", [(2, None, 0, 512), (3, None, 0, 128), (5, None, 0, 16),
                                            (2, dict(l_dp=2, n_mb=8), 0, 256)])
def test_order4_mode_parity(D, O, presets, k, over, c0, c1):
    """DFLOP_MODE_ORDER4 (N4(a) per candidate, R37): per-candidate T bit-exact against the
    oracle's ORDER4 mode, never above the slot-order T."""
    p = presets[k]
    pl = dict(p.plan, **over) if over else p.plan
    (t, f, x), (dt, df, dx) = feats(p)
    _, ticks = D.predict_costs(p.model, pl, dt, df, dx, want_f32=False)
    q = host_u32(ticks)
    g, o = check_balance(D, O, q, pl, p.K, p.R, p.G, p.seed(0), c0, c1, mode=16)
    g0 = gpu_balance(D, dev_u32(q), pl, p.K, p.R, p.G, p.seed(0), c0, c1)
    assert (g["cT"] <= g0["cT"]).all() and (g["cC"] == g0["cC"]).all()


def test_order4_search_and_winner_order(D, O, presets):
    p = presets[3]
    (t, f, x), (dt, df, dx) = feats(p)
    res = D.search_plans(p.model, dt, df, dx, K=1024, R=p.R, G=p.G, seed=p.seed(0), plan=p.plan, order4=True)
    _, ticks = D.predict_costs(p.model, p.plan, dt, df, dx, want_f32=False)
    o = O.balance_threaded(host_u32(ticks), p.plan, 1024, p.R, p.G, p.seed(0), mode=16, per_candidate=False)
    assert res["makespan"] == o["T"] and res["cand"] == o["c"]
    # the winner's slot orders: the rounds = 0 order search of its assignment
    g = D.order_search(ticks, p.plan, res["assign"], rounds=0)
    assert g["makespan"] == res["makespan"]


def test_fuzz_random_shapes(D, O):
    """Random shapes through every balance code path (packed / plain / 64-bit variants, narrow
    and wide assignments, one- and two-sample LPT steps, CSR overflow and rebuilds, ORDER4)
    against the oracle, per candidate."""
    rng = np.random.default_rng(2026)
    for trial in range(80):
        n_mb = int(rng.choice([1, 2, 3, 5, 8, 16, 33, 64, 150]))
        l_dp = int(rng.choice([1, 1, 2, 3]))
        e_pp, l_pp = int(rng.integers(1, 4)), int(rng.integers(1, 6))
        pl = dict(e_tp=1, e_pp=e_pp, e_dp=1, l_tp=1, l_pp=l_pp, l_dp=l_dp, n_mb=n_mb)
        m = n_mb * l_dp
        n = int(rng.integers(0, 900))
        hi = int(rng.choice([50, 5000, 2 ** 20, 2 ** 27]))   # 2^27: 64-bit sums, makespans < 2^40
        q = rng.integers(0, hi, (4, n), dtype=np.uint64).astype(np.uint32)
        if rng.random() < 0.3 and n:                          # heavy tail
            q[:, rng.integers(0, n)] = np.uint32(min(hi * 40, 2 ** 31))
        G = int(rng.choice([1, 4, 8, 16]))
        R = int(rng.choice([0, 1, 6, 16]))
        mode = int(rng.choice([0, 0, 16]))
        K = 96
        c0 = int(rng.integers(0, K - 24))
        check_balance(D, O, q, pl, K, R, G, (trial, 7), c0, c0 + 24, mode=mode)


def test_makespan_overflow_flag(D):
    """Makespans >= 2^40 ticks do not fit the packed argmin key: the device status carries
    DFLOP_DEV_MAKESPAN_OVERFLOW (include/dflop.h) and the search reports OVERFLOW."""
    rng = np.random.default_rng(1)
    pl = dict(e_tp=1, e_pp=1, e_dp=1, l_tp=1, l_pp=2, l_dp=1, n_mb=4)
    q = rng.integers(2 ** 30, 2 ** 31, (4, 2000), dtype=np.uint64).astype(np.uint32)
    r = D.balance_microbatches(dev_u32(q), pl, 64, 2, 8, (1, 1))
    assert D.cand_result(r["best"])["status"] & D.DEV_MAKESPAN_OVERFLOW


def test_split_pipeline_selected_for_config5(D, presets, monkeypatch):
    """The bench workload runs the split pipeline by default (profile counts its chunks), and
    DFLOP_SPLIT=0 turns it off -- with the same winner."""
    monkeypatch.delenv("DFLOP_SPLIT", raising=False)
    p = presets[5]
    (t, f, x), (dt, df, dx) = feats(p, 0)
    _, ticks = D.predict_costs(p.model, p.plan, dt, df, dx, want_f32=False)
    K = 20000
    D.profile_read(reset=True)
    D.profile_enable(True)
    a = D.cand_result(D.balance_microbatches(ticks, p.plan, K, p.R, p.G, p.seed(0))["best"])
    pr = D.profile_read(reset=True)
    monkeypatch.setenv("DFLOP_SPLIT", "0")
    b = D.cand_result(D.balance_microbatches(ticks, p.plan, K, p.R, p.G, p.seed(0))["best"])
    pr0 = D.profile_read(reset=True)
    D.profile_enable(False)
    assert pr["split_chunks"] >= 1 and pr0["split_chunks"] == 0
    assert a == b


def test_split_pipeline_order4(D, O, presets, monkeypatch):
    """DFLOP_MODE_ORDER4 through the split pipeline (the ORDER4 instantiation of its candidate
    kernel): every candidate of a 3,000-candidate family equals the merged kernel's, and a
    window equals the oracle's ORDER4 mode."""
    p = presets[5]
    q = O.predict(p.model, p.plan, *p.features(3))[1]
    qd = dev_u32(q)
    K, seed = 3000, (5, 6)
    monkeypatch.setenv("DFLOP_SPLIT", "0")
    merged = gpu_balance(D, qd, p.plan, K, p.R, p.G, seed, 0, K, mode=16)
    monkeypatch.setenv("DFLOP_SPLIT", "2")
    monkeypatch.setenv("DFLOP_SPLIT_CHUNK", "1000")
    split = gpu_balance(D, qd, p.plan, K, p.R, p.G, seed, 0, K, mode=16)
    assert (split["cT"] == merged["cT"]).all() and (split["cC"] == merged["cC"]).all()
    assert split["best"] == merged["best"] and (split["assign"] == merged["assign"]).all()
    check_balance(D, O, q, p.plan, K, p.R, p.G, seed, 990, 1010, mode=16)


def test_split_pipeline_workspace_bound(D, presets):
    """The split pipeline's entries (n + 8m bytes per candidate) are sized for the chunk, which
    is capped at 2^20 candidates: config 5 at K = 10^6 holds them all, at K = 2^22 the chunk
    (and the workspace) stops growing."""
    p = presets[5]
    entry = p.n + 8 * p.plan["n_mb"] * p.plan["l_dp"]
    w1 = D.balance_workspace_bytes(p.n, p.plan, 10 ** 6, p.R, p.G)
    w4 = D.balance_workspace_bytes(p.n, p.plan, 1 << 22, p.R, p.G)
    assert w1 >= 10 ** 6 * entry
    assert w4 <= (1 << 20) * entry + (w1 - 10 ** 6 * entry) + (1 << 26)
