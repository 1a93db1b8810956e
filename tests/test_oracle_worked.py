"""Pins of the oracle's a1 (per-item durations) and Stage-A arithmetic at NON-UNIT model
shapes, against hand-derived worked examples (tests/golden/predict_worked.txt,
tests/golden/stage_a_worked.txt; each derivation written out in the file, from S:233,
P:486).  The unit-model pins of test_oracle_pins.py cannot tell 24*h^2
from 24*h, the encoder throughput queried at b from one queried at s, E_tp from L_tp, or
n-bar*s-bar^2 from t_seq^2; these fixtures can (test_worked_examples_reject_planted_errors compiles
mutated copies of the oracle and checks that each one fails them).
-m "not gpu".
"""
import os
from fractions import Fraction

import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _num(tok):
    """'57456/187' -> Fraction; '604.8' -> Fraction('604.8'); exact rationals throughout."""
    return Fraction(tok)


def _kv(tokens):
    out = {}
    for t in tokens:
        k, v = t.split("=")
        out[k] = v
    return out


def load_predict_fixture():
    model, plan, items, costs = {}, {}, [], []
    for raw in open(os.path.join(GOLD, "predict_worked.txt")):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        head, rest = line.split(None, 1)
        if head == "model":
            kv = _kv(rest.split())
            for k in ("e_layers", "e_hidden", "e_seq", "l_layers", "l_hidden", "tau_tile", "tau_frame"):
                model[k] = int(kv[k])
            model["bwd_ratio"] = float(kv["bwd_ratio"])
            model["tick_ns"] = float(kv["tick_ns"])
        elif head == "grid":
            name, xs, tps, vals = [p.strip() for p in rest.split("|")]
            x = [float(v) for v in xs.split("=")[1].split(",")]
            tp = [float(v) for v in tps.split("=")[1].split(",")]
            v = [[float(t) for t in row.split(",")] for row in vals.split(";")]
            assert len(v) == len(tp) and all(len(r) == len(x) for r in v)
            model[name] = dict(x=x, tp=tp, v=v)
        elif head == "plan":
            plan = {k: int(v) for k, v in _kv(rest.split()).items()}
        elif head == "item":
            nm, t, f, x = rest.split()
            items.append((nm, int(t), int(f), int(x)))
        elif head == "cost":
            left, right = rest.split("|")
            lt = left.split()
            costs.append(dict(e_attn=int(lt[0]), name=lt[1], ns=[_num(v) for v in lt[2:6]],
                              ticks=[int(v) for v in right.split()]))
    return model, plan, items, costs


def load_stage_a_fixture():
    rows = []
    for raw in open(os.path.join(GOLD, "stage_a_worked.txt")):
        line = raw.strip()
        if not line or line.startswith("#"):
            continue
        head, rest = line.split(None, 1)
        assert head == "pair"
        a, b, c = rest.split("|")
        t = a.split()
        rows.append(dict(name=t[0], e_attn=int(t[1]), cfg=[int(v) for v in t[2].split(",")], i=int(t[3]),
                         gbs=int(t[4]), b_bar=float(t[5]), s_bar=float(t[6]),
                         dur=[_num(v) for v in b.split()], want=[int(v) for v in c.split()]))
    return rows


def zero_mem():
    z = dict(l=[1.0, 2.0], tp=[1.0], x=[0.0], v=[[[0.0]], [[0.0]]])
    return dict(ms_e=dict(z), as_e=dict(z), ms_l=dict(z), as_l=dict(z), mem_per_gpu=1.0)


def test_fixture_self_consistent():
    """The fixture's tick columns are round-half-even of its exact ns columns, and the
    backward columns are twice the forward ones -- a typo guard on the file."""
    _, _, _, costs = load_predict_fixture()
    assert len(costs) == 10
    for c in costs:
        ef, eb, lf, lb = c["ns"]
        assert eb == 2 * ef and lb == 2 * lf
        assert c["ticks"] == [round(v) for v in c["ns"]]        # Python round() is half-even
    for r in load_stage_a_fixture():
        e, l = (round(v) for v in r["dur"])
        assert [e, l] == r["want"][:2]
        assert r["want"][2] == (r["i"] + r["cfg"][1] + r["cfg"][4] - 1) * max(e, l)


@pytest.mark.parametrize("e_attn", [0, 1])
def test_predict_worked_example(O, e_attn):
    model, plan, items, costs = load_predict_fixture()
    model = dict(model, e_attn=e_attn)
    t = [it[1] for it in items]
    f = [it[2] for it in items]
    x = [it[3] for it in items]
    cf, q, st, _ = O.predict(model, plan, t, f, x)
    assert st == 0
    want = [c for c in costs if c["e_attn"] == e_attn]
    assert [c["name"] for c in want] == [it[0] for it in items]
    for i, c in enumerate(want):
        for k in range(4):
            exact = float(c["ns"][k])
            if exact == 0.0:
                assert cf[k, i] == 0.0, (c["name"], k)              # b = 0 -> exactly 0
            else:
                assert abs(cf[k, i] - exact) <= 1e-12 * exact, (c["name"], k, cf[k, i], exact)
        assert [int(v) for v in q[:, i]] == c["ticks"], c["name"]


@pytest.mark.parametrize("row", range(4))
def test_stage_a_worked_example(O, row):
    model, _, _, _ = load_predict_fixture()
    r = load_stage_a_fixture()[row]
    model = dict(model, e_attn=r["e_attn"])
    res = O.stage_a_pair(model, zero_mem(), r["cfg"], r["i"], r["gbs"], r["b_bar"], r["s_bar"])
    assert res["feasible"]
    assert [res["e_dur"], res["l_dur"], res["T_A"]] == r["want"], (r["name"], r["e_attn"], res)


# ---------------------------------------------------------------- plant detection
# Mutation test: each plant is a plausible transcription error of the oracle's a1 /
# Stage-A arithmetic, applied textually to a copy of oracle/dflop_oracle.c, compiled, and run
# against the worked examples above; every mutant must FAIL them (VERDICT r01 "Next 1").
ORACLE_SRC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "dflop_oracle.c")


def _swap(text, a, b):
    return text.replace(a, "\x00").replace(b, a).replace("\x00", b)


PLANTS = {
    # 24*h instead of 24*h^2 -- encoder and LLM linear terms, a1 and Stage A
    "24h": lambda s: s.replace("24.0 * (double)m->e_hidden * (double)m->e_hidden", "24.0 * (double)m->e_hidden")
                      .replace("24.0 * (double)m->l_hidden * (double)m->l_hidden", "24.0 * (double)m->l_hidden"),
    # E_thr queried at the LLM length s instead of the encoder batch b ("b(d)")
    "E_thr_at_s": lambda s: s.replace("orc_interp_thr(&m->thr_e, bd,", "orc_interp_thr(&m->thr_e, sd,")
                             .replace("orc_interp_thr(&m->thr_e, t_bsz,", "orc_interp_thr(&m->thr_e, t_seq,"),
    # E_tp and L_tp swapped (query and divisor)
    "swap_tp": lambda s: _swap(s, "p->e_tp", "p->l_tp").replace(
        "uint32_t e_tp = cfg[0], e_pp = cfg[1], e_dp = cfg[2], l_tp = cfg[3],",
        "uint32_t e_tp = cfg[3], e_pp = cfg[1], e_dp = cfg[2], l_tp = cfg[0],"),
    # the encoder/LLM DP ratio of R13 dropped from a1
    "no_dp_ratio": lambda s: s.replace(" * ((double)p->l_dp / (double)p->e_dp)", ""),
    # Stage A's t_bsz divided by L_dp instead of E_dp
    "t_bsz_l_dp": lambda s: s.replace("(mean_b * (double)gbs) / ((double)i * (double)e_dp)",
                                      "(mean_b * (double)gbs) / ((double)i * (double)l_dp)"),
    # pipeline degree missing from the LLM divisor
    "no_l_pp": lambda s: s.replace("/ ((double)p->l_tp * (double)p->l_pp)", "/ ((double)p->l_tp)")
                          .replace("/ ((double)l_tp * (double)l_pp)", "/ ((double)l_tp)"),
    # t_seq^2 instead of n-bar * s-bar^2 for Stage-A attention (R5)
    "t_seq_sq": lambda s: s.replace("nbar * (c_att * mean_s * mean_s)", "(c_att * t_seq * t_seq)"),
}
EXPECT = {"24h": ("predict", "stage_a"), "E_thr_at_s": ("predict", "stage_a"), "swap_tp": ("predict", "stage_a"),
          "t_seq_sq": ("stage_a",), "no_dp_ratio": ("predict",), "t_bsz_l_dp": ("stage_a",),
          "no_l_pp": ("predict", "stage_a")}


def _fails(fn, *a):
    try:
        fn(*a)
    except AssertionError:
        return True
    return False


@pytest.mark.parametrize("plant", sorted(PLANTS))
def test_worked_examples_reject_planted_errors(O, monkeypatch, plant):
    src = open(ORACLE_SRC).read()
    mutated = PLANTS[plant](src)
    assert mutated != src, f"plant {plant} no longer applies to the oracle source"
    handle = O.load(O.build_variant(mutated, plant))
    monkeypatch.setattr(O, "_lib", handle)
    fails = {
        "predict": any(_fails(test_predict_worked_example, O, ea) for ea in (0, 1)),
        "stage_a": any(_fails(test_stage_a_worked_example, O, r) for r in range(4)),
    }
    for which in EXPECT[plant]:
        assert fails[which], f"plant {plant} survives the {which} worked example"
