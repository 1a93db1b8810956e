"""Host-side checks of the C-ABI library (no compute calls, no GPU): it loads, exports every
symbol include/dflop.h declares, and the ctypes struct layouts match the C header
(sizeof/offsetof printed by a gcc-compiled probe of include/dflop.h).  -m "not gpu".
"""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dflop.h")


@pytest.fixture(scope="module")
def D():
    from paper_2603_25120_b200 import _build, dflop
    _build.build()
    return dflop


def declared_functions():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:dflop_status|uint32_t|uint64_t|const char\*)\s+(dflop_\w+)\(", src, re.M)))


def test_exports_every_declared_symbol(D):
    names = declared_functions()
    assert len(names) == 21
    assert sorted(names) == sorted(D.EXPORTS)
    out = subprocess.run(["nm", "-D", "--defined-only", D.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (dflop_\w+)", out))
    assert set(names) <= exported


def test_abi_version_and_last_error(D):
    assert D.abi_version() == 5
    assert D.lib().dflop_last_error() == b""


def test_validation_without_gpu(D, presets):
    # argument validation happens before any CUDA call: a bad struct_size is rejected
    m = D.cost_model_struct(presets[1].model)
    m.struct_size = 3
    pl = D.plan_struct(presets[1].plan)
    code = D.lib().dflop_predict_costs(C.byref(m), C.byref(pl), None, None, None, 0, None, None, None, None)
    assert code == 1 and b"struct_size" in D.lib().dflop_last_error()
    m = D.cost_model_struct(presets[1].model)
    m.thr_e.v[0][3] = -1.0
    code = D.lib().dflop_predict_costs(C.byref(m), C.byref(pl), None, None, None, 0, None, None, None, None)
    assert code == 1 and b"thr_e" in D.lib().dflop_last_error()
    code = D.lib().dflop_simulate_1f1b(None, None, 1, 0, 4, None, None, None)
    assert code == 2
    # exact solver: m = n_mb * l_dp computed in 64 bits (65536 * 65536 must not wrap to 0)
    big = D.plan_struct(dict(e_tp=1, e_pp=1, e_dp=1, l_tp=1, l_pp=1, l_dp=65536, n_mb=65536))
    need = C.c_size_t(0)
    code = D.lib().dflop_exact_cmax(None, 0, C.byref(big), C.c_uint64(1), None, None, C.byref(need), None, None, None)
    assert code == 1 and b"65535" in D.lib().dflop_last_error()
    wide = D.plan_struct(dict(e_tp=1, e_pp=1, e_dp=1, l_tp=1, l_pp=1, l_dp=2, n_mb=200))
    code = D.lib().dflop_exact_cmax(None, 0, C.byref(wide), C.c_uint64(1), None, None, C.byref(need), None, None, None)
    assert code == 1 and b"> 256" in D.lib().dflop_last_error()
    # the library's caches are released (nothing allocated on a CPU-only host)
    assert D.lib().dflop_release_caches() == 0


PROBE = r"""
#include <stdio.h>
#include <stddef.h>
#include "dflop.h"
#define S(t) printf(#t " %zu\n", sizeof(t));
#define F(t, f) printf(#t "." #f " %zu\n", offsetof(t, f));
int main(void) {
  S(dflop_grid) S(dflop_mem_grid) S(dflop_cost_model) S(dflop_mem_model) S(dflop_plan) S(dflop_cluster)
  S(dflop_balance_params) S(dflop_cand_result) S(dflop_search_params) S(dflop_plan_result) S(dflop_profile)
  S(dflop_correction) F(dflop_correction, rho) S(dflop_exact_result) F(dflop_exact_result, makespan)
  F(dflop_cost_model, bwd_ratio) F(dflop_cost_model, thr_e) F(dflop_cost_model, thr_lin)
  F(dflop_cost_model, correction)
  F(dflop_mem_model, ms_e) F(dflop_mem_model, mem_per_gpu) F(dflop_balance_params, id_base)
  F(dflop_search_params, fixed_plan) F(dflop_search_params, seed) F(dflop_plan_result, makespan)
  F(dflop_plan_result, alg1_plan) F(dflop_plan_result, alg1_makespan) F(dflop_plan_result, n_candidates)
  return 0;
}
"""


def test_struct_layouts_match_header(D, tmp_path):
    src = tmp_path / "probe.c"
    src.write_text(PROBE)
    exe = tmp_path / "probe"
    subprocess.check_call(["gcc", "-std=c11", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    got = dict(line.split() for line in subprocess.check_output([str(exe)], text=True).splitlines())
    m = {"dflop_grid": D.Grid, "dflop_mem_grid": D.MemGrid, "dflop_cost_model": D.CostModel,
         "dflop_mem_model": D.MemModel, "dflop_plan": D.Plan, "dflop_cluster": D.Cluster,
         "dflop_balance_params": D.BalanceParams, "dflop_cand_result": D.CandResult,
         "dflop_search_params": D.SearchParams, "dflop_plan_result": D.PlanResult, "dflop_profile": D.Profile,
         "dflop_correction": D.Correction, "dflop_exact_result": D.ExactResult}
    for k, v in got.items():
        if "." in k:
            s, f = k.split(".")
            assert getattr(m[s], f).offset == int(v), k
        else:
            assert C.sizeof(m[k]) == int(v), k
