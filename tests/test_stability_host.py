"""Stability analysis (Sec. 4): the library's host-side fmm_rule_quantities / fmm_plan_stability
/ fmm_choose_variants (product code, no GPU) against the oracle's exact Fraction analysis and
the values the paper prints (Table 1)."""
import itertools
from fractions import Fraction

import numpy as np
import pytest

import paper_1507_00687_b200 as fb
from oracle import rules as R
from test_gpu_rules import to_gpu_rule
from test_oracle_rules import _perm323, app_b_323, app_c_442


def test_xi_simplified_equals_unsimplified_definition():
    # P:449-453 vs the simplified product form P:455-463 (oracle pinned against itself by
    # two different formulas) on uniform, D'Alberto and random Castrapel-Gustafson plans
    s, w = R.strassen(), R.winograd()
    cg = [R.castrapel_gustafson(w, x, y, z) for x in (1, 2) for y in (1, 2) for z in (1, 2)]
    plans = [[[s], [s] * 7], R.Plan.dalberto_two_level().levels, [[w], [cg[(3 * r) % 8] for r in range(7)]]]
    for pl in plans:
        assert R.xi_nonuniform(pl) == R.xi_nonuniform_full(pl)


def test_delta_closed_forms():
    # L = 1: delta = K/K0 + max_k (gamma_k + max_r (alpha_r + beta_r) I(w_kr != 0)) = K/K0 + Q
    for rule in (R.strassen(), R.winograd(), R.classical222(), app_b_323()):
        assert R.delta_nonuniform([[rule]], 1024) == Fraction(1024, rule.k0) + R.quantities(rule).Q
    # uniform plans: delta <= K/prod K0 + sum Q (the Thm 4.4 first factor)
    s = R.strassen()
    assert R.delta_nonuniform([[s], [s] * 7], 4096) <= 1024 + 2 * 8


@pytest.mark.parametrize("maker", [R.classical222, R.strassen, R.winograd, R.strassen_dalberto,
                                   app_b_323, app_c_442])
def test_rule_quantities_match_oracle(maker):
    rule = maker()
    g = to_gpu_rule(fb, rule).quantities()
    q = R.quantities(rule)
    assert g["nnz"] == q.nnz and g["Q"] == q.Q and g["E"] == q.E
    assert list(g["q"]) == [float(x) for x in q.q] and list(g["e"]) == [float(x) for x in q.e]


def test_rule_quantities_table1_values():
    # Table 1: (nnz, Q, E) for classical, Strassen, <3,2,3>, <4,4,2>
    want = {"classical222": (24, 4, 2), "strassen": (36, 8, 12)}
    for name, (nnz, Q, E) in want.items():
        g = fb.Rule.builtin(name).quantities()
        assert (g["nnz"], g["Q"], g["E"]) == (nnz, Q, E)
    g = to_gpu_rule(fb, app_b_323()).quantities()
    assert (g["nnz"], g["Q"], g["E"]) == (94, 10, 20)
    g = to_gpu_rule(fb, app_c_442()).quantities()
    assert (g["nnz"], g["Q"], g["E"]) == (257, 22, 89)


def _gplan(rules_by_level, dims=(1024, 1024, 1024)):
    nodes = [to_gpu_rule(fb, r) for lvl in rules_by_level for r in lvl]
    return fb.Plan(nodes, *dims, uniform=False, levels=len(rules_by_level))


def test_plan_xi_paper_examples():
    s = R.strassen()
    # uniform two-level Strassen 144, D'Alberto 96
    assert _gplan([[s], [s] * 7]).stability()["xi"] == 144
    assert _gplan(R.Plan.dalberto_two_level().levels).stability()["xi"] == 96
    # <3,2,3> uniform 400, three-variant plan 352
    b = app_b_323()
    v1 = _perm323([[1, 0, 0], [0, 0, 1], [0, 1, 0]], b)
    v2 = _perm323([[0, 1, 0], [0, 0, 1], [1, 0, 0]], b)
    lvl2 = [v1 if r in (1, 3, 10, 11) else v2 if r in (4, 5, 7, 9, 12, 13) else b for r in range(1, 16)]
    assert _gplan([[b], [b] * 15], (3 * 9 * 8, 4 * 8, 9 * 8)).stability()["xi"] == 400
    assert _gplan([[b], lvl2], (3 * 9 * 8, 4 * 8, 9 * 8)).stability()["xi"] == 352


def test_plan_stability_matches_oracle_on_random_plans():
    w = R.winograd()
    cg = [R.castrapel_gustafson(w, x, y, z) for x in (1, 2) for y in (1, 2) for z in (1, 2)]
    rng = np.random.default_rng(0)
    for _ in range(5):
        lvl2 = [cg[i] for i in rng.integers(0, 8, 7)]
        lvl3 = [cg[i] for i in rng.integers(0, 8, 49)]
        levels = [[w], lvl2, lvl3]
        st = _gplan(levels, (512, 512, 512)).stability()
        assert st["xi"] == R.xi_nonuniform(levels)
        assert st["delta"] == R.delta_nonuniform(levels, 512)
        assert np.isnan(st["uniform_bound"])
    # uniform: the Thm 4.4 factor
    st = fb.Plan([fb.Rule.builtin("winograd")] * 3, 4096, 4096, 4096).stability()
    assert st["uniform_bound"] == R.uniform_bound_factor([w] * 3, 4096)
    assert st["xi"] == R.quantities(w).E ** 3


def test_choose_variants_is_the_brute_force_minimum():
    s, d = R.strassen(), R.strassen_dalberto()
    choice, xi = fb.choose_variants(fb.Rule.builtin("strassen"),
                                    [fb.Rule.builtin("strassen"), fb.Rule.builtin("strassen_dalberto")])
    brute = min(R.xi_nonuniform([[s], [[s, d][c] for c in combo]])
                for combo in itertools.product(range(2), repeat=7))
    assert xi == brute <= 96  # the paper's D'Alberto plan reaches 96
    assert R.xi_nonuniform([[s], [[s, d][c] for c in choice]]) == xi
    # Strassen-Winograd with the eight Castrapel-Gustafson variants
    w = R.winograd()
    cg = [R.castrapel_gustafson(w, x, y, z) for x in (1, 2) for y in (1, 2) for z in (1, 2)]
    choice, xi = fb.choose_variants(to_gpu_rule(fb, w), [to_gpu_rule(fb, v) for v in cg])
    assert R.xi_nonuniform([[w], [cg[c] for c in choice]]) == xi
    assert xi <= R.quantities(w).E ** 2


def test_rule_transforms_validate_and_match_table1():
    # App. A: Strassen's rotations share Q, E; App. B: [[W,U,V]] is the <3,3,2> row of
    # Table 1 (nnz 94, Q 11, E 23); App. C: transposition keeps E = 89, the
    # rotations give (26, 102) and the <4,2,4> row (23, 92) (reading A21)
    s = fb.Rule.builtin("strassen")
    for kind in ("rotate", "rotate2", "transpose"):
        q = s.transform(kind).quantities()
        assert (q["Q"], q["E"]) == (8, 12)
    b = to_gpu_rule(fb, app_b_323())
    r1 = b.transform("rotate")
    assert (r1.info()["m0"], r1.info()["k0"], r1.info()["n0"]) == (3, 3, 2)
    q = r1.quantities()
    assert (q["nnz"], q["Q"], q["E"]) == (94, 11, 23)
    c = to_gpu_rule(fb, app_c_442())
    assert c.transform("transpose").quantities()["E"] == 89
    q1, q2 = c.transform("rotate").quantities(), c.transform("rotate2").quantities()
    assert (q1["Q"], q1["E"]) == (26, 102) and (q2["Q"], q2["E"]) == (23, 92)
    # transposition is an involution up to the table itself
    t2 = c.transform("transpose").transform("transpose").info()
    ci = c.info()
    for key in ("U", "V", "W"):
        assert np.array_equal(t2[key], ci[key])
