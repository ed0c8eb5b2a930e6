"""Pins for oracle/rules.py: Brent identities, the App. A convention, Table 1, the Sec. 4.4
stability factors and the Thm 4.3 / 4.4 bound formulas.  Every expected value here is printed
in the paper (cited) or is a closed form the paper states."""
from fractions import Fraction

import numpy as np
import pytest

from oracle import rules as R
from fmm_testutil import golden, read_golden_matrices


def _golden_rule(name, fname, m0, k0, n0):
    g = read_golden_matrices(fname)
    return R.make_rule(name, m0, k0, n0, g["U"], g["V"], g["W"])


def app_b_323():
    return _golden_rule("app_b_323", "app_b_323.txt", 3, 2, 3)


@pytest.mark.parametrize("name", sorted(R.BUILTINS))
def test_builtin_rules_satisfy_brent(name):
    # Eq. eqn:bilinear_alg holds for all A, B iff the Brent equations hold.
    assert R.brent_violations(R.builtin(name)) == []


def test_app_a_printed_is_transposed_convention():
    # P:1993 states U/V column-major, W row-major; the printed table only satisfies the Brent
    # equations with U/V row-major and W column-major (reading A1).
    g = read_golden_matrices("app_a_strassen_printed.txt")
    printed = R.make_rule("printed", 2, 2, 2, g["U"], g["V"], g["W"])
    assert len(R.brent_violations(printed, ("col", "col", "row"))) > 0
    assert R.brent_violations(printed, ("row", "row", "col")) == []
    # the oracle's Strassen = printed with rows 2 and 3 (1-based) swapped
    s = R.strassen()
    for X, P in ((s.U, g["U"]), (s.V, g["V"]), (s.W, g["W"])):
        P = [P[0], P[2], P[1], P[3]]
        assert [[int(x) for x in row] for row in X] == P


def test_app_b_323_is_valid_under_stated_convention():
    assert R.brent_violations(app_b_323()) == []


def test_brent_check_detects_a_single_sign_flip():
    s = R.strassen()
    W = [list(r) for r in s.W]
    W[0][3] = -W[0][3]
    bad = R.make_rule("bad", 2, 2, 2, s.U, s.V, W)
    assert len(R.brent_violations(bad)) > 0


def test_table1_principal_quantities():
    # Table 1: R, nnz, Q, E
    rows = {}
    for line in golden("table1.txt").read_text().splitlines():
        if line.strip() and not line.startswith("#"):
            n, *v = line.split()
            rows[n] = tuple(int(x) for x in v)
    rules = {"classical222": R.classical222(), "strassen": R.strassen(), "app_b_323": app_b_323()}
    for name, (Rk, nnz, Q, E) in rows.items():
        q = R.quantities(rules[name])
        assert (rules[name].R, q.nnz, q.Q, q.E) == (Rk, nnz, Q, E), name


def test_stability_vectors_printed_in_sec_4_4():
    # Strassen e = [12 4 4 12]; <3,2,3> e printed as [20 20 2 12 4 20 4 12 20],
    # which is the column-major order of C (reading A20).
    assert R.quantities(R.strassen()).e == [12, 4, 4, 12]
    e = R.quantities(app_b_323()).e  # row-major k = ia*3 + jb
    col_major = [e[ia * 3 + jb] for jb in range(3) for ia in range(3)]
    assert col_major == [20, 20, 2, 12, 4, 20, 4, 12, 20]


def test_abg_equal_ab_for_unit_coefficients():
    # when U and V have +-1 entries, alpha = a and beta = b.
    for name in R.BUILTINS:
        q = R.quantities(R.builtin(name))
        assert q.alpha == q.a and q.beta == q.b


def test_dalberto_xi():
    # uniform two-level Strassen xi = 12^2 = 144; D'Alberto's plan gives 96.
    s = R.strassen()
    assert R.xi_nonuniform([[s], [s] * 7]) == 144
    assert R.xi_nonuniform(R.Plan.dalberto_two_level().levels) == 96
    assert R.brent_violations(R.strassen_dalberto()) == []


def _perm323(P, base):
    P = np.array(P)
    I2 = np.eye(2, dtype=int)
    U = R._kron_rows(I2, P, base.U)
    V = R._kron_rows(P, I2, base.V)
    W = R._kron_rows(P, P, base.W)
    return R.make_rule(base.name + "_v", 3, 2, 3, U, V, W)


def test_323_three_variant_plan_xi():
    # uniform two-level xi = 400, three-variant plan = 352.
    b = app_b_323()
    v1 = _perm323([[1, 0, 0], [0, 0, 1], [0, 1, 0]], b)
    v2 = _perm323([[0, 1, 0], [0, 0, 1], [1, 0, 0]], b)
    assert R.brent_violations(v1) == [] and R.brent_violations(v2) == []
    assert R.xi_nonuniform([[b], [b] * 15]) == 400
    lvl2 = []
    for r1 in range(1, 16):
        if r1 in (1, 3, 10, 11):
            lvl2.append(v1)
        elif r1 in (4, 5, 7, 9, 12, 13):
            lvl2.append(v2)
        else:
            lvl2.append(b)
    assert R.xi_nonuniform([[b], lvl2]) == 352


@pytest.mark.parametrize("xyz", [(x, y, z) for x in (1, 2) for y in (1, 2) for z in (1, 2)])
def test_castrapel_gustafson_variants_valid(xyz):
    # all eight (P^x (x) P^y)U, (P^z (x) P^x)V, (P^y (x) P^z)W variants are algorithms.
    for base in (R.winograd(), R.strassen()):
        assert R.brent_violations(R.castrapel_gustafson(base, *xyz)) == []


def test_bound_closed_forms():
    s = R.strassen()
    # L = 0: K^2
    assert R.stationary_bound_factor(s, 0, 1000) == 1000 ** 2
    # full recursion: (1 + Q L) E^{log_K0 K}
    assert R.stationary_bound_factor(s, 10, 1024) == (1 + 8 * 10) * 12 ** 10
    # L = 1, K = 1024: (512 + 8) * 512 * 12 (Thm stationary_analysis)
    assert R.stationary_bound_factor(s, 1, 1024) == (512 + 8) * 512 * 12
    # uniform non-stationary with one rule repeated = stationary (P:395-397 vs P:270)
    for L in range(4):
        assert R.uniform_bound_factor([s] * L, 4096) == R.stationary_bound_factor(s, L, 4096)
    # empty sequence = K^2
    assert R.uniform_bound_factor([], 77) == 77 ** 2


def test_winograd_derived_quantities():
    # Not printed in the paper (P:474 only says "slightly larger stability factor" than 12);
    # derived from the Brent-valid table: nnz 42, Q 10, E 18.
    q = R.quantities(R.winograd())
    assert (q.nnz, q.Q, q.E) == (42, 10, 18)
    assert q.E > 12


# ---- App. C <4,4,2;26> ------------------------------------------------------------
# DESIGN.md reading A27: the printed rows are a relabelling of A's, B's and C's entries; these
# labels (found by matching each row's Brent slice) make the printed table an exact algorithm.
APP_C_LABELS = {
    "U": [(0, 0), (2, 0), (1, 0), (3, 0), (0, 2), (2, 2), (1, 2), (3, 2),
          (0, 1), (2, 1), (1, 1), (3, 1), (0, 3), (2, 3), (1, 3), (3, 3)],
    "V": [(0, 0), (1, 0), (0, 1), (1, 1), (2, 0), (3, 0), (2, 1), (3, 1)],
    "W": [(0, 0), (1, 0), (0, 1), (1, 1), (2, 0), (3, 0), (2, 1), (3, 1)],
}


def app_c_442():
    g = read_golden_matrices("app_c_442.txt")
    return R.make_rule_labelled("app_c_442", 4, 4, 2, g["U"], g["V"], g["W"],
                                APP_C_LABELS["U"], APP_C_LABELS["V"], APP_C_LABELS["W"],
                                u_den=2, v_den=2)


def test_app_c_442_printed_order_is_not_the_stated_convention():
    g = read_golden_matrices("app_c_442.txt")
    half = lambda X: [[Fraction(x, 2) for x in r] for r in X]
    printed = R.make_rule("printed442", 4, 4, 2, half(g["U"]), half(g["V"]), g["W"])
    assert len(R.brent_violations(printed)) > 0


def test_app_c_442_relabelled_is_exact_and_matches_table1():
    rule = app_c_442()
    assert R.brent_violations(rule) == []
    q = R.quantities(rule)
    # Table 1 row <4,4,2>: R 26, nnz 257, Q 22, E 89; Ex. better_emax: E = 89
    assert (rule.R, q.nnz, q.Q, q.E) == (26, 257, 22, 89)
    # U and V carry +-1/2 entries, so a, b (1-norms) differ from alpha, beta (counts)
    assert q.a != q.alpha


def test_app_c_442_transpose_via_vec_permutation_keeps_E():
    # <P42 V, P44 U, P24 W> is a <2,4,4> algorithm with the same E; its cyclic
    # rotation [[V, W, U]] is the <4,2,4> row of Table 1 (Q 23, E 92; A21).
    rule = app_c_442()
    rot = R.make_rule("rot424", 4, 2, 4, rule.V, rule.W, rule.U)
    assert R.brent_violations(rot) == []
    q = R.quantities(rot)
    assert (q.nnz, q.Q, q.E) == (257, 23, 92)
