"""Pins for the oracle executor (oracle/fmm_oracle.c via oracle.fmm) and the double-double
reference.  Anchors: exact integer products, brute-force rationals, the classical definition,
the summation-order reading A3 on a hand-computed case, the Thm 4.3/4.4 bounds against the
double-double reference, and structural invariants (row sampling, padding, determinism)."""
from fractions import Fraction

import numpy as np
import pytest

import fmm_inputs as fi
from oracle import rules as R
from oracle.rules import Plan

EPS64 = 2.0 ** -53


def _plans():
    s, w, c = R.strassen(), R.winograd(), R.classical222()
    return {
        "strassen_L1": Plan.stationary(s, 1),
        "strassen_L3": Plan.stationary(s, 3),
        "winograd_L2": Plan.stationary(w, 2),
        "winograd_L3": Plan.stationary(w, 3),
        "classical_L2": Plan.stationary(c, 2),
        "C3_mix": Plan.uniform([w, c, s]),
        "dalberto": Plan.dalberto_two_level(),
    }


@pytest.mark.parametrize("pname", sorted(_plans()))
def test_integer_inputs_give_exact_product(orc, pname):
    # SPEC S:292-294 / S:317: integer inputs with all intermediates < 2^53 -> exact A@B.
    plan = _plans()[pname]
    A, B = fi.integer_pair(48, 64, 40, seed=11)
    Cx = orc.fmm(A, B, plan)  # padded internally when dims are not multiples of 2^L
    Ci = A.astype(np.int64) @ B.astype(np.int64)
    assert np.array_equal(Cx, Ci.astype(np.float64))


def test_identity_exact(orc):
    # I x I = I exactly.
    I = np.eye(16)
    for plan in _plans().values():
        assert np.array_equal(orc.fmm(I, I, plan), I)


def test_brute_force_rationals_tiny(orc):
    # Exact rational A@B vs the FMM in double: within the Thm 4.3 bound, with dyadic inputs.
    rng = np.random.default_rng(5)
    for n in (2, 4, 8):
        A = rng.integers(-1000, 1000, (n, n)) / 1024.0
        B = rng.integers(-1000, 1000, (n, n)) / 512.0
        exact = [[sum(Fraction(A[i, k]) * Fraction(B[k, j]) for k in range(n)) for j in range(n)]
                 for i in range(n)]
        for rule in (R.strassen(), R.winograd()):
            L = int(np.log2(n))
            Cx = orc.fmm(A, B, Plan.stationary(rule, L))
            err = max(abs(Fraction(Cx[i, j]) - exact[i][j]) for i in range(n) for j in range(n))
            f = R.stationary_bound_factor(rule, L, n)
            assert float(err) <= float(f) * np.abs(A).max() * np.abs(B).max() * EPS64


def test_L0_is_the_classical_sequential_loop(orc):
    # L = 0: the classical algorithm, k ascending from 0.0 (reading A4).
    A, B = fi.random_pair(7, 9, 5, seed=3)
    Cx = orc.fmm(A, B, Plan([]))
    for i in range(7):
        for j in range(5):
            c = np.float64(0.0)
            for k in range(9):
                c = c + A[i, k] * B[k, j]
            assert Cx[i, j] == c


def test_summation_order_is_ascending_index():
    # Reading A3: S_r = sum_i u_ir A_i accumulated sequentially with i ascending.  Winograd
    # column M3 has U = (A11:+1, A21:-1, A12:+1, A22:-1) (i = ia + 2 ja).  With 1x1 blocks
    # A11 = 2^53, A21 = -1, A12 = -2^53, A22 = -1:
    #   ((2^53 - (-1)) + (-2^53)) - (-1) = (2^53 + 0) - 2^53 + 1 = 1   (2^53 + 1 rounds to 2^53)
    # whereas the exact value is 2.  Hand-computed, not taken from the oracle.
    import oracle
    w = R.winograd()
    A = np.array([[2.0 ** 53, -(2.0 ** 53)], [-1.0, -1.0]])  # [[A11, A12], [A21, A22]]
    B = np.ones((2, 2))
    S, _ = oracle.node_st(w, A, B)
    assert S[2, 0, 0] == 1.0
    # and C accumulation r ascending: Winograd C12 = M1 + M3 + M5 + M6; with M = (2^53, 0, 1, 0,
    # -2^53, 1, 0): ((2^53 + 1) + (-2^53)) + 1 = 2^53 - 2^53 + 1 = 1 (exact: 2)
    Ms = np.array([2.0 ** 53, 0.0, 1.0, 0.0, -(2.0 ** 53), 1.0, 0.0]).reshape(7, 1, 1)
    Cn = oracle.node_c(w, Ms)
    assert Cn[0, 1] == 1.0


def test_uniform_tree_equals_stationary_bitwise(orc):
    # a tree plan whose nodes hold the same rule (here as distinct Rule objects with equal
    # coefficients) is bitwise identical to the stationary plan.
    s = R.strassen()
    s2 = R.make_rule("strassen_copy", 2, 2, 2, s.U, s.V, s.W)
    A, B = fi.random_pair(64, 64, 64, seed=2)
    tree = Plan([[s], [s2 if r % 2 else s for r in range(7)]])
    assert np.array_equal(orc.fmm(A, B, tree), orc.fmm(A, B, Plan.stationary(s, 2)))


def test_deterministic_across_calls(orc):
    A, B = fi.random_pair(128, 128, 128, seed=9)
    p = Plan.stationary(R.winograd(), 2)
    assert np.array_equal(orc.fmm(A, B, p), orc.fmm(A, B, p))


def test_padding_neutral(orc):
    # unpadded dims = crop of a manual zero-padded run.
    A, B = fi.random_pair(37, 50, 29, seed=4)
    p = Plan.stationary(R.winograd(), 2)
    Ap = np.zeros((40, 52))
    Ap[:37, :50] = A
    Bp = np.zeros((52, 32))
    Bp[:50, :29] = B
    assert np.array_equal(orc.fmm(A, B, p), orc.fmm(Ap, Bp, p)[:37, :29])


def test_row_sampling_is_bitwise(orc):
    # the oracle on A[G,:] with all of B equals rows G of the full oracle run.
    A, B = fi.random_pair(256, 128, 96, seed=6)
    for plan in (Plan.stationary(R.winograd(), 3), Plan.uniform([R.winograd(), R.classical222(),
                                                                   R.strassen()])):
        full = orc.fmm(A, B, plan)
        G = orc.lift_rows(256, plan, [0, 5, 31])
        assert len(G) == 8 * 3
        assert np.array_equal(orc.fmm_rows(A, B, plan, G), full[G])


def test_row_col_sampling_is_bitwise(orc):
    A, B = fi.random_pair(128, 64, 256, seed=16)
    for plan in (Plan.stationary(R.winograd(), 3), Plan.dalberto_two_level()):
        full = orc.fmm(A, B, plan)
        G = orc.lift_rows(128, plan, [1, 7])
        H = orc.lift_cols(256, plan, [0, 3, 30])
        assert np.array_equal(orc.fmm_sub(A, B, plan, G, H), full[np.ix_(G, H)])


@pytest.mark.parametrize("pname", ["winograd_L2", "strassen_L3", "C3_mix", "dalberto",
                                   "classical_L2"])
def test_bound_holds_against_double_double(orc, pname):
    # Thm stationary_analysis / non_stationary: ||C^ - C|| <= f ||A|| ||B|| eps.
    plan = _plans()[pname]
    A, B = fi.random_pair(256, 256, 256, seed=8)
    Cx = orc.fmm(A, B, plan)
    hi, lo = orc.ref_dd(A, B)
    err = np.max(np.abs((Cx - hi) - lo))
    f = R.uniform_bound_factor([lv[0] for lv in plan.levels], 256) if pname != "dalberto" else \
        R.stationary_bound_factor(R.strassen(), 2, 256)
    assert err <= float(f) * np.abs(A).max() * np.abs(B).max() * EPS64
    assert err > 0  # the computation really rounds


def test_C1_full_size_bound(orc):
    # C1 (BASELINE configs[0]): S-W L=2, 512^3, U(-1,1) seed 0.
    A, B = fi.config_inputs("C1")
    plan = Plan.stationary(R.winograd(), 2)
    Cx = orc.fmm(A, B, plan)
    hi, lo = orc.ref_dd(A, B)
    err = np.max(np.abs((Cx - hi) - lo))
    f = float(R.stationary_bound_factor(R.winograd(), 2, 512))
    assert err <= f * np.abs(A).max() * np.abs(B).max() * EPS64


def test_f32_executor_integer_exact_and_bound(orc):
    A, B = fi.integer_pair(64, 64, 64, seed=1)
    p = Plan.stationary(R.winograd(), 3)
    Cx = orc.fmm(A.astype(np.float32), B.astype(np.float32), p)
    assert Cx.dtype == np.float32
    assert np.array_equal(Cx.astype(np.int64), A.astype(np.int64) @ B.astype(np.int64))
    A, B = fi.random_pair(128, 128, 128, seed=1, dtype=np.float32)
    Cx = orc.fmm(A, B, p)
    hi, lo = orc.ref_dd(A.astype(np.float64), B.astype(np.float64))
    err = np.max(np.abs((Cx.astype(np.float64) - hi) - lo))
    f = float(R.stationary_bound_factor(R.winograd(), 3, 128))
    assert err <= f * np.abs(A).max() * np.abs(B).max() * 2.0 ** -24


# ---- double-double reference pins ---------------------------------------------------------

def test_dd_exact_on_integers(orc):
    # exact on integer inputs < 2^25 with K <= 2^10.
    g = np.random.default_rng(0)
    A = g.integers(-(2 ** 24), 2 ** 24, (8, 1024)).astype(np.float64)
    B = g.integers(-(2 ** 24), 2 ** 24, (1024, 8)).astype(np.float64)
    hi, lo = orc.ref_dd(A, B)
    exact = [[sum(int(A[i, k]) * int(B[k, j]) for k in range(1024)) for j in range(8)]
             for i in range(8)]
    for i in range(8):
        for j in range(8):
            assert Fraction(hi[i, j]) + Fraction(lo[i, j]) == exact[i][j]


def test_dd_matches_fractions(orc):
    A, B = fi.random_pair(3, 200, 4, seed=12)
    hi, lo = orc.ref_dd(A, B)
    for i in range(3):
        for j in range(4):
            ex = sum(Fraction(A[i, k]) * Fraction(B[k, j]) for k in range(200))
            s = sum(abs(Fraction(A[i, k]) * Fraction(B[k, j])) for k in range(200))
            assert abs(Fraction(hi[i, j]) + Fraction(lo[i, j]) - ex) <= s * Fraction(1, 2 ** 100)
            assert hi[i, j] == float(Fraction(hi[i, j]) + Fraction(lo[i, j]))


def test_dd_row_subset(orc):
    A, B = fi.random_pair(16, 32, 8, seed=2)
    hi, lo = orc.ref_dd(A, B)
    hs, ls = orc.ref_dd(A, B, rows=[3, 11])
    assert np.array_equal(hs, hi[[3, 11]]) and np.array_equal(ls, lo[[3, 11]])


def _three_level_nonuniform():
    """Root S-W; level 1 (7 nodes, BFS index r1) and level 2 (49 nodes, BFS index 7 r1 + r2,
    P:147-149) draw from ten 7-product 2x2x2 rules -- Strassen, its D'Alberto variant and the
    eight Castrapel-Gustafson variants of S-W -- by a function of the index that
    is not symmetric in (r1, r2), so a wrong mixed-radix node order changes which rule runs
    where."""
    w = R.winograd()
    pool = [R.strassen(), R.strassen_dalberto()] + [
        R.castrapel_gustafson(w, x, y, z) for x in (1, 2) for y in (1, 2) for z in (1, 2)]
    lvl1 = [pool[(3 * r1 + 1) % 10] for r1 in range(7)]
    lvl2 = [pool[(idx * idx + 3 * idx) % 10] for idx in range(49)]
    return w, lvl1, lvl2


def test_three_level_nonuniform_node_order(orc):
    # The oracle's node -> rule mapping (BFS index idx * R + r at every level) at
    # three levels, where idx = r1 (level 1) and idx = 7 r1 + r2 (level 2) differ from any
    # other order.  Expectation composed here, level by level, from the oracle's building
    # blocks (node_st, the classical leaf, node_c) with the BFS index written out explicitly.
    import oracle
    w, lvl1, lvl2 = _three_level_nonuniform()
    A, B = fi.random_pair(64, 64, 64, seed=31)

    def compose(order):
        S0, T0 = oracle.node_st(w, A, B)
        M1 = []
        for r1 in range(7):
            S1, T1 = oracle.node_st(lvl1[r1], S0[r1], T0[r1])
            M2 = []
            for r2 in range(7):
                rule = lvl2[order(r1, r2)]
                S2, T2 = oracle.node_st(rule, S1[r2], T1[r2])
                leaves = np.stack([oracle.fmm(S2[r3], T2[r3], Plan([])) for r3 in range(7)])
                M2.append(oracle.node_c(rule, leaves))
            M1.append(oracle.node_c(lvl1[r1], np.stack(M2)))
        return oracle.node_c(w, np.stack(M1))

    want = compose(lambda r1, r2: 7 * r1 + r2)
    got = oracle.fmm(A, B, Plan([[w], lvl1, lvl2]))
    assert np.array_equal(got, want)
    # the pin is sensitive: the transposed mixed-radix order gives a different rounding
    assert not np.array_equal(compose(lambda r1, r2: 7 * r2 + r1), want)
    # and the plan is still a correct product (Brent-exact rules): exact on small integers
    Ai, Bi = fi.integer_pair(64, 64, 64, seed=9, lo=-4, hi=4)
    Ci = oracle.fmm(Ai, Bi, Plan([[w], lvl1, lvl2]))
    assert np.array_equal(Ci, (Ai.astype(np.int64) @ Bi.astype(np.int64)).astype(np.float64))
