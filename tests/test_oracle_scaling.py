"""Pins for the oracle's diagonal scaling (Sec. 6, Alg. 1-3): the paper's worked examples (with
the corrections listed in DESIGN.md readings A17-A19), the Lemma alt-scaling-example closed
form, the stopping criterion, the theorem invariants, and the accuracy contrasts of Exs. 5.1 /
5.2 (reading A25: non-dyadic z = 1e-10)."""
import math

import numpy as np
import pytest

import fmm_inputs as fi
from oracle import rules as R
from oracle.rules import Plan

Z = 2.0 ** -40  # exact-value pins
EPS = 2.0 ** -53


def test_ex51_outside_scaling_gives_ones(orc):
    # Ex. out_scaling: A' = B' = ones.
    A = np.array([[1.0, 1.0], [1.0, 1.0]])
    for z in (Z, 1e-10):
        B = np.array([[z, 1.0], [z, 1.0]])
        Ap, Bp, dA, dB = orc.scale_outside(A, B)
        assert np.array_equal(Ap, np.ones((2, 2))) and np.array_equal(Bp, np.ones((2, 2)))
        assert np.array_equal(dA, [1, 1]) and np.array_equal(dB, [z, 1])


def test_ex52_inside_scaling(orc):
    # Ex. in_scaling: D = diag(sqrt z, 1/sqrt z), A' = B' = sqrt(z) ones;
    # outside scaling does nothing (D_A = D_B = I).
    A = np.array([[1.0, Z], [1.0, Z]])
    B = np.array([[Z, Z], [1.0, 1.0]])
    Ap, Bp, d = orc.scale_inside(A, B)
    sz = 2.0 ** -20
    assert np.array_equal(d, [sz, 1 / sz])
    assert np.array_equal(Ap, sz * np.ones((2, 2))) and np.array_equal(Bp, sz * np.ones((2, 2)))
    Ao, Bo, dA, dB = orc.scale_outside(A, B)
    assert np.array_equal(Ao, A) and np.array_equal(Bo, B)
    assert np.array_equal(dA, [1, 1]) and np.array_equal(dB, [1, 1])


def test_ex69_both_orders(orc):
    # Ex. inout_outin_scaling: printed A', B' of both orders (reading A18 corrects
    # only the printed C' of the in->out case, which is not checked here).
    A = np.array([[1.0, 1 / Z], [1.0, 1.0]])
    B = np.array([[Z, 1.0], [Z, 1.0]])
    r = orc.scale_repeated(A, B, first_O=True, tau=0.0, max_steps=2)
    assert np.array_equal(r["A"], [[Z, 1], [1, 1]]) and np.array_equal(r["B"], np.ones((2, 2)))
    r = orc.scale_repeated(A, B, first_O=False, tau=0.0, max_steps=2)
    s = 2.0 ** -20
    assert np.array_equal(r["A"], [[s, 1], [1, s]]) and np.array_equal(r["B"], [[s, s], [1, 1]])


def test_ex610_in_out_half_and_corrected_out_in(orc):
    # Ex. outin_inout_scaling: the in->out half is as printed; the out->in half
    # follows Alg. 1/2 as A' = [[sqrt z, z], [sqrt z, 1]], B' = [[sqrt z, sqrt z], [1, 1]]
    # (reading A19: the printed out->in matrices row-scaled B).
    A = np.array([[1.0, Z], [Z, Z]])
    B = np.array([[Z, 1.0], [1.0, 1 / Z]])
    r = orc.scale_repeated(A, B, first_O=False, tau=0.0, max_steps=2)
    assert np.array_equal(r["A"], [[1, 1], [Z, 1]]) and np.array_equal(r["B"], np.ones((2, 2)))
    r = orc.scale_repeated(A, B, first_O=True, tau=0.0, max_steps=2)
    s = 2.0 ** -20
    assert np.array_equal(r["A"], [[s, Z], [s, 1]]) and np.array_equal(r["B"], [[s, s], [1, 1]])


def test_scaling_fails_is_fixed_point(orc):
    # Ex. scaling_fails: outside and inside scaling leave A, B unchanged.
    for z in (Z, 1e-10):
        A = np.array([[1.0, z], [z, 1.0]])
        Ao, Bo, dA, dB = orc.scale_outside(A, A)
        assert np.array_equal(Ao, A) and np.array_equal(Bo, A)
        Ai, Bi, d = orc.scale_inside(A, A)
        assert np.array_equal(Ai, A) and np.array_equal(Bi, A) and np.array_equal(d, [1, 1])
        r = orc.scale_repeated(A, A, tau=1.0, max_steps=10)
        assert np.array_equal(r["A"], A) and r["steps"] == 2  # stops at the first tested step


@pytest.mark.parametrize("v", [1, 2, 3])
def test_lemma_alt_scaling_example_closed_form(orc, v):
    # Lemma alt-scaling-example: A = [[1,0],[1,2^-2^v]], B = I, first step O:
    # mu_22^{(t)} = 2^{2^{v-(t-t0)/2}} - 1 for t = t0, t0+2, ...; mu^{(t+1)} = mu^{(t)};
    # limits r* = (1,1), s* = (1, 2^-2^v), ||A*|| = ||B*|| = 1.
    A = np.array([[1.0, 0.0], [1.0, 2.0 ** -(2 ** v)]])
    B = np.eye(2)
    n = 2 * (v + 2)
    r = orc.scale_repeated(A, B, first_O=True, tau=0.0, max_steps=n, trace=True)
    assert r["steps"] == n
    s_star = 2.0 ** -(2 ** v)
    for t in range(n):
        mu = abs(r["tdA"][t][1] * r["tdB"][t][1] * r["normA"][t] * r["normB"][t] - s_star) / s_star
        expect = 2.0 ** (2.0 ** (v - (t // 2))) - 1.0  # t0 = 0 (0-based), pairs (t0, t0+1) equal
        assert mu == pytest.approx(expect, rel=4e-16, abs=4e-16), (t, mu, expect)


def _mu_max(orc, A, B, first_O, upto):
    """max_ij mu_ij^{(t)} for t < upto against the numerically converged limit (Thm
    stopping-criterion diagnostic; the limit is estimated by iterating to stagnation)."""
    lim = orc.scale_repeated(A, B, first_O=first_O, tau=0.0, max_steps=200, trace=True)
    rs = lim["tdA"][-1][:, None] * lim["tdB"][-1][None, :] * lim["normA"][-1] * lim["normB"][-1]
    tr = orc.scale_repeated(A, B, first_O=first_O, tau=0.0, max_steps=upto, trace=True)
    out = []
    for t in range(tr["steps"]):
        cur = tr["tdA"][t][:, None] * tr["tdB"][t][None, :] * tr["normA"][t] * tr["normB"][t]
        out.append(float(np.max(np.abs(cur - rs) / rs)))
    return out


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_stopping_criterion_guarantee_and_monotonicity(orc, seed):
    # Thm stopping-criterion: when the test fires at tau, mu <= tau.
    # Thm accuracy-alt-scaling: r_i s_j ||A|| ||B|| is nonincreasing in t.
    A, B = fi.config_inputs("C4", scale_div=256)  # 16 x 16, the C4 recipe (log-uniform skew)
    for tau in (1.0, 0.1):
        res = orc.scale_repeated(A, B, first_O=True, tau=tau, max_steps=200, trace=True)
        assert res["steps"] < 200
        mus = _mu_max(orc, A, B, True, res["steps"])
        assert mus[-1] <= tau * (1 + 1e-12)
    tr = orc.scale_repeated(A, B, first_O=True, tau=0.0, max_steps=30, trace=True)
    prev = None
    for t in range(tr["steps"]):
        cur = tr["tdA"][t][:, None] * tr["tdB"][t][None, :] * tr["normA"][t] * tr["normB"][t]
        if prev is not None:
            assert np.all(cur <= prev * (1 + 8 * EPS))
        prev = cur


def test_step_postconditions(orc):
    A, B = fi.config_inputs("C4", scale_div=128)  # 32 x 32
    Ao, Bo, _, _ = orc.scale_outside(A, B)
    # O step: every row of A' and column of B' has max-abs exactly 1
    assert np.all(np.abs(Ao).max(axis=1) == 1.0) and np.all(np.abs(Bo).max(axis=0) == 1.0)
    Ai, Bi, p = orc.scale_inside(A, B)
    # I step: column k of A' and row k of B' have equal max-norms, to rounding
    ca, rb = np.abs(Ai).max(axis=0), np.abs(Bi).max(axis=1)
    assert np.allclose(ca, rb, rtol=4 * EPS, atol=0)
    assert np.allclose(ca, np.sqrt(np.abs(A).max(axis=0) * np.abs(B).max(axis=1)), rtol=4 * EPS)


def test_pow2_round():
    import oracle
    assert oracle.pow2_round(1.0) == 1.0
    assert oracle.pow2_round(3.0) == 4.0  # log2 3 = 1.58
    assert oracle.pow2_round(0.75) == 1.0  # log2 0.75 = -0.415
    assert oracle.pow2_round(2.0 ** -30 * 1.4) == 2.0 ** -30  # 1.4 < sqrt 2
    assert oracle.pow2_round(2.0 ** 70 * 1.42) == 2.0 ** 71  # 1.42 > sqrt 2
    s = math.sqrt(2.0)  # the double nearest sqrt(2) is above sqrt(2)
    assert s * s > 2.0 or math.fsum([s * s]) > 2.0
    assert oracle.pow2_round(s) == 2.0
    assert oracle.pow2_round(np.nextafter(s, 0)) == 1.0  # just below sqrt(2)


def test_pow2_scaling_is_exact(orc):
    # with power-of-two factors, applying and removing the scaling is exact.
    A, B = fi.config_inputs("C4", scale_div=128)
    Ao, Bo, dA, dB = orc.scale_outside(A, B, pow2=True)
    assert np.array_equal(Ao * dA[:, None], A) and np.array_equal(Bo * dB[None, :], B)
    assert np.all(np.frexp(dA)[0] == 0.5) and np.all(np.frexp(dB)[0] == 0.5)


def test_zero_row_precondition(orc):
    import oracle
    A = np.ones((3, 3))
    A[1] = 0
    with pytest.raises(oracle.ScalingError, match="row of A at index 1"):
        orc.scale_outside(A, np.ones((3, 3)))
    with pytest.raises(oracle.ScalingError, match="column of A at index 2"):
        B = np.ones((3, 3))
        A2 = np.ones((3, 3))
        A2[:, 2] = 0
        orc.scale_inside(A2, B)


def _strassen_rel_err(orc, A, B, mode, entry):
    C, _ = orc.scaled_fmm(A, B, Plan.stationary(R.strassen(), 1), mode=mode)
    hi, lo = orc.ref_dd(A, B)
    i, j = entry
    return abs((C[i, j] - hi[i, j]) - lo[i, j]) / abs(hi[i, j])


def test_ex51_ex52_accuracy_contrast(orc):
    # P:698-712 / P:776: unscaled Strassen has O(eps/z) relative error on c11 of Ex. 5.1, outside
    # scaling O(eps); Ex. 5.2 c12 likewise with inside scaling.
    z = 1e-10  # reading A25: non-dyadic so that the unscaled run really rounds
    A = np.ones((2, 2))
    B = np.array([[z, 1.0], [z, 1.0]])
    assert _strassen_rel_err(orc, A, B, "none", (0, 0)) > 1e3 * EPS / 1  # O(eps/z)
    assert _strassen_rel_err(orc, A, B, "outside", (0, 0)) <= 4 * EPS
    A = np.array([[1.0, z], [1.0, z]])
    B = np.array([[z, z], [1.0, 1.0]])
    assert _strassen_rel_err(orc, A, B, "none", (0, 1)) > 1e3 * EPS
    assert _strassen_rel_err(orc, A, B, "inside", (0, 1)) <= 4 * EPS
