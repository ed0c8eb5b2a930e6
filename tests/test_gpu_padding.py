"""GPU: zero padding of dims that the plan's base cases do not divide ("we can
always pad the matrices with zeros"; SPEC pad_dims S:306-314).  The library copies A, B into
zero-padded workspace buffers, runs the recursion on the padded dims and crops C -- exactly
what the oracle's fmm() does -- so the parity bar is unchanged, and with unit leaf inner
dimension (after padding) the result is bitwise the oracle's."""
import numpy as np
import pytest
import torch

import fmm_inputs as fi
import oracle
from oracle import rules as R
from oracle.rules import Plan as OPlan

pytestmark = pytest.mark.gpu
TOL64, TOL32 = 1e-13, 5e-5


@pytest.fixture(scope="module")
def fb():
    import paper_1507_00687_b200 as fb
    assert torch.cuda.is_available()
    return fb


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


@pytest.mark.parametrize("dims", [(5, 5, 5), (500, 300, 260), (131, 67, 99), (1, 9, 3)])
@pytest.mark.parametrize("names", [("strassen", "strassen"), ("winograd", "classical222", "strassen")])
@pytest.mark.parametrize("fusion", ["off", "on"])
def test_padded_parity(fb, dims, names, fusion):
    M, K, N = dims
    A, B = fi.random_pair(M, K, N, seed=M * 7 + K)
    p = fb.Plan([fb.Rule.builtin(n) for n in names], M, K, N)
    p.set_fusion(fusion)
    Cg = p.execute(dev(A), dev(B)).cpu().numpy()
    assert Cg.shape == (M, N)
    Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
    assert oracle.parity_metric(Cg, Co, np.abs(A).max(), np.abs(B).max(), K) <= TOL64
    p.set_schedule("hybrid")  # padding wraps any schedule
    assert np.array_equal(p.execute(dev(A), dev(B)).cpu().numpy(), Cg)


@pytest.mark.parametrize("fusion", ["off", "on"])
def test_padded_unit_leaf_bitwise(fb, fusion):
    # K = 3 pads to 4 = 2^2: every leaf has inner dimension 1 (the padded column is zero)
    A, B = fi.random_pair(37, 3, 29, seed=3)
    names = ("winograd", "strassen")
    p = fb.Plan([fb.Rule.builtin(n) for n in names], 37, 3, 29)
    p.set_fusion(fusion)
    Cg = p.execute(dev(A), dev(B)).cpu().numpy()
    assert np.array_equal(Cg, oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names])))


def test_padded_strided_output_and_guard(fb):
    M, K, N = 203, 101, 77
    A, B = fi.random_pair(M, K, N, seed=4)
    p = fb.Plan([fb.Rule.builtin("winograd")] * 3, M, K, N)
    big = torch.full((M + 4, N + 5), 777.0, dtype=torch.float64, device="cuda")
    Cv = big[2:2 + M, :N]
    p.execute(dev(A), dev(B), Cv)
    torch.cuda.synchronize()
    g = big.clone()
    g[2:2 + M, :N] = 777.0
    assert torch.all(g == 777.0)
    Co = oracle.fmm(A, B, OPlan.stationary(R.winograd(), 3))
    assert oracle.parity_metric(Cv.cpu().numpy(), Co, np.abs(A).max(), np.abs(B).max(), K) <= TOL64


def test_padded_f32(fb):
    A, B = fi.random_pair(300, 200, 100, seed=5, dtype=np.float32)
    for leaf in (fb.fmm.LEAF_NATIVE, fb.fmm.LEAF_3XTF32):
        p = fb.Plan([fb.Rule.builtin("winograd")] * 3, 300, 200, 100, dtype="f32", leaf=leaf)
        Cg = p.execute(dev(A), dev(B)).cpu().numpy()
        Co = oracle.fmm(A, B, OPlan.stationary(R.winograd(), 3))
        assert oracle.parity_metric(Cg, Co, np.abs(A).max(), np.abs(B).max(), 200) <= TOL32


@pytest.mark.parametrize("mode", ["outside", "repeated"])
def test_padded_with_scaling(fb, mode):
    # scaling runs on the unpadded matrices (a zero padding row would violate its
    # precondition); the scaled A', B' are then padded.  The paper's experiment size
    # N = 3500 is not divisible by 2^L for L >= 3.
    A, B = fi.draw("skew", 100, 70, 90, 3)
    names = ("strassen",) * 3
    p = fb.Plan([fb.Rule.builtin(n) for n in names], 100, 70, 90,
                scaling={"mode": mode, "pow2": 1, "tau": 1.0, "max_steps": 20})
    Cg = p.execute(dev(A), dev(B)).cpu().numpy()
    Co, _ = oracle.scaled_fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]), mode=mode, pow2=True)
    ref_hi, ref_lo = oracle.ref_dd(A, B)
    # componentwise: GPU and oracle agree to the accuracy the scaled FMM itself has
    rel_g = np.max(np.abs((Cg - ref_hi) - ref_lo) / np.abs(ref_hi))
    rel_o = np.max(np.abs((Co - ref_hi) - ref_lo) / np.abs(ref_hi))
    assert rel_g <= 10 * rel_o + 1e-15
    assert np.max(np.abs(Cg - Co) / np.abs(Co)) <= 10 * rel_o + 1e-15
