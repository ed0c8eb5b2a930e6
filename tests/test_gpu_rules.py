"""GPU: base cases other than 2x2x2 and stability-driven variants through the C ABI (rules
created from the paper's printed tables).  The kernels are
rule-generic (K1 / K3 / K2F read the coefficient tables), so the same parity bar applies:
tolerance against the oracle, bitwise with unit leaf inner dimension, fused = unfused."""
from fractions import Fraction

import numpy as np
import pytest
import torch

import fmm_inputs as fi
import oracle
from oracle import rules as R
from oracle.rules import Plan as OPlan
from test_oracle_rules import app_b_323, app_c_442

pytestmark = pytest.mark.gpu
TOL64 = 1e-13


@pytest.fixture(scope="module")
def fb():
    import paper_1507_00687_b200 as fb
    assert torch.cuda.is_available()
    return fb


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def to_gpu_rule(fb, rule):
    """fmm_rule_create from an oracle rule: integer numerators over a common 2^s."""
    den = 1
    for X in (rule.U, rule.V, rule.W):
        for row in X:
            for x in row:
                den = max(den, Fraction(x).denominator)
    s = den.bit_length() - 1
    assert 1 << s == den
    num = lambda X: np.array([[int(Fraction(x) * den) for x in row] for row in X])
    return fb.Rule.create(rule.m0, rule.k0, rule.n0, num(rule.U), num(rule.V), num(rule.W),
                          log2_den=s, name=rule.name)


def run_both(fb, orules, M, K, N, A, B, fusion):
    p = fb.Plan([to_gpu_rule(fb, r) for r in orules], M, K, N)
    p.set_fusion(fusion)
    C = p.execute(dev(A), dev(B))
    torch.cuda.synchronize()
    return C.cpu().numpy()


CASES = {
    "323": ([app_b_323], (3 * 64, 2 * 96, 3 * 40)),
    "323_strassen": ([app_b_323, R.strassen], (6 * 40, 4 * 32, 6 * 30)),
    "442": ([app_c_442], (4 * 48, 4 * 40, 2 * 64)),
    "442_winograd": ([app_c_442, R.winograd], (8 * 24, 8 * 20, 4 * 32)),
    "winograd_323": ([R.winograd, app_b_323], (6 * 32, 4 * 32, 6 * 20)),
}


@pytest.mark.parametrize("case", sorted(CASES))
def test_other_base_cases_parity_and_fusion(fb, case):
    makers, (M, K, N) = CASES[case]
    orules = [m() for m in makers]
    A, B = fi.random_pair(M, K, N, seed=M + K)
    Cu = run_both(fb, orules, M, K, N, A, B, "off")
    Cf = run_both(fb, orules, M, K, N, A, B, "on")
    assert np.array_equal(Cf, Cu)
    Co = oracle.fmm(A, B, OPlan.uniform(orules))
    assert oracle.parity_metric(Cu, Co, np.abs(A).max(), np.abs(B).max(), K) <= TOL64


@pytest.mark.parametrize("case", sorted(CASES))
def test_other_base_cases_unit_leaf_bitwise(fb, case):
    makers, _ = CASES[case]
    orules = [m() for m in makers]
    pm = int(np.prod([r.m0 for r in orules]))
    pk = int(np.prod([r.k0 for r in orules]))
    pn = int(np.prod([r.n0 for r in orules]))
    M, K, N = 8 * pm, pk, 6 * pn
    A, B = fi.random_pair(M, K, N, seed=pk)
    Co = oracle.fmm(A, B, OPlan.uniform(orules))
    for fusion in ("off", "on"):
        assert np.array_equal(run_both(fb, orules, M, K, N, A, B, fusion), Co)


def test_442_integer_inputs_exact(fb):
    # +-1/2 coefficients: every intermediate is dyadic, so integer inputs give the exact product
    rule = app_c_442()
    A, B = fi.integer_pair(4 * 32, 4 * 16, 2 * 32, seed=5)
    Ci = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float64)
    assert np.array_equal(run_both(fb, [rule], *A.shape, B.shape[1], A, B, "on"), Ci)


def test_castrapel_gustafson_nonuniform_plan(fb):
    # stability-driven non-uniform plan: S-W at the root, a different
    # Castrapel-Gustafson variant of S-W at each level-2 node
    w = R.winograd()
    variants = [R.castrapel_gustafson(w, x, y, z) for x in (1, 2) for y in (1, 2) for z in (1, 2)]
    lvl2 = [variants[r % 8] for r in range(7)]
    nodes = [to_gpu_rule(fb, w)] + [to_gpu_rule(fb, v) for v in lvl2]
    oplan = OPlan([[w], lvl2])
    for (M, K, N), check in (((256, 192, 128), "parity"), ((64, 4, 32), "bitwise")):
        A, B = fi.random_pair(M, K, N, seed=K)
        Co = oracle.fmm(A, B, oplan)
        for fusion, sched in (("off", "auto"), ("on", "auto"), ("on", "hybrid"), ("off", "depth")):
            p = fb.Plan(nodes, M, K, N, uniform=False, levels=2)
            p.set_fusion(fusion)
            p.set_schedule(sched)
            Cg = p.execute(dev(A), dev(B)).cpu().numpy()
            if check == "parity":
                assert oracle.parity_metric(Cg, Co, np.abs(A).max(), np.abs(B).max(), K) <= TOL64
            else:
                assert np.array_equal(Cg, Co)


@pytest.mark.parametrize("kind", ["rotate", "rotate2"])
def test_rotated_323_through_the_abi(fb, kind):
    # App. B rotations: [[W,U,V]] is <3,3,2>, [[V,W,U]] is <2,3,3>; the GPU rule
    # comes from fmm_rule_transform, the oracle's is built independently from App. B's tables
    b = app_b_323()
    if kind == "rotate":
        orule = R.make_rule("rot", 3, 3, 2, b.W, b.U, b.V)
    else:
        orule = R.make_rule("rot2", 2, 3, 3, b.V, b.W, b.U)
    grule = to_gpu_rule(fb, b).transform(kind)
    gi = grule.info()
    assert (gi["m0"], gi["k0"], gi["n0"]) == (orule.m0, orule.k0, orule.n0)
    M, K, N = orule.m0 * 40, orule.k0 * 36, orule.n0 * 44
    A, B = fi.random_pair(M, K, N, seed=9)
    p = fb.Plan([grule, fb.Rule.builtin("strassen")], 2 * M, 2 * K, 2 * N)
    A2, B2 = fi.random_pair(2 * M, 2 * K, 2 * N, seed=10)
    Cg = p.execute(dev(A2), dev(B2)).cpu().numpy()
    Co = oracle.fmm(A2, B2, OPlan.uniform([orule, R.strassen()]))
    assert oracle.parity_metric(Cg, Co, np.abs(A2).max(), np.abs(B2).max(), 2 * K) <= TOL64


def test_three_level_nonuniform_plan(fb):
    # the 3-level non-uniform plan pinned on the oracle (test_oracle_exec.
    # test_three_level_nonuniform_node_order): 57 node rules in BFS order through the C ABI,
    # every schedule and fusion mode -- parity at a generic size, bitwise with leaf inner
    # dimension 1 (the node -> rule order of the GPU plan must match the oracle's exactly)
    from test_oracle_exec import _three_level_nonuniform
    w, lvl1, lvl2 = _three_level_nonuniform()
    nodes = [to_gpu_rule(fb, w)] + [to_gpu_rule(fb, r) for r in lvl1] + [to_gpu_rule(fb, r) for r in lvl2]
    oplan = OPlan([[w], lvl1, lvl2])
    for (M, K, N), check in (((512, 384, 256), "parity"), ((128, 8, 64), "bitwise")):
        A, B = fi.random_pair(M, K, N, seed=K + 5)
        Co = oracle.fmm(A, B, oplan)
        for fusion, sched in (("off", "breadth"), ("on", "breadth"), ("on", "hybrid"), ("off", "depth"),
                              ("auto", "auto")):
            p = fb.Plan(nodes, M, K, N, uniform=False, levels=3)
            p.set_fusion(fusion)
            p.set_schedule(sched)
            Cg = p.execute(dev(A), dev(B)).cpu().numpy()
            if check == "parity":
                assert oracle.parity_metric(Cg, Co, np.abs(A).max(), np.abs(B).max(), K) <= TOL64
            else:
                assert np.array_equal(Cg, Co), (fusion, sched)
