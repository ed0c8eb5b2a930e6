"""GPU: two recursion levels per pass -- S / T formation (K1X2, fmm_plan_set_k1_levels) and the
W-combination (K3X2, fmm_plan_set_k3_levels).

K1X2 evaluates S_{r1 r2} = sum_i2 u2_{i2 r2} (sum_i1 u1_{i1 r1} A[i1][i2]) and K3X2
C[k1][k2] = sum_r1 w1_{k1 r1} (sum_r2 w2_{k2 r2} M_{r1 r2}) in registers in the order of two
one-level passes (Eq. eqn:recursive_alg P:116-125 applied at two consecutive levels; sequential
summation P:241-246, reading A3), so plans with one and two levels per pass must agree
BITWISE, and with unit leaf inner dimension (every leaf product one multiplication) both must
equal the oracle bitwise."""
import numpy as np
import pytest
import torch

import fmm_inputs as fi
import oracle
from oracle import rules as R
from oracle.rules import Plan as OPlan

pytestmark = pytest.mark.gpu

TOL64 = 1e-13
TOL32 = 5e-5

PLANS = {
    "winograd_L2": ("winograd",) * 2,
    "winograd_L3": ("winograd",) * 3,           # pair (1, 2) + a one-level pass at the root
    "strassen_L4": ("strassen",) * 4,           # pairs (2, 3) and (0, 1): C2's plan
    "strassen_L5": ("strassen",) * 5,
    "classical_L2": ("classical222",) * 2,
    "C3_mix": ("winograd", "classical222", "strassen"),
    "mix_pairs": ("strassen", "winograd", "classical222", "winograd"),
}


@pytest.fixture(scope="module")
def fb():
    import paper_1507_00687_b200 as fb
    assert torch.cuda.is_available()
    return fb


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def run(fb, names, A, B, levels, dtype="f64", fusion="auto", schedule="auto", leaf=None, k3=None):
    M, K = A.shape
    N = B.shape[1]
    kw = {} if leaf is None else {"leaf": leaf}
    p = fb.Plan([fb.Rule.builtin(n) for n in names], M, K, N, dtype=dtype, **kw)
    p.set_k1_levels(levels)
    p.set_k3_levels(levels if k3 is None else k3)
    p.set_fusion(fusion)
    p.set_schedule(schedule)
    C = p.execute(dev(A), dev(B))
    torch.cuda.synchronize()
    return C.cpu().numpy(), p


@pytest.mark.parametrize("pname", sorted(PLANS))
def test_unit_leaf_equals_oracle_bitwise(fb, pname):
    # leaf inner dimension 1: every M_r = S_r T_r is one rounded product, so the whole
    # recursion is a fixed sequence of roundings the oracle reproduces exactly
    names = PLANS[pname]
    L = len(names)
    M, K, N = 3 * 2 ** L, 2 ** L, 5 * 2 ** L
    A, B = fi.random_pair(M, K, N, seed=31 + L)
    Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
    for fusion in ("off", "on"):
        C2, p = run(fb, names, A, B, 2, fusion=fusion)
        assert np.array_equal(C2, Co), (pname, fusion)


@pytest.mark.parametrize("pname", sorted(PLANS))
@pytest.mark.parametrize("schedule", ["breadth", "depth", "hybrid"])
def test_two_level_equals_one_level_bitwise(fb, pname, schedule):
    names = PLANS[pname]
    L = len(names)
    # ragged tiles in every dim at the leaves; vectorised path (K, N multiples of 2^L)
    M, K, N = 2 ** L * 37, 2 ** L * 20, 2 ** L * 26
    A, B = fi.random_pair(M, K, N, seed=7 * L)
    C1, p1 = run(fb, names, A, B, 1, schedule=schedule)
    C2, p2 = run(fb, names, A, B, 2, schedule=schedule)
    assert np.array_equal(C1, C2)
    assert p2.launch_count() <= p1.launch_count()  # equal where a level forms nothing (classical)
    Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
    assert oracle.parity_metric(C2, Co, np.abs(A).max(), np.abs(B).max(), K) <= TOL64


@pytest.mark.parametrize("pname", ["strassen_L4", "C3_mix", "mix_pairs"])
@pytest.mark.parametrize("fusion", ["off", "auto"])
def test_k1_k3_levels_independent_bitwise(fb, pname, fusion):
    # every combination of one / two levels per K1 and K3 pass gives the same bits
    names = PLANS[pname]
    L = len(names)
    M, K, N = 2 ** L * 21, 2 ** L * 12, 2 ** L * 18
    A, B = fi.random_pair(M, K, N, seed=3 * L)
    outs = [run(fb, names, A, B, k1, fusion=fusion, k3=k3)[0] for k1 in (1, 2) for k3 in (1, 2)]
    for C in outs[1:]:
        assert np.array_equal(outs[0], C)


@pytest.mark.parametrize("dims", [(509, 383, 257), (250, 130, 66), (64, 64, 63)])
def test_padded_and_unvectorised(fb, dims):
    # zero padding of non-divisible dims, and odd K / N (scalar path)
    M, K, N = dims
    A, B = fi.random_pair(M, K, N, seed=M)
    names = ("winograd", "strassen", "winograd")
    C1, _ = run(fb, names, A, B, 1)
    C2, _ = run(fb, names, A, B, 2)
    assert np.array_equal(C1, C2)


@pytest.mark.parametrize("leaf", ["native", "3xtf32"])
def test_f32(fb, leaf):
    lf = {"native": fb.fmm.LEAF_NATIVE, "3xtf32": fb.fmm.LEAF_3XTF32}[leaf]
    names = ("strassen",) * 4
    A, B = fi.random_pair(512, 512, 512, seed=12, dtype=np.float32)
    C1, _ = run(fb, names, A, B, 1, dtype="f32", leaf=lf)
    C2, _ = run(fb, names, A, B, 2, dtype="f32", leaf=lf)
    assert np.array_equal(C1, C2)
    Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
    assert oracle.parity_metric(C2, Co, np.abs(A).max(), np.abs(B).max(), 512) <= TOL32


def test_partition_partials(fb):
    # virtual ranks (multi-GPU partition, depth-first top level): partials agree bitwise
    A, B = fi.random_pair(512, 256, 384, seed=5)
    names = ("winograd",) * 3
    for nranks in (2, 3):
        for rank in range(nranks):
            outs = []
            for levels in (1, 2):
                p = fb.Plan([fb.Rule.builtin(n) for n in names], 512, 256, 384)
                p.set_k1_levels(levels)
                p.set_k3_levels(levels)
                p.set_partition(rank, nranks)
                outs.append(p.execute(dev(A), dev(B)).cpu().numpy())
            assert np.array_equal(outs[0], outs[1])


def test_ineligible_rules_fall_back(fb):
    # <3,2,3;15> (App. B) splits A into 6 blocks (> 4): a pair containing its level keeps the
    # one-level passes, with the same schedule and results as levels = 1
    from test_gpu_rules import to_gpu_rule
    from test_oracle_rules import app_b_323
    w = fb.Rule.builtin("winograd")
    b = to_gpu_rule(fb, app_b_323())
    M, K, N = 6 * 32, 4 * 32, 6 * 20
    A, B = fi.random_pair(M, K, N, seed=3)
    outs, counts = [], []
    for levels in (1, 2):
        p = fb.Plan([w, b], M, K, N)
        p.set_k1_levels(levels)
        p.set_k3_levels(levels)
        counts.append(p.launch_count())
        outs.append(p.execute(dev(A), dev(B)).cpu().numpy())
    assert counts[0] == counts[1]
    assert np.array_equal(outs[0], outs[1])
    # and an eligible pair drops one launch
    p = fb.Plan([w, w], 256, 256, 256)
    p.set_single_launch(False)  # (else the whole plan is one kernel)
    n2 = p.launch_count()
    p.set_k1_levels(1)
    assert p.launch_count() == n2 + 1


@pytest.mark.parametrize("names", [("strassen",) * 4, ("winograd", "classical222", "strassen"),
                                   ("classical222", "winograd", "winograd")])
def test_hybrid_schedule_bitwise(fb, names):
    # hybrid top level (root S / T at once, subtrees in turn, root + level-1 combination as one
    # K3X2 at the end) against breadth-first, fused and unfused
    L = len(names)
    M, K, N = 2 ** L * 24, 2 ** L * 10, 2 ** L * 16
    A, B = fi.random_pair(M, K, N, seed=L + 40)
    for fusion in ("off", "on"):
        Cb, _ = run(fb, names, A, B, 2, fusion=fusion, schedule="breadth")
        Ch, _ = run(fb, names, A, B, 2, fusion=fusion, schedule="hybrid")
        assert np.array_equal(Cb, Ch)


def test_workspace_smaller(fb):
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w] * 3, 4096, 4096, 4096)
    ws2 = p.workspace_bytes()
    p.set_k1_levels(1)
    assert ws2 < p.workspace_bytes()


@pytest.mark.parametrize("leaf", ["3xtf32", "tf32"])
@pytest.mark.parametrize("names,dims,sched", [
    (("winograd",) * 2, (512, 512, 512), "auto"),
    (("winograd",) * 3, (1024, 512, 768), "hybrid"),     # C5's schedule in miniature
    (("winograd",) * 3, (1024, 512, 768), "depth"),
    (("strassen",) * 4, (1024, 1024, 1024), "breadth"),
    (("winograd", "classical222", "strassen"), (1024, 512, 1024), "auto"),  # C3's rules
    (("winograd",) * 2, (512, 4 * 72, 4 * 90), "auto"),  # leaf k, n not multiples of 32
])
def test_leaf_split_in_pass(fb, leaf, names, dims, sched):
    # FP32 tensor-core leaves: the leaf level's K1X2 writes every leaf
    # operand's TF32 hi / lo pair straight into the GEMM's arena (views included) instead of
    # S_r / T_r + a split kernel: the same elementwise split of the same sums, so bitwise the
    # split-kernel path; and within the FP32 tolerance of the oracle
    M, K, N = dims
    lf = {"3xtf32": fb.fmm.LEAF_3XTF32, "tf32": fb.fmm.LEAF_TF32}[leaf]
    A, B = fi.random_pair(M, K, N, seed=M + K, dtype=np.float32)
    outs = []
    for in_pass in (True, False):
        p = fb.Plan([fb.Rule.builtin(n) for n in names], M, K, N, dtype="f32", leaf=lf)
        p.set_schedule(sched)
        p.set_leaf_split(in_pass)
        outs.append(p.execute(dev(A), dev(B)).cpu().numpy())
    assert np.array_equal(outs[0], outs[1])
    if leaf == "3xtf32":
        Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
        assert oracle.parity_metric(outs[0], Co, np.abs(A).max(), np.abs(B).max(), K) <= TOL32


def test_leaf_split_in_pass_partition(fb):
    # virtual ranks of a multi-GPU partition: each rank's partial is the split-kernel path's
    A, B = fi.random_pair(1024, 512, 512, seed=9, dtype=np.float32)
    for rank in range(3):
        outs = []
        for in_pass in (True, False):
            p = fb.Plan([fb.Rule.builtin("winograd")] * 3, 1024, 512, 512, dtype="f32",
                        leaf=fb.fmm.LEAF_3XTF32)
            p.set_partition(rank, 3)
            p.set_leaf_split(in_pass)
            outs.append(p.execute(dev(A), dev(B)).cpu().numpy())
        assert np.array_equal(outs[0], outs[1])
