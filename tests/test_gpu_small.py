"""The single-launch small plan (kernels_small.cu): a two-level plan compiled
to K1X2 -> leaf products -> K3X2 runs as one cooperative kernel.  Its arithmetic is the
three-launch schedule's element by element, so the result is bitwise equal to it; it matches the
oracle within the north-star tolerance, and bitwise when the leaf inner dimension is 1."""
import numpy as np
import pytest
import torch

import fmm_inputs as fi
import oracle
from oracle import rules as R
from oracle.rules import Plan as OPlan

pytestmark = pytest.mark.gpu
TOL64 = 1e-13


@pytest.fixture(scope="module")
def fb():
    import paper_1507_00687_b200 as fb
    assert torch.cuda.is_available()
    return fb


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def exe(p, A, B):
    C = p.execute(dev(A), dev(B))
    torch.cuda.synchronize()
    return C.cpu().numpy()


# (the classical rule forms no S / T -- its operands are views -- so a classical-only plan has no
# K1X2 pass and keeps its two launches)
PAIRS = [("winograd", "winograd"), ("strassen", "strassen"), ("winograd", "classical222"),
         ("strassen", "winograd"), ("classical222", "strassen")]


@pytest.mark.parametrize("names", PAIRS)
@pytest.mark.parametrize("dims", [(512, 512, 512), (4 * 37, 4 * 21, 4 * 45), (256, 1024, 128),
                                  (4 * 100, 4 * 64, 4 * 36)])
def test_single_launch_bitwise_three_launches(fb, names, dims):
    M, K, N = dims
    A, B = fi.random_pair(M, K, N, seed=M + N)
    rules = [fb.Rule.builtin(n) for n in names]
    p1 = fb.Plan(rules, M, K, N)
    p3 = fb.Plan(rules, M, K, N)
    p3.set_single_launch(False)
    assert p1.launch_count() == 1 and p3.launch_count() == 3
    C1 = exe(p1, A, B)
    assert np.array_equal(C1, exe(p3, A, B))
    assert np.array_equal(C1, exe(p1, A, B))  # deterministic across calls
    Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
    assert oracle.parity_metric(C1, Co, np.abs(A).max(), np.abs(B).max(), K) <= TOL64


@pytest.mark.parametrize("names", PAIRS)
def test_single_launch_unit_leaf_bitwise_oracle(fb, names):
    A, B = fi.random_pair(256, 4, 192, seed=5)
    p = fb.Plan([fb.Rule.builtin(n) for n in names], 256, 4, 192)
    assert p.launch_count() == 1
    assert np.array_equal(exe(p, A, B), oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names])))


def test_single_launch_C1_and_graph(fb):
    A, B = fi.config_inputs("C1")
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w, w], 512, 512, 512)
    ref = exe(p, A, B)
    Co = oracle.fmm(A, B, OPlan.stationary(R.winograd(), 2))
    assert oracle.parity_metric(ref, Co, np.abs(A).max(), np.abs(B).max(), 512) <= TOL64
    p.set_graph(True)  # the cooperative launch captured and replayed
    Ad, Bd = dev(A), dev(B)
    C = torch.empty((512, 512), dtype=torch.float64, device="cuda")
    for _ in range(3):
        C.fill_(float("nan"))
        p.execute(Ad, Bd, C)
        torch.cuda.synchronize()
        assert np.array_equal(C.cpu().numpy(), ref)


def test_single_launch_strided_output_no_oob(fb):
    M, K, N = 4 * 40, 4 * 24, 4 * 36
    A, B = fi.random_pair(M, K, N, seed=9)
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w, w], M, K, N)
    assert p.launch_count() == 1
    ldc = N + 6
    big = torch.full((M + 8, ldc), 12345.0, dtype=torch.float64, device="cuda")
    Cv = big[4:4 + M, :N]
    nb = p.workspace_bytes()
    wsb = torch.full((nb + 4096,), 0xA5, dtype=torch.uint8, device="cuda")
    p.execute(dev(A), dev(B), Cv, ws=wsb[:nb])
    torch.cuda.synchronize()
    g = big.clone()
    g[4:4 + M, :N] = 12345.0
    assert torch.all(g == 12345.0), "write outside C[:, :N]"
    assert torch.all(wsb[nb:] == 0xA5), "write past the workspace"
    p3 = fb.Plan([w, w], M, K, N)
    p3.set_single_launch(False)
    assert np.array_equal(Cv.cpu().numpy(), exe(p3, A, B))
