"""GPU parity: the CUDA path (through the C ABI) against the oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): ||C_gpu - C_oracle||max / (||A||max ||B||max K) <= 1e-13
(FP64) and <= 5e-5 (FP32).  Kernel-level checks whose order is fixed (K1 linear combinations,
K3 combinations, scaling) are bitwise, and so is the whole recursion when the leaf inner
dimension is 1 (the leaf is then a single correctly rounded product on both sides)."""
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


def gpu_plan(fb, names, M, K, N, dtype="f64", **kw):
    return fb.Plan([fb.Rule.builtin(n) for n in names], M, K, N, dtype=dtype, **kw)


def run(fb, names, A, B, dtype="f64", **kw):
    M, K = A.shape
    N = B.shape[1]
    p = gpu_plan(fb, names, M, K, N, dtype=dtype, **kw)
    Cg = p.execute(dev(A), dev(B))
    torch.cuda.synchronize()
    return Cg.cpu().numpy()


def parity(Cg, Co, A, B):
    return oracle.parity_metric(Cg, Co, np.abs(A).max(), np.abs(B).max(), A.shape[1])


# ---- K2 alone ---------------------------------------------------------------------------------

@pytest.mark.parametrize("shape", [(128, 128, 128), (256, 512, 384), (1, 1, 1), (7, 13, 5),
                                   (129, 257, 131), (300, 17, 260), (64, 0, 64)])
def test_leaf_gemm_f64(fb, shape):
    M, K, N = shape
    A, B = fi.random_pair(M, K, N, seed=M + K + N)
    Cg = fb.gemm(dev(A), dev(B)).cpu().numpy()
    Co = oracle.fmm(A, B, OPlan([]))
    if K == 0:
        assert np.all(Cg == 0)
        return
    assert parity(Cg, Co, A, B) <= TOL64
    # componentwise classical bound gamma_K sum |a||b| for any order
    g = K * 2.0 ** -53 / (1 - K * 2.0 ** -53)
    assert np.all(np.abs(Cg - Co) <= 2 * g * (np.abs(A) @ np.abs(B)) + 1e-300)


def test_leaf_gemm_f64_unaligned_ld(fb):
    A, B = fi.random_pair(100, 70, 90, seed=1)
    Ab = torch.zeros((100, 71), dtype=torch.float64, device="cuda")
    Ab[:, :70] = dev(A)
    Bb = torch.zeros((70, 93), dtype=torch.float64, device="cuda")
    Bb[:, :90] = dev(B)
    Cg = fb.gemm(Ab[:, :70], Bb[:, :90]).cpu().numpy()
    assert parity(Cg, oracle.fmm(A, B, OPlan([])), A, B) <= TOL64


@pytest.mark.parametrize("leaf", ["3xtf32", "native"])
def test_leaf_gemm_f32_unaligned_ld(fb, leaf):
    # operands whose rows are not 16-byte aligned (ld % 4 != 0): the scalar split path of the
    # tensor-core leaf; an output with ld > n
    lf = {"3xtf32": fb.fmm.LEAF_3XTF32, "native": fb.fmm.LEAF_NATIVE}[leaf]
    A, B = fi.random_pair(100, 70, 90, seed=1, dtype=np.float32)
    Ab = torch.zeros((100, 71), dtype=torch.float32, device="cuda")
    Ab[:, :70] = dev(A)
    Bb = torch.zeros((70, 93), dtype=torch.float32, device="cuda")
    Bb[:, :90] = dev(B)
    Cb = torch.full((100, 97), float("nan"), dtype=torch.float32, device="cuda")
    fb.gemm(Ab[:, :70], Bb[:, :90], leaf=lf, C_out=Cb[:, :90])
    Cg = Cb.cpu().numpy()
    assert parity(Cg[:, :90], oracle.fmm(A, B, OPlan([])), A, B) <= TOL32
    assert np.all(np.isnan(Cg[:, 90:]))  # nothing written past n


def test_leaf_gemm_f32(fb):
    A, B = fi.random_pair(200, 300, 100, seed=3, dtype=np.float32)
    Cg = fb.gemm(dev(A), dev(B)).cpu().numpy()
    assert parity(Cg, oracle.fmm(A, B, OPlan([])), A, B) <= TOL32


@pytest.mark.parametrize("shape", [(128, 32, 256), (256, 512, 384), (200, 300, 100), (7, 5, 3),
                                   (1024, 1024, 1024)])
def test_leaf_gemm_tf32_tensor_core(fb, shape):
    # tcgen05 kind::tf32 leaf: 3xTF32 must pass the FP32 parity tolerance against the FP32
    # oracle leaf; single-pass TF32 is a labelled variant (error ~ 2^-11 per product).
    M, K, N = shape
    A, B = fi.random_pair(M, K, N, seed=K, dtype=np.float32)
    Co = oracle.fmm(A, B, OPlan([]))
    C3 = fb.gemm(dev(A), dev(B), leaf=fb.fmm.LEAF_3XTF32).cpu().numpy()
    C1 = fb.gemm(dev(A), dev(B), leaf=fb.fmm.LEAF_TF32).cpu().numpy()
    p3, p1 = parity(C3, Co, A, B), parity(C1, Co, A, B)
    assert p3 <= TOL32
    assert p3 < p1  # the lo terms are really applied
    exact = A.astype(np.float64) @ B.astype(np.float64)
    absab = np.abs(A).astype(np.float64) @ np.abs(B).astype(np.float64)
    # 3xTF32 with FP32 tensor-core accumulation: componentwise within K * 2^-22 sum|a||b|
    assert np.all(np.abs(C3 - exact) <= K * 2.0 ** -22 * absab + 1e-30)
    assert np.all(np.abs(C1 - exact) <= K * 2.0 ** -9 * absab + 1e-30)


@pytest.mark.parametrize("K", [4096, 4096 + 96])
def test_tf32_chunked_accumulation_accuracy(fb, K):
    # k2p_tf32 drains 128-deep TMEM chunks into round-to-nearest register totals (DESIGN.md
    # §6.3): against the exact product its error must stay within 2x that of the FP32 oracle's
    # leaf (the paper's classical base case, in FP32: sequential round-to-nearest dot
    # products).  Accumulating all of K in the truncating TMEM adds fails this (~13x at K=4096).
    M = N = 256
    A, B = fi.random_pair(M, K, N, seed=5, dtype=np.float32)
    C3 = fb.gemm(dev(A), dev(B), leaf=fb.fmm.LEAF_3XTF32).cpu().numpy().astype(np.float64)
    exact = A.astype(np.float64) @ B.astype(np.float64)
    Co = oracle.fmm(A, B, OPlan([])).astype(np.float64)
    den = np.abs(exact).max()
    e_gpu = np.abs(C3 - exact).max() / den
    e_oracle = np.abs(Co - exact).max() / den
    assert e_gpu <= 2.0 * e_oracle, (e_gpu, e_oracle)


@pytest.mark.parametrize("names", [("winograd", "winograd"), ("strassen",) * 3])
def test_f32_recursion_3xtf32(fb, names):
    A, B = fi.random_pair(512, 512, 512, seed=14, dtype=np.float32)
    p = fb.Plan([fb.Rule.builtin(n) for n in names], 512, 512, 512, dtype="f32",
                leaf=fb.fmm.LEAF_3XTF32)
    Cg = p.execute(dev(A), dev(B)).cpu().numpy()
    Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
    assert parity(Cg, Co, A, B) <= TOL32


# ---- K1 / K3 bitwise -----------------------------------------------------------------------------

@pytest.mark.parametrize("name", sorted(R.BUILTINS))
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("dims", [(64, 96, 32), (6, 10, 14)])
def test_node_st_bitwise(fb, name, dtype, dims):
    m, k, n = dims
    A, B = fi.random_pair(m, k, n, seed=5, dtype=dtype)
    Sg, Tg = fb.node_st(fb.Rule.builtin(name), dev(A), dev(B))
    So, To = oracle.node_st(R.builtin(name), A, B)
    assert np.array_equal(Sg.cpu().numpy(), So) and np.array_equal(Tg.cpu().numpy(), To)


@pytest.mark.parametrize("name", sorted(R.BUILTINS))
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_node_c_bitwise(fb, name, dtype):
    r = R.builtin(name)
    g = np.random.default_rng(7)
    Ms = g.standard_normal((r.R, 24, 40)).astype(dtype)
    Cg = fb.node_c(fb.Rule.builtin(name), dev(Ms)).cpu().numpy()
    assert np.array_equal(Cg, oracle.node_c(r, Ms))


def test_summation_order_case_on_gpu(fb):
    # the hand-computed order pin of tests/test_oracle_exec.py, through the CUDA K1 / K3
    A = np.array([[2.0 ** 53, -(2.0 ** 53)], [-1.0, -1.0]])
    S, _ = fb.node_st(fb.Rule.builtin("winograd"), dev(A), dev(np.ones((2, 2))))
    assert S[2, 0, 0].item() == 1.0
    Ms = np.array([2.0 ** 53, 0.0, 1.0, 0.0, -(2.0 ** 53), 1.0, 0.0]).reshape(7, 1, 1)
    assert fb.node_c(fb.Rule.builtin("winograd"), dev(Ms))[0, 1].item() == 1.0


# ---- whole recursion ----------------------------------------------------------------------------

PLANS = {
    "winograd_L2": ("winograd", "winograd"),
    "strassen_L3": ("strassen",) * 3,
    "classical_L2": ("classical222",) * 2,
    "C3_mix": ("winograd", "classical222", "strassen"),
}


@pytest.mark.parametrize("pname", sorted(PLANS))
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_recursion_bitwise_with_unit_leaf_k(fb, pname, dtype):
    # K = 2^L: every leaf has inner dimension 1, so the leaf is one rounded product on both
    # sides and the whole result is fixed by the S/T/C summation order (reading A3).
    names = PLANS[pname]
    L = len(names)
    A, B = fi.random_pair(16 * 2 ** L, 2 ** L, 8 * 2 ** L, seed=L, dtype=dtype)
    Cg = run(fb, names, A, B, dtype="f64" if dtype == np.float64 else "f32")
    Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
    assert np.array_equal(Cg, Co)


@pytest.mark.parametrize("pname", sorted(PLANS))
def test_recursion_parity_f64(fb, pname):
    names = PLANS[pname]
    A, B = fi.random_pair(512, 384, 256, seed=11)
    Cg = run(fb, names, A, B)
    Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
    assert parity(Cg, Co, A, B) <= TOL64


def test_integer_inputs_exact(fb):
    A, B = fi.integer_pair(256, 256, 256, seed=2)
    Ci = (A.astype(np.int64) @ B.astype(np.int64)).astype(np.float64)
    for names in PLANS.values():
        assert np.array_equal(run(fb, names, A, B), Ci)


def test_dalberto_nonuniform(fb):
    s, d = fb.Rule.builtin("strassen"), fb.Rule.builtin("strassen_dalberto")
    nodes = [s] + [d if r in (0, 2, 3) else s for r in range(7)]
    A, B = fi.random_pair(256, 256, 256, seed=3)
    p = fb.Plan(nodes, 256, 256, 256, uniform=False, levels=2)
    Cg = p.execute(dev(A), dev(B)).cpu().numpy()
    Co = oracle.fmm(A, B, OPlan.dalberto_two_level())
    assert parity(Cg, Co, A, B) <= TOL64
    # unit-leaf bitwise variant
    A, B = fi.random_pair(64, 4, 64, seed=4)
    p = fb.Plan(nodes, 64, 4, 64, uniform=False, levels=2)
    assert np.array_equal(p.execute(dev(A), dev(B)).cpu().numpy(),
                          oracle.fmm(A, B, OPlan.dalberto_two_level()))


def test_C1_full_size(fb):
    A, B = fi.config_inputs("C1")
    Cg = run(fb, ("winograd", "winograd"), A, B)
    Co = oracle.fmm(A, B, OPlan.stationary(R.winograd(), 2))
    assert parity(Cg, Co, A, B) <= TOL64
    # and the Thm 4.3 bound against the double-double reference
    hi, lo = oracle.ref_dd(A, B)
    f = float(R.stationary_bound_factor(R.winograd(), 2, 512))
    assert np.max(np.abs((Cg - hi) - lo)) <= f * np.abs(A).max() * np.abs(B).max() * 2.0 ** -53


def test_C2_reduced(fb):
    A, B = fi.config_inputs("C2", scale_div=4)  # 1024^3, Strassen L=4 -> 64^3 leaves
    for names in (("strassen",) * 4, ("classical222",) * 4):
        Cg = run(fb, names, A, B)
        Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
        assert parity(Cg, Co, A, B) <= TOL64


def test_C3_reduced(fb):
    A, B = fi.config_inputs("C3", scale_div=8)  # 1024 x 512 x 1024
    names = ("winograd", "classical222", "strassen")
    Cg = run(fb, names, A, B)
    Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
    assert parity(Cg, Co, A, B) <= TOL64


def test_f32_recursion_parity(fb):
    A, B = fi.random_pair(512, 512, 512, seed=4, dtype=np.float32)
    Cg = run(fb, ("winograd",) * 3, A, B, dtype="f32")
    Co = oracle.fmm(A, B, OPlan.stationary(R.winograd(), 3))
    assert parity(Cg, Co, A, B) <= TOL32


def test_deterministic(fb):
    A, B = fi.random_pair(512, 512, 512, seed=6)
    p = gpu_plan(fb, ("winograd",) * 2, 512, 512, 512)
    c1 = p.execute(dev(A), dev(B)).cpu().numpy()
    c2 = p.execute(dev(A), dev(B)).cpu().numpy()
    assert np.array_equal(c1, c2)


@pytest.mark.parametrize("dtype,fusion", [("f64", "auto"), ("f64", "off"), ("f32", "auto")])
def test_split_schedule_matches_breadth_first(fb, dtype, fusion):
    # depth-first top level (used for big problems and sharding) with nranks = 1 is bitwise
    # equal to the breadth-first schedule: same kernels, same per-element orders.  The hybrid
    # top level combines levels 0-1 in one pass after fused leaf parents, else levels 1-2 per
    # subtree and the root alone (FP32 tensor-core leaves, unfused FP64): same sums, same order.
    npdt = np.float64 if dtype == "f64" else np.float32
    A, B = fi.random_pair(256, 256, 256, seed=8, dtype=npdt)
    p = gpu_plan(fb, ("winograd",) * 3, 256, 256, 256, dtype=dtype)
    p.set_fusion(fusion)
    bf = p.execute(dev(A), dev(B)).cpu().numpy()
    p.set_schedule("depth")
    assert np.array_equal(p.execute(dev(A), dev(B)).cpu().numpy(), bf)
    p.set_schedule("hybrid")  # root S / T at once, root (+ level 1) combination at the end
    assert np.array_equal(p.execute(dev(A), dev(B)).cpu().numpy(), bf)
    p.set_schedule("auto")
    parts = []
    for rank in range(3):
        p.set_partition(rank, 3)
        parts.append(p.execute(dev(A), dev(B)).cpu().numpy())
    # virtual ranks: the partial sums add up to the product (parity), each rank's set of blocks
    # is exact w.r.t. its own owned products
    total = parts[0] + parts[1] + parts[2]
    assert parity(total, bf, A, B) <= (TOL64 if dtype == "f64" else TOL32)
    p.set_partition(0, 1)
    assert np.array_equal(p.execute(dev(A), dev(B)).cpu().numpy(), bf)


def test_empty_and_degenerate(fb):
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w], 0, 4, 4)
    p.execute(torch.empty((0, 4), dtype=torch.float64, device="cuda"),
              torch.zeros((4, 4), dtype=torch.float64, device="cuda"))
    p = fb.Plan([w], 4, 0, 4)
    Cg = p.execute(torch.empty((4, 0), dtype=torch.float64, device="cuda"),
                   torch.empty((0, 4), dtype=torch.float64, device="cuda"))
    assert torch.all(Cg == 0)
    # identity exact
    I = np.eye(64)
    assert np.array_equal(run(fb, ("strassen",) * 3, I, I), I)


@pytest.mark.parametrize("leaf", ["3xtf32", "tf32"])
def test_tf32_empty_and_degenerate(fb, leaf):
    # FP32 tensor-core leaves: an empty inner dimension gives C = 0 (no chunk reaches TMEM, the
    # epilogue stores zeros); an empty plan is a no-op; a leaf GEMM of one row / one column and
    # identity operands are exact (products of TF32-exact values, sums of zeros)
    lf = {"3xtf32": fb.fmm.LEAF_3XTF32, "tf32": fb.fmm.LEAF_TF32}[leaf]
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w, w], 64, 0, 96, dtype="f32", leaf=lf)
    Cg = p.execute(torch.empty((64, 0), dtype=torch.float32, device="cuda"),
                   torch.empty((0, 96), dtype=torch.float32, device="cuda"))
    assert Cg.shape == (64, 96) and torch.all(Cg == 0)
    Cg = fb.gemm(torch.empty((5, 0), dtype=torch.float32, device="cuda"),
                 torch.empty((0, 7), dtype=torch.float32, device="cuda"), leaf=lf)
    assert torch.all(Cg == 0)
    p = fb.Plan([w], 0, 8, 8, dtype="f32", leaf=lf)
    p.execute(torch.empty((0, 8), dtype=torch.float32, device="cuda"),
              torch.zeros((8, 8), dtype=torch.float32, device="cuda"))
    I = np.eye(256, dtype=np.float32)
    X = fi.random_pair(256, 256, 256, seed=3, dtype=np.float32)[0]
    # multiples of 1/8 in [-1, 1]: every S / T sum (<= 16 terms) and product stays TF32-exact
    X = (np.round(X * 8) / 8).astype(np.float32)
    for names in (("winograd",) * 2, ("strassen",) * 3):
        p = fb.Plan([fb.Rule.builtin(n) for n in names], 256, 256, 256, dtype="f32", leaf=lf)
        assert np.array_equal(p.execute(dev(I), dev(X)).cpu().numpy(), run_exact_ref(I, X))
    row = fb.gemm(dev(X[:1]), dev(I), leaf=lf).cpu().numpy()
    assert np.array_equal(row, X[:1])


def run_exact_ref(A, B):
    return (A.astype(np.float64) @ B.astype(np.float64)).astype(np.float32)


@pytest.mark.parametrize("schedule", ["breadth", "depth", "hybrid"])
@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_execute_host_overlapped(fb, schedule, dtype):
    # fmm_execute_host (pinned host buffers; the depth-first schedule overlaps block copies with
    # the compute) returns exactly what fmm_execute returns on device buffers.
    npdt = np.float64 if dtype == "f64" else np.float32
    A, B = fi.random_pair(256, 512, 384, seed=31, dtype=npdt)
    w = fb.Rule.builtin("winograd")
    leaf = fb.fmm.LEAF_NATIVE if dtype == "f64" else fb.fmm.LEAF_3XTF32
    p = fb.Plan([w, w], 256, 512, 384, dtype=dtype, leaf=leaf)
    p.set_schedule(schedule)
    Cd = p.execute(dev(A), dev(B)).cpu().numpy()
    Ah = torch.from_numpy(A).pin_memory()
    Bh = torch.from_numpy(B).pin_memory()
    Ch = torch.full((256, 384), float("nan"), dtype=Ah.dtype).pin_memory()
    Ad, Bd = torch.empty_like(Ah, device="cuda"), torch.empty_like(Bh, device="cuda")
    Cdd = torch.empty((256, 384), dtype=Ah.dtype, device="cuda")
    for _ in range(2):  # twice: buffers reused across calls
        p.execute_host(Ah, Bh, Ch, Ad, Bd, Cdd)
        torch.cuda.synchronize()
        assert np.array_equal(Ch.numpy(), Cd)
    Co = oracle.fmm(A, B, OPlan.stationary(R.winograd(), 2))
    assert parity(Ch.numpy(), Co, A, B) <= (TOL64 if dtype == "f64" else TOL32)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_cuda_graph_replay(fb, dtype):
    # FP32: the tensor-core leaf (tensor maps encoded at capture, the in-pass split) replayed
    npdt = np.float64 if dtype == "f64" else np.float32
    A, B = fi.random_pair(512, 512, 512, seed=40, dtype=npdt)
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w, w], 512, 512, 512, dtype=dtype)
    ref = p.execute(dev(A), dev(B)).cpu().numpy()
    p.set_graph(True)
    Ad, Bd = dev(A), dev(B)
    C1 = torch.empty((512, 512), dtype=Ad.dtype, device="cuda")
    for _ in range(3):
        C1.zero_()
        p.execute(Ad, Bd, C1)
        torch.cuda.synchronize()
        assert np.array_equal(C1.cpu().numpy(), ref)
    C2 = torch.empty_like(C1)  # new buffers -> a second captured graph
    p.execute(Ad, Bd, C2)
    torch.cuda.synchronize()
    assert np.array_equal(C2.cpu().numpy(), ref)


@pytest.mark.parametrize("dtype,leaf", [("f64", 0), ("f32", 0), ("f32", 2)])
@pytest.mark.parametrize("dims", [(256, 128, 192), (200, 136, 72), (256, 128, 256)])  # last: in-pass split
def test_no_out_of_bounds_writes(fb, dtype, leaf, dims):
    # compute-sanitizer is closed on this pool: guard bands instead.  C has padding columns
    # (ldc > N) and guard rows before / after; the workspace has guard bytes after its end.
    # Nothing outside C[:, :N] and ws may change.
    M, K, N = dims
    L = 2 if all(d % 4 == 0 for d in dims) else 1
    if any(d % (2 ** L) for d in dims):
        pytest.skip("dims not divisible")
    npdt = np.float64 if dtype == "f64" else np.float32
    A, B = fi.random_pair(M, K, N, seed=50, dtype=npdt)
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w] * L, M, K, N, dtype=dtype, leaf=leaf)
    tdt = torch.float64 if dtype == "f64" else torch.float32
    ldc = N + 6
    big = torch.full((M + 8, ldc), 12345.0, dtype=tdt, device="cuda")
    Cv = big[4:4 + M, :N]
    nb = p.workspace_bytes()
    wsb = torch.full((nb + 4096,), 0xA5, dtype=torch.uint8, device="cuda")
    p.execute(dev(A), dev(B), Cv, ws=wsb[:nb])
    torch.cuda.synchronize()
    g = big.clone()
    g[4:4 + M, :N] = 12345.0
    assert torch.all(g == 12345.0), "write outside C[:, :N]"
    assert torch.all(wsb[nb:] == 0xA5), "write past the workspace"
    Co = oracle.fmm(A, B, OPlan.stationary(R.winograd(), L))
    assert parity(Cv.cpu().numpy(), Co, A, B) <= (TOL64 if dtype == "f64" else TOL32)


@pytest.mark.parametrize("names,sched,fusion", [(("winograd",) * 3, "hybrid", "on"),
                                                (("winograd",) * 3, "depth", "off"),
                                                (("strassen",) * 4, "breadth", "on")])
def test_no_out_of_bounds_writes_deep(fb, names, sched, fusion):
    # the same guard bands around the two-level passes (K1X2 / K3X2), the fused leaf kernel,
    # the hybrid and per-r depth-first top levels, with ragged 64 x 64 leaf tiles
    L = len(names)
    M, K, N = 2 ** L * 36, 2 ** L * 20, 2 ** L * 28
    A, B = fi.random_pair(M, K, N, seed=70 + L)
    p = fb.Plan([fb.Rule.builtin(n) for n in names], M, K, N)
    p.set_schedule(sched)
    p.set_fusion(fusion)
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
    Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
    assert parity(Cv.cpu().numpy(), Co, A, B) <= TOL64


def test_matmul_convenience_api(fb):
    # fb.matmul: cached plans; FP64 parity, FP32 (3xTF32) parity, scaling, padding
    A, B = fi.random_pair(300, 260, 200, seed=61)
    C1 = fb.matmul(dev(A), dev(B), rules=("strassen", "winograd")).cpu().numpy()
    Co = oracle.fmm(A, B, OPlan.uniform([R.strassen(), R.winograd()]))
    assert parity(C1, Co, A, B) <= TOL64
    C2 = fb.matmul(dev(A), dev(B), rules=("strassen", "winograd")).cpu().numpy()
    assert np.array_equal(C1, C2) and len(fb.fmm._PLAN_CACHE) >= 1
    A32, B32 = A.astype(np.float32), B.astype(np.float32)
    C3 = fb.matmul(dev(A32), dev(B32), rules=("winograd",) * 2).cpu().numpy()
    assert parity(C3, oracle.fmm(A32, B32, OPlan.stationary(R.winograd(), 2)), A32, B32) <= TOL32
    As, Bs = fi.draw("skew", 128, 64, 96, 3)
    Cs = fb.matmul(dev(As), dev(Bs), rules=("winograd",) * 2, scaling="repeated").cpu().numpy()
    Cso, _ = oracle.scaled_fmm(As, Bs, OPlan.stationary(R.winograd(), 2), mode="repeated", pow2=True)
    hi, lo = oracle.ref_dd(As, Bs)
    rel = lambda X: np.max(np.abs((X - hi) - lo) / np.abs(hi))
    assert rel(Cs) <= 10 * max(rel(Cso), 1e-15)


@pytest.mark.parametrize("fusion", ["off", "on"])
def test_deep_recursion_node_chunks(fb, fusion):
    # Strassen L = 6 on 128^3: 7^6 = 117649 leaves of 2 x 2 x 2 -- more nodes than a grid
    # dimension holds (65535), so the steps launch in node chunks (P:111-129 allows any depth)
    A, B = fi.random_pair(128, 128, 128, seed=66)
    p = fb.Plan([fb.Rule.builtin("strassen")] * 6, 128, 128, 128)
    p.set_fusion(fusion)
    Cg = p.execute(dev(A), dev(B)).cpu().numpy()
    Co = oracle.fmm(A, B, OPlan.stationary(R.strassen(), 6))
    assert parity(Cg, Co, A, B) <= TOL64
    Ai, Bi = fi.integer_pair(128, 128, 128, seed=3, lo=-2, hi=2)
    Ci = (Ai.astype(np.int64) @ Bi.astype(np.int64)).astype(np.float64)
    assert np.array_equal(p.execute(dev(Ai), dev(Bi)).cpu().numpy(), Ci)


def test_execute_host_batch_f32_hybrid(fb):
    # FP32 (3xTF32 leaves) through a hybrid-schedule plan (the host path uses its depth-first
    # twin), a stream of 4 problems over 2 buffer sets
    M = K = N = 512
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w, w, w], M, K, N, dtype="f32", leaf=fb.fmm.LEAF_3XTF32)
    p.set_schedule("hybrid")
    pairs = [fi.random_pair(M, K, N, seed=200 + i, dtype=np.float32) for i in range(4)]
    want = [p.execute(dev(A), dev(B)).cpu().numpy() for A, B in pairs]
    Ah = [torch.from_numpy(A).pin_memory() for A, _ in pairs]
    Bh = [torch.from_numpy(B).pin_memory() for _, B in pairs]
    Ch = [torch.empty((M, N), dtype=torch.float32).pin_memory() for _ in pairs]
    dv = lambda r, c: [torch.empty((r, c), dtype=torch.float32, device="cuda") for _ in range(2)]
    p.execute_host_batch(Ah, Bh, Ch, dv(M, K), dv(K, N), dv(M, N))
    torch.cuda.synchronize()
    for c, w_ in zip(Ch, want):
        assert np.array_equal(c.numpy(), w_)


@pytest.mark.parametrize("nbuf", [1, 2, 3])
@pytest.mark.parametrize("shape,scaling", [((256, 512, 384), None), ((250, 130, 66), None),
                                           ((256, 256, 256), "repeated")])
def test_execute_host_batch(fb, nbuf, shape, scaling):
    # fmm_execute_host_batch: a stream of different problems, pipelined over nbuf device buffer
    # sets, each result exactly fmm_execute's (the padded and the scaled plans take the
    # whole-operand copy path)
    M, K, N = shape
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w, w], M, K, N, scaling=scaling)
    n = 5
    pairs = [fi.random_pair(M, K, N, seed=100 + i) for i in range(n)]
    want = [p.execute(dev(A), dev(B)).cpu().numpy() for A, B in pairs]
    Ah = [torch.from_numpy(A).pin_memory() for A, _ in pairs]
    Bh = [torch.from_numpy(B).pin_memory() for _, B in pairs]
    Ch = [torch.full((M, N), float("nan"), dtype=torch.float64).pin_memory() for _ in range(n)]
    Ad = [torch.empty((M, K), dtype=torch.float64, device="cuda") for _ in range(nbuf)]
    Bd = [torch.empty((K, N), dtype=torch.float64, device="cuda") for _ in range(nbuf)]
    Cd = [torch.empty((M, N), dtype=torch.float64, device="cuda") for _ in range(nbuf)]
    for _ in range(2):  # twice: buffers and events reused across calls
        for c in Ch:
            c.fill_(float("nan"))
        p.execute_host_batch(Ah, Bh, Ch, Ad, Bd, Cd)
        torch.cuda.synchronize()
        for c, w_ in zip(Ch, want):
            assert np.array_equal(c.numpy(), w_)
    p.execute_host_batch([], [], [], Ad, Bd, Cd)  # empty batch


@pytest.mark.parametrize("names,dtype", [(("winograd",), "f64"), (("winograd",) * 2, "f64"),
                                         (("strassen",) * 3, "f64"), (("winograd", "classical222"), "f64"),
                                         (("winograd",) * 2, "f32")])
@pytest.mark.parametrize("P", [2, 3, 4])
def test_p2p_combine_virtual_ranks(fb, names, dtype, P):
    # comm mode 3 on virtual ranks: each rank's plan writes its owned top-level products into
    # its symmetric buffer; the combine over the P buffers (here local pointers standing in for
    # the IPC-mapped peers) gives, row slice by row slice, exactly the single-GPU C (ascending r)
    L = len(names)
    M, K, N = 2 ** L * 40, 2 ** L * 24, 2 ** L * 32
    npdt = np.float64 if dtype == "f64" else np.float32
    A, B = fi.random_pair(M, K, N, seed=50 + L + P, dtype=npdt)
    rules = [fb.Rule.builtin(n) for n in names]
    ref = fb.Plan(rules, M, K, N, dtype=dtype).execute(dev(A), dev(B)).cpu().numpy()
    plans, ptrs = [], []
    for rank in range(P):
        p = fb.Plan(rules, M, K, N, dtype=dtype)
        p.set_partition(rank, P)
        p.set_comm_mode("p2p")
        R = rules[0].info()["R"]
        assert p.sym_bytes() == -(-R // P) * (M >> 1) * (N >> 1) * A.itemsize + 256
        p.sym_alloc()
        p.execute(dev(A), dev(B))  # no communicator: only the owned products, into the buffer
        plans.append(p)
        ptrs.append(p.sym_ptr())
    torch.cuda.synchronize()
    C = torch.full((M, N), float("nan"), dtype=torch.from_numpy(A).dtype, device="cuda")
    for rank in range(P):
        plans[rank].p2p_combine(ptrs, C, M * rank // P, M * (rank + 1) // P)
    torch.cuda.synchronize()
    assert np.array_equal(C.cpu().numpy(), ref)


def test_p2p_mode_errors(fb):
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w, w], 256, 256, 256)
    p.set_partition(0, 2)
    p.set_comm_mode("p2p")
    with pytest.raises(fb.FmmError):  # no symmetric buffer
        p.execute(dev(np.zeros((256, 256))), dev(np.zeros((256, 256))))
    q = fb.Plan([w, w], 250, 256, 256)  # padded: not supported in mode 3
    q.set_partition(0, 2)
    q.set_comm_mode("p2p")
    q.sym_alloc()
    with pytest.raises(fb.FmmError):
        q.execute(dev(np.zeros((250, 256))), dev(np.zeros((256, 256))))
