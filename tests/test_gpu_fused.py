"""GPU: the accumulation step fused into the leaf-product epilogue (K2F, fmm_plan_set_fusion).

The fused kernel runs a parent's R leaf products in ascending r per output tile and updates
C_k = w_kr M_r / C_k + w_kr M_r after each one -- the K3 / ACC sequence of roundings (Eq.
eqn:recursive_alg P:116-125, sequential summation P:241-246, reading A3) -- so fused
and unfused plans must agree BITWISE, and with unit leaf inner dimension both must equal the
oracle bitwise."""
import numpy as np
import pytest
import torch

import fmm_inputs as fi
import oracle
from oracle import rules as R
from oracle.rules import Plan as OPlan

pytestmark = pytest.mark.gpu

TOL64 = 1e-13

PLANS = {
    "winograd_L1": ("winograd",),
    "winograd_L2": ("winograd", "winograd"),
    "strassen_L3": ("strassen",) * 3,
    "classical_L2": ("classical222",) * 2,
    "C3_mix": ("winograd", "classical222", "strassen"),
}


@pytest.fixture(scope="module")
def fb():
    import paper_1507_00687_b200 as fb
    assert torch.cuda.is_available()
    return fb


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def plan(fb, names, M, K, N, fusion, schedule="auto"):
    p = fb.Plan([fb.Rule.builtin(n) for n in names], M, K, N)
    p.set_fusion(fusion)
    p.set_schedule(schedule)
    return p


def exe(p, A, B):
    C = p.execute(dev(A), dev(B))
    torch.cuda.synchronize()
    return C.cpu().numpy()


@pytest.mark.parametrize("pname", sorted(PLANS))
@pytest.mark.parametrize("schedule", ["breadth", "depth", "hybrid"])
def test_fused_equals_unfused_bitwise(fb, pname, schedule):
    names = PLANS[pname]
    A, B = fi.random_pair(512, 384, 256, seed=21)
    pf = plan(fb, names, 512, 384, 256, "on", schedule)
    assert pf.fused_launches() >= 1
    pu = plan(fb, names, 512, 384, 256, "off", schedule)
    assert pu.fused_launches() == 0
    Cf, Cu = exe(pf, A, B), exe(pu, A, B)
    assert np.array_equal(Cf, Cu)
    Co = oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]))
    assert oracle.parity_metric(Cf, Co, np.abs(A).max(), np.abs(B).max(), 384) <= TOL64


@pytest.mark.parametrize("pname", sorted(PLANS))
def test_fused_unit_leaf_bitwise_vs_oracle(fb, pname):
    names = PLANS[pname]
    L = len(names)
    A, B = fi.random_pair(16 * 2 ** L, 2 ** L, 8 * 2 ** L, seed=L + 3)
    Cf = exe(plan(fb, names, *A.shape, B.shape[1], "on"), A, B)
    assert np.array_equal(Cf, oracle.fmm(A, B, OPlan.uniform([R.builtin(n) for n in names])))


@pytest.mark.parametrize("dims", [(4 * 33, 4 * 17, 4 * 45), (4 * 129, 4 * 3, 4 * 65), (8, 4, 12)])
def test_fused_ragged_and_scalar_path(fb, dims):
    # leaf dims not multiples of the tile (ragged tiles) and odd leaf columns (8-byte path)
    M, K, N = dims
    A, B = fi.random_pair(M, K, N, seed=M + N)
    names = ("winograd", "strassen")
    Cf = exe(plan(fb, names, M, K, N, "on"), A, B)
    Cu = exe(plan(fb, names, M, K, N, "off"), A, B)
    assert np.array_equal(Cf, Cu)


def test_fused_dalberto_nonuniform(fb):
    s, d = fb.Rule.builtin("strassen"), fb.Rule.builtin("strassen_dalberto")
    nodes = [s] + [d if r in (0, 2, 3) else s for r in range(7)]
    A, B = fi.random_pair(64, 4, 64, seed=4)
    p = fb.Plan(nodes, 64, 4, 64, uniform=False, levels=2)
    p.set_fusion("on")
    assert p.fused_launches() == 1
    assert np.array_equal(exe(p, A, B), oracle.fmm(A, B, OPlan.dalberto_two_level()))


@pytest.mark.parametrize("L", [1, 2])
def test_fused_partition_partials(fb, L):
    # virtual ranks: each rank's partial C is the same with and without fusion
    A, B = fi.random_pair(256, 256, 256, seed=9)
    names = ("winograd",) * L
    for nranks in (2, 3):
        for rank in range(nranks):
            ps = [plan(fb, names, 256, 256, 256, f) for f in ("on", "off")]
            for p in ps:
                p.set_partition(rank, nranks)
            assert np.array_equal(exe(ps[0], A, B), exe(ps[1], A, B))


def test_fused_empty_inner_dimension(fb):
    p = plan(fb, ("winograd",), 8, 0, 8, "on")
    C = p.execute(torch.empty((8, 0), dtype=torch.float64, device="cuda"),
                  torch.empty((0, 8), dtype=torch.float64, device="cuda"))
    assert torch.all(C == 0)


def test_fused_no_out_of_bounds_writes(fb):
    M, K, N = 264, 136, 200
    A, B = fi.random_pair(M, K, N, seed=51)
    p = plan(fb, ("winograd", "winograd"), M, K, N, "on")
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
    Cu = exe(plan(fb, ("winograd", "winograd"), M, K, N, "off"), A, B)
    assert np.array_equal(Cv.cpu().numpy(), Cu)


def test_fused_C2_full_size_equals_unfused(fb):
    # C2 at full size (auto mode fuses it): bitwise equal to the unfused schedule
    A, B = fi.config_inputs("C2")
    pa = plan(fb, ("strassen",) * 4, 4096, 4096, 4096, "auto")
    assert pa.fused_launches() == 1
    Cf = exe(pa, A, B)
    Cu = exe(plan(fb, ("strassen",) * 4, 4096, 4096, 4096, "off"), A, B)
    assert np.array_equal(Cf, Cu)


@pytest.mark.parametrize("depth,nranks", [(2, 2), (2, 4), (2, 8), (3, 8)])
def test_shard_depth_virtual_ranks(fb, depth, nranks):
    # finer sharding (units = paths of the first `depth` levels): the ranks' partial C sum to
    # the product (parity), every unit is owned once, and rank partials are deterministic
    A, B = fi.random_pair(256, 256, 256, seed=12)
    names = ("winograd",) * 3
    ref = exe(plan(fb, names, 256, 256, 256, "auto"), A, B)
    total = np.zeros_like(ref)
    units = []
    for rank in range(nranks):
        p = plan(fb, names, 256, 256, 256, "auto")
        p.set_shard_depth(depth)
        p.set_partition(rank, nranks)
        units += p.owned(rank, nranks)
        part = exe(p, A, B)
        assert np.array_equal(part, exe(p, A, B))
        total += part
    assert sorted(units) == list(range(7 ** depth))
    assert oracle.parity_metric(total, ref, np.abs(A).max(), np.abs(B).max(), 256) <= TOL64


@pytest.mark.parametrize("dims,names", [((2048, 2048, 2048), ("winograd",) * 3),
                                        ((3072, 3072, 3072), ("winograd",) * 2)])
def test_split_chains_equal_unfused(fb, dims, names):
    # units whose R-product chain is split over 2-3 CTAs ordered by per-unit turnstiles (the
    # split is chosen by the plan's makespan model): bitwise the unfused K2 + K3, deterministic
    M, K, N = dims
    A, B = fi.random_pair(M, K, N, seed=K // 64)
    pa = plan(fb, names, M, K, N, "on")
    assert pa.fused_launches() == 1
    Cf = exe(pa, A, B)
    assert np.array_equal(Cf, exe(plan(fb, names, M, K, N, "off"), A, B))
    assert np.array_equal(Cf, exe(pa, A, B))


@pytest.mark.parametrize("split", [0x0706, 0x0701, 0x070301, 0x070502, 0x07060504])
def test_forced_split_equal_unfused(fb, monkeypatch, split):
    # non-uniform chain splits (byte g = end of group g's products, FMM_K2F_SPLIT tuning knob):
    # every grouping keeps each C element's ascending-r sum, so bitwise the unfused K2 + K3
    M = K = N = 1024
    names = ("strassen",) * 3
    A, B = fi.random_pair(M, K, N, seed=split % 97)
    monkeypatch.setenv("FMM_K2F_SPLIT", str(split))
    pa = plan(fb, names, M, K, N, "on")
    assert pa.fused_launches() == 1  # compiles the plan with the forced split
    Cf = exe(pa, A, B)
    assert np.array_equal(Cf, exe(plan(fb, names, M, K, N, "off"), A, B))
    assert np.array_equal(Cf, exe(pa, A, B))


@pytest.mark.parametrize("leaf", ["3xtf32", "tf32"])
@pytest.mark.parametrize("pname", ["winograd_L2", "C3_mix"])
def test_tf32_leaves_never_fuse(fb, leaf, pname):
    # the FP32 tensor-core leaves keep their products in TMEM chunk buffers + register totals
    # (k2p_tf32) and are combined by K3: fusion "on" compiles no fused launch and gives the
    # unfused result (the fused FP32 epilogue of round 1 was removed in round 2)
    names = PLANS[pname]
    M, K, N = 512, 384, 512
    A, B = fi.random_pair(M, K, N, seed=K, dtype=np.float32)
    lf = {"3xtf32": fb.fmm.LEAF_3XTF32, "tf32": fb.fmm.LEAF_TF32}[leaf]
    out = []
    for fusion in ("on", "off"):
        p = fb.Plan([fb.Rule.builtin(n) for n in names], M, K, N, dtype="f32", leaf=lf)
        p.set_fusion(fusion)
        assert p.fused_launches() == 0
        out.append(exe(p, A, B))
    assert np.array_equal(out[0], out[1])