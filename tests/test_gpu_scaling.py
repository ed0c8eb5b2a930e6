"""GPU diagonal scaling (K4) against the oracle: factors and scaled matrices bitwise (the max
reductions are exact, divisions / sqrt correctly rounded, same operation order), the stopping
test's step count equal, and scaled FMM products at the C4 recipe (componentwise check, since
the normalised parity metric is vacuous for C4's skewed magnitudes -- SURVEY §8(c) C-tol)."""
import numpy as np
import pytest
import torch

import fmm_inputs as fi
import oracle
from oracle import rules as R
from oracle.rules import Plan as OPlan

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fb():
    import paper_1507_00687_b200 as fb
    return fb


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def host(t):
    return t.cpu().numpy()


INPUTS = {
    "c4_small": lambda: fi.config_inputs("C4", scale_div=64),  # 64^3, C4 recipe
    "c4_rect": lambda: fi.draw("skew", 96, 40, 72, 3),
    "ex69": lambda: (np.array([[1.0, 2.0 ** 40], [1.0, 1.0]]), np.array([[2.0 ** -40, 1.0], [2.0 ** -40, 1.0]])),
}


@pytest.mark.parametrize("name", sorted(INPUTS))
@pytest.mark.parametrize("pow2", [False, True])
def test_outside_inside_bitwise(fb, name, pow2):
    A, B = INPUTS[name]()
    Ao, Bo, dA, dB = fb.scale_outside(dev(A), dev(B), pow2=pow2)
    ra, rb, rdA, rdB = oracle.scale_outside(A, B, pow2=pow2)
    for g, o in ((Ao, ra), (Bo, rb), (dA, rdA), (dB, rdB)):
        assert np.array_equal(host(g), o)
    Ai, Bi, d = fb.scale_inside(dev(A), dev(B), pow2=pow2)
    ra, rb, rd = oracle.scale_inside(A, B, pow2=pow2)
    for g, o in ((Ai, ra), (Bi, rb), (d, rd)):
        assert np.array_equal(host(g), o)


@pytest.mark.parametrize("name", sorted(INPUTS))
@pytest.mark.parametrize("first_O", [True, False])
@pytest.mark.parametrize("tau,pow2", [(1.0, False), (0.1, False), (1.0, True), (0.0, False)])
def test_repeated_bitwise(fb, name, first_O, tau, pow2):
    A, B = INPUTS[name]()
    g = fb.scale_repeated(dev(A), dev(B), first_O=first_O, tau=tau, max_steps=12, pow2=pow2)
    o = oracle.scale_repeated(A, B, first_O=first_O, tau=tau, max_steps=12, pow2=pow2)
    assert g["steps"] == o["steps"]
    for k in ("A", "B", "dA", "dB", "dI"):
        assert np.array_equal(host(g[k]), o[k]), k


def test_lemma_sequence_on_gpu(fb):
    # Lemma alt-scaling-example, v = 2: the cumulative s_2 factor sequence.
    A = np.array([[1.0, 0.0], [1.0, 2.0 ** -4]])
    B = np.eye(2)
    for n, want in ((1, 1.0), (3, 0.25), (5, 0.125)):
        g = fb.scale_repeated(dev(A), dev(B), first_O=True, tau=0.0, max_steps=n)
        assert host(g["dB"])[1] == want


def test_zero_row_precondition(fb):
    A = np.ones((8, 8))
    A[3] = 0
    with pytest.raises(fb.FmmError) as e:
        fb.scale_outside(dev(A), dev(np.ones((8, 8))))
    assert e.value.status == "FMM_E_PRECOND" and "index 3" in str(e.value)


@pytest.mark.parametrize("mode", ["none", "outside", "inside", "out_in", "in_out", "repeated"])
def test_scaled_fmm_C4_recipe(fb, mode):
    # C4 recipe at 512^3 (S-W L=3, 64^3 leaves), pow2 factors (reading A7)
    A, B = fi.config_inputs("C4", scale_div=8)
    M, K = A.shape
    N = B.shape[1]
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w, w, w], M, K, N, scaling={"mode": mode, "tau": 1.0, "max_steps": 20, "pow2": 1})
    Cg = host(p.execute(dev(A), dev(B)))
    steps = p.last_scaling_steps()
    plan = OPlan.stationary(R.winograd(), 3)
    Co, info = oracle.scaled_fmm(A, B, plan, mode=mode, pow2=True, tau=1.0, max_steps=20)
    assert steps == info["steps"]
    hi, lo = oracle.ref_dd(A, B)
    rel = lambda X: np.max(np.abs((X - hi) - lo) / np.abs(hi))
    rel_o = rel(Co)
    # componentwise GPU vs oracle at the level of the mode's own relative error
    d = np.max(np.abs(Cg - Co) / np.abs(hi))
    assert d <= 10 * max(rel_o, 1e-13), (mode, d, rel_o)
    assert oracle.parity_metric(Cg, Co, np.abs(A).max(), np.abs(B).max(), K) <= 1e-13
    if mode == "repeated":
        assert rel(Cg) < 1e-10  # repeated O-I is accurate on this skew
    # the scaling wraps any schedule: depth-first and hybrid top levels give the same bits
    for sched in ("depth", "hybrid"):
        p.set_schedule(sched)
        assert np.array_equal(host(p.execute(dev(A), dev(B))), Cg), sched


@pytest.mark.parametrize("pow2", [True, False])
def test_extreme_magnitudes_bitwise(fb, pow2):
    # rows / columns near the top and bottom of the FP64 range: the power-of-two factors 2^1023
    # and subnormal powers of two have no normal reciprocal, so the library falls back from
    # the multiply-by-reciprocal pass to true division (flags[F_INEXACT]); results stay bitwise
    # the oracle's (reading A9)
    g = np.random.default_rng(3)
    A = g.uniform(0.5, 1.0, (64, 96))
    B = g.uniform(0.5, 1.0, (96, 80))
    A[5] *= 1.2e308                 # rounds to 2^1023: reciprocal subnormal
    A[7] *= 2.0 ** -1060            # subnormal row
    B[:, 3] *= 1.2e308
    B[:, 9] *= 2.0 ** -1065
    for first_O in (True, False):
        gg = fb.scale_repeated(dev(A), dev(B), first_O=first_O, tau=1.0, max_steps=6, pow2=pow2)
        o = oracle.scale_repeated(A, B, first_O=first_O, tau=1.0, max_steps=6, pow2=pow2)
        assert gg["steps"] == o["steps"]
        for k in ("A", "B", "dA", "dB", "dI"):
            assert np.array_equal(host(gg[k]), o[k]), k
    Ao, Bo, dA, dB = fb.scale_outside(dev(A), dev(B), pow2=pow2)
    ra, rb, rdA, rdB = oracle.scale_outside(A, B, pow2=pow2)
    for x, y in ((Ao, ra), (Bo, rb), (dA, rdA), (dB, rdB)):
        assert np.array_equal(host(x), y)


def test_scale_apply_definition_and_roundtrip(fb):
    # fmm_scale_apply: a' = (a / dA_i) * d_k, b' = (b / d_k) / dB_j, each correctly rounded --
    # bitwise numpy's IEEE operations; with the cumulative pow2 factors of Alg. 3 it reproduces
    # the scaled matrices of fmm_scale_repeated exactly (eqn:scaling)
    A, B = fi.draw("skew", 96, 40, 72, 3)
    g = np.random.default_rng(1)
    dA, d, dB = g.uniform(0.5, 3, 96), g.uniform(0.5, 3, 40), g.uniform(0.5, 3, 72)
    Ao, Bo = fb.scale_apply(dev(A), dev(B), dev(dA), dev(d), dev(dB))
    assert np.array_equal(host(Ao), (A / dA[:, None]) * d[None, :])
    assert np.array_equal(host(Bo), (B / d[:, None]) / dB[None, :])
    r = fb.scale_repeated(dev(A), dev(B), first_O=True, tau=1.0, max_steps=12, pow2=True)
    Ao, Bo = fb.scale_apply(dev(A), dev(B), r["dA"], r["dI"], r["dB"])
    assert np.array_equal(host(Ao), host(r["A"])) and np.array_equal(host(Bo), host(r["B"]))


def _extreme_pair():
    # rows / columns whose power-of-two factors have no normal reciprocal (2^1023, subnormal),
    # and a row whose scaled entries become subnormal after the first O step (max 2^600, an
    # entry 2^-430 (1 + 2^-20) -> 2^-1030 (1 + 2^-20): not representable) -- both force the
    # one-kernel scaling run from its virtual form to the materialised one, on device
    g = np.random.default_rng(3)
    A = g.uniform(0.5, 1.0, (64, 96))
    B = g.uniform(0.5, 1.0, (96, 80))
    A[5] *= 1.2e308
    A[7] *= 2.0 ** -1060
    B[:, 3] *= 1.2e308
    B[:, 9] *= 2.0 ** -1065
    return A, B


def _subnormal_after_step_pair():
    g = np.random.default_rng(4)
    A = g.uniform(0.5, 1.0, (64, 96))
    B = g.uniform(0.5, 1.0, (96, 80))
    A[11, :] *= 2.0 ** 600
    A[11, 17] = 2.0 ** -430 * (1 + 2.0 ** -20)
    return A, B


SCALED_PLANS = {
    "L1_fused": (("winograd",), "auto", "on"),
    "L2": (("winograd",) * 2, "auto", "auto"),
    "L3_breadth": (("winograd",) * 3, "breadth", "auto"),
    "L3_depth": (("winograd",) * 3, "depth", "off"),
    "L3_hybrid": (("winograd", "classical222", "strassen"), "hybrid", "on"),
}


@pytest.mark.parametrize("pname", sorted(SCALED_PLANS))
@pytest.mark.parametrize("mode", ["outside", "inside", "out_in", "in_out", "repeated"])
def test_virtual_scaling_equals_materialised(fb, pname, mode):
    # virtual scaling (pow2 factors applied while the root K1 reads A, B; unscale folded into the
    # root combination) is bitwise the materialised form, on every schedule
    names, sched, fusion = SCALED_PLANS[pname]
    L = len(names)
    M, K, N = 2 ** L * 48, 2 ** L * 40, 2 ** L * 36
    A, B = fi.draw("skew", M, K, N, 3)
    rules = [fb.Rule.builtin(n) for n in names]
    sc = {"mode": mode, "tau": 1.0, "max_steps": 20, "pow2": 1}
    pv = fb.Plan(rules, M, K, N, scaling=sc)
    pm = fb.Plan(rules, M, K, N, scaling=sc)
    pm.set_virtual_scaling(False)
    for p in (pv, pm):
        p.set_schedule(sched)
        p.set_fusion(fusion)
    Cv = host(pv.execute(dev(A), dev(B)))
    Cm = host(pm.execute(dev(A), dev(B)))
    assert np.array_equal(Cv, Cm)
    assert pv.last_scaling_steps() == pm.last_scaling_steps()
    Co, info = oracle.scaled_fmm(A, B, OPlan.uniform([R.builtin(n) for n in names]), mode=mode,
                                 pow2=True, tau=1.0, max_steps=20)
    assert pv.last_scaling_steps() == info["steps"]
    assert oracle.parity_metric(Cv, Co, np.abs(A).max(), np.abs(B).max(), K) <= 1e-13


@pytest.mark.parametrize("pair", ["extreme", "subnormal_after_step"])
@pytest.mark.parametrize("mode", ["outside", "out_in", "repeated"])
def test_virtual_scaling_falls_back_bitwise(fb, pair, mode):
    # inputs the virtual form cannot carry: the run switches to the materialised form on
    # device; the entry point's A', B', factors and steps stay bitwise the oracle's, and a
    # scaled plan's C is bitwise the materialised plan's
    A, B = _extreme_pair() if pair == "extreme" else _subnormal_after_step_pair()
    first_O = True
    steps = {"outside": 1, "out_in": 2, "repeated": 12}[mode]
    tau = 1.0 if mode == "repeated" else -1.0
    gg = fb.scale_repeated(dev(A), dev(B), first_O=first_O, tau=tau, max_steps=steps, pow2=True)
    o = oracle.scale_repeated(A, B, first_O=first_O, tau=tau, max_steps=steps, pow2=True)
    assert gg["steps"] == o["steps"]
    for k in ("A", "B", "dA", "dB", "dI"):
        assert np.array_equal(host(gg[k]), o[k]), k
    w = fb.Rule.builtin("winograd")
    sc = {"mode": mode, "tau": 1.0, "max_steps": 12, "pow2": 1}
    pv = fb.Plan([w, w], 64, 96, 80, scaling=sc)
    pm = fb.Plan([w, w], 64, 96, 80, scaling=sc)
    pm.set_virtual_scaling(False)
    Cv = host(pv.execute(dev(A), dev(B)))
    Cm = host(pm.execute(dev(A), dev(B)))
    assert np.array_equal(Cv, Cm, equal_nan=True)


def test_virtual_scaling_in_cuda_graph(fb):
    # the one-kernel scaling run is a cooperative launch: captured and replayed in a graph
    A, B = fi.draw("skew", 256, 256, 256, 3)
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w, w, w], 256, 256, 256, scaling={"mode": "repeated", "pow2": 1})
    ref = host(p.execute(dev(A), dev(B)))
    p.set_graph(True)
    Ad, Bd = dev(A), dev(B)
    C = torch.empty((256, 256), dtype=torch.float64, device="cuda")
    for _ in range(3):
        C.zero_()
        p.execute(Ad, Bd, C)
        torch.cuda.synchronize()
        assert np.array_equal(host(C), ref)


@pytest.mark.parametrize("dims", [(1536, 2200, 700), (600, 4096, 1100)])
def test_repeated_wide_matrices_bitwise(fb, dims):
    # rows / columns wider than one reduction tile (512 / 256 columns): factors, steps and the
    # scaled matrices bitwise the oracle's (a tiling bug that skips columns changes the steps)
    M, K, N = dims
    A, B = fi.draw("skew", M, K, N, 3)
    for first_O in (True, False):
        g = fb.scale_repeated(dev(A), dev(B), first_O=first_O, tau=1.0, max_steps=20, pow2=True)
        o = oracle.scale_repeated(A, B, first_O=first_O, tau=1.0, max_steps=20, pow2=True)
        assert g["steps"] == o["steps"]
        for k in ("A", "B", "dA", "dB", "dI"):
            assert np.array_equal(host(g[k]), o[k]), k


@pytest.mark.parametrize("dims", [(300, 4094, 500), (257, 4097, 300), (96, 2, 64), (40, 3, 50),
                                  (5000, 512, 64)])
def test_repeated_fused_pass_edges_bitwise(fb, dims):
    # the fused A pass before an O step (whole rows, K <= 4096 even) at its
    # edges: a ragged last 512-column segment, K past the limit or odd (the unfused passes run),
    # tiny K, and more rows than blocks x 16 (several rows per tile)
    M, K, N = dims
    A, B = fi.draw("skew", M, K, N, 5)
    for first_O in (True, False):
        g = fb.scale_repeated(dev(A), dev(B), first_O=first_O, tau=0.0, max_steps=7, pow2=True)
        o = oracle.scale_repeated(A, B, first_O=first_O, tau=0.0, max_steps=7, pow2=True)
        assert g["steps"] == o["steps"]
        for k in ("A", "B", "dA", "dB", "dI"):
            assert np.array_equal(host(g[k]), o[k]), k


@pytest.mark.parametrize("first_O", [True, False])
def test_fused_pass_fallback_at_later_step(fb, first_O):
    # a value that turns subnormal only after a later O step: with first_O = False the first
    # fused pass is the one before step 1, so its speculative column maxima (F_BADX) are what
    # sends the run to the materialised form there; bitwise the oracle either way
    A, B = _subnormal_after_step_pair()
    gg = fb.scale_repeated(dev(A), dev(B), first_O=first_O, tau=0.0, max_steps=6, pow2=True)
    o = oracle.scale_repeated(A, B, first_O=first_O, tau=0.0, max_steps=6, pow2=True)
    assert gg["steps"] == o["steps"]
    for k in ("A", "B", "dA", "dB", "dI"):
        assert np.array_equal(host(gg[k]), o[k]), k


@pytest.mark.parametrize("M", [160000, 180000])
def test_repeated_fused_pass_tall_bitwise(fb, M):
    # tall A: about 1000 rows per fused tile at 160000 rows (the tile's exponents staged in
    # shared memory hold 1024), past that the run falls back to the unfused passes; bitwise the
    # oracle either way
    K, N = 64, 48
    A, B = fi.draw("skew", M, K, N, 6)
    for first_O in (True, False):
        g = fb.scale_repeated(dev(A), dev(B), first_O=first_O, tau=0.0, max_steps=5, pow2=True)
        o = oracle.scale_repeated(A, B, first_O=first_O, tau=0.0, max_steps=5, pow2=True)
        assert g["steps"] == o["steps"]
        for k in ("A", "B", "dA", "dB", "dI"):
            assert np.array_equal(host(g[k]), o[k]), k


@pytest.mark.parametrize("dims", [(300, 4094, 200), (96, 2, 64), (257, 600, 300), (1100, 4096, 520)])
def test_repeated_guard_band_bitwise(fb, dims):
    # A and B as views into larger buffers whose padding (columns past K / N and rows past
    # M / K) holds a huge finite sentinel: a pass that read past a row's end or the last row
    # would change a maximum, hence the factors and the steps.  Row pitches stay even (the
    # fused pass and the TMA rings need 16-byte aligned rows).
    M, K, N = dims
    A, B = fi.draw("skew", M, K, N, 7)
    Ab = torch.full((M + 3, K + 6), 1e300, dtype=torch.float64, device="cuda")
    Bb = torch.full((K + 3, N + 6), 1e300, dtype=torch.float64, device="cuda")
    Ab[:M, :K] = dev(A)
    Bb[:K, :N] = dev(B)
    for first_O in (True, False):
        g = fb.scale_repeated(Ab[:M, :K], Bb[:K, :N], first_O=first_O, tau=0.0, max_steps=6, pow2=True)
        o = oracle.scale_repeated(A, B, first_O=first_O, tau=0.0, max_steps=6, pow2=True)
        assert g["steps"] == o["steps"]
        for k in ("A", "B", "dA", "dB", "dI"):
            assert np.array_equal(host(g[k]), o[k]), k
    assert bool((Ab[M:, :] == 1e300).all()) and bool((Ab[:, K:] == 1e300).all())  # inputs untouched
    assert bool((Bb[K:, :] == 1e300).all()) and bool((Bb[:, N:] == 1e300).all())
