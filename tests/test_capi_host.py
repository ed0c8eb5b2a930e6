"""Host-side (no GPU) checks of the C-ABI library: it loads, exports every symbol include/fmm.h
declares, its rule tables / Brent check / plan logic behave, and its built-in rules equal the
oracle's independently written tables."""
import ctypes
import re

import numpy as np
import pytest

import paper_1507_00687_b200 as fb
from fmm_testutil import ROOT
from oracle import rules as R


def _declared_symbols():
    src = (ROOT / "include" / "fmm.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fmm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = fb.lib()
    syms = _declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s
    # the binding mirrors the header one-to-one
    assert set(fb.fmm.SIGNATURES) == set(syms)


@pytest.mark.parametrize("name", sorted(R.BUILTINS))
def test_builtin_rules_match_oracle_tables(name):
    info = fb.Rule.builtin(name).info()
    ref = R.builtin(name)
    for key in ("U", "V", "W"):
        want = np.array([[int(x) for x in row] for row in getattr(ref, key)])
        assert np.array_equal(info[key], want), (name, key)
    assert info["log2_den"] == 0


def test_rule_create_rejects_brent_violation():
    s = R.strassen()
    U = np.array([[int(x) for x in r] for r in s.U])
    V = np.array([[int(x) for x in r] for r in s.V])
    W = np.array([[int(x) for x in r] for r in s.W])
    ok = fb.Rule.create(2, 2, 2, U, V, W, name="mystrassen")
    assert ok.info()["R"] == 7
    W2 = W.copy()
    W2[0, 3] = -W2[0, 3]
    with pytest.raises(fb.FmmError) as e:
        fb.Rule.create(2, 2, 2, U, V, W2)
    assert e.value.status == "FMM_E_RULE" and e.value.n_violations > 0
    # App. A as printed (transposed convention) is rejected
    from fmm_testutil import read_golden_matrices
    g = read_golden_matrices("app_a_strassen_printed.txt")
    with pytest.raises(fb.FmmError):
        fb.Rule.create(2, 2, 2, g["U"], g["V"], g["W"])


def test_rule_create_dyadic_coefficients():
    # classical with all coefficients scaled: U*2, V*2, W/4 -> numerators (2,2,1) / 2^2? Use a
    # denominator: U = 2/2, V = 2/2, W = 2/2 represents the same rule (coefficient 1).
    c = R.classical222()
    U = np.array([[int(x) * 2 for x in r] for r in c.U])
    V = np.array([[int(x) * 2 for x in r] for r in c.V])
    W = np.array([[int(x) * 2 for x in r] for r in c.W])
    fb.Rule.create(2, 2, 2, U, V, W, log2_den=1)
    with pytest.raises(fb.FmmError):
        fb.Rule.create(2, 2, 2, U, V, W, log2_den=0)  # = 8x the classical product


def test_plan_shape_errors_and_workspace():
    w = fb.Rule.builtin("winograd")
    # non-divisible dims are zero-padded: 510 -> 512 costs the padded copies
    pp = fb.Plan([w, w], 510, 512, 512)
    p = fb.Plan([w, w], 512, 512, 512)
    assert p.launch_count() == 1  # the single-launch small plan (K1X2, leaves, K3X2 in one kernel)
    p.set_single_launch(False)
    assert pp.launch_count() == p.launch_count() + 3 == 6  # pad A, pad B, crop C
    assert pp.workspace_bytes() == p.workspace_bytes() + 3 * 512 * 512 * 8
    ws = p.workspace_bytes()
    # breadth-first, two levels per K1 pass (default): level 1: 7 M blocks of 256^2 (its S / T
    # are never formed); level 2: 40 S + 40 T (49 minus the 3 x 3 products whose U / V columns
    # are trivial at both levels: views of A, B) + 49 M of 128^2
    exp = 7 * 256 * 256 * 8 + (40 + 40 + 49) * 128 * 128 * 8
    assert exp <= ws <= exp + (1 << 16)
    assert p.launch_count() == 1 + 1 + 1  # one K1X2 (S and T of both levels), K2, one K3X2
    p.set_k3_levels(1)
    assert p.launch_count() == 1 + 1 + 2  # K3 one level per pass
    with pytest.raises(fb.FmmError):
        p.set_k3_levels(0)
    # one level per pass: level 1: 4 S + 4 T + 7 M of 256^2; level 2: 28 + 28 + 49 of 128^2
    p.set_k1_levels(1)
    exp = (4 + 4 + 7) * 256 * 256 * 8 + (28 + 28 + 49) * 128 * 128 * 8
    assert exp <= p.workspace_bytes() <= exp + (1 << 16)
    assert p.launch_count() == 2 + 1 + 2  # K1 x2 levels (S and T in one launch), K2, K3 x2
    with pytest.raises(fb.FmmError):
        p.set_k1_levels(3)


def test_partition_ownership():
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w, w, w], 1024, 1024, 1024)
    for P in (1, 2, 4, 8):
        owned = [p.owned(r, P) for r in range(P)]
        flat = sorted(x for o in owned for x in o)
        assert flat == list(range(7))  # every top-level product exactly once
        for r in range(P):
            assert owned[r] == [x for x in range(7) if x % P == r]
    p.set_partition(1, 4)
    assert p.workspace_bytes() > 0


def test_nonuniform_plan_validation():
    s, d = fb.Rule.builtin("strassen"), fb.Rule.builtin("strassen_dalberto")
    nodes = [s] + [d if r in (0, 2, 3) else s for r in range(7)]
    fb.Plan(nodes, 256, 256, 256, uniform=False, levels=2)
    with pytest.raises(fb.FmmError):
        fb.Plan(nodes[:5], 256, 256, 256, uniform=False, levels=2)
    c = fb.Rule.builtin("classical222")
    with pytest.raises(fb.FmmError):  # rank differs within a level
        fb.Plan([s] + [c] + [s] * 6, 256, 256, 256, uniform=False, levels=2)


def test_fusion_auto_policy():
    # auto (FP64): fuse the leaf-parent level when parents x 128^2 leaf tiles fill >= 4 waves
    # of 148 SMs at >= 90 % wave efficiency (the grid kernel K2F)
    w, s, c = (fb.Rule.builtin(n) for n in ("winograd", "strassen", "classical222"))
    cases = [([w, w], (512,) * 3, 0),                 # C1: 7 parents x 1 tile
             ([s] * 4, (4096,) * 3, 1),               # C2: 343 x 4 = 1372 (9.3 waves, 93 %)
             ([w, c, s], (8192, 4096, 8192), 1),     # C3: 56 x 64 = 3584 (97 %)
             ([w] * 3, (4096,) * 3, 1),               # C4: 49 x 16 = 784: chains split in 2 (turnstiles)
             ([w] * 3, (32768,) * 3, 7)]              # C5: depth-first, 7 x 1024 per subtree
    for rules, (M, K, N), want in cases:
        p = fb.Plan(rules, M, K, N)
        assert p.fused_launches() == want, (M, want)
    p = fb.Plan([w] * 3, 4096, 4096, 4096)
    p.set_fusion("on")
    ws_fused = p.workspace_bytes()
    p.set_fusion("off")
    assert p.fused_launches() == 0
    assert p.workspace_bytes() > ws_fused  # leaf M_r buffers are not allocated when fused
    p32 = fb.Plan([w] * 3, 4096, 4096, 4096, dtype="f32")
    assert p32.fused_launches() == 0


def test_shard_depth_units_and_balance():
    # finer units improve the R = 7 balance cap 7 / (P ceil(7/P)) = 87.5 %
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w] * 3, 1024, 1024, 1024)
    for depth, P, cap in ((1, 8, 7 / 8), (2, 4, 49 / (4 * 13)), (2, 2, 49 / 50), (3, 8, 343 / (8 * 43))):
        p.set_shard_depth(depth)
        owned = [p.owned(r, P) for r in range(P)]
        assert sorted(u for o in owned for u in o) == list(range(7 ** depth))
        assert abs(7 ** depth / (P * max(len(o) for o in owned)) - cap) < 1e-12
    with pytest.raises(fb.FmmError):
        p.set_shard_depth(4)


def test_bench_pass_byte_model():
    # bench.py's pipeline roofline counts the algorithmic pass bytes: one S-W
    # level on n^3: K1 reads the 4 quarter blocks of A and B and writes 4 non-trivial S and T;
    # K3 reads 7 products and writes 4 quarters; a fused leaf level writes its output only;
    # classical levels form nothing (all operands are aliases)
    import bench
    w = fb.Rule.builtin("winograd").info()
    c = fb.Rule.builtin("classical222").info()
    n, q = 1024, (512 * 512) * 8
    assert bench.pass_bytes([w], n, n, n, 8, False) == (4 + 4) * q * 2 + (7 + 4) * q
    assert bench.pass_bytes([w], n, n, n, 8, True) == (4 + 4) * q * 2 + 4 * q
    assert bench.pass_bytes([c], n, n, n, 8, False) == (8 + 4) * q


def test_execute_host_batch_argument_errors():
    # checked before any CUDA call: null arrays, nbuf < 1, count < 0, ld < cols
    lib = fb.lib()
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w], 64, 64, 64)
    P = ctypes.c_void_p
    one = (P * 1)(P(16))
    args = lambda count, nbuf, ld: (p._h, count, one, ld, one, ld, one, ld, one, one, one, nbuf,
                                    None, ctypes.c_size_t(0), None)
    assert lib.fmm_execute_host_batch(*args(1, 0, 64)) == 1   # nbuf < 1
    assert lib.fmm_execute_host_batch(*args(-1, 1, 64)) == 1  # count < 0
    assert lib.fmm_execute_host_batch(*args(1, 1, 32)) == 1   # ld < cols
    assert lib.fmm_execute_host_batch(p._h, 1, None, 64, one, 64, one, 64, one, one, one, 1,
                                      None, ctypes.c_size_t(0), None) == 1
    assert b"fmm_execute_host_batch" in lib.fmm_last_error()


def test_hybrid_schedule_structure():
    # hybrid (schedule 3): one root K1, per top-level r a K1X2 (levels 1-2) and a K2F, one
    # K3X2 (levels 0-1) at the end; auto picks it for single-rank plans whose breadth-first
    # workspace exceeds 24 GiB (C5), and depth-first when partitioned
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w] * 3, 1024, 1024, 1024)
    p.set_fusion("on")
    p.set_schedule("hybrid")
    assert p.launch_count() == 1 + 7 * 2 + 1
    big = fb.Plan([w] * 3, 32768, 32768, 32768)
    assert big.launch_count() == 1 + 7 * 2 + 1
    assert big.workspace_bytes() <= 64 << 30
    big.set_partition(0, 2)
    assert big.launch_count() != 1 + 7 * 2 + 1
    with pytest.raises(fb.FmmError):
        fb.fmm._call("fmm_plan_set_schedule", p._h, 4)


def test_p2p_comm_mode_schedule():
    # comm mode 3: owned top-level products go to the symmetric buffer (no ACC into a partial
    # C, no zeroing); its size is ceil(R / P) products plus the barrier scratch
    w = fb.Rule.builtin("winograd")
    p = fb.Plan([w, w], 512, 512, 512)
    p.set_partition(0, 2)
    n_reduce = p.launch_count()
    p.set_comm_mode("p2p")
    assert p.launch_count() == n_reduce - 4  # rank 0 owns r = 0, 2, 4, 6: four ACC launches
    assert p.sym_bytes() == 4 * 256 * 256 * 8 + 256
    p.set_comm_mode("reduce")
    assert p.launch_count() == n_reduce
    with pytest.raises(fb.FmmError):
        fb.fmm._call("fmm_plan_set_comm_mode", p._h, 4)


def test_leaf_split_and_shard_order_host():
    # host-only plan structure of the round-2 options (no GPU needed to compile a plan)
    w = fb.Rule.builtin("winograd")
    # FP32 tensor-core leaves: the in-pass split removes no launch (the split kernel runs inside
    # the leaf step) but the plan compiles both ways; other values are argument errors
    p = fb.Plan([w, w], 512, 512, 512, dtype="f32", leaf=fb.fmm.LEAF_3XTF32)
    n1 = p.launch_count()
    p.set_leaf_split(False)
    assert p.launch_count() == n1
    with pytest.raises(fb.FmmError):
        fb.fmm._call("fmm_plan_set_leaf_split", p._h, 2)
    with pytest.raises(fb.FmmError):
        fb.fmm._call("fmm_plan_set_shard_order", p._h, 2)
    # block units at depth 3 over 8 ranks: rank 0 owns units 0..42 = six whole level-2 subtrees
    # (each run breadth-first: one S / T pass + one fused leaf launch) and one single unit
    q = fb.Plan([w] * 3, 1024, 1024, 1024)
    q.set_fusion("on")
    q.set_shard_depth(3)
    q.set_shard_order("block")
    assert q.owned(0, 8) == list(range(43))
    q.set_partition(0, 8)
    blocks = q.launch_count()
    q.set_shard_order("cyclic")
    assert q.launch_count() > blocks  # round-robin: every unit formed and combined on its own


def test_header_is_plain_c():
    # the boundary header compiles as C99 and as C++ (no torch / C++ types in the signatures)
    import shutil
    import subprocess
    hdr = ROOT / "include" / "fmm.h"
    for cc, lang, std in (("gcc", "c", "-std=c99"), ("g++", "c++", "-std=c++17")):
        if shutil.which(cc) is None:
            pytest.skip(f"{cc} not available")
        r = subprocess.run([cc, "-x", lang, std, "-fsyntax-only", "-Wall", "-Werror", str(hdr)],
                           capture_output=True, text=True)
        assert r.returncode == 0, r.stderr
