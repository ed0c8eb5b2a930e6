"""Host logic of bench.py that feeds reported numbers: the algorithmic pass bytes of the
whole-step pipeline roofline, checked against hand counts for Strassen-Winograd
(products and combinations in DESIGN.md reading A2; 4 non-trivial U and V columns, all 4 blocks
read; 3 trivial columns; W row nonzeros 2 + 4 + 4 + 4)."""
import sys

import pytest

from fmm_testutil import ROOT

sys.path.insert(0, str(ROOT))
import bench  # noqa: E402
import paper_1507_00687_b200 as fb  # noqa: E402


@pytest.fixture(scope="module")
def sw():
    return fb.Rule.builtin("winograd").info()


def test_one_level_counts(sw):
    n, e = 1024, 8
    q = (n // 2) ** 2  # one quarter block
    # K1: A's 4 blocks read once + 4 formed S, same for B; K3: 7 products read + C written
    k1 = 2 * (4 * q + 4 * q)
    assert bench.pass_bytes([sw], n, n, n, e, False, False, False) == (k1 + 7 * q + 4 * q) * e
    # fused leaf-parent level: the output written once instead of K3
    assert bench.pass_bytes([sw], n, n, n, e, True, False, False) == (k1 + 4 * q) * e


def test_two_level_counts(sw):
    n, e = 1024, 8
    s = (n // 4) ** 2  # one level-2 block
    # K1X2 per operand: the 16 sub-blocks read once, the 49 - 3*3 = 40 formed grandchildren
    k1x2 = 2 * (16 + 40) * s
    # K3X2 from the 49 level-2 products into C (16 sub-blocks)
    k3x2 = (49 + 16) * s
    assert bench.pass_bytes([sw, sw], n, n, n, e, False, True, True) == (k1x2 + k3x2) * e
    # one level per pass: level 0 (4 + 4 blocks of 4s per operand) then 7 nodes x (4 + 4) s,
    # K3 at level 1 (7 nodes x (7 + 4) s) and at level 0 (7 x 4s + 16 s)
    one = 2 * (4 * 4 * s + 4 * 4 * s) + 2 * 7 * (4 * s + 4 * s) + 7 * (7 * s + 4 * s) + (7 * 4 * s + 16 * s)
    assert bench.pass_bytes([sw, sw], n, n, n, e, False, False, False) == one * e


def test_depth_first_top_level_not_paired(sw):
    # the per-r depth-first top level combines with ACC, so K3 pairing starts at level 1
    n, e = 4096, 8
    paired = bench.pass_bytes([sw] * 3, n, n, n, e, True, True, True, False)
    unpaired_top = bench.pass_bytes([sw] * 3, n, n, n, e, True, True, True, True)
    assert paired < unpaired_top


def test_cpu_baseline_reports_parity_and_dd_errors():
    # the CPU-baseline leg on a small problem: the sampled parity against the oracle and both
    # paths' errors against the double-double reference are reported (here "GPU" = the oracle's
    # own full result, so the parity is 0 and the two errors coincide)
    import numpy as np
    import oracle
    from oracle import rules as OR
    import fmm_inputs as fi
    oracle.build()
    M = K = N = 128
    A, B = fi.random_pair(M, K, N, seed=5)
    full = oracle.fmm(A, B, OR.Plan.uniform([OR.builtin("winograd")] * 2))
    out = bench.cpu_baseline(A, B, ("winograd", "winograd"), M, K, N, C_gpu_host=full, target_s=0.01)
    assert out["kind"] == "oracle" and out["parity_sampled"] == 0.0
    e = out["error_vs_dd"]
    assert e["gpu"] == e["oracle"] and 0.0 < e["gpu"] < 1e-13


def test_tf32_split_counts(sw):
    # FP32 tensor-core leaves, two levels, 4-byte elements
    n, e = 1024, 4
    s = (n // 4) ** 2
    k3x2 = (49 + 16) * s
    # split in the leaf level's K1X2: all 49 grandchildren formed (views too), hi + lo written,
    # the 16 sub-blocks read once, per operand
    in_pass = 2 * (16 + 2 * 49) * s
    assert bench.pass_bytes([sw, sw], n, n, n, e, False, True, True, False, "pass") == (in_pass + k3x2) * e
    # split kernel: the 40 formed grandchildren written by K1X2, then all 49 leaf operands read
    # and their hi + lo written, per operand
    kernel = 2 * (16 + 40) * s + 2 * 3 * 49 * s
    assert bench.pass_bytes([sw, sw], n, n, n, e, False, True, True, False, "kernel") == (kernel + k3x2) * e


def test_default_shard():
    # bench.py's multi-GPU partition (profiles/r02_partition_times.md): one rank unsharded;
    # otherwise depth-3 units (or the plan's depth) in contiguous blocks
    assert bench.default_shard(1, 3) == (1, "cyclic")
    assert bench.default_shard(2, 3) == (3, "block")
    assert bench.default_shard(8, 3) == (3, "block")
    assert bench.default_shard(4, 2) == (2, "block")
