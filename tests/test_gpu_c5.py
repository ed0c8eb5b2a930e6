"""Full-size parity at BASELINE config C5 (32768^3, S-W L=3) in the launch configuration bench.py
times (the hybrid top-level schedule the auto plan picks, same plan, same stream usage; also
bitwise against the per-r depth-first schedule), against the oracle on a
row/column sample it computes bitwise-exactly (oracle.fmm_sub on lifted rows / columns), plus a
whole-matrix property: the FMM result agrees with the library's own classical product within
the sum of the two Thm 4.3 bounds."""
import numpy as np
import pytest
import torch

import fmm_inputs as fi
import oracle
from oracle import rules as R

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N = 32768


@pytest.fixture(scope="module")
def c5():
    A, B = fi.draw_torch("u(-1,1)", N, N, N, 4)
    return A, B


def test_c5_f64_sampled_parity_and_bound(c5):
    import paper_1507_00687_b200 as fb
    A, B = c5
    Ad, Bd = A.cuda(), B.cuda()
    w = fb.Rule.builtin("winograd")
    plan = fb.Plan([w, w, w], N, N, N)
    assert plan.launch_count() == 1 + 7 * 2 + 1  # hybrid: root K1, 7 x (K1X2 + K2F), K3X2
    Cd = plan.execute(Ad, Bd)
    torch.cuda.synchronize()
    pdf = fb.Plan([w, w, w], N, N, N)
    pdf.set_schedule("depth")  # per-r depth-first (the multi-GPU and host-pipeline form)
    assert torch.equal(pdf.execute(Ad, Bd), Cd)
    del pdf
    torch.cuda.empty_cache()
    An, Bn = A.numpy(), B.numpy()
    amax, bmax = float(np.abs(An).max()), float(np.abs(Bn).max())
    op = R.Plan.stationary(R.winograd(), 3)
    G = oracle.lift_rows(N, op, [0, 1, 2047, 4095])
    H = oracle.lift_cols(N, op, [0, 5, 4095])
    Co = oracle.fmm_sub(An, Bn, op, G, H)
    Cg = Cd[torch.from_numpy(G).cuda()][:, torch.from_numpy(H).cuda()].cpu().numpy()
    assert oracle.parity_metric(Cg, Co, amax, bmax, N) <= 1e-13
    # whole-matrix property vs the classical leaf kernel on the full problem
    Cc = fb.gemm(Ad, Bd)
    diff = (Cd - Cc).abs().max().item()
    eps = 2.0 ** -53
    f_fmm = float(R.stationary_bound_factor(R.winograd(), 3, N))
    f_cls = float(N) ** 2
    assert diff <= (f_fmm + f_cls) * amax * bmax * eps
    # and against the double-double reference on the sampled rows (Thm 4.3 bound)
    hi, lo = oracle.ref_dd(An, np.ascontiguousarray(Bn[:, H]), rows=G[:8])
    err = np.max(np.abs((Cg[:8] - hi) - lo))
    assert err <= f_fmm * amax * bmax * eps


def test_c5_f32_3xtf32_sampled_parity(c5):
    # the FP32 variant of C5 (FP64 draws cast to FP32), 3xTF32 tensor-core leaves
    import paper_1507_00687_b200 as fb
    A, B = c5
    A32, B32 = A.float(), B.float()
    w = fb.Rule.builtin("winograd")
    plan = fb.Plan([w, w, w], N, N, N, dtype="f32", leaf=fb.fmm.LEAF_3XTF32)
    Cd = plan.execute(A32.cuda(), B32.cuda())
    torch.cuda.synchronize()
    An, Bn = A32.numpy(), B32.numpy()
    op = R.Plan.stationary(R.winograd(), 3)
    G = oracle.lift_rows(N, op, [0, 4095])
    H = oracle.lift_cols(N, op, [3, 2048])
    Co = oracle.fmm_sub(An, Bn, op, G, H)
    Cg = Cd[torch.from_numpy(G).cuda()][:, torch.from_numpy(H).cuda()].cpu().numpy()
    assert oracle.parity_metric(Cg, Co, float(np.abs(An).max()), float(np.abs(Bn).max()), N) <= 5e-5
