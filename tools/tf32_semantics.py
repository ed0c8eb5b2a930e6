"""Experiment: how does tcgen05 kind::tf32 treat the low 13 mantissa bits of its FP32 inputs?
Single-pass TF32 on inputs x = 1 + d (d below TF32 precision) against exact products, and the
3xTF32 error and its mean (a bias shows truncating accumulation).  Round 1 compared three hi / lo
split modes here (profiles/r01_tf32_variants.md); the library keeps the round-to-nearest split."""
import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1507_00687_b200 as fb
# probe: A = [1 + 0.75 ulp_tf32] (1x32, first element only), B = [1] -> C = tf32-treatment of A
ulp = 2.0 ** -10
vals = [1 + 0.75 * ulp, 1 + 0.25 * ulp, 1 + 0.5 * ulp, -(1 + 0.75 * ulp)]
out = []
for v in vals:
    A = torch.zeros((128, 32), dtype=torch.float32); A[0, 0] = v
    B = torch.zeros((32, 256), dtype=torch.float32); B[0, 0] = 1.0
    C = fb.gemm(A.cuda(), B.cuda(), leaf=fb.fmm.LEAF_TF32)
    out.append((v, float(C[0, 0])))
print("single-pass TF32 of x*1:", [(f"{a:.10f}", f"{c:.10f}") for a, c in out])
rng = np.random.default_rng(0)
for K in (256, 4096):
    A = rng.uniform(-1, 1, (256, K)).astype(np.float32)
    B = rng.uniform(-1, 1, (K, 256)).astype(np.float32)
    exact = A.astype(np.float64) @ B.astype(np.float64)
    C = fb.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), leaf=fb.fmm.LEAF_3XTF32).cpu().numpy()
    print("K", K, "3xTF32 max|err|", float(np.abs(C - exact).max()),
          "mean err", float((C - exact).mean()))
