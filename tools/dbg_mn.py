import os, sys
sys.path.insert(0, '.')
import numpy as np, torch
import paper_1507_00687_b200 as fb
M, K, N = 128, 32, 256
A = np.zeros((M, K), np.float32)
for i in range(K): A[i, i] = 1.0
B = (np.arange(K * N, dtype=np.float32).reshape(K, N) % 1000) + 1
C = fb.gemm(torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda(), leaf=1).cpu().numpy()
ok = np.array_equal(C[:K], B)
print({k: os.environ.get(k) for k in ("FMM_MN_LBO", "FMM_MN_SBO", "FMM_MN_LAYOUT", "FMM_MN_SW128_PLAIN")}, "equal", ok, "C[0,:4]", C[0, :4], "C[1,:4]", C[1, :4])
rng = np.random.default_rng(0)
for (M2, K2, N2) in [(256, 512, 384), (200, 300, 100)]:
    A2 = rng.uniform(-1, 1, (M2, K2)).astype(np.float32); B2 = rng.uniform(-1, 1, (K2, N2)).astype(np.float32)
    C2 = fb.gemm(torch.from_numpy(A2).cuda(), torch.from_numpy(B2).cuda(), leaf=2).cpu().numpy()
    print("  3xtf32", (M2, K2, N2), "max err", float(np.abs(C2 - A2.astype(np.float64) @ B2.astype(np.float64)).max()))
