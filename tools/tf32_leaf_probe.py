"""FP32 tensor-core leaf probe: time and accuracy of one 3xTF32 leaf GEMM through fmm_gemm
(k2p_tf32) for the chunk length in the environment (FMM_TF32_CHUNK is read once per process,
so run one process per setting).

Accuracy: max |C - C_ref| / max |C_ref| over a 64 x 64 sample, C_ref the exact (fp64) product of
the FP32 inputs; beside it the same figure for a sequential round-to-nearest FP32 dot product
(numpy cumsum in float32: the FP32 oracle's leaf order).  Measurement tool only.

  python tools/tf32_leaf_probe.py [n] [batch]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1507_00687_b200 as fb  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    g = torch.Generator(device="cuda").manual_seed(4)
    A = torch.rand(n, n, dtype=torch.float32, device="cuda", generator=g) * 2 - 1
    B = torch.rand(n, n, dtype=torch.float32, device="cuda", generator=g) * 2 - 1
    C = torch.empty_like(A)
    fb.gemm(A, B, leaf=fb.fmm.LEAF_3XTF32, C_out=C)
    torch.cuda.synchronize()
    reps = max(3, int(4e12 / (2 * n ** 3)))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fb.gemm(A, B, leaf=fb.fmm.LEAF_3XTF32, C_out=C)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    rows = torch.arange(0, n, n // 64, device="cuda")[:64]
    Ad = A[rows].double().cpu().numpy()
    Bd = B[:, rows].double().cpu().numpy()
    ref = Ad @ Bd
    got = C[rows][:, rows].double().cpu().numpy()
    a32 = A[rows].cpu().numpy()
    b32 = B[:, rows].cpu().numpy()
    seq = np.empty_like(ref)
    for j in range(64):
        prod = (a32 * b32[:, j][None, :]).astype(np.float32)  # exact products rounded to FP32
        seq[:, j] = np.cumsum(prod, axis=1, dtype=np.float32)[:, -1]
    den = np.abs(ref).max()
    print(json.dumps({"n": n,
                      "chunk": os.environ.get("FMM_TF32_CHUNK", "default"), "ms": round(ms, 3),
                      "tflops_3x": round(2 * n ** 3 / ms / 1e9, 1),
                      "err_gpu": float(np.abs(got - ref).max() / den),
                      "err_seq_fp32": float(np.abs(seq - ref).max() / den)}))


if __name__ == "__main__":
    main()
