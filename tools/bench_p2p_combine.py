"""Comm mode 3's combine kernel (k_p2p_combine) timed on one GPU over virtual ranks: P plans
with set_partition(rank, P) fill their symmetric product buffers, then every rank's row slice of
C is combined from the P buffers -- here all local, so the loads come from HBM instead of over
NVLink; algorithmic bytes = the W-weighted products each C element reads + C written once.

    python tools/bench_p2p_combine.py [--n 32768] [--P 2] [--reps 5]
"""
import argparse
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_1507_00687_b200 as fb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=32768)
ap.add_argument("--P", type=int, default=2)
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
n, P = a.n, a.P
w = fb.Rule.builtin("winograd")
A = torch.rand(n, n, dtype=torch.float64, device="cuda")
B = torch.rand(n, n, dtype=torch.float64, device="cuda")
plans, ptrs = [], []
for r in range(P):
    p = fb.Plan([w] * 3, n, n, n)
    p.set_partition(r, P)
    p.set_comm_mode("p2p")
    p.sym_alloc()
    p.execute(A, B)
    torch.cuda.synchronize()
    p._ws = None
    torch.cuda.empty_cache()
    plans.append(p)
    ptrs.append(p.sym_ptr())
C = torch.empty(n, n, dtype=torch.float64, device="cuda")
ref = fb.Plan([w] * 3, n, n, n).execute(A, B)
torch.cuda.synchronize()
for _ in range(2):
    for r in range(P):
        plans[r].p2p_combine(ptrs, C, n * r // P, n * (r + 1) // P)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(a.reps):
    for r in range(P):
        plans[r].p2p_combine(ptrs, C, n * r // P, n * (r + 1) // P)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / a.reps
nnz = sum(1 for k in range(4) for q in range(7) if w.info()["W"][k][q] != 0)  # 14 for S-W
bytes_ = (nnz / 4 + 1) * n * n * 8
print(json.dumps({"n": n, "P": P, "ms_all_rows": ms, "GBps": bytes_ / ms / 1e6,
                  "bytes": bytes_, "bitwise_equal_single_gpu": bool(torch.equal(C, ref))}))
