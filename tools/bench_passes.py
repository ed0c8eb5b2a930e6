"""HBM-pass microbenchmark (not the bench): K1 (S/T formation) and K3 (W-combination) timed
through one-level Strassen-Winograd plans whose shapes make one pass dominate, reported as
algorithmic GB/s (bytes each pass must move: needed input blocks read once, non-trivial
outputs written once) against the measured copy bandwidth.

    python tools/bench_passes.py [--n 16384] [--reps 5]
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_1507_00687_b200 as fb  # noqa: E402


def run(plan, A, B, C, reps):
    ws = plan.workspace()
    for _ in range(2):
        plan.execute(A, B, C, ws=ws)
    torch.cuda.synchronize()
    plan.set_timing(True)
    plan.step_times()
    for _ in range(reps):
        plan.execute(A, B, C, ws=ws)
    t = plan.step_times()
    plan.set_timing(False)
    return {k: (ms / reps, n // reps) for k, (ms, n) in t.items()}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=16384)
    ap.add_argument("--thin", type=int, default=256)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--only", default="", help="k4: only the scaling passes; k1: no scaling passes")
    a = ap.parse_args()
    n, t = a.n, a.thin
    w = fb.Rule.builtin("winograd")
    out = {"K1_variant": os.environ.get("FMM_K1_VARIANT", "default")}
    q = (n // 2) ** 2 * 8  # bytes of one quarter block of the big operand
    if a.only != "k4":
        passes_k1_k3(a, n, t, w, q, out)
    if a.only != "k1":
        k4(a, n, w, out)
    print(json.dumps(out))


def passes_k1_k3(a, n, t, w, q, out):
    # K1: A is n x n, B is n x t (S-W: all 4 A blocks needed, 4 non-trivial S; same for T)
    A = torch.rand(n, n, dtype=torch.float64, device="cuda")
    B = torch.rand(n, t, dtype=torch.float64, device="cuda")
    C = torch.empty(n, t, dtype=torch.float64, device="cuda")
    p = fb.Plan([w], n, n, t)
    r = run(p, A, B, C, a.reps)
    bytes_k1 = 8 * q + 8 * (n // 2) * (t // 2) * 8
    out["K1"] = {"ms": r["K1"][0], "GBps": bytes_k1 / r["K1"][0] / 1e6, "bytes": bytes_k1}
    del A, B, C, p
    # K3: C is n x n, K = t (reads 7 quarter-size M_r, writes 4 quarters)
    A = torch.rand(n, t, dtype=torch.float64, device="cuda")
    B = torch.rand(t, n, dtype=torch.float64, device="cuda")
    C = torch.empty(n, n, dtype=torch.float64, device="cuda")
    p = fb.Plan([w], n, t, n)
    p.set_fusion("off")  # time the K3 pass itself
    r = run(p, A, B, C, a.reps)
    bytes_k3 = 11 * q
    out["K3"] = {"ms": r["K3"][0], "GBps": bytes_k3 / r["K3"][0] / 1e6, "bytes": bytes_k3}
    p.set_schedule("depth")
    r = run(p, A, B, C, a.reps)
    bytes_acc = (7 + 14 + 10) * q  # read M_r x7, write 14 (nnz W), read 10 (non-first)
    out["ACC"] = {"ms": r["ACC"][0], "GBps": bytes_acc / r["ACC"][0] / 1e6, "bytes": bytes_acc}


def k4(a, n, w, out):
    # K4: repeated scaling without the stop test (steps fixed) on n/4 x n/4 x n/4 FP64:
    # initial max reductions read A, B; every step reads + writes A and B once (apply fused with
    # the next step's reductions); the unscale reads + writes C.
    for m4 in sorted({n // 4, n}):
        k4_size(a, m4, w, out)


def k4_size(a, m4, w, out):
    steps = 10
    A = torch.rand(m4, m4, dtype=torch.float64, device="cuda") + 0.5
    B = torch.rand(m4, m4, dtype=torch.float64, device="cuda") + 0.5
    C = torch.empty(m4, m4, dtype=torch.float64, device="cuda")
    for pow2 in (0, 1):
        p = fb.Plan([w], m4, m4, m4, scaling={"mode": "repeated", "tau": -1.0, "max_steps": steps,
                                              "pow2": pow2})
        r = run(p, A, B, C, a.reps)
        mat = m4 * m4 * 8
        bytes_k4 = 2 * mat + steps * 4 * mat + 2 * mat
        out[f"K4_{m4}_pow2_{pow2}"] = {"ms": r["SCALE"][0], "GBps": bytes_k4 / r["SCALE"][0] / 1e6,
                                  "bytes": bytes_k4, "steps": steps}
        del p


if __name__ == "__main__":
    main()
