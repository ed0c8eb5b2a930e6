"""The paper's scaling experiment (Sec. 6.5, Fig. fig:scaling) on the GPU
path: one pair of N x N matrices from each of the three distributions, Strassen
with L = 1..6 recursion levels (N = 3500 is zero-padded for L >= 3), every scaling
mode of the C ABI, and the largest relative error |c^ - c| / |c| against the double-double
classical reference (the stand-in for the paper's quadruple precision).

    python tools/scaling_experiment.py [--n 3500] [--levels 1..6] [--out profiles/r01_scaling_experiment.md]

Modes: none, outside (Alg. 1), inside (Alg. 2), out_in / in_out (one O then one I step, or
reverse), repeated x2 (O I O I, no stopping test), repeated x10 (20 steps, no test),
repeated tau=1 (Alg. 3 with the Thm stopping test, <= 20 steps).  Factors are rounded to
powers of two (reading A7).  The classical leaf alone (L = 0) is the
reference point for "relatively accurate".
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import fmm_inputs as fi  # noqa: E402
import oracle  # noqa: E402  (test infrastructure: the high-precision reference)
import paper_1507_00687_b200 as fb  # noqa: E402

MODES = [
    ("none", {"mode": "none"}),
    ("outside", {"mode": "outside", "pow2": 1}),
    ("inside", {"mode": "inside", "pow2": 1}),
    ("out_in", {"mode": "out_in", "pow2": 1}),
    ("in_out", {"mode": "in_out", "pow2": 1}),
    ("rep_x2", {"mode": "repeated", "pow2": 1, "tau": -1.0, "max_steps": 4}),
    ("rep_x10", {"mode": "repeated", "pow2": 1, "tau": -1.0, "max_steps": 20}),
    ("rep_tau1", {"mode": "repeated", "pow2": 1, "tau": 1.0, "max_steps": 20}),
]
DISTS = [("1: U(0,1)", "u(0,1)"), ("2: Ex. 5.2-like", "paper2"), ("3: Ex. 6.9-like", "paper3")]


def max_rel(Chat, hi, lo):
    d = np.abs((Chat - hi) - lo)
    c = np.abs(hi)
    nz = c > 0
    return float(np.max(d[nz] / c[nz]))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=3500)
    ap.add_argument("--levels", default="1,2,3,4,5,6")
    ap.add_argument("--seed", type=int, default=7)
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    n = a.n
    levels = [int(x) for x in a.levels.split(",")]
    s = fb.Rule.builtin("strassen")
    rows = []
    for dname, dist in DISTS:
        A, B = fi.draw(dist, n, n, n, a.seed)
        t0 = time.time()
        hi, lo = oracle.ref_dd(A, B)
        tref = time.time() - t0
        Ad, Bd = torch.from_numpy(A).cuda(), torch.from_numpy(B).cuda()
        C0 = fb.gemm(Ad, Bd).cpu().numpy()  # classical leaf on the whole problem (L = 0)
        res = {"dist": dname, "classical": max_rel(C0, hi, lo), "ref_s": tref}
        for L in levels:
            for mname, sc in MODES:
                p = fb.Plan([s] * L, n, n, n, scaling=sc if sc["mode"] != "none" else None)
                C = p.execute(Ad, Bd)
                torch.cuda.synchronize()
                res[(L, mname)] = max_rel(C.cpu().numpy(), hi, lo)
                if mname == "rep_tau1":
                    res[(L, "rep_tau1_steps")] = p.last_scaling_steps()
                del p
        rows.append(res)
        print(json.dumps({k if isinstance(k, str) else f"L{k[0]}_{k[1]}": v for k, v in res.items()}),
              flush=True)
    lines = [f"# Paper Sec. 6.5 scaling experiment on the GPU path (N = {n}, Strassen, seed {a.seed})", "",
             "Largest relative error |c^ - c| / |c| over all entries against the double-double classical",
             "reference (P:1858-1859).  `classical` = the DMMA leaf GEMM on the whole problem (no recursion).",
             "Command: `python tools/scaling_experiment.py`.  Modes: see the tool's docstring.", ""]
    for r in rows:
        lines.append(f"## Distribution {r['dist']}  (classical: {r['classical']:.2e})")
        lines.append("")
        lines.append("| L | " + " | ".join(m for m, _ in MODES) + " | tau=1 steps |")
        lines.append("|---|" + "---|" * (len(MODES) + 1))
        for L in levels:
            lines.append(f"| {L} | " + " | ".join(f"{r[(L, m)]:.1e}" for m, _ in MODES)
                         + f" | {r[(L, 'rep_tau1_steps')]} |")
        lines.append("")
    text = "\n".join(lines)
    print(text)
    if a.out:
        Path(a.out).write_text(text + "\n")


if __name__ == "__main__":
    main()
