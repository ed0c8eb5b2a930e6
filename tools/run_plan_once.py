"""Run one BASELINE config's plan a few times (a target for ncu captures, not a benchmark).

    python tools/run_plan_once.py C2 [--levels 2] [--reps 1]
"""
import argparse
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import fmm_inputs as fi  # noqa: E402
import paper_1507_00687_b200 as fb  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("config")
ap.add_argument("--levels", type=int, default=2)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
c = fi.CONFIGS[a.config]
A = torch.rand(c.M, c.K, dtype=torch.float64, device="cuda")
B = torch.rand(c.K, c.N, dtype=torch.float64, device="cuda")
p = fb.Plan([fb.Rule.builtin(r) for r in c.rules], c.M, c.K, c.N)
p.set_k1_levels(a.levels)
for _ in range(a.reps):
    p.execute(A, B)
torch.cuda.synchronize()
print("ok")
