"""K1 / K3 microbenchmark (not the bench): the S / T formation and W-combination passes of a plan
timed alone (CUDA events the library records per launch kind), with one or two recursion levels
per pass (K1 reported as algorithmic GB/s: bench.pass_bytes' K1 part, needed input blocks read
once, formed outputs written once, against the measured copy bandwidth; K3 as time).

    python tools/bench_k1x2.py [--configs C2,C4,C5] [--reps 5]   (FMM_K1X2_RPB / FMM_K3X2_RPB: rows per CTA)
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import bench  # noqa: E402
import fmm_inputs as fi  # noqa: E402
import paper_1507_00687_b200 as fb  # noqa: E402


def k1_bytes(infos, M, K, N, esz, two):
    tot = bench.pass_bytes(infos, M, K, N, esz, False, two, False)  # K3 one level: subtracted below
    k3, nodes, m, n = 0, 1, M, N
    for r in infos:
        mb, nb = m // r["m0"], n // r["n0"]
        k3 += nodes * (r["R"] * mb * nb + m * n) * esz
        nodes *= r["R"]
        m, n = mb, nb
    return tot - k3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C3,C4,C5")
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    out = {"variant": os.environ.get("FMM_K1X2_VARIANT", "0")}
    for cfg in a.configs.split(","):
        c = fi.CONFIGS[cfg]
        M, K, N = c.M, c.K, c.N
        infos = [fb.Rule.builtin(r).info() for r in c.rules]
        A = torch.rand(M, K, dtype=torch.float64, device="cuda")
        B = torch.rand(K, N, dtype=torch.float64, device="cuda")
        Cm = torch.empty(M, N, dtype=torch.float64, device="cuda")
        for levels in (1, 2):
            p = fb.Plan([fb.Rule.builtin(r) for r in c.rules], M, K, N)
            p.set_k1_levels(levels)
            p.set_k3_levels(levels)
            ws = p.workspace()
            for _ in range(2):
                p.execute(A, B, Cm, ws=ws)
            torch.cuda.synchronize()
            p.set_timing(True)
            p.step_times()
            for _ in range(a.reps):
                p.execute(A, B, Cm, ws=ws)
            t = p.step_times()
            p.set_timing(False)
            ms = t["K1"][0] / a.reps
            nb = k1_bytes(infos, M, K, N, 8, levels == 2)
            out[f"{cfg}_L{levels}"] = {"k1_ms": ms, "k1_GB": nb / 1e9, "GBps": nb / ms / 1e6,
                                       "launches": t["K1"][1] // a.reps,
                                       "k3_ms": t.get("K3", (0.0, 0))[0] / a.reps,
                                       "k3_launches": t.get("K3", (0.0, 0))[1] // a.reps}
            del ws, p
            torch.cuda.empty_cache()
        del A, B, Cm
        torch.cuda.empty_cache()
    print(json.dumps(out))


if __name__ == "__main__":
    main()
