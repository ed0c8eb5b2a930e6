"""Quick device-side timing probe (not the bench): leaf GEMM and whole-plan throughput.

    python tools/probe.py [--c5] [--sizes 4096,8192]
"""
import argparse
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

import paper_1507_00687_b200 as fb  # noqa: E402


def timeit(fn, reps=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="2048,4096,8192")
    ap.add_argument("--c5", action="store_true")
    ap.add_argument("--plans", action="store_true")
    a = ap.parse_args()
    out = {}
    for n in map(int, a.sizes.split(",")):
        A = torch.rand(n, n, dtype=torch.float64, device="cuda")
        B = torch.rand(n, n, dtype=torch.float64, device="cuda")
        C = torch.empty_like(A)
        ms = timeit(lambda: fb.gemm(A, B, C_out=C))
        out[f"gemm_f64_{n}"] = {"ms": ms, "tflops": 2 * n ** 3 / ms / 1e9}
        A32, B32 = A.float(), B.float()
        C32 = torch.empty_like(A32)
        ms = timeit(lambda: fb.gemm(A32, B32, C_out=C32))
        out[f"gemm_f32simt_{n}"] = {"ms": ms, "tflops": 2 * n ** 3 / ms / 1e9}
        del A, B, C, A32, B32, C32
        print(json.dumps(out), flush=True)
    if a.plans:
        w = fb.Rule.builtin("winograd")
        s = fb.Rule.builtin("strassen")
        c = fb.Rule.builtin("classical222")
        for name, rules, (M, K, N) in [("C1", [w, w], (512,) * 3), ("C2", [s] * 4, (4096,) * 3),
                                       ("C2c", [c] * 4, (4096,) * 3),
                                       ("C3", [w, c, s], (8192, 4096, 8192)),
                                       ("C4none", [w] * 3, (4096,) * 3)]:
            A = torch.rand(M, K, dtype=torch.float64, device="cuda")
            B = torch.rand(K, N, dtype=torch.float64, device="cuda")
            p = fb.Plan(rules, M, K, N)
            Cm = torch.empty(M, N, dtype=torch.float64, device="cuda")
            ms = timeit(lambda: p.execute(A, B, Cm), reps=10 if M < 1000 else 5)
            out[name] = {"ms": ms, "eff_tflops": 2 * M * N * K / ms / 1e9}
            print(json.dumps(out), flush=True)
            del A, B, Cm, p
            torch.cuda.empty_cache()
    if a.c5:
        n = 32768
        A = torch.rand(n, n, dtype=torch.float64, device="cuda") * 2 - 1
        B = torch.rand(n, n, dtype=torch.float64, device="cuda") * 2 - 1
        C = torch.empty_like(A)
        w = fb.Rule.builtin("winograd")
        p = fb.Plan([w, w, w], n, n, n)
        print("ws GiB", p.workspace_bytes() / 2 ** 30, flush=True)
        t0 = time.time()
        p.execute(A, B, C)
        p.set_timing(True)
        p.step_times()
        ms = timeit(lambda: p.execute(A, B, C), reps=2, warm=0)
        kinds = p.step_times()
        out["C5"] = {"ms": ms, "eff_tflops": 2 * n ** 3 / ms / 1e9, "wall": time.time() - t0,
                     "kinds_ms_per_step": {k: v[0] / 2 for k, v in kinds.items()},
                     "k2_tflops": (7 ** 3 * 2 * 4096 ** 3 * 2) / (kinds["K2"][0] * 1e-3) / 1e12}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
