"""Per-rank compute of the multi-GPU partitions on ONE GPU (the box has one): for P = 2, 4, 8
ranks, the shard depth / unit order bench.py uses and the alternatives, every rank's plan
(`set_partition(rank, P)`, the same units and schedule a real rank runs, no communicator) is timed
on the C5 operands.  The slowest rank bounds the P-GPU step from below (the collective comes on
top); the sum over ranks against the one-GPU step shows the work each extra rank repeats (the
root K1 columns of its units).  Measurement tool only, not a multi-GPU number.

    python tools/partition_times.py [--config C5] [--reps 2]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_1507_00687_b200 as fb  # noqa: E402


def time_plan(plan, A, B, C, ws, reps):
    plan.execute(A, B, C, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        plan.execute(A, B, C, ws=ws)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C5")
    ap.add_argument("--reps", type=int, default=2)
    a = ap.parse_args()
    torch.cuda.set_device(0)
    Ah, Bh = bench.make_inputs(a.config, "f64")
    A, B = Ah.cuda(), Bh.cuda()
    del Ah, Bh
    C = torch.empty((A.shape[0], B.shape[1]), dtype=A.dtype, device="cuda")
    one = bench.make_plan(fb, a.config)
    ws = one.workspace(A.device)
    t1 = time_plan(one, A, B, C, ws, a.reps)
    flops = 2.0 * A.shape[0] * A.shape[1] * B.shape[1]
    out = {"config": a.config, "one_gpu_ms": t1, "partitions": []}
    del ws, one
    variants = [(P, d, o) for P in (2, 4, 8) for d, o in ((2 if P in (2, 4) else 1, "cyclic"),
                                                         (3, "block"), (2, "block"))]
    for P, depth, order in variants:
        ranks = []
        for r in range(P):
            p = bench.make_plan(fb, a.config)
            if depth > 1:
                p.set_shard_depth(depth)
            p.set_shard_order(order)
            p.set_partition(r, P)
            ws = p.workspace(A.device)
            ranks.append(time_plan(p, A, B, C, ws, a.reps))
            del ws, p
            torch.cuda.empty_cache()
        mx = max(ranks)
        out["partitions"].append({
            "ranks": P, "shard_depth": depth, "order": order, "rank_ms": ranks, "max_rank_ms": mx,
            "sum_rank_ms": sum(ranks),
            "compute_bound_eff": t1 / (P * mx),
            "compute_bound_tflops": flops / (mx * 1e-3) / 1e12})
        print(json.dumps(out["partitions"][-1]), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
