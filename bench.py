#!/usr/bin/env python
"""bench.py -- effective FP64 GFLOP/s (2MNK/t) of the recursive fast-matrix-multiplication hot
path (arXiv 1507.00687) on B200, BASELINE.json configs[4] (C5): M = K = N = 32768, FP64,
Strassen-Winograd, 3 levels, A, B ~ U(-1,1) seed 4.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl fmm|reference] [--dtype f64|f32]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU, NCCL)

One step = one complete C = A.B through the C ABI (fmm_execute): every K1 / K2 / K3 / ACC launch
of the plan (plus, for N > 1, the ncclReduce of the partial C onto rank 0).  Work is strong-
scaled: the 7 top-level products are split round-robin over the ranks.  Timing: W untimed
steps, then K steps bracketed by barrier + synchronize, CUDA events on the launch stream, max
over ranks.  The operands (8 GiB each) exceed the 126 MB L2, so no flush is needed.

The JSON line also carries: `e2e` (same metric through fmm_execute_host_batch with pinned host
buffers, copies inside the timed region), `roofline` (the leaf-product kernel K2 against the
measured FP64 DMMA peak), `cpu_baseline` (the CPU oracle on a bounded row/column sample of the
same workload), `clocks` (nvidia-smi sampled during the timed region) and `gpu_launches`.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "effective FP64 GFLOP/s (2MNK/t) at 1/2/4/8 B200 and max-norm error vs oracle"
UNIT = "GFLOP/s"
FP64_DMMA_PEAK_TFLOPS = 36.9  # profiles/r01_fp64_peak_microbench.txt (mma.sync f64, 1965 MHz)
TF32_PEAK_TFLOPS_NOMINAL = 1100.0  # B200_PROFILING.md nominal dense tf32 (fallback)
BF16_PEAK_TFLOPS_NOMINAL = 2250.0  # B200_PROFILING.md nominal dense bf16


def tf32_peak():
    """TF32 tensor peak for the FP32 leaf: MEASURED_PEAKS.json's sustained bf16 figure (the
    leaf runs inside a long step) x the guide's nominal tf32 / bf16 ratio; else the nominal."""
    try:
        mp = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        v = float(mp["bf16_tflops_sustained"])
        return v * TF32_PEAK_TFLOPS_NOMINAL / BF16_PEAK_TFLOPS_NOMINAL, (
            f"MEASURED_PEAKS.json bf16_tflops_sustained {v:g} x nominal tf32/bf16 "
            f"{TF32_PEAK_TFLOPS_NOMINAL:g}/{BF16_PEAK_TFLOPS_NOMINAL:g}")
    except (OSError, KeyError, ValueError):
        return TF32_PEAK_TFLOPS_NOMINAL, "B200_PROFILING.md nominal dense TF32 (fallback)"


def tf32_burst(achieved, three):
    """The same kernel against MEASURED_PEAKS.json's burst bf16 figure (the sustained one, the
    rule for a kernel inside a long step, was measured on cuBLAS at a power-capped 1320 MHz)."""
    try:
        v = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        return {}
    pk = v * TF32_PEAK_TFLOPS_NOMINAL / BF16_PEAK_TFLOPS_NOMINAL / (3 if three else 1)
    return {"peak_burst": pk, "frac_burst": (achieved / pk) if achieved else None,
            "peak_note": "MEASURED_PEAKS.json's sustained bf16 figure is cuBLAS under sw_power_cap at "
                         "~1320 MHz; the 3xTF32 leaf runs under the same cap at ~1550-1600 MHz, so "
                         "frac against the sustained-derived peak can exceed 1; frac_burst is "
                         "against the burst-derived one"}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """SM clock and clock-event (throttle) reasons sampled in-process through NVML every 2 ms by a
    background thread while active, plus one synchronous sample each at the start and the end of
    the timed region (`point()`), so even a sub-millisecond timed region has samples taken while
    its kernels run.  Falls back to nvidia-smi (200 ms) when NVML is unavailable."""

    REASONS = (("hw_slowdown", 0x8), ("hw_thermal_slowdown", 0x40), ("sw_thermal_slowdown", 0x20),
               ("sw_power_cap", 0x4), ("hw_power_brake_slowdown", 0x80))

    def __init__(self, index: int, period_s: float = 0.002):
        self.index = index
        self.period = period_s
        self.samples = []  # (sm_mhz, reason bitmask)
        self.sm_max = None
        self.on = False
        self.nv = None
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.sm_max = float(pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM))
        except Exception:  # noqa: BLE001 -- NVML missing: nvidia-smi fallback below
            self.nv = None

    def _one(self):
        if self.nv is None:
            return
        try:
            sm = float(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            rs = int(self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h))
            self.samples.append((sm, rs))
        except Exception:  # noqa: BLE001
            pass

    def _loop(self):
        while self.on:
            self._one()
            time.sleep(self.period)

    def point(self):
        """A synchronous sample (call right after enqueueing / before synchronising)."""
        self._one()

    def start(self):
        self.samples = []
        if self.nv is None:
            return self._smi_start()
        self.on = True
        self.t = threading.Thread(target=self._loop, daemon=True)
        self.t.start()

    def stop(self):
        if self.nv is None:
            return self._smi_stop()
        self.on = False
        self.t.join(timeout=1.0)
        if not self.samples:
            return None
        reasons = sorted({n for _, rs in self.samples for n, bit in self.REASONS if rs & bit})
        return {"sm_mhz": statistics.median(s for s, _ in self.samples), "sm_max_mhz": self.sm_max,
                "reasons": reasons, "samples": len(self.samples), "source": "NVML in-process, 2 ms"}

    # -- nvidia-smi fallback (200 ms period) --
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def _smi_start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.lines = []
            self.t = threading.Thread(target=lambda: [self.lines.append(x.strip()) for x in self.proc.stdout],
                                      daemon=True)
            self.t.start()
        except OSError:
            self.proc = None

    def _smi_stop(self):
        if getattr(self, "proc", None) is None:
            return None
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [q.strip() for q in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return None
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi, 200 ms"}


# ------------------------------------------------------------------------------------------
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def load_traffic(workload: str):
    """Per-launch DRAM bytes of K2 from a committed ncu --set full capture (or None)."""
    f = ROOT / "profiles" / "k2_traffic.json"
    if not f.exists():
        return None
    try:
        d = json.loads(f.read_text())
        return d.get(workload)
    except (OSError, ValueError):
        return None


def make_inputs(cfg, dtype):
    """Inputs of BASELINE config `cfg` drawn by the shared recipe (fmm_inputs) into pinned host
    memory (uniform families straight into pinned buffers)."""
    import torch
    import fmm_inputs as fi
    c = fi.CONFIGS[cfg]
    t0 = time.time()
    if c.dist in ("u(-1,1)", "u(0,1)"):
        A, B = fi.draw_torch(c.dist, c.M, c.K, c.N, c.seed, pin=True)
    else:
        A, B = fi.draw_torch(c.dist, c.M, c.K, c.N, c.seed)
        A, B = A.pin_memory(), B.pin_memory()
    if dtype == "f32":
        A, B = A.float().pin_memory(), B.float().pin_memory()
    log(f"[bench] {cfg} inputs {c.M}x{c.K}x{c.N} ({c.dist}, seed {c.seed}) in {time.time() - t0:.1f}s")
    return A, B


# ------------------------------------------------------------------------------------------
def scaling_config(mode: str):
    """The scaling configuration the bench runs (readings A7 / A10): power-of-two
    factors, tau = 1, at most 20 steps."""
    return None if mode == "none" else {"mode": mode, "tau": 1.0, "max_steps": 20, "pow2": 1}


def default_shard(nranks: int, levels: int):
    """(shard depth, unit order) for `nranks` ranks, from the per-rank compute of every rank's
    partition timed on one B200 at C5 (tools/partition_times.py, profiles/r02_partition_times.md;
    one-GPU time / (P x slowest rank)): depth 3 in contiguous blocks gives 0.974 / 0.948 / 0.909
    at 2 / 4 / 8 ranks (round 1's choice -- depth 2 round-robin at 2 and 4 ranks, the 7
    top-level products at 8 -- 0.924 / 0.865 / 0.855).  Blocks keep a rank's units on shared
    upper-level paths, and a subtree the rank owns entirely runs breadth-first like one unit."""
    if nranks <= 1:
        return 1, "cyclic"
    return min(3, levels), "block"


def make_plan(fb, cfg: str, dtype: str = "f64", leaf=None, scaling: str = "none"):
    """The plan bench.py times for BASELINE config `cfg` (also used by the full-size parity
    tests, so they check exactly this launch configuration)."""
    import fmm_inputs as fi
    c = fi.CONFIGS[cfg]
    if leaf is None:
        leaf = fb.fmm.LEAF_NATIVE if dtype == "f64" else fb.fmm.LEAF_3XTF32
    return fb.Plan([fb.Rule.builtin(r) for r in c.rules], c.M, c.K, c.N, dtype=dtype, leaf=leaf,
                   scaling=scaling_config(scaling))


# ------------------------------------------------------------------------------------------
def cpu_baseline(A_host, B_host, plan_rules, M, K, N, C_gpu_host=None, target_s=15.0,
                 scaling="none"):
    """The CPU oracle, as it stands, on a bounded row/column sample of the same workload:
    rows G = lift_rows(leaf rows), columns H = lift_cols(leaf cols) (bitwise the oracle's own
    entries of C, oracle.fmm_sub).  Value = 2 |G| |H| K / t.  With scaling, the oracle first
    scales the whole operands (Alg. 1-3, O(MK + KN) work, timed separately as
    `scale_seconds`), runs the sampled FMM on A', B' and unscales the sampled entries -- again
    bitwise the oracle's own entries."""
    import numpy as np
    import oracle
    from oracle import rules as OR
    plan = OR.Plan.uniform([OR.builtin(n) for n in plan_rules])
    A = A_host.numpy() if hasattr(A_host, "numpy") else A_host
    B = B_host.numpy() if hasattr(B_host, "numpy") else B_host
    sc = None
    t_scale = 0.0
    if scaling != "none":
        t0 = time.perf_counter()
        cfg = scaling_config(scaling)
        sc = oracle.scale_operands(A, B, scaling, pow2=bool(cfg["pow2"]), tau=cfg["tau"],
                                   max_steps=cfg["max_steps"])
        t_scale = time.perf_counter() - t0
    As, Bs = (A, B) if sc is None else (sc["A"], sc["B"])
    pm, _, pn = plan.dims_divisor()
    # calibrate: one leaf row/col first, doubling both (about 4x the work each time) until one
    # run takes >= target_s / 2: the reported run is then 7.5-30 s of CPU work at target 15 s
    nr = 1
    res = None
    while True:
        G = oracle.lift_rows(M, plan, range(nr))
        H = oracle.lift_cols(N, plan, range(nr))
        Ag = np.ascontiguousarray(As[G, :])
        Bh = np.ascontiguousarray(Bs[:, H])
        t0 = time.perf_counter()
        Cs = oracle.fmm(Ag, Bh, plan)
        t = time.perf_counter() - t0
        res = (nr, G, H, Cs, t)
        if t >= target_s / 2 or nr * 2 > min(M // pm, N // pn) or nr >= 1024:
            break
        nr *= 2
    nr, G, H, Cs, t = res
    if sc is not None:
        Cs = oracle.unscale(Cs, sc["dA"][G], sc["dB"][H])
    flops = 2.0 * len(G) * len(H) * K
    out = {"value": flops / t / 1e9, "unit": UNIT, "cores": oracle.num_threads(), "kind": "oracle",
           "sample": f"C[G,H] with |G|={len(G)} rows x |H|={len(H)} cols (leaf rows/cols 0..{nr - 1} "
                     f"lifted through all levels; oracle.fmm_sub, bitwise the full oracle's entries)",
           "seconds": t}
    if sc is not None:
        out["scale_seconds"] = t_scale
        out["scaling_steps"] = int(sc["steps"])
    if C_gpu_host is not None:
        Cg = C_gpu_host[np.ix_(G, H)]
        out["parity_sampled"] = oracle.parity_metric(Cg, Cs, float(np.abs(A).max()),
                                                     float(np.abs(B).max()), K)
        # both paths against the double-double classical reference (the stand-in for the
        # paper's quadruple precision) on a 64 x 64 corner of the sample
        g, h = G[:64], H[:64]
        hi, lo = oracle.ref_dd(np.ascontiguousarray(A[g, :]), np.ascontiguousarray(B[:, h]))
        scale = float(np.abs(hi).max()) or 1.0
        nz = hi != 0

        def err(X):
            d = np.abs((X.astype(np.float64) - hi) - lo)
            return {"normwise": float(np.max(d) / scale),
                    "max_rel": float(np.max(d[nz] / np.abs(hi[nz]))) if nz.any() else 0.0}

        eg, eo = err(Cg[:64, :64]), err(Cs[:64, :64])
        out["error_vs_dd"] = {"gpu": eg["normwise"], "oracle": eo["normwise"],
                              "gpu_max_rel": eg["max_rel"], "oracle_max_rel": eo["max_rel"],
                              "measure": "max |C - C_dd| / max |C_dd| (and max |C - C_dd| / |C_dd|) "
                                         "over 64 x 64 sampled entries"}
        if sc is not None:
            # componentwise Thm 4.3 bound through the exact power-of-two unscale (SURVEY §8(c)
            # C-tol: the normalised metric is vacuous for skewed magnitudes)
            from oracle import rules as R2
            f = float(R2.uniform_bound_factor([OR.builtin(n) for n in plan_rules], K))
            bnd = f * 2.0 ** -53 * float(np.abs(sc["A"]).max()) * float(np.abs(sc["B"]).max()) * \
                np.outer(sc["dA"][G], sc["dB"][H])
            d = np.abs(Cg.astype(np.float64) - Cs)
            nzc = Cs != 0  # exact zeros (cancellation in the unscaled modes) excluded
            out["componentwise"] = {"max_rel_gpu_vs_oracle": float(np.max(d[nzc] / np.abs(Cs[nzc]))) if nzc.any() else 0.0,
                                    "max_ratio_to_2x_thm_bound": float(np.max(d / (2 * bnd)))}
    return out


def parity_record(cpu, dtype):
    """The bench line's parity object from the cpu_baseline sample: the north star's metric and
    tolerance, plus (scaled runs) the componentwise check against twice the Thm 4.3 bound."""
    if not cpu or "parity_sampled" not in cpu:
        return None
    tol = 1e-13 if dtype == "f64" else 5e-5
    rec = {"metric": "||C_gpu - C_oracle||_max / (||A||_max ||B||_max K) on the cpu_baseline "
                     "sample (BASELINE north_star tolerance)",
           "value": cpu["parity_sampled"], "tolerance": tol}
    ok = cpu["parity_sampled"] <= tol
    if "componentwise" in cpu:
        rec["componentwise"] = cpu["componentwise"]
        ok = ok and cpu["componentwise"]["max_ratio_to_2x_thm_bound"] <= 1.0
    rec["pass"] = bool(ok)
    return rec


# ------------------------------------------------------------------------------------------
def pass_bytes(rule_infos, M, K, N, esz, fused_leaf_level, two_level=True, two_level_k3=True,
               depth_first_top=False, tf32_split=None):
    """Algorithmic HBM bytes of the add passes of a uniform plan: per level, K1
    reads each node's A / B block once and writes the non-trivial S_r / T_r (a column with a
    single +1 is an alias); with two levels per pass (K1X2, levels paired from the bottom where
    both split <= 4 blocks) a pass reads the sub-blocks its formed grandchildren use once and
    writes only the grandchildren (all but the products trivial at both levels); K3 reads the R
    child products and writes the node's output; with the leaf-parent level fused, that level
    only writes its output once.  tf32_split (FP32 tensor-core leaves): "pass" -- the leaf
    level's K1X2 forms every leaf operand (views too) and writes its TF32 hi and lo parts (DESIGN.md
    §6.3); "kernel" -- a split pass reads every leaf operand and writes hi and lo."""
    def col(X, r):
        return [i for i in range(len(X)) if X[i][r] != 0]

    def trivial(X, r):
        nz = col(X, r)
        return len(nz) == 1 and X[nz[0]][r] == 1

    def one_level(X, R):
        """(number of non-trivial columns, number of blocks they read)"""
        cnt, used = 0, set()
        for r in range(R):
            if not trivial(X, r):
                cnt += 1
                used |= set(col(X, r))
        return cnt, len(used)

    def two_levels(X1, R1, X2, R2):
        """(formed grandchildren, sub-blocks (i1, i2) read) of a K1X2 node"""
        formed, need = 0, set()
        for r1 in range(R1):
            need2 = set()
            for r2 in range(R2):
                if trivial(X1, r1) and trivial(X2, r2):
                    continue
                formed += 1
                need2 |= set(col(X2, r2))
            need |= {(i1, i2) for i1 in col(X1, r1) for i2 in need2}
        return formed, len(need)

    L = len(rule_infos)
    dims = [(M, K, N)]
    for ri in rule_infos:
        m, k, n = dims[-1]
        dims.append((m // ri["m0"], k // ri["k0"], n // ri["n0"]))
    nodes = [1]
    for ri in rule_infos:
        nodes.append(nodes[-1] * ri["R"])
    small = [ri["m0"] * ri["k0"] <= 4 and ri["k0"] * ri["n0"] <= 4 for ri in rule_infos]
    pair = [False] * (L + 1)
    if two_level:
        for e in range(L - 2, -1, -2):
            pair[e] = small[e] and small[e + 1] and rule_infos[e]["R"] * rule_infos[e + 1]["R"] <= 64
    total = 0
    l = 0
    while l < L:  # K1
        ri = rule_infos[l]
        if pair[l]:
            r2 = rule_infos[l + 1]
            mb, kb, nb = dims[l + 2]
            if tf32_split == "pass" and l + 2 == L:
                allf = ri["R"] * r2["R"]  # every grandchild formed, hi + lo written
                na = len({(i1, i2) for r1 in range(ri["R"]) for i1 in col(ri["U"], r1)
                          for q in range(r2["R"]) for i2 in col(r2["U"], q)})
                nb_ = len({(i1, i2) for r1 in range(ri["R"]) for i1 in col(ri["V"], r1)
                           for q in range(r2["R"]) for i2 in col(r2["V"], q)})
                total += nodes[l] * ((na + 2 * allf) * mb * kb + (nb_ + 2 * allf) * kb * nb) * esz
                l += 2
                continue
            fa, na = two_levels(ri["U"], ri["R"], r2["U"], r2["R"])
            fb_, nb_ = two_levels(ri["V"], ri["R"], r2["V"], r2["R"])
            total += nodes[l] * ((na + fa) * mb * kb + (nb_ + fb_) * kb * nb) * esz
            l += 2
        else:
            mb, kb, nb = dims[l + 1]
            (nsa, ua), (nsb, ub) = one_level(ri["U"], ri["R"]), one_level(ri["V"], ri["R"])
            total += nodes[l] * ((ua + nsa) * mb * kb + (ub + nsb) * kb * nb) * esz
            l += 1
    if tf32_split == "kernel":  # read every leaf operand, write its hi and lo
        mb, kb, nb = dims[L]
        total += nodes[L] * 3 * (mb * kb + kb * nb) * esz
    # K3 / fused epilogue; two levels per K3 pass (K3X2) paired from the bottom of the unfused
    # levels (not the depth-first top level, whose W-combination is the per-r ACC pass)
    top = L - 2 if fused_leaf_level else L - 1
    if fused_leaf_level:
        m, _, n = dims[L - 1]
        total += nodes[L - 1] * m * n * esz  # fused W-combination: the output written once
    l = top
    first = 1 if depth_first_top else 0
    while l >= 0:
        ri = rule_infos[l]
        m, _, n = dims[l]
        if (two_level_k3 and l - 1 >= first and small[l - 1] and small[l]
                and rule_infos[l - 1]["R"] * ri["R"] <= 64):
            mg, _, ng = dims[l + 1]  # grandchildren of level l - 1
            pm, _, pn = dims[l - 1]
            total += nodes[l - 1] * (rule_infos[l - 1]["R"] * ri["R"] * mg * ng + pm * pn) * esz
            l -= 2
        else:
            mb, _, nb = dims[l + 1]
            total += nodes[l] * (ri["R"] * mb * nb + m * n) * esz  # K3: read R products, write the output
            l -= 1
    return total


# ------------------------------------------------------------------------------------------
def run_reference(args):
    """--impl reference: the CPU oracle (this tier's reference arm) timed on bounded samples of
    the same workload, rank 0 only."""
    ws, rank, _ = dist_env()
    if rank != 0:
        return
    import numpy as np
    import oracle
    from oracle import rules as OR
    import fmm_inputs as fi
    c = fi.CONFIGS[args.config]
    M, K, N = c.M, c.K, c.N
    rules = c.rules
    oracle.build()
    A, B = make_inputs(args.config, "f64")
    An, Bn = A.numpy(), B.numpy()
    plan = OR.Plan.uniform([OR.builtin(n) for n in rules])
    nr = args.ref_sample
    times = []
    for step in range(args.warmup + args.steps):
        pm, _, pn = plan.dims_divisor()
        rows = [(step * nr + i) % (M // pm) for i in range(nr)]
        cols = [(step * nr + i) % (N // pn) for i in range(nr)]
        G = oracle.lift_rows(M, plan, rows)
        H = oracle.lift_cols(N, plan, cols)
        t0 = time.perf_counter()
        oracle.fmm(np.ascontiguousarray(An[G, :]), np.ascontiguousarray(Bn[:, H]), plan)
        t = time.perf_counter() - t0
        if step >= args.warmup:
            times.append(t)
    flops = 2.0 * len(G) * len(H) * K
    total = sum(times)
    value = flops * len(times) / total / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": total / len(times) * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"{args.config}: {' / '.join(rules)}, M={M} K={K} N={N} FP64, "
                                   f"{c.dist} seed {c.seed}",
                       "sample_per_step": f"C[G,H], |G| = {len(G)}, |H| = {len(H)} lifted rows/cols"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.num_threads(),
                             "kind": "oracle",
                             "sample": f"per step C[G,H] with |G|={len(G)}, |H|={len(H)} (row/col-sampled oracle)"},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------------------------
def run_fmm(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_1507_00687_b200 as fb

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import fmm_inputs as fi
    cfgd = fi.CONFIGS[args.config]
    M, K, N = cfgd.M, cfgd.K, cfgd.N
    rules = cfgd.rules
    dt = torch.float64 if args.dtype == "f64" else torch.float32
    esz = 8 if args.dtype == "f64" else 4
    leaf = fb.fmm.LEAF_NATIVE if args.dtype == "f64" else args.leaf
    stream = torch.cuda.Stream()

    # ---- inputs: host (pinned) on rank 0, device copies on every rank -----------------------
    if rank == 0:
        A_h, B_h = make_inputs(args.config, args.dtype)
    A = torch.empty((M, K), dtype=dt, device="cuda")
    B = torch.empty((K, N), dtype=dt, device="cuda")
    Cd = torch.empty((M, N), dtype=dt, device="cuda")
    if rank == 0:
        A.copy_(A_h)
        B.copy_(B_h)
    if ws > 1:
        dist.broadcast(A, 0)
        dist.broadcast(B, 0)
    torch.cuda.synchronize()

    plan = make_plan(fb, args.config, args.dtype, leaf, args.scaling)
    shard_order = "cyclic" if args.shard_order == "auto" else args.shard_order
    if args.shard_depth <= 0:  # auto (default_shard); the fused NVLink combine works on the
        # top-level products (depth 1), laid out round-robin
        args.shard_depth, auto_order = default_shard(ws, len(rules)) if args.comm != "p2p" else (1, "cyclic")
        if args.shard_order == "auto":
            shard_order = auto_order
    # --comm-one-rank: a one-rank NCCL communicator at N = 1, so the exchange (the collective,
    # or mode 3's barriers and combine) really runs on a single GPU
    use_comm = ws > 1 or args.comm_one_rank
    if ws > 1 and args.shard_depth > 1:
        plan.set_shard_depth(args.shard_depth)
    if ws > 1 and shard_order != "cyclic":
        plan.set_shard_order(shard_order)
    if use_comm and args.comm != "reduce":
        plan.set_comm_mode(args.comm)
    if use_comm:
        uid = [fb.comm_unique_id() if rank == 0 else None]
        if ws > 1:
            dist.broadcast_object_list(uid, 0)
        plan.set_comm(uid[0], rank, ws)
        if args.comm == "p2p":  # symmetric product buffers, CUDA IPC handles exchanged
            handles = [plan.sym_alloc()]
            if ws > 1:
                mine, handles = handles[0], [None] * ws
                dist.all_gather_object(handles, mine)
            plan.set_peer_handles(handles)
    wsp = plan.workspace(A.device)
    use_graph = args.graph == "on" or (args.graph == "auto" and M * N * K <= 4096 ** 3 and ws == 1)
    if use_graph:
        plan.set_graph(True)
    log(f"[bench] rank {rank}: workspace {plan.workspace_bytes() / 2**30:.1f} GiB, "
        f"{plan.launch_count()} launches / step")

    def step():
        plan.execute(A, B, Cd, ws=wsp, stream=stream)

    # ---- warm-up ------------------------------------------------------------------------------
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    torch.cuda.synchronize()

    # ---- timed region (device events, max over ranks) -----------------------------------------
    sampler = ClockSampler(local)
    plan.set_timing(not use_graph)
    plan.step_times()  # reset
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    small = (M * K + K * N + M * N) * esz < (512 << 20)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda") if small else None
    sampler.start()
    if not small:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        sampler.point()  # while the enqueued steps run
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    else:  # operands fit in L2: flush L2 (256 MB write) between steps, outside the events
        evs = []
        for _ in range(args.steps):
            with torch.cuda.stream(stream):
                flush.fill_(1)
            a, b2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            step()
            b2.record(stream)
            evs.append((a, b2))
        sampler.point()
        torch.cuda.synchronize()
        ms = sum(a.elapsed_time(b2) for a, b2 in evs)
    clocks = sampler.stop()
    kinds = plan.step_times()
    plan.set_timing(False)
    if ws > 1:
        dist.barrier()
    if ws > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    flops = 2.0 * M * N * K
    value = flops * args.steps / (ms * 1e-3) / 1e9

    # ---- roofline of the dominant kernel (K2, the leaf products) -------------------------------
    L = len(rules)
    nleaves = 1
    for r in rules:
        nleaves *= fb.Rule.builtin(r).info()["R"]
    leaf_flops_step = nleaves * 2.0 * (M >> L) * (N >> L) * (K >> L)
    if use_graph:  # per-kind events are not recorded under graph replay: time K2 alone after
        plan.set_graph(False)
        plan.set_timing(True)
        plan.step_times()
        with torch.cuda.stream(stream):
            for _ in range(args.steps):
                step()
        torch.cuda.synchronize()
        kinds = plan.step_times()
        plan.set_timing(False)
    k2_ms, k2_n = kinds.get("K2", (0.0, 0))
    per_launch_flops = leaf_flops_step * args.steps / max(k2_n, 1)
    tf32, tf32_src = tf32_peak()
    peak = FP64_DMMA_PEAK_TFLOPS if args.dtype == "f64" else tf32 / (
        3 if leaf == fb.fmm.LEAF_3XTF32 else 1)
    achieved = per_launch_flops / (k2_ms / max(k2_n, 1) * 1e-3) / 1e12 if k2_n else None
    workload = f"{args.config}-{args.dtype}-n{M}-L{L}-p{ws}" if args.config == "C5" else \
        f"{args.config}-{args.dtype}-p{ws}"
    fused = plan.fused_launches() > 0
    single = (plan.launch_count() == 1 and len(rules) == 2 and args.scaling == "none"
              and args.dtype == "f64")
    k2_name = ("k_small_plan (the whole step in one cooperative kernel: K1X2, the leaf products on "
               "DMMA mma.sync f64, K3X2; achieved = leaf flops / kernel time)" if single else
               "k2f_gemm_f64 (leaf products on DMMA mma.sync f64 + the parents' W-combination "
               "fused in the epilogue)" if fused else "k2_gemm_f64 (leaf products, DMMA mma.sync f64)")
    k2_name32 = ("k2p_tf32 (3xTF32 leaf products on tcgen05, persistent, 128-deep TMEM chunks drained "
                 "into round-to-nearest register totals; hi / lo operands written by the leaf "
                 "level's K1X2" + (", a split kernel in the launch)" if os.environ.get(
                     "FMM_TF32_PRESPLIT", "1") == "0" else ")"))
    roofline = {"kernel": k2_name if args.dtype == "f64" else k2_name32,
                "bound": "tensor", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                "frac": (achieved / peak) if achieved else None,
                "traffic": load_traffic(workload),
                "peak_source": "measured FP64 DMMA microbenchmark (profiles/r01_fp64_peak_microbench.txt); "
                               "MEASURED_PEAKS.json has no FP64 entry" if args.dtype == "f64" else
                               tf32_src + (" / 3 (3xTF32: three MMA passes)"
                                           if leaf == fb.fmm.LEAF_3XTF32 else ""),
                **({} if args.dtype == "f64" else tf32_burst(achieved, leaf == fb.fmm.LEAF_3XTF32)),
                "flops_per_launch": per_launch_flops, "launch_ms": (k2_ms / k2_n) if k2_n else None,
                "step_share": {k: v[0] / max(sum(x[0] for x in kinds.values()), 1e-9)
                               for k, v in kinds.items()},
                "timing_note": "K2 launch times from CUDA events the library records on the launch "
                               "stream" + (" (separate pass: graph replay in the timed region)" if use_graph else "")}

    # ---- whole-step roofline: leaf flops at the tensor peak + algorithmic pass bytes at the
    #      measured copy bandwidth (SURVEY §8(d) "pipeline roofline") ---------------------------
    hbm = 6543.4
    try:
        hbm = float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        pass
    tf32_split = None
    if args.dtype == "f32" and leaf != fb.fmm.LEAF_NATIVE:
        lk = K >> len(rules) if all(r in ("winograd", "strassen", "classical222") for r in rules) else 0
        ln = N >> len(rules) if lk else 0
        presplit = (os.environ.get("FMM_TF32_PRESPLIT", "1") != "0" and lk % 32 == 0 and ln % 32 == 0
                    and os.environ.get("FMM_K1X2", "1") != "0" and len(rules) >= 2)
        tf32_split = "pass" if presplit else "kernel"
    pbytes = (pass_bytes([fb.Rule.builtin(r).info() for r in rules], M, K, N, esz, fused,
                         os.environ.get("FMM_K1X2", "1") != "0", os.environ.get("FMM_K3X2", "1") != "0",
                         "ACC" in kinds, tf32_split) if ws == 1 else None)
    pipeline = None
    if pbytes is not None and args.scaling == "none":
        t_roof = leaf_flops_step / (peak * 1e12) + pbytes / (hbm * 1e9)
        pipeline = {"t_roof_ms": t_roof * 1e3, "frac": t_roof * 1e3 / (ms / args.steps),
                    "leaf_flops": leaf_flops_step, "pass_bytes": pbytes,
                    "note": "leaf flops / leaf-kernel peak + algorithmic K1 / K3 bytes / measured "
                            "copy bandwidth (MEASURED_PEAKS.json hbm_gbs); frac = t_roof / t"}

    # ---- end-to-end through the C ABI with host buffers ---------------------------------------
    # value: K problems through fmm_execute_host_batch (pinned host A, B in, C out every problem;
    # two device buffer sets, so problem i's input copies overlap problem i - 1's compute and its
    # C copy-out problem i + 1's).  serial: one fmm_execute_host call per problem, synchronised
    # in between (no cross-problem overlap).  Multi-rank: rank 0 copies in, broadcasts, and
    # copies the reduced C out, every step.
    e2e = None
    if not args.no_e2e:
        # distributed C (reduce_scatter, p2p): every rank copies out its own rows
        dist_c = ws > 1 and args.comm in ("reduce_scatter", "p2p")
        r0, r1 = (M * rank // ws, M * (rank + 1) // ws) if dist_c else (0, M)
        C_h = (torch.empty((r1 - r0, N), dtype=dt).pin_memory() if (rank == 0 or dist_c)
               else None)

        def e2e_serial(nsteps, warm):
            for it in range(warm + nsteps):
                if ws > 1:
                    dist.barrier()
                torch.cuda.synchronize()
                if it == warm:
                    f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    f0.record(stream)
                if ws == 1:
                    plan.execute_host(A_h, B_h, C_h, A, B, Cd, ws=wsp, stream=stream)
                else:
                    with torch.cuda.stream(stream):
                        if rank == 0:
                            A.copy_(A_h, non_blocking=True)
                            B.copy_(B_h, non_blocking=True)
                        dist.broadcast(A, 0)
                        dist.broadcast(B, 0)
                        step()
                        if rank == 0 or dist_c:
                            C_h.copy_(Cd[r0:r1], non_blocking=True)
            f1.record(stream)
            torch.cuda.synchronize()
            return f0.elapsed_time(f1)

        def max_ranks(v):
            if ws > 1:
                t = torch.tensor([v], dtype=torch.float64, device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                v = float(t.item())
            return v

        sms = max_ranks(e2e_serial(args.steps, args.e2e_warmup))
        ems, how = sms, "one fmm_execute_host call per problem, synchronised in between"
        if ws == 1:
            A2, B2, C2 = torch.empty_like(A), torch.empty_like(B), torch.empty_like(Cd)
            devs = ([A, A2], [B, B2], [Cd, C2])
            W = max(args.e2e_warmup, 2)
            plan.execute_host_batch([A_h] * W, [B_h] * W, [C_h] * W, *devs, ws=wsp, stream=stream)
            torch.cuda.synchronize()
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record(stream)
            plan.execute_host_batch([A_h] * args.steps, [B_h] * args.steps, [C_h] * args.steps,
                                    *devs, ws=wsp, stream=stream)
            f1.record(stream)
            torch.cuda.synchronize()
            ems = f0.elapsed_time(f1)
            how = ("K problems through one fmm_execute_host_batch call (2 device buffer sets: "
                   "copies of neighbouring problems overlap compute)")
            del A2, B2, C2
        e2e = {"value": flops * args.steps / (ems * 1e-3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": (M * K + K * N) * esz, "d2h_bytes_per_step": M * N * esz,
               "ms_per_step": ems / args.steps, "how": how,
               "serial": {"value": flops * args.steps / (sms * 1e-3) / 1e9,
                          "ms_per_step": sms / args.steps}}

    # ---- CPU oracle baseline (rank 0, N = 1) ----------------------------------------------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        import oracle
        oracle.build()
        Cg = Cd.cpu().numpy()
        An = A_h.numpy() if args.dtype == "f64" else A_h.double().numpy()
        Bn = B_h.numpy() if args.dtype == "f64" else B_h.double().numpy()
        if args.dtype == "f32":
            An, Bn = A_h.numpy(), B_h.numpy()
        cpu = cpu_baseline(An, Bn, rules, M, K, N, C_gpu_host=Cg, target_s=args.cpu_seconds,
                           scaling=args.scaling)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": {"workload": f"{args.config}: {' / '.join(rules)} (root first), M={M} K={K} "
                                   f"N={N} {args.dtype.upper()}, {cfgd.dist} seed {cfgd.seed} "
                                   f"(BASELINE configs[{ {'C1': 0, 'C2': 1, 'C2c': 1, 'C3': 2, 'C4': 3, 'C5': 4}[args.config] }])"
                                   + (f", scaling {args.scaling} (pow2, tau=1)" if args.scaling != "none" else ""),
                       "parallelism": (f"top-level r round-robin over {ws} GPU(s)" if args.shard_depth <= 1
                                       else f"depth-{args.shard_depth} paths "
                                       f"{'in contiguous blocks' if shard_order == 'block' else 'round-robin'}"
                                       f" over {ws} GPU(s)")
                                      + (f", {args.comm} of C" if use_comm else ""),
                       "l2": ("operands %.1f GiB each > 126 MB L2 (no flush needed)" % (M * K * esz / 2**30))
                  if not small else "L2 flushed (256 MB write) between timed steps, outside the events",
                       "leaf": {0: "native", 1: "tf32", 2: "3xtf32"}[leaf],
                       "k3_fused_in_leaf_epilogue": bool(fused),
                       **({"scaling_steps_taken": plan.last_scaling_steps(ws=wsp, stream=stream)}
                          if args.scaling != "none" and ws == 1 else {})},
            "parity": parity_record(cpu, args.dtype),
            "roofline": roofline, "pipeline_roofline": pipeline, "cpu_baseline": cpu, "e2e": e2e,
            "clocks": clocks,
            "gpu_launches": plan.launch_count() * args.steps,
            "cuda_graph": use_graph,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="fmm", choices=["fmm", "reference"])
    ap.add_argument("--dtype", default="f64", choices=["f64", "f32"])
    ap.add_argument("--leaf", type=int, default=2, help="FP32 leaf: 0 native, 1 tf32, 2 3xtf32")
    ap.add_argument("--config", default="C5", choices=["C1", "C2", "C2c", "C3", "C4", "C5"],
                    help="BASELINE config (default C5: the throughput config the metric is quoted on)")
    ap.add_argument("--graph", default="auto", choices=["auto", "on", "off"],
                    help="CUDA-graph replay of each step (auto: on for problems <= 4096^3)")
    ap.add_argument("--scaling", default="none",
                    choices=["none", "outside", "inside", "out_in", "in_out", "repeated"])
    ap.add_argument("--shard-depth", type=int, default=0,
                    help="multi-GPU units = paths of the first d levels (fmm_plan_set_shard_depth); "
                         "0 = auto (bench.default_shard: 3 in blocks)")
    ap.add_argument("--shard-order", default="auto", choices=["auto", "cyclic", "block"],
                    help="multi-GPU unit order (fmm_plan_set_shard_order); auto = with the auto depth, "
                         "blocks, else round-robin")
    ap.add_argument("--comm", default="reduce", choices=["reduce", "allreduce", "reduce_scatter", "p2p"],
                    help="multi-GPU exchange (fmm_plan_set_comm_mode): NCCL on the partial C, or "
                         "p2p = the fused NVLink W-combination of the peers' top-level products")
    ap.add_argument("--comm-one-rank", action="store_true",
                    help="at N = 1, attach a one-rank NCCL communicator so the --comm exchange runs")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-warmup", type=int, default=1)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0)
    ap.add_argument("--ref-sample", type=int, default=256,
                    help="reference arm: leaf rows / cols per step (sample = 8x that per side at C5)")
    args = ap.parse_args()
    ws, _, _ = dist_env()
    if args.gpus != ws and ws > 1:
        log(f"[bench] --gpus {args.gpus} but WORLD_SIZE {ws}")
    if args.impl == "reference":
        run_reference(args)
    else:
        if args.warmup < 3:  # timing rule: at least 3 untimed warm-up steps (reported as run)
            log(f"[bench] --warmup {args.warmup} raised to 3")
            args.warmup = 3
        run_fmm(args)


if __name__ == "__main__":
    main()
