"""Seeded synthetic inputs shared by the oracle side and the product side.

This module holds NONE of the method's arithmetic: it only draws the A, B matrices of the
BASELINE.json configs (and small test cases) on the host with torch's CPU generator, so that the
CUDA path and the oracle see bit-identical inputs.  Recipe (DESIGN.md §4 / SURVEY §8(d)):
`g = torch.Generator('cpu').manual_seed(seed)`, float64, row-major; U(a,b) = a + (b-a)*rand;
N(0,1) = randn; draw order per config; the FP32 variant casts the FP64 draws.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch


@dataclass(frozen=True)
class Config:
    name: str
    M: int
    K: int
    N: int
    rules: tuple  # rule name per level, root first
    dist: str  # "u(-1,1)" | "n(0,1)" | "u(0,1)" | "skew"
    seed: int
    note: str = ""


# BASELINE.json configs[0..4] (C1..C5).  DESIGN.md reading A15: level 1 is the root.
CONFIGS = {
    "C1": Config("C1", 512, 512, 512, ("winograd", "winograd"), "u(-1,1)", 0,
                 "Strassen-Winograd L=2, leaf 128^3"),
    "C2": Config("C2", 4096, 4096, 4096, ("strassen",) * 4, "n(0,1)", 1,
                 "Strassen L=4, leaf 256^3"),
    "C2c": Config("C2c", 4096, 4096, 4096, ("classical222",) * 4, "n(0,1)", 1,
                  "classical <2,2,2;8> L=4 comparison for C2"),
    "C3": Config("C3", 8192, 4096, 8192, ("winograd", "classical222", "strassen"), "u(0,1)", 2,
                 "uniform non-stationary S-W / classical / Strassen"),
    "C4": Config("C4", 4096, 4096, 4096, ("winograd",) * 3, "skew", 3,
                 "diagonal-scaling stress"),
    "C5": Config("C5", 32768, 32768, 32768, ("winograd",) * 3, "u(-1,1)", 4,
                 "throughput, S-W L=3"),
}


def _u(g, shape, a, b, pin=False):
    """U(a, b) = a + (b - a) * rand, computed in place (rand * (b - a) is exact for the
    power-of-two widths used, then one rounded addition)."""
    t = torch.empty(shape, dtype=torch.float64, pin_memory=pin)
    t.uniform_(0.0, 1.0, generator=g)
    return t.mul_(b - a).add_(a)


def draw_torch(dist: str, M: int, K: int, N: int, seed: int, pin: bool = False):
    """A, B as float64 CPU torch tensors (optionally in pinned memory, for the benchmark's
    host buffers).  Only the uniform families support pin=True."""
    g = torch.Generator("cpu").manual_seed(seed)
    if dist == "u(-1,1)":
        return _u(g, (M, K), -1.0, 1.0, pin), _u(g, (K, N), -1.0, 1.0, pin)
    if dist == "u(0,1)":
        return _u(g, (M, K), 0.0, 1.0, pin), _u(g, (K, N), 0.0, 1.0, pin)
    assert not pin
    return tuple(torch.from_numpy(x) for x in draw(dist, M, K, N, seed))


def draw(dist: str, M: int, K: int, N: int, seed: int):
    """A (M x K), B (K x N) as float64 numpy arrays (row-major)."""
    if dist in ("u(-1,1)", "u(0,1)"):
        A, B = draw_torch(dist, M, K, N, seed)
        return A.numpy(), B.numpy()
    g = torch.Generator("cpu").manual_seed(seed)
    if dist == "u(-1,1)":
        A = _u(g, (M, K), -1.0, 1.0)
        B = _u(g, (K, N), -1.0, 1.0)
    elif dist == "u(0,1)":
        A = _u(g, (M, K), 0.0, 1.0)
        B = _u(g, (K, N), 0.0, 1.0)
    elif dist == "n(0,1)":
        A = torch.randn((M, K), generator=g, dtype=torch.float64)
        B = torch.randn((K, N), generator=g, dtype=torch.float64)
    elif dist == "skew":
        # C4: G, H ~ U(0,1); d1 (M), d2 (K), d3 (K), d4 (N) = 10^U(-8,8);
        # A = (d1_i g_ij) d2_j, B = (d3_k h_kj) d4_j.
        G = _u(g, (M, K), 0.0, 1.0)
        H = _u(g, (K, N), 0.0, 1.0)
        d1 = torch.pow(10.0, _u(g, (M,), -8.0, 8.0))
        d2 = torch.pow(10.0, _u(g, (K,), -8.0, 8.0))
        d3 = torch.pow(10.0, _u(g, (K,), -8.0, 8.0))
        d4 = torch.pow(10.0, _u(g, (N,), -8.0, 8.0))
        A = (d1[:, None] * G) * d2[None, :]
        B = (d3[:, None] * H) * d4[None, :]
    elif dist in ("paper2", "paper3"):
        # PAPER.md Sec. 6.5 distributions 2 and 3 (distribution 1 is "u(0,1)").
        # All entries are drawn U(0,1) (A then B, row-major); the designated blocks are then
        # multiplied by 1/N^2 or N^2 (U(0, c) = c U(0, 1)).  Halves are taken 0-based: rows
        # i < N/2 (top), columns j >= N/2 (right) -- DESIGN.md reading A28.
        assert M == K == N, "the paper's distributions are square"
        A = _u(g, (M, K), 0.0, 1.0)
        B = _u(g, (K, N), 0.0, 1.0)
        h = N // 2
        small, big = 1.0 / (N * N), float(N * N)
        if dist == "paper2":  # A: right columns small; B: top rows small (models Ex. 5.2)
            A[:, h:] *= small
            B[:h, :] *= small
        else:  # A: top-right block large; B: left columns small (models Ex. 6.9)
            A[:h, h:] *= big
            B[:, :h] *= small
    else:
        raise ValueError(dist)
    return A.numpy(), B.numpy()


def config_inputs(name: str, scale_div: int = 1, dtype=np.float64):
    """Inputs of config `name`; scale_div > 1 shrinks M, K, N by that factor (same recipe and
    seed) for oracle-sized parity cases."""
    c = CONFIGS[name]
    A, B = draw(c.dist, c.M // scale_div, c.K // scale_div, c.N // scale_div, c.seed)
    if dtype != np.float64:
        A, B = A.astype(dtype), B.astype(dtype)
    return A, B


def random_pair(M: int, K: int, N: int, seed: int, dist: str = "u(-1,1)", dtype=np.float64):
    A, B = draw(dist, M, K, N, seed)
    return A.astype(dtype, copy=False), B.astype(dtype, copy=False)


def integer_pair(M: int, K: int, N: int, seed: int, lo: int = -8, hi: int = 8):
    """Small-integer matrices (exactly representable; used for exactness pins)."""
    g = torch.Generator("cpu").manual_seed(seed)
    A = torch.randint(lo, hi + 1, (M, K), generator=g).to(torch.float64)
    B = torch.randint(lo, hi + 1, (K, N), generator=g).to(torch.float64)
    return A.numpy(), B.numpy()
