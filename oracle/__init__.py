"""CPU ORACLE for the recursive fast-matrix-multiplication hot path of arXiv 1507.00687.

THIS PACKAGE IS TEST INFRASTRUCTURE.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s
`cpu_baseline` / `--impl reference` legs may import it.  The product (`paper_1507_00687_b200`)
never imports, links or executes anything here, and nothing here imports the product: the two
share no code, tables or constants.  Inputs shared by both come from `fmm_inputs`, which holds
none of the method's arithmetic.

Layout
  rules.py        exact <U,V,W> tables, Brent check, principal quantities, bounds (Python,
                  Fractions)
  fmm_oracle.c    the executor / double-double reference / scaling, plain C + OpenMP, compiled
                  with -O2 -fno-fast-math -ffp-contract=off into liboracle.so
  __init__.py     ctypes marshalling + error metrics (this file)

Parity pins are in tests/test_oracle_*.py.  Functions without a pin: none.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

from . import rules as rules  # noqa: F401
from .rules import Plan, Rule

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "fmm_oracle.c"
_LIB = _HERE / "liboracle.so"
CFLAGS = ["-O2", "-std=c11", "-fno-fast-math", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared"]


def build(force: bool = False) -> Path:
    """Compile liboracle.so with gcc (the oracle is plain C; no CUDA)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(["gcc", *CFLAGS, str(_SRC), "-o", str(tmp), "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


class _CRule(C.Structure):
    _fields_ = [("m0", C.c_int), ("k0", C.c_int), ("n0", C.c_int), ("R", C.c_int),
                ("U", C.POINTER(C.c_double)), ("V", C.POINTER(C.c_double)),
                ("W", C.POINTER(C.c_double))]


class _CPlan(C.Structure):
    _fields_ = [("L", C.c_int), ("rules", C.POINTER(_CRule)), ("node_rule", C.POINTER(C.c_int)),
                ("level_off", C.POINTER(C.c_int64))]


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(str(build()))
        P, I64, I = C.c_void_p, C.c_int64, C.c_int
        for suf in ("f64", "f32"):
            f = getattr(_lib, f"orc_fmm_{suf}")
            f.argtypes = [C.POINTER(_CPlan), I64, I64, I64, P, I64, P, I64, P, I64]
            f.restype = I
            f = getattr(_lib, f"orc_node_st_{suf}")
            f.argtypes = [C.POINTER(_CRule), I64, I64, I64, P, I64, P, I64, P, P]
            f.restype = None
            f = getattr(_lib, f"orc_node_c_{suf}")
            f.argtypes = [C.POINTER(_CRule), I64, I64, P, P, I64]
            f.restype = None
        _lib.orc_ref_dd.argtypes = [I64, I64, P, I64, P, I64, P, I64, P, P, I64]
        _lib.orc_ref_dd.restype = None
        _lib.orc_pow2_round.argtypes = [C.c_double]
        _lib.orc_pow2_round.restype = C.c_double
        _lib.orc_step_O.argtypes = [I64, I64, I64, P, I64, P, I64, I, P, P, C.POINTER(I)]
        _lib.orc_step_O.restype = I
        _lib.orc_step_I.argtypes = [I64, I64, I64, P, I64, P, I64, I, P, C.POINTER(I)]
        _lib.orc_step_I.restype = I
        _lib.orc_scale_repeated.argtypes = [I64, I64, I64, P, I64, P, I64, I, C.c_double, I, I,
                                            P, P, P, P, P, P, P, P, P, C.POINTER(I)]
        _lib.orc_scale_repeated.restype = I
        _lib.orc_unscale.argtypes = [I64, I64, P, I64, P, P]
        _lib.orc_unscale.restype = None
        _lib.orc_num_threads.restype = I
    return _lib


def num_threads() -> int:
    return int(lib().orc_num_threads())


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


class _RuleHolder:
    """Keeps the float64 coefficient arrays alive while C holds pointers to them."""

    def __init__(self, rule: Rule):
        self.arrays = [np.ascontiguousarray(x) for x in rule.as_float()]
        dp = C.POINTER(C.c_double)
        self.c = _CRule(rule.m0, rule.k0, rule.n0, rule.R,
                        *(a.ctypes.data_as(dp) for a in self.arrays))


class _PlanHolder:
    def __init__(self, plan: Plan):
        plan.validate()
        uniq, idx = [], {}
        node_rule, level_off = [], []
        for lv in plan.levels:
            level_off.append(len(node_rule))
            for r in lv:
                key = id(r) if r.name not in idx else r.name
                if r.name not in idx:
                    idx[r.name] = len(uniq)
                    uniq.append(_RuleHolder(r))
                node_rule.append(idx[r.name])
        level_off.append(len(node_rule))
        self.holders = uniq
        self.rules_arr = (_CRule * max(1, len(uniq)))(*[h.c for h in uniq])
        self.node_rule = np.array(node_rule or [0], dtype=np.int32)
        self.level_off = np.array(level_off, dtype=np.int64)
        self.c = _CPlan(plan.L, self.rules_arr, self.node_rule.ctypes.data_as(C.POINTER(C.c_int)),
                        self.level_off.ctypes.data_as(C.POINTER(C.c_int64)))


def _check2d(a: np.ndarray, dtype) -> np.ndarray:
    assert a.ndim == 2 and a.dtype == dtype, (a.shape, a.dtype)
    assert a.strides[1] == a.itemsize, "rows must be contiguous"
    return a


def fmm(A: np.ndarray, B: np.ndarray, plan: Plan) -> np.ndarray:
    """C = A @ B by the recursive algorithm of `plan` (Eq. eqn:recursive_alg) in the
    working precision of A/B (float64 or float32).  Zero-pads to the plan's divisors and crops
    (P:114-115)."""
    dt = A.dtype
    assert dt in (np.float64, np.float32) and B.dtype == dt
    M, K = A.shape
    K2, N = B.shape
    assert K == K2
    if M == 0 or N == 0 or K == 0:
        return np.zeros((M, N), dt)  # empty sum
    pm, pk, pn = plan.dims_divisor()
    Mp, Kp, Np = -(-M // pm) * pm, -(-K // pk) * pk, -(-N // pn) * pn
    if (Mp, Kp, Np) != (M, K, N):
        Ap = np.zeros((Mp, Kp), dt)
        Ap[:M, :K] = A
        Bp = np.zeros((Kp, Np), dt)
        Bp[:K, :N] = B
        return fmm(Ap, Bp, plan)[:M, :N].copy()
    A = _check2d(np.ascontiguousarray(A), dt)
    B = _check2d(np.ascontiguousarray(B), dt)
    Cm = np.empty((M, N), dt)
    ph = _PlanHolder(plan)
    fn = lib().orc_fmm_f64 if dt == np.float64 else lib().orc_fmm_f32
    rc = fn(C.byref(ph.c), M, K, N, _ptr(A), A.strides[0] // A.itemsize, _ptr(B),
            B.strides[0] // B.itemsize, _ptr(Cm), N)
    if rc != 0:
        raise RuntimeError("orc_fmm failed")
    return Cm


def node_st(rule: Rule, A: np.ndarray, B: np.ndarray):
    """All S_r (R x mb x kb) and T_r (R x kb x nb) of one node (Eq. eqn:bilinear_alg)."""
    dt = A.dtype
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B)
    m, k = A.shape
    n = B.shape[1]
    S = np.empty((rule.R, m // rule.m0, k // rule.k0), dt)
    T = np.empty((rule.R, k // rule.k0, n // rule.n0), dt)
    h = _RuleHolder(rule)
    fn = lib().orc_node_st_f64 if dt == np.float64 else lib().orc_node_st_f32
    fn(C.byref(h.c), m, k, n, _ptr(A), k, _ptr(B), n, _ptr(S), _ptr(T))
    return S, T


def node_c(rule: Rule, Ms: np.ndarray) -> np.ndarray:
    """C (M0*mb x N0*nb) = the W-combination of R blocks Ms (R x mb x nb), r ascending."""
    Ms = np.ascontiguousarray(Ms)
    R, mb, nb = Ms.shape
    m, n = mb * rule.m0, nb * rule.n0
    Cm = np.empty((m, n), Ms.dtype)
    h = _RuleHolder(rule)
    fn = lib().orc_node_c_f64 if Ms.dtype == np.float64 else lib().orc_node_c_f32
    fn(C.byref(h.c), m, n, _ptr(Ms), _ptr(Cm), n)
    return Cm


def ref_dd(A: np.ndarray, B: np.ndarray, rows=None):
    """Classical A@B in double-double (compensated Dot2, k ascending); returns (hi, lo) with
    hi = fl(hi + lo).  Stand-in for the paper's quad-precision reference."""
    A = _check2d(np.ascontiguousarray(A, dtype=np.float64), np.float64)
    B = _check2d(np.ascontiguousarray(B, dtype=np.float64), np.float64)
    M, K = A.shape
    N = B.shape[1]
    if rows is None:
        rows_a, nr, rp = None, M, None
    else:
        rows_a = np.ascontiguousarray(np.asarray(rows, dtype=np.int64))
        nr, rp = len(rows_a), _ptr(rows_a)
    hi = np.empty((nr, N))
    lo = np.empty((nr, N))
    lib().orc_ref_dd(K, N, _ptr(A), K, _ptr(B), N, rp, nr, _ptr(hi), _ptr(lo), N)
    return hi, lo


def pow2_round(x: float) -> float:
    return float(lib().orc_pow2_round(float(x)))


class ScalingError(ValueError):
    pass


_WHICH = {0: "row of A", 1: "column of B", 2: "column of A", 3: "row of B"}


def _raise(rc, which):
    raise ScalingError(f"all-zero {_WHICH.get(which.value, '?')} at index {-rc - 1}")


def scale_outside(A, B, pow2=False):
    """Alg. 1 lines 1-4.  Returns (A', B', dA, dB)."""
    A = np.array(A, dtype=np.float64, order="C", copy=True)
    B = np.array(B, dtype=np.float64, order="C", copy=True)
    M, K = A.shape
    N = B.shape[1]
    r, s, w = np.empty(M), np.empty(N), C.c_int(-1)
    rc = lib().orc_step_O(M, K, N, _ptr(A), K, _ptr(B), N, int(pow2), _ptr(r), _ptr(s), C.byref(w))
    if rc:
        _raise(rc, w)
    return A, B, r, s


def scale_inside(A, B, pow2=False):
    """Alg. 2 lines 1-3.  Returns (A', B', d)."""
    A = np.array(A, dtype=np.float64, order="C", copy=True)
    B = np.array(B, dtype=np.float64, order="C", copy=True)
    M, K = A.shape
    N = B.shape[1]
    p, w = np.empty(K), C.c_int(-1)
    rc = lib().orc_step_I(M, K, N, _ptr(A), K, _ptr(B), N, int(pow2), _ptr(p), C.byref(w))
    if rc:
        _raise(rc, w)
    return A, B, p


def scale_repeated(A, B, first_O=True, tau=1.0, max_steps=20, pow2=False, trace=False):
    """Alg. 3 with the Thm stopping-criterion test.
    Returns dict(A, B, dA, dB, dI, steps, [kind, normA, normB, w, tdA, tdB])."""
    A = np.array(A, dtype=np.float64, order="C", copy=True)
    B = np.array(B, dtype=np.float64, order="C", copy=True)
    M, K = A.shape
    N = B.shape[1]
    dA, dB, dI = np.empty(M), np.empty(N), np.empty(K)
    ms = max(1, max_steps)
    kind = C.create_string_buffer(ms)
    nA, nB, ww = np.zeros(ms), np.zeros(ms), np.zeros(ms)
    tdA = np.zeros((ms, M)) if trace else None
    tdB = np.zeros((ms, N)) if trace else None
    w = C.c_int(-1)
    rc = lib().orc_scale_repeated(M, K, N, _ptr(A), K, _ptr(B), N, int(first_O), float(tau),
                                  int(max_steps), int(pow2), _ptr(dA), _ptr(dB), _ptr(dI), kind,
                                  _ptr(nA), _ptr(nB), _ptr(ww),
                                  _ptr(tdA) if trace else None, _ptr(tdB) if trace else None,
                                  C.byref(w))
    if rc < 0:
        _raise(rc, w)
    out = dict(A=A, B=B, dA=dA, dB=dB, dI=dI, steps=rc)
    if trace:
        out.update(kind=kind.raw[:rc].decode(), normA=nA[:rc], normB=nB[:rc], w=ww[:rc],
                   tdA=tdA[:rc], tdB=tdB[:rc])
    return out


def unscale(Cp, dA, dB):
    """C = D_A C' D_B as (dA_i * c'_ij) * dB_j."""
    Cm = np.array(Cp, dtype=np.float64, order="C", copy=True)
    M, N = Cm.shape
    dA = np.ascontiguousarray(dA, dtype=np.float64)
    dB = np.ascontiguousarray(dB, dtype=np.float64)
    lib().orc_unscale(M, N, _ptr(Cm), N, _ptr(dA), _ptr(dB))
    return Cm


SCALE_MODES = ("none", "outside", "inside", "out_in", "in_out", "repeated")


def scale_operands(A, B, mode="none", pow2=False, tau=1.0, max_steps=20):
    """The scaling half of Alg. 1-3: returns dict(A=A', B=B', dA, dB, steps) with
    A' = D_A^-1 A D, B' = D^-1 B D_B^-1 (D folded into A', B'; P:745-748, P:862-866,
    P:940-956).  out_in / in_out = one O then one I step (or reverse) = Alg. 3 with
    max_steps=2 and no stop test reached."""
    A = np.asarray(A, dtype=np.float64)
    B = np.asarray(B, dtype=np.float64)
    M, K = A.shape
    N = B.shape[1]
    if mode == "none":
        return dict(A=A, B=B, dA=np.ones(M), dB=np.ones(N), steps=0)
    if mode == "outside":
        Ap, Bp, dA, dB = scale_outside(A, B, pow2)
        return dict(A=Ap, B=Bp, dA=dA, dB=dB, steps=1)
    if mode == "inside":
        Ap, Bp, _ = scale_inside(A, B, pow2)
        return dict(A=Ap, B=Bp, dA=np.ones(M), dB=np.ones(N), steps=1)
    first_O = mode in ("out_in", "repeated")
    steps = 2 if mode in ("out_in", "in_out") else max_steps
    tau_eff = tau if mode == "repeated" else -1.0  # fixed 2-step modes: no stop test
    res = scale_repeated(A, B, first_O=first_O, tau=tau_eff, max_steps=steps, pow2=pow2)
    return dict(A=res["A"], B=res["B"], dA=res["dA"], dB=res["dB"], steps=res["steps"])


def scaled_fmm(A, B, plan: Plan, mode="none", pow2=False, tau=1.0, max_steps=20):
    """Scaling wrapper + FMM + unscale (Alg. 1-3; Alg. 1 line 5 read as C' = A'B', DESIGN.md
    reading A5).  Returns (C, info); info holds the step count, the factors dA, dB and the
    scaled operands A', B' the FMM ran on."""
    info = scale_operands(A, B, mode, pow2, tau, max_steps)
    Cp = fmm(info["A"], info["B"], plan)
    if mode == "none":
        return Cp, info
    return unscale(Cp, info["dA"], info["dB"]), info


# ---------------------------------------------------------------------------------------------
# Row sampling: the recursion commutes with restricting to rows that are
# consistent across every level's block split.
# ---------------------------------------------------------------------------------------------

def lift_rows(M: int, plan: Plan, leaf_rows) -> np.ndarray:
    """Rows G of A/C whose restriction the oracle can run exactly: every leaf-local row in
    `leaf_rows` lifted through all levels' row splits (sorted).  |G| = prod(M0) * |leaf_rows|."""
    pm, _, _ = plan.dims_divisor()
    mleaf = M // pm
    G = np.asarray(sorted(set(int(r) for r in leaf_rows)), dtype=np.int64)
    assert G.size and G.max() < mleaf
    offs = np.array([0], dtype=np.int64)
    m = M
    for lv in plan.levels:
        m0 = lv[0].m0
        m //= m0
        offs = (offs[:, None] + (np.arange(m0) * m)[None, :]).ravel()
    return np.sort((offs[:, None] + G[None, :]).ravel())


def lift_cols(N: int, plan: Plan, leaf_cols) -> np.ndarray:
    """Columns H of B/C consistent with every level's column split (the transpose of
    lift_rows): column j of every T_r, M_r and C_k depends only on column j of the B blocks."""
    _, _, pn = plan.dims_divisor()
    nleaf = N // pn
    H = np.asarray(sorted(set(int(c) for c in leaf_cols)), dtype=np.int64)
    assert H.size and H.max() < nleaf
    offs = np.array([0], dtype=np.int64)
    n = N
    for lv in plan.levels:
        n0 = lv[0].n0
        n //= n0
        offs = (offs[:, None] + (np.arange(n0) * n)[None, :]).ravel()
    return np.sort((offs[:, None] + H[None, :]).ravel())


def fmm_sub(A: np.ndarray, B: np.ndarray, plan: Plan, rows: np.ndarray, cols: np.ndarray) -> np.ndarray:
    """C_oracle[rows][:, cols] from A[rows, :] and B[:, cols] alone (rows / cols from lift_rows /
    lift_cols): bitwise equal to the same entries of the full oracle run, because the leaf is
    row- and column-independent and every S / T / C sum is elementwise."""
    return fmm(np.ascontiguousarray(A[rows, :]), np.ascontiguousarray(B[:, cols]), plan)


def fmm_rows(A: np.ndarray, B: np.ndarray, plan: Plan, rows: np.ndarray) -> np.ndarray:
    """C_oracle[rows, :] computed by running the oracle on A[rows, :] with all of B.  `rows`
    must come from lift_rows (bitwise equal to the same rows of the full oracle run)."""
    return fmm(np.ascontiguousarray(A[rows, :]), B, plan)


# ---------------------------------------------------------------------------------------------
# Metrics (BASELINE.json north_star tolerance)
# ---------------------------------------------------------------------------------------------

def parity_metric(Cx, Cy, A_maxabs, B_maxabs, K) -> float:
    """||Cx - Cy||max / (||A||max ||B||max K)."""
    d = np.max(np.abs(np.asarray(Cx, np.float64) - np.asarray(Cy, np.float64))) if np.size(Cx) else 0.0
    return float(d / (A_maxabs * B_maxabs * K))


def error_report(Chat, hi, lo, A_maxabs, B_maxabs):
    """Error of Chat against the double-double reference (hi + lo)."""
    Chat = np.asarray(Chat, np.float64)
    d = np.abs((Chat - hi) - lo)
    nz = hi != 0
    rel = float(np.max(d[nz] / np.abs(hi[nz]))) if nz.any() else 0.0
    return {"max_abs": float(d.max()) if d.size else 0.0,
            "normalised": float(d.max() / (A_maxabs * B_maxabs)) if d.size else 0.0,
            "max_rel": rel, "zero_entries": int((~nz).sum())}
