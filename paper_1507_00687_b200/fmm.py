"""Thin ctypes binding of libfmm_b200.so (include/fmm.h): same names, argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module only converts torch
tensors to (pointer, leading dimension) pairs and picks the current CUDA stream.  There is no
fallback: if the library is missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from pathlib import Path
from typing import Optional, Sequence

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "libfmm_b200.so"

# enums (include/fmm.h)
FMM_OK = 0
STATUS = {0: "FMM_OK", 1: "FMM_E_ARG", 2: "FMM_E_RULE", 3: "FMM_E_SHAPE", 4: "FMM_E_ALIGN",
          5: "FMM_E_PRECOND", 6: "FMM_E_UNSUPPORTED", 7: "FMM_E_CUDA", 8: "FMM_E_NCCL",
          9: "FMM_E_OOM", 10: "FMM_E_NOT_CONVERGED"}
F64, F32 = 0, 1
LEAF_NATIVE, LEAF_TF32, LEAF_3XTF32 = 0, 1, 2
SCALE_MODES = {"none": 0, "outside": 1, "inside": 2, "out_in": 3, "in_out": 4, "repeated": 5}

# every function declared in include/fmm.h: name -> (restype, argtypes)
_P, _I, _I64, _SZ, _D = C.c_void_p, C.c_int, C.c_int64, C.c_size_t, C.c_double


class fmm_scaling(C.Structure):
    _fields_ = [("mode", C.c_int), ("first_step_is_O", C.c_int), ("tau", C.c_double),
                ("max_steps", C.c_int), ("pow2", C.c_int)]


SIGNATURES = {
    "fmm_rule_create": (_I, [_I, _I, _I, _I, _P, _P, _P, _I, C.c_char_p, C.POINTER(_P), C.POINTER(_I64)]),
    "fmm_rule_builtin": (_I, [C.c_char_p, C.POINTER(_P)]),
    "fmm_rule_info": (_I, [_P, C.POINTER(_I), C.POINTER(_I), C.POINTER(_I), C.POINTER(_I), _P, _P, _P, C.POINTER(_I)]),
    "fmm_rule_destroy": (None, [_P]),
    "fmm_plan_create": (_I, [C.POINTER(_P), _I, _I, _I, _I64, _I64, _I64, _I, _I, C.POINTER(fmm_scaling), C.POINTER(_P)]),
    "fmm_plan_destroy": (None, [_P]),
    "fmm_plan_set_partition": (_I, [_P, _I, _I]),
    "fmm_plan_set_schedule": (_I, [_P, _I]),
    "fmm_plan_set_fusion": (_I, [_P, _I]),
    "fmm_plan_set_shard_depth": (_I, [_P, _I]),
    "fmm_plan_set_comm_mode": (_I, [_P, _I]),
    "fmm_rule_transform": (_I, [_P, _I, C.POINTER(_P)]),
    "fmm_plan_set_k1_levels": (_I, [_P, _I]),
    "fmm_plan_set_leaf_split": (_I, [_P, _I]),
    "fmm_plan_set_shard_order": (_I, [_P, _I]),
    "fmm_plan_sym_bytes": (_I, [_P, _P]),
    "fmm_plan_sym_alloc": (_I, [_P, _P]),
    "fmm_plan_sym_ptr": (_I, [_P, _P]),
    "fmm_plan_set_peer_handles": (_I, [_P, _P, _I]),
    "fmm_plan_p2p_combine": (_I, [_P, _P, _I, _P, _I64, _I64, _I64, _P]),
    "fmm_plan_set_k3_levels": (_I, [_P, _I]),
    "fmm_scale_apply": (_I, [_I, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _P, _P, _P, _I64, _P, _I64, _P]),
    "fmm_rule_quantities": (_I, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_double), C.POINTER(C.c_double), _P, _P]),
    "fmm_plan_stability": (_I, [_P, C.POINTER(C.c_double), C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "fmm_choose_variants": (_I, [_P, _P, _I, _P, C.POINTER(C.c_double)]),
    "fmm_plan_fused_launches": (_I, [_P, C.POINTER(C.c_int64)]),
    "fmm_plan_owned": (_I, [_P, _I, _I, _P, C.POINTER(_I)]),
    "fmm_plan_workspace_bytes": (_I, [_P, C.POINTER(_SZ)]),
    "fmm_plan_launch_count": (_I, [_P, C.POINTER(_I64)]),
    "fmm_plan_set_timing": (_I, [_P, _I]),
    "fmm_plan_set_graph": (_I, [_P, _I]),
    "fmm_plan_step_times": (_I, [_P, _P, _P]),
    "fmm_execute": (_I, [_P, _P, _I64, _P, _I64, _P, _I64, _P, _SZ, _P]),
    "fmm_execute_host": (_I, [_P, _P, _I64, _P, _I64, _P, _I64, _P, _P, _P, _P, _SZ, _P]),
    "fmm_execute_host_batch": (_I, [_P, _I, _P, _I64, _P, _I64, _P, _I64, _P, _P, _P, _I, _P, _SZ, _P]),
    "fmm_node_st": (_I, [_P, _I, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _P, _P]),
    "fmm_node_c": (_I, [_P, _I, _I64, _I64, _P, _P, _I64, _P]),
    "fmm_gemm": (_I, [_I, _I, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P]),
    "fmm_scale_outside": (_I, [_I, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P, _I64, _P, _P, _I, _P]),
    "fmm_scale_inside": (_I, [_I, _I64, _I64, _I64, _P, _I64, _P, _I64, _P, _I64, _P, _I64, _P, _I, _P]),
    "fmm_scale_repeated": (_I, [_I, _I64, _I64, _I64, _P, _I64, _P, _I64, C.POINTER(fmm_scaling), _P, _I64, _P, _I64, _P, _P, _P, _P, _P, _SZ, _P]),
    "fmm_scale_workspace_bytes": (_I, [_I64, _I64, _I64, C.POINTER(_SZ)]),
    "fmm_unscale": (_I, [_I, _I64, _I64, _P, _I64, _P, _P, _P]),
    "fmm_plan_last_scaling_steps": (_I, [_P, _P, C.POINTER(_I), _P]),
    "fmm_comm_unique_id": (_I, [_P]),
    "fmm_plan_set_comm": (_I, [_P, _P, _I, _I]),
    "fmm_plan_set_barrier": (_I, [_P, _P, _P]),
    "fmm_plan_set_virtual_scaling": (_I, [_P, _I]),
    "fmm_plan_set_single_launch": (_I, [_P, _I]),
    "fmm_last_error": (C.c_char_p, []),
    "fmm_version": (C.c_char_p, []),
}

_lib = None


class FmmError(RuntimeError):
    def __init__(self, fn, code, msg):
        super().__init__(f"{fn}: {STATUS.get(code, code)}: {msg}")
        self.code = code
        self.status = STATUS.get(code, str(code))


def lib():
    """Load libfmm_b200.so (built in-tree by `paper_1507_00687_b200.build`).  Raises if absent:
    the product path has no CPU or library fallback."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_1507_00687_b200.build`")
        h = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
    return _lib


def _check(fn: str, code: int):
    if code != FMM_OK:
        raise FmmError(fn, code, lib().fmm_last_error().decode())


def _call(fn: str, *args):
    _check(fn, getattr(lib(), fn)(*args))


def _stream(stream=None):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _dtype_code(t) -> int:
    import torch
    if t.dtype == torch.float64:
        return F64
    if t.dtype == torch.float32:
        return F32
    raise TypeError(f"unsupported dtype {t.dtype}")


def _mat(t, name):
    """(pointer, ld) of a row-major CUDA matrix (unit column stride)."""
    if t.dim() != 2 or (t.numel() > 0 and t.shape[1] > 1 and t.stride(1) != 1):
        raise ValueError(f"{name} must be a 2-D row-major tensor")
    return C.c_void_p(t.data_ptr()), max(t.stride(0), t.shape[1], 1)


# ---------------------------------------------------------------------------------------------
class Rule:
    """fmm_rule wrapper (<U,V,W>)."""

    def __init__(self, handle, name):
        self._h = C.c_void_p(handle)
        self.name = name

    @classmethod
    def builtin(cls, name: str) -> "Rule":
        h = C.c_void_p()
        _call("fmm_rule_builtin", name.encode(), C.byref(h))
        return cls(h.value, name)

    @classmethod
    def create(cls, m0, k0, n0, U, V, W, log2_den=0, name="custom") -> "Rule":
        import numpy as np
        U = np.ascontiguousarray(U, dtype=np.int32)
        V = np.ascontiguousarray(V, dtype=np.int32)
        W = np.ascontiguousarray(W, dtype=np.int32)
        R = U.shape[1]
        h = C.c_void_p()
        nv = C.c_int64(0)
        code = lib().fmm_rule_create(m0, k0, n0, R, U.ctypes.data, V.ctypes.data, W.ctypes.data,
                                     log2_den, name.encode(), C.byref(h), C.byref(nv))
        if code != FMM_OK:
            err = FmmError("fmm_rule_create", code, lib().fmm_last_error().decode())
            err.n_violations = nv.value
            raise err
        return cls(h.value, name)

    def info(self):
        import numpy as np
        m0, k0, n0, R, den = C.c_int(), C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _call("fmm_rule_info", self._h, C.byref(m0), C.byref(k0), C.byref(n0), C.byref(R), None,
              None, None, C.byref(den))
        U = np.zeros((m0.value * k0.value, R.value), np.int32)
        V = np.zeros((k0.value * n0.value, R.value), np.int32)
        W = np.zeros((m0.value * n0.value, R.value), np.int32)
        _call("fmm_rule_info", self._h, None, None, None, None, U.ctypes.data, V.ctypes.data,
              W.ctypes.data, None)
        return dict(m0=m0.value, k0=k0.value, n0=n0.value, R=R.value, U=U, V=V, W=W,
                    log2_den=den.value)

    def transform(self, kind: str) -> "Rule":
        """'rotate' ([[W,U,V]]: <n0,m0,k0>), 'rotate2' ([[V,W,U]]: <k0,n0,m0>) or 'transpose'
        (<n0,k0,m0>), validated (fmm_rule_transform)."""
        h = C.c_void_p()
        _call("fmm_rule_transform", self._h, {"rotate": 1, "rotate2": 2, "transpose": 3}[kind],
              C.byref(h))
        return Rule(h.value, f"{self.name}_{kind}")

    def quantities(self):
        """nnz, Q, E, q (m0*n0), e (m0*n0) of the rule (Sec. 4.1)."""
        import numpy as np
        info = self.info()
        nw = info["m0"] * info["n0"]
        nnz, Q, E = C.c_int64(), C.c_double(), C.c_double()
        q, e = np.zeros(nw), np.zeros(nw)
        _call("fmm_rule_quantities", self._h, C.byref(nnz), C.byref(Q), C.byref(E), q.ctypes.data,
              e.ctypes.data)
        return dict(nnz=nnz.value, Q=Q.value, E=E.value, q=q, e=e)

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.fmm_rule_destroy(self._h)
            self._h = None


def choose_variants(root: "Rule", variants: Sequence["Rule"]):
    """Two-level plan minimising xi: (choice per child r of the root, xi) (fmm_choose_variants)."""
    import numpy as np
    R = root.info()["R"]
    arr = (C.c_void_p * len(variants))(*[v._h.value for v in variants])
    ch = np.zeros(R, np.int32)
    xi = C.c_double()
    _call("fmm_choose_variants", root._h, C.cast(arr, C.c_void_p), len(variants), ch.ctypes.data,
          C.byref(xi))
    return [int(c) for c in ch], xi.value


def _scaling(scaling) -> Optional[fmm_scaling]:
    if scaling is None:
        return None
    if isinstance(scaling, str):
        scaling = {"mode": scaling}
    mode = SCALE_MODES[scaling.get("mode", "none")] if isinstance(scaling.get("mode"), str) else scaling.get("mode", 0)
    return fmm_scaling(mode, int(scaling.get("first_step_is_O", 1)), float(scaling.get("tau", 1.0)),
                       int(scaling.get("max_steps", 20)), int(scaling.get("pow2", 0)))


class Plan:
    """fmm_plan wrapper.  `rules`: one Rule per level (uniform=True) or one per internal node in
    BFS order (uniform=False)."""

    def __init__(self, rules: Sequence[Rule], M: int, K: int, N: int, dtype: str = "f64",
                 leaf: int = LEAF_NATIVE, uniform: bool = True, levels: Optional[int] = None,
                 scaling=None):
        self.rules = list(rules)
        self.levels = len(self.rules) if (uniform and levels is None) else levels
        if self.levels is None:
            raise ValueError("levels required for a non-uniform plan")
        self.M, self.K, self.N = M, K, N
        self.dtype = {"f64": F64, "f32": F32}[dtype]
        arr = (C.c_void_p * max(1, len(self.rules)))(*[r._h.value for r in self.rules])
        sc = _scaling(scaling)
        h = C.c_void_p()
        _call("fmm_plan_create", C.cast(arr, C.POINTER(C.c_void_p)), len(self.rules), self.levels,
              int(uniform), M, K, N, self.dtype, leaf, C.byref(sc) if sc is not None else None,
              C.byref(h))
        self._h = h
        self.scaling = sc
        self._ws = None

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.fmm_plan_destroy(self._h)
            self._h = None

    def workspace_bytes(self) -> int:
        b = C.c_size_t()
        _call("fmm_plan_workspace_bytes", self._h, C.byref(b))
        return b.value

    def launch_count(self) -> int:
        n = C.c_int64()
        _call("fmm_plan_launch_count", self._h, C.byref(n))
        return n.value

    STEP_KINDS = {1: "K1", 2: "K2", 3: "K3", 4: "ACC", 5: "ZERO", 6: "SCALE", 7: "REDUCE"}  # K2 includes K2F / the single-launch kernel

    def set_single_launch(self, enable: bool = True):
        """Small two-level plans as one cooperative kernel (default) or three launches."""
        _call("fmm_plan_set_single_launch", self._h, int(enable))
        self._ws = None

    def set_virtual_scaling(self, enable: bool = True):
        """Power-of-two scaling applied on the fly by the root K1 (default) or materialised."""
        _call("fmm_plan_set_virtual_scaling", self._h, int(enable))
        self._ws = None

    def set_graph(self, enable: bool = True):
        """Replay fmm_execute as a CUDA graph for repeated calls with the same buffers."""
        _call("fmm_plan_set_graph", self._h, int(enable))

    def set_timing(self, enable: bool = True):
        _call("fmm_plan_set_timing", self._h, int(enable))

    def step_times(self):
        """{kind: (total ms, launches)} since the previous call (synchronises)."""
        import numpy as np
        ms = np.zeros(8)
        n = np.zeros(8, np.int64)
        _call("fmm_plan_step_times", self._h, ms.ctypes.data, n.ctypes.data)
        return {self.STEP_KINDS[k]: (float(ms[k]), int(n[k])) for k in range(1, 8) if n[k]}

    def set_partition(self, rank: int, nranks: int):
        _call("fmm_plan_set_partition", self._h, rank, nranks)
        self._ws = None

    def set_schedule(self, schedule: str):
        """'auto' | 'breadth' | 'depth' (top-level depth-first, per-r accumulation) | 'hybrid'
        (root S / T at once, subtrees in turn, root combination at the end)."""
        _call("fmm_plan_set_schedule", self._h,
              {"auto": 0, "breadth": 1, "depth": 2, "hybrid": 3}[schedule])
        self._ws = None

    def stability(self):
        """{'xi', 'delta', 'uniform_bound'} of the plan's recursion tree (fmm_plan_stability)."""
        xi, de, ub = C.c_double(), C.c_double(), C.c_double()
        _call("fmm_plan_stability", self._h, C.byref(xi), C.byref(de), C.byref(ub))
        return {"xi": xi.value, "delta": de.value, "uniform_bound": ub.value}

    def set_fusion(self, mode):
        """Leaf-product epilogue fusion of the parents' W-combination: 'off' | 'on' | 'auto'."""
        _call("fmm_plan_set_fusion", self._h, {"off": 0, "on": 1, "auto": 2}[mode])
        self._ws = None

    def set_k1_levels(self, levels: int = 2):
        """S / T formation: 2 = two recursion levels per K1 pass (K1X2, default), 1 = one."""
        _call("fmm_plan_set_k1_levels", self._h, int(levels))
        self._ws = None

    def set_leaf_split(self, in_pass: bool = True):
        """FP32 tensor-core leaves: hi / lo operand split written by the leaf level's K1X2
        (True, default where it applies) or by a separate split pass (False)."""
        _call("fmm_plan_set_leaf_split", self._h, int(bool(in_pass)))
        self._ws = None

    def set_k3_levels(self, levels: int = 2):
        """W-combination: 2 = two recursion levels per K3 pass (K3X2, default), 1 = one."""
        _call("fmm_plan_set_k3_levels", self._h, int(levels))
        self._ws = None

    def fused_launches(self) -> int:
        n = C.c_int64()
        _call("fmm_plan_fused_launches", self._h, C.byref(n))
        return n.value

    def set_comm_mode(self, mode: str):
        """Multi-GPU exchange: 'reduce' (C on rank 0), 'allreduce', 'reduce_scatter' (rows), or
        'p2p' (fused NVLink combine of the peers' top-level products into this rank's rows)."""
        _call("fmm_plan_set_comm_mode", self._h,
              {"reduce": 0, "allreduce": 1, "reduce_scatter": 2, "p2p": 3}[mode])
        self._ws = None

    def sym_bytes(self) -> int:
        n = C.c_size_t()
        _call("fmm_plan_sym_bytes", self._h, C.byref(n))
        return n.value

    def sym_alloc(self) -> bytes:
        """Allocate this rank's symmetric product buffer; returns its 64-byte CUDA IPC handle."""
        h = C.create_string_buffer(64)
        _call("fmm_plan_sym_alloc", self._h, h)
        return h.raw

    def sym_ptr(self) -> int:
        v = C.c_void_p()
        _call("fmm_plan_sym_ptr", self._h, C.byref(v))
        return v.value or 0

    def set_peer_handles(self, handles):
        """Every rank's sym_alloc() handle, in rank order."""
        buf = b"".join(handles)
        _call("fmm_plan_set_peer_handles", self._h, C.c_char_p(buf), len(handles))

    def p2p_combine(self, peer_ptrs, C_out, row0: int, row1: int, stream=None):
        """Rows [row0, row1) of C = sum_r w_kr M_r from the products at peer_ptrs (building block)."""
        arr = (C.c_void_p * len(peer_ptrs))(*peer_ptrs)
        _call("fmm_plan_p2p_combine", self._h, arr, len(peer_ptrs), C.c_void_p(C_out.data_ptr()),
              C_out.stride(0), row0, row1, _stream(stream))
        return C_out

    def set_shard_depth(self, depth: int):
        """Multi-GPU units = paths of the first `depth` levels (fmm_plan_set_shard_depth)."""
        _call("fmm_plan_set_shard_depth", self._h, depth)
        self._ws = None

    def set_shard_order(self, order: str = "cyclic"):
        """Multi-GPU unit order: "cyclic" (unit u on rank u mod P, default) or "block"
        (contiguous blocks of units per rank)."""
        _call("fmm_plan_set_shard_order", self._h, {"cyclic": 0, "block": 1}[order])
        self._ws = None

    def owned(self, rank: int, nranks: int):
        import numpy as np
        R = C.c_int()
        _call("fmm_plan_owned", self._h, rank, nranks, None, C.byref(R))
        out = np.zeros(R.value, np.int32)
        _call("fmm_plan_owned", self._h, rank, nranks, out.ctypes.data, C.byref(R))
        return [r for r in range(R.value) if out[r]]

    def set_comm(self, uid: bytes, rank: int, nranks: int):
        buf = C.create_string_buffer(bytes(uid), 128)
        _call("fmm_plan_set_comm", self._h, buf, rank, nranks)
        self._ws = None

    BARRIER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p)

    def set_barrier(self, fn):
        """Comm mode 3's barrier as a Python callable fn(stream_ptr) -> None (raising = failure),
        or None for the NCCL barrier (fmm_plan_set_barrier)."""
        if fn is None:
            self._barrier = None
            _call("fmm_plan_set_barrier", self._h, None, None)
        else:
            def tramp(_user, stream):
                try:
                    fn(stream)
                    return 0
                except Exception:  # noqa: BLE001 -- reported as FMM_E_NCCL by the library
                    return 1
            self._barrier = self.BARRIER_FN(tramp)  # kept alive with the plan
            _call("fmm_plan_set_barrier", self._h, C.cast(self._barrier, C.c_void_p), None)
        self._ws = None

    def workspace(self, device=None):
        """A cached device workspace tensor of workspace_bytes()."""
        import torch
        nb = self.workspace_bytes()
        if self._ws is None or self._ws.numel() < nb:
            self._ws = torch.empty(nb, dtype=torch.uint8, device=device or "cuda")
        return self._ws

    def execute(self, A, B, C_out=None, ws=None, stream=None):
        """C = A.B on the device (torch CUDA tensors, row-major)."""
        import torch
        if C_out is None:
            C_out = torch.empty((self.M, self.N), dtype=A.dtype, device=A.device)
        ws = self.workspace(A.device) if ws is None else ws
        a, lda = _mat(A, "A")
        b, ldb = _mat(B, "B")
        c, ldc = _mat(C_out, "C")
        _call("fmm_execute", self._h, a, lda, b, ldb, c, ldc, C.c_void_p(ws.data_ptr()),
              ws.numel() * ws.element_size(), _stream(stream))
        return C_out

    def execute_host(self, A_host, B_host, C_host, A_dev, B_dev, C_dev, ws=None, stream=None):
        """End-to-end call with host (pinned) buffers; copies are enqueued on the stream."""
        ws = self.workspace(A_dev.device) if ws is None else ws
        a, lda = C.c_void_p(A_host.data_ptr()), A_host.stride(0)
        b, ldb = C.c_void_p(B_host.data_ptr()), B_host.stride(0)
        c, ldc = C.c_void_p(C_host.data_ptr()), C_host.stride(0)
        _call("fmm_execute_host", self._h, a, lda, b, ldb, c, ldc, C.c_void_p(A_dev.data_ptr()),
              C.c_void_p(B_dev.data_ptr()), C.c_void_p(C_dev.data_ptr()),
              C.c_void_p(ws.data_ptr()), ws.numel() * ws.element_size(), _stream(stream))
        return C_host

    def execute_host_batch(self, A_hosts, B_hosts, C_hosts, A_devs, B_devs, C_devs, ws=None,
                           stream=None):
        """A stream of products C_i = A_i B_i with host (pinned) buffers, pipelined across
        problems over the device buffer sets A_devs / B_devs / C_devs (problem i uses set
        i mod len(A_devs)); returns without synchronising."""
        n, nbuf = len(A_hosts), len(A_devs)
        if n == 0:
            return C_hosts
        if not (len(B_hosts) == len(C_hosts) == n and len(B_devs) == len(C_devs) == nbuf):
            raise ValueError("execute_host_batch: list lengths differ")
        ws = self.workspace(A_devs[0].device) if ws is None else ws
        arr = lambda ts: (C.c_void_p * max(len(ts), 1))(*[t.data_ptr() for t in ts])
        _call("fmm_execute_host_batch", self._h, n, arr(A_hosts), A_hosts[0].stride(0),
              arr(B_hosts), B_hosts[0].stride(0), arr(C_hosts), C_hosts[0].stride(0),
              arr(A_devs), arr(B_devs), arr(C_devs), nbuf, C.c_void_p(ws.data_ptr()),
              ws.numel() * ws.element_size(), _stream(stream))
        return C_hosts

    def last_scaling_steps(self, ws=None, stream=None) -> int:
        ws = self._ws if ws is None else ws
        n = C.c_int()
        _call("fmm_plan_last_scaling_steps", self._h, C.c_void_p(ws.data_ptr()), C.byref(n),
              _stream(stream))
        return n.value


# ---------------------------------------------------------------------------------------------
def gemm(A, B, leaf=LEAF_NATIVE, C_out=None, stream=None):
    """Classical C = A.B with the leaf kernel alone."""
    import torch
    M, K = A.shape
    N = B.shape[1]
    if C_out is None:
        C_out = torch.empty((M, N), dtype=A.dtype, device=A.device)
    a, lda = _mat(A, "A")
    b, ldb = _mat(B, "B")
    c, ldc = _mat(C_out, "C")
    _call("fmm_gemm", _dtype_code(A), leaf, M, K, N, a, lda, b, ldb, c, ldc, _stream(stream))
    return C_out


_PLAN_CACHE = {}


def matmul(A, B, rules=("winograd",) * 3, scaling=None, leaf=None, C_out=None, stream=None):
    """C = A @ B by recursive fast matrix multiplication: `rules` is one built-in rule name (or
    Rule) per level, root first; `scaling` None / 'outside' / 'inside' / 'out_in' /
    'in_out' / 'repeated' or a dict (fmm_scaling fields), FP64 only.  Plans are cached per
    (rules, dims, dtype, leaf, scaling, device).  A, B: row-major CUDA tensors (float64 or
    float32; FP32 defaults to the 3xTF32 tensor-core leaf)."""
    import torch
    if A.dtype != B.dtype or A.dtype not in (torch.float64, torch.float32):
        raise ValueError("A and B must both be float64 or float32")
    dtype = "f64" if A.dtype == torch.float64 else "f32"
    if leaf is None:
        leaf = LEAF_NATIVE if dtype == "f64" else LEAF_3XTF32
    M, K = A.shape
    N = B.shape[1]
    rl = tuple(r if isinstance(r, Rule) else Rule.builtin(r) for r in rules)
    sc = scaling if (scaling is None or isinstance(scaling, dict)) else {"mode": scaling, "pow2": 1}
    key = (tuple(r.name for r in rl), M, K, N, dtype, leaf,
           tuple(sorted(sc.items())) if sc else None, A.device.index)
    plan = _PLAN_CACHE.get(key)
    if plan is None:
        plan = Plan(list(rl), M, K, N, dtype=dtype, leaf=leaf, scaling=sc)
        _PLAN_CACHE[key] = plan
    return plan.execute(A, B, C_out=C_out, stream=stream)


def node_st(rule: Rule, A, B, stream=None):
    """All S_r, T_r of one node (R x mb x kb, R x kb x nb)."""
    import torch
    info = rule.info()
    m, k = A.shape
    n = B.shape[1]
    S = torch.empty((info["R"], m // info["m0"], k // info["k0"]), dtype=A.dtype, device=A.device)
    T = torch.empty((info["R"], k // info["k0"], n // info["n0"]), dtype=A.dtype, device=A.device)
    a, lda = _mat(A, "A")
    b, ldb = _mat(B, "B")
    _call("fmm_node_st", rule._h, _dtype_code(A), m, k, n, a, lda, b, ldb,
          C.c_void_p(S.data_ptr()), C.c_void_p(T.data_ptr()), _stream(stream))
    return S, T


def node_c(rule: Rule, Ms, stream=None):
    """C = sum_r w_kr M_r of one node from R contiguous blocks."""
    import torch
    info = rule.info()
    R, mb, nb = Ms.shape
    Cm = torch.empty((mb * info["m0"], nb * info["n0"]), dtype=Ms.dtype, device=Ms.device)
    Ms = Ms.contiguous()
    _call("fmm_node_c", rule._h, _dtype_code(Ms), Cm.shape[0], Cm.shape[1],
          C.c_void_p(Ms.data_ptr()), C.c_void_p(Cm.data_ptr()), Cm.shape[1], _stream(stream))
    return Cm


def scale_outside(A, B, pow2=False, stream=None):
    """Alg. 1 lines 1-4: returns (A', B', dA, dB)."""
    import torch
    M, K = A.shape
    N = B.shape[1]
    Ao, Bo = torch.empty_like(A), torch.empty_like(B)
    dA = torch.empty(M, dtype=torch.float64, device=A.device)
    dB = torch.empty(N, dtype=torch.float64, device=A.device)
    a, lda = _mat(A, "A")
    b, ldb = _mat(B, "B")
    _call("fmm_scale_outside", F64, M, K, N, a, lda, b, ldb, C.c_void_p(Ao.data_ptr()), K,
          C.c_void_p(Bo.data_ptr()), N, C.c_void_p(dA.data_ptr()), C.c_void_p(dB.data_ptr()),
          int(pow2), _stream(stream))
    return Ao, Bo, dA, dB


def scale_inside(A, B, pow2=False, stream=None):
    """Alg. 2 lines 1-3: returns (A', B', d)."""
    import torch
    M, K = A.shape
    N = B.shape[1]
    Ao, Bo = torch.empty_like(A), torch.empty_like(B)
    d = torch.empty(K, dtype=torch.float64, device=A.device)
    a, lda = _mat(A, "A")
    b, ldb = _mat(B, "B")
    _call("fmm_scale_inside", F64, M, K, N, a, lda, b, ldb, C.c_void_p(Ao.data_ptr()), K,
          C.c_void_p(Bo.data_ptr()), N, C.c_void_p(d.data_ptr()), int(pow2), _stream(stream))
    return Ao, Bo, d


def scale_repeated(A, B, first_O=True, tau=1.0, max_steps=20, pow2=False, stream=None):
    """Alg. 3: returns dict(A, B, dA, dB, dI, steps) (steps read back: synchronises)."""
    import torch
    M, K = A.shape
    N = B.shape[1]
    Ao, Bo = torch.empty_like(A), torch.empty_like(B)
    dev = A.device
    dA = torch.empty(M, dtype=torch.float64, device=dev)
    dB = torch.empty(N, dtype=torch.float64, device=dev)
    dI = torch.empty(K, dtype=torch.float64, device=dev)
    steps = torch.zeros(1, dtype=torch.int32, device=dev)
    nb = C.c_size_t()
    _call("fmm_scale_workspace_bytes", M, K, N, C.byref(nb))
    ws = torch.empty(nb.value, dtype=torch.uint8, device=dev)
    cfg = fmm_scaling(5, int(first_O), float(tau), int(max_steps), int(pow2))
    a, lda = _mat(A, "A")
    b, ldb = _mat(B, "B")
    _call("fmm_scale_repeated", F64, M, K, N, a, lda, b, ldb, C.byref(cfg),
          C.c_void_p(Ao.data_ptr()), K, C.c_void_p(Bo.data_ptr()), N, C.c_void_p(dA.data_ptr()),
          C.c_void_p(dB.data_ptr()), C.c_void_p(dI.data_ptr()), C.c_void_p(steps.data_ptr()),
          C.c_void_p(ws.data_ptr()), nb.value, _stream(stream))
    return dict(A=Ao, B=Bo, dA=dA, dB=dB, dI=dI, steps=int(steps.item()))


def scale_apply(A, B, dA, d, dB, stream=None):
    """A' = D_A^-1 A D, B' = D^-1 B D_B^-1 for given factor vectors (fmm_scale_apply)."""
    import torch
    M, K = A.shape
    N = B.shape[1]
    Ao, Bo = torch.empty_like(A), torch.empty_like(B)
    a, lda = _mat(A, "A")
    b, ldb = _mat(B, "B")
    _call("fmm_scale_apply", F64, M, K, N, a, lda, b, ldb, C.c_void_p(dA.data_ptr()),
          C.c_void_p(d.data_ptr()), C.c_void_p(dB.data_ptr()), C.c_void_p(Ao.data_ptr()), K,
          C.c_void_p(Bo.data_ptr()), N, _stream(stream))
    return Ao, Bo


def unscale(Cm, dA, dB, stream=None):
    """In place C <- D_A C D_B."""
    c, ldc = _mat(Cm, "C")
    _call("fmm_unscale", F64, Cm.shape[0], Cm.shape[1], c, ldc, C.c_void_p(dA.data_ptr()),
          C.c_void_p(dB.data_ptr()), _stream(stream))
    return Cm


def comm_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _call("fmm_comm_unique_id", buf)
    return buf.raw


def version() -> str:
    return lib().fmm_version().decode()
