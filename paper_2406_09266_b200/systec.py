"""Thin ctypes binding of libsystec (include/systec.h).  Argument marshalling
only: every step of the computation runs in the library's CUDA kernels.
PyTorch provides device memory and streams.  There is no CPU fallback: if the
shared library is missing or cannot be loaded this module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libsystec.so")

OK, ERR_ARG, ERR_UNSUPPORTED, ERR_INDEX, ERR_ALIAS, ERR_NOMEM, ERR_CUDA = range(7)
_ERRORS = {ERR_ARG: ValueError, ERR_UNSUPPORTED: NotImplementedError, ERR_INDEX: IndexError,
           ERR_ALIAS: ValueError, ERR_NOMEM: MemoryError, ERR_CUDA: RuntimeError}


class SystecStats(ctypes.Structure):
    _fields_ = [("nnz", ctypes.c_int64), ("dim", ctypes.c_int64), ("order", ctypes.c_int32),
                ("key_bits", ctypes.c_int32), ("G", ctypes.c_int64), ("expanded", ctypes.c_int64),
                ("pattern_hist", ctypes.c_int64 * 16), ("lead_runs", ctypes.c_int64),
                ("max_lead_run", ctypes.c_int64), ("pos1_runs", ctypes.c_int64),
                ("input_was_sorted", ctypes.c_int32), ("band_shift", ctypes.c_int32),
                ("bad_entry", ctypes.c_int64), ("bandwidth", ctypes.c_int64), ("window_blocks", ctypes.c_int64)]


class SystecExecOpts(ctypes.Structure):
    _fields_ = [("warps_per_block", ctypes.c_int32), ("blocks_per_sm", ctypes.c_int32),
                ("pos1_accumulate", ctypes.c_int32), ("force_scalar", ctypes.c_int32),
                ("no_zero", ctypes.c_int32), ("l2_hints", ctypes.c_int32),
                ("chunk_k", ctypes.c_int32), ("stages", ctypes.c_int32), ("vpl", ctypes.c_int32),
                ("prefetch", ctypes.c_int32), ("copies", ctypes.c_int32), ("ablation", ctypes.c_int32),
                ("static_ranges", ctypes.c_int32), ("occupancy", ctypes.c_int32), ("fixed_rank", ctypes.c_int32),
                ("window", ctypes.c_int32), ("lane_bytes", ctypes.c_int32)]


class SystecPlanOpts(ctypes.Structure):
    _fields_ = [("band_shift", ctypes.c_int32), ("general", ctypes.c_int32), ("window", ctypes.c_int32),
                ("reserved", ctypes.c_int32 * 5)]


EXPORTS = ["systec_mttkrp", "systec_mttkrp_host", "systec_plan_create", "systec_plan_execute",
           "systec_plan_execute_ex", "systec_plan_stats", "systec_plan_prepared",
           "systec_plan_copy_prepared", "systec_plan_last_launch", "systec_plan_destroy",
           "systec_status_string", "systec_last_cuda_error", "systec_version", "systec_last_bad_entry",
           "systec_plan_create_general", "systec_expand_symmetric", "systec_plan_minplus",
           "systec_cp_als_sym", "systec_plan_ttm", "systec_ttm_unpack", "systec_plan_sssp",
           "systec_plan_create_ex", "systec_testing_cpd_pass"]

_lib = None


def load(path: str | None = None):
    """Load libsystec.so (fails loudly when it is missing)."""
    global _lib
    if _lib is not None:
        return _lib
    p = path or os.environ.get("SYSTEC_LIB") or LIB_PATH   # SYSTEC_LIB: experiment builds
    if not os.path.exists(p):
        raise ImportError(f"libsystec.so not built at {p}; run __graft_entry__.build() "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(p)
    i32, i64, vp = ctypes.c_int, ctypes.c_int64, ctypes.c_void_p
    lib.systec_mttkrp.argtypes = [i32, i64, i64, vp, vp, vp, i32, vp, vp]
    lib.systec_mttkrp_host.argtypes = [i32, i64, i64, vp, vp, vp, i32, vp, vp]
    lib.systec_plan_create.argtypes = [ctypes.POINTER(vp), i32, i64, i64, vp, vp, vp]
    lib.systec_plan_execute.argtypes = [vp, vp, i32, vp, vp]
    lib.systec_plan_create_ex.argtypes = [ctypes.POINTER(vp), i32, i64, i64, vp, vp, ctypes.POINTER(SystecPlanOpts), vp]
    lib.systec_plan_create_general.argtypes = [ctypes.POINTER(vp), i32, i64, i64, vp, vp, vp]
    lib.systec_plan_minplus.argtypes = [vp, vp, vp, vp]
    lib.systec_plan_ttm.argtypes = [vp, vp, i32, vp, vp]
    lib.systec_plan_sssp.argtypes = [vp, i64, vp, i32, ctypes.POINTER(i32), vp]
    lib.systec_ttm_unpack.argtypes = [i64, i32, vp, vp, vp]
    lib.systec_cp_als_sym.argtypes = [vp, vp, i32, vp, i32, ctypes.c_double, vp, ctypes.POINTER(i32), vp]
    lib.systec_testing_cpd_pass.argtypes = [i32, i64, vp, vp, vp, vp, i32, vp]
    lib.systec_expand_symmetric.argtypes = [i32, i64, i64, vp, vp, i64, vp, vp, ctypes.POINTER(i64), vp]
    lib.systec_plan_execute_ex.argtypes = [vp, vp, i32, vp, ctypes.POINTER(SystecExecOpts), vp]
    lib.systec_plan_stats.argtypes = [vp, ctypes.POINTER(SystecStats)]
    lib.systec_plan_prepared.argtypes = [vp, ctypes.POINTER(vp), ctypes.POINTER(vp)]
    lib.systec_plan_copy_prepared.argtypes = [vp, vp, vp, vp]
    lib.systec_plan_last_launch.argtypes = [vp] + [ctypes.POINTER(ctypes.c_int32)] * 5
    lib.systec_plan_destroy.argtypes = [vp]
    lib.systec_status_string.argtypes = [i32]
    lib.systec_status_string.restype = ctypes.c_char_p
    lib.systec_last_cuda_error.argtypes = []
    lib.systec_version.argtypes = []
    lib.systec_last_bad_entry.argtypes = []
    lib.systec_last_bad_entry.restype = i64
    for name in EXPORTS:
        if name not in ("systec_status_string", "systec_last_bad_entry"):
            getattr(lib, name).restype = i32
    _lib = lib
    return lib


class SystecError(RuntimeError):
    pass


def _check(rc: int, what: str):
    if rc == OK:
        return
    lib = load()
    msg = f"{what}: {lib.systec_status_string(rc).decode()}"
    if rc == ERR_CUDA:
        msg += f" (cudaError {lib.systec_last_cuda_error()})"
    if rc == ERR_INDEX:
        msg += f" (first bad entry {lib.systec_last_bad_entry()})"
    raise _ERRORS.get(rc, SystecError)(msg)


def _stream_handle(stream):
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def _dev(t, dtype, name):
    import torch
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return ctypes.c_void_p(t.data_ptr() if t.numel() else 0)


def _opts(**kw) -> SystecExecOpts:
    o = SystecExecOpts()
    alias = {"K": "chunk_k"}
    names = {f for f, _ in SystecExecOpts._fields_}
    for k, v in kw.items():
        k = alias.get(k, k)
        if k not in names or k == "reserved":
            raise TypeError(f"unknown execute option {k!r}")
        setattr(o, k, int(v))
    return o


class Plan:
    """A prepared (validated, canonicalised, sorted) symmetric tensor on the GPU:
    ``systec_plan_create``.  ``idx`` [nnz][order] int32 and ``vals`` [nnz] fp32
    are CUDA tensors; they may be freed after construction.  ``window``
    (order 2): also build the atomic-free windowed kernel's pointers.  ``band_shift``
    (``systec_plan_create_ex``): None/0 = auto, -1 = lexicographic stream,
    s > 0 = band-major by c_{n-1} >> s."""

    def __init__(self, order: int, dim: int, idx, vals, stream=None, general: bool = False,
                 band_shift: int | None = None, window: bool = False):
        import torch
        lib = load()
        nnz = int(vals.shape[0])
        if idx.dim() != 2 or idx.shape[1] != order or idx.shape[0] != nnz:
            raise ValueError("idx must be [nnz][order]")
        h = ctypes.c_void_p()
        ip, vp_ = _dev(idx, torch.int32, "idx"), _dev(vals, torch.float32, "vals")
        if band_shift is not None or window:
            po = SystecPlanOpts(band_shift=band_shift or 0, general=int(general), window=int(window))
            _check(lib.systec_plan_create_ex(ctypes.byref(h), order, dim, nnz, ip, vp_, ctypes.byref(po),
                                             _stream_handle(stream)), "systec_plan_create_ex")
        else:
            fn, name = ((lib.systec_plan_create_general, "systec_plan_create_general") if general
                        else (lib.systec_plan_create, "systec_plan_create"))
            _check(fn(ctypes.byref(h), order, dim, nnz, ip, vp_, _stream_handle(stream)), name)
        self.general = general
        self._h = h
        self.order, self.dim, self.nnz = order, dim, nnz

    def execute(self, B, C=None, stream=None, **opts):
        """``systec_plan_execute(_ex)``: returns C [dim][R] fp32 (overwritten)."""
        import torch
        lib = load()
        if B.dim() != 2 or B.shape[0] != self.dim:
            raise ValueError("B must be [dim][R]")
        R = int(B.shape[1])
        if C is None:
            C = torch.empty((self.dim, R), dtype=torch.float32, device=B.device)
        if tuple(C.shape) != (self.dim, R):
            raise ValueError("C must be [dim][R]")
        bp, cp = _dev(B, torch.float32, "B"), _dev(C, torch.float32, "C")
        s = _stream_handle(stream)
        if opts:
            o = _opts(**opts)
            _check(lib.systec_plan_execute_ex(self._h, bp, R, cp, ctypes.byref(o), s), "systec_plan_execute_ex")
        else:
            _check(lib.systec_plan_execute(self._h, bp, R, cp, s), "systec_plan_execute")
        return C

    def minplus(self, d, y=None, stream=None):
        """``systec_plan_minplus`` (order-2 plans): y[i] = min(d[i], min_j A[i,j] + d[j])."""
        import torch
        if d.dim() != 1 or d.shape[0] != self.dim:
            raise ValueError("d must be [dim]")
        if y is None:
            y = torch.empty_like(d)
        _check(load().systec_plan_minplus(self._h, _dev(d, torch.float32, "d"), _dev(y, torch.float32, "y"),
                                          _stream_handle(stream)), "systec_plan_minplus")
        return y

    def cp_als(self, B, max_iters: int = 50, tol: float = 1e-7, stream=None):
        """``systec_cp_als_sym``: symmetric CP-ALS from the initial factor B (CUDA
        tensor [dim][R], updated in place).  Returns (B, lambda, fits)."""
        import torch
        if B.dim() != 2 or B.shape[0] != self.dim:
            raise ValueError("B must be [dim][R]")
        R = int(B.shape[1])
        lam = torch.empty(R, dtype=torch.float32, device=B.device)
        fits = np.zeros(max(max_iters, 1), np.float64)
        done = ctypes.c_int()
        _check(load().systec_cp_als_sym(self._h, _dev(B, torch.float32, "B"), R, _dev(lam, torch.float32, "lambda"),
                                        max_iters, tol, fits.ctypes.data_as(ctypes.c_void_p), ctypes.byref(done),
                                        _stream_handle(stream)), "systec_cp_als_sym")
        return B, lam, fits[:done.value]

    def sssp(self, source: int, max_iters: int | None = None, stream=None):
        """``systec_plan_sssp`` (order-2 plans): Bellman-Ford distances from
        ``source``; returns (dist CUDA tensor [dim], relaxations done)."""
        import torch
        dist = torch.empty(self.dim, dtype=torch.float32, device="cuda")
        done = ctypes.c_int()
        it = self.dim if max_iters is None else max_iters
        _check(load().systec_plan_sssp(self._h, source, ctypes.c_void_p(dist.data_ptr()), it, ctypes.byref(done),
                                       _stream_handle(stream)), "systec_plan_sssp")
        return dist, done.value

    def ttm(self, B, packed=None, full: bool = False, stream=None):
        """``systec_plan_ttm`` (order-3 plans): packed canonical half
        [dim(dim+1)/2][R]; with full=True also ``systec_ttm_unpack`` -> [dim][dim][R]."""
        import torch
        R = int(B.shape[1])
        rows = self.dim * self.dim if getattr(self, "general", False) else self.dim * (self.dim + 1) // 2
        if packed is None:
            packed = torch.empty((rows, R), dtype=torch.float32, device=B.device)
        s = _stream_handle(stream)
        _check(load().systec_plan_ttm(self._h, _dev(B, torch.float32, "B"), R, _dev(packed, torch.float32, "C"), s),
               "systec_plan_ttm")
        if not full or getattr(self, "general", False):
            return packed
        Cf = torch.empty((self.dim, self.dim, R), dtype=torch.float32, device=B.device)
        _check(load().systec_ttm_unpack(self.dim, R, ctypes.c_void_p(packed.data_ptr()),
                                        ctypes.c_void_p(Cf.data_ptr()), s), "systec_ttm_unpack")
        return Cf

    def stats(self) -> dict:
        st = SystecStats()
        _check(load().systec_plan_stats(self._h, ctypes.byref(st)), "systec_plan_stats")
        d = {k: getattr(st, k) for k, _ in SystecStats._fields_}
        d["pattern_hist"] = list(st.pattern_hist)
        return d

    def prepared(self):
        """Copy of the prepared stream: (coords [order][nnz] int32, vals [nnz] fp32) CUDA tensors."""
        import torch
        coords = torch.empty((self.order, self.nnz), dtype=torch.int32, device="cuda")
        vals = torch.empty(self.nnz, dtype=torch.float32, device="cuda")
        if self.nnz:
            _check(load().systec_plan_copy_prepared(self._h, ctypes.c_void_p(coords.data_ptr()),
                                                    ctypes.c_void_p(vals.data_ptr()), _stream_handle(None)),
                   "systec_plan_copy_prepared")
        return coords, vals

    def last_launch(self) -> dict:
        vals = [ctypes.c_int32() for _ in range(5)]
        _check(load().systec_plan_last_launch(self._h, *[ctypes.byref(v) for v in vals]), "systec_plan_last_launch")
        d = dict(zip(["grid_x", "grid_y", "block", "smem_bytes", "kernel_id"], [v.value for v in vals]))
        kid = d["kernel_id"]
        if kid >= 0:   # decimal fields: general | copies (2) | pf + 2 dynamic + 4 fixed-rank | order | vw | lpe (2) | vpl | pos1
            d.update(general=kid // 1000000000, copies=kid // 10000000 % 100, prefetch=kid // 1000000 % 2,
                     dynamic=kid // 1000000 % 10 // 2 % 2, fixed_rank=kid // 1000000 % 10 // 4,
                     order=kid // 100000 % 10,
                     vw=kid // 10000 % 10, lpe=kid // 100 % 100, vpl=kid // 10 % 10, pos1=kid % 10)
        return d

    def destroy(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            load().systec_plan_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass


def plan_create(order, dim, idx, vals, stream=None) -> Plan:
    return Plan(order, dim, idx, vals, stream)


def plan_create_general(order, dim, idx, vals, stream=None) -> Plan:
    """``systec_plan_create_general``: the non-symmetric baseline plan."""
    return Plan(order, dim, idx, vals, stream, general=True)


def expand_symmetric(order: int, dim: int, idx, vals, stream=None):
    """``systec_expand_symmetric``: (idx_exp [m][order] int32, vals_exp [m] fp32) CUDA tensors."""
    import torch
    lib = load()
    nnz = int(vals.shape[0])
    cnt = ctypes.c_int64()
    ip, vp_ = _dev(idx, torch.int32, "idx"), _dev(vals, torch.float32, "vals")
    s = _stream_handle(stream)
    _check(lib.systec_expand_symmetric(order, dim, nnz, ip, vp_, 0, None, None, ctypes.byref(cnt), s),
           "systec_expand_symmetric")
    m = cnt.value
    out_i = torch.empty((m, order), dtype=torch.int32, device=idx.device)
    out_v = torch.empty(m, dtype=torch.float32, device=idx.device)
    if m:
        _check(lib.systec_expand_symmetric(order, dim, nnz, ip, vp_, m, ctypes.c_void_p(out_i.data_ptr()),
                                           ctypes.c_void_p(out_v.data_ptr()), ctypes.byref(cnt), s),
               "systec_expand_symmetric")
    return out_i, out_v


def mttkrp(order: int, dim: int, idx, vals, B, C=None, stream=None):
    """One-shot ``systec_mttkrp`` on CUDA tensors; returns C [dim][R] (overwritten)."""
    import torch
    lib = load()
    nnz = int(vals.shape[0])
    if idx.dim() != 2 or idx.shape[1] != order or idx.shape[0] != nnz:
        raise ValueError("idx must be [nnz][order]")
    R = int(B.shape[1])
    if C is None:
        C = torch.empty((dim, R), dtype=torch.float32, device=B.device)
    _check(lib.systec_mttkrp(order, dim, nnz, _dev(idx, torch.int32, "idx"), _dev(vals, torch.float32, "vals"),
                             _dev(B, torch.float32, "B"), R, _dev(C, torch.float32, "C"), _stream_handle(stream)),
           "systec_mttkrp")
    return C


def mttkrp_host(order: int, dim: int, idx, vals, B, C=None, stream=None):
    """``systec_mttkrp_host`` on host arrays (numpy or pinned CPU tensors); returns C."""
    lib = load()

    import torch

    def host_ptr(a, dtype, name, shape):
        if hasattr(a, "data_ptr"):          # torch CPU tensor (possibly pinned): used in place, so it must
            tdt = torch.int32 if dtype == np.int32 else torch.float32    # already be what the ABI reads
            if a.is_cuda or not a.is_contiguous():
                raise TypeError(f"{name} must be a contiguous host tensor")
            if a.dtype != tdt:
                raise TypeError(f"{name} must be {tdt}, got {a.dtype}")
            if tuple(a.shape) != shape:
                raise TypeError(f"{name} must have shape {shape}, got {tuple(a.shape)}")
            return ctypes.c_void_p(a.data_ptr() if a.numel() else 0), a
        arr = np.ascontiguousarray(a, dtype=dtype)
        if arr.size != int(np.prod(shape)):
            raise ValueError(f"{name} must have shape {shape}, got {arr.shape}")
        return ctypes.c_void_p(arr.ctypes.data if arr.size else 0), arr

    nnz = int(vals.shape[0])
    R = int(B.shape[1])
    if C is None:
        C = np.empty((dim, R), np.float32)
    ip, _i = host_ptr(idx, np.int32, "idx", (nnz, order))
    vp_, _v = host_ptr(vals, np.float32, "vals", (nnz,))
    bp, _b = host_ptr(B, np.float32, "B", (dim, R))
    cp, _c = host_ptr(C, np.float32, "C", (dim, R))
    if not hasattr(C, "data_ptr") and _c is not C:
        raise ValueError("C must be a contiguous float32 array")
    _check(lib.systec_mttkrp_host(order, dim, nnz, ip, vp_, bp, R, cp, _stream_handle(stream)),
           "systec_mttkrp_host")
    return C


def testing_cpd_pass(form: int, M, F, W, store: bool = True, stream=None):
    """``systec_testing_cpd_pass``: one R = 32 CP-ALS dense pass in kernel form
    ``form`` (0 mma.sync, 1 tcgen05).  Returns (G [32][32] = M^T M, dots [32]
    = sum_i M o F) as fp64 CUDA tensors summed over the blocks; F is
    overwritten with M W when ``store``."""
    import torch
    if M.dim() != 2 or M.shape[1] != 32 or F.shape != M.shape or tuple(W.shape) != (32, 32):
        raise ValueError("M, F must be [dim][32] and W [32][32]")
    part = torch.zeros((1024, 32 * 32 + 32), dtype=torch.float64, device=M.device)
    rc = load().systec_testing_cpd_pass(form, int(M.shape[0]), _dev(M, torch.float32, "M"), _dev(F, torch.float32, "F"),
                                        _dev(W, torch.float32, "W"), _dev(part, torch.float64, "part"), int(store),
                                        _stream_handle(stream))
    if rc < 0:
        _check(-rc, "systec_testing_cpd_pass")
    tot = part[:rc].sum(dim=0)
    return tot[:1024].reshape(32, 32), tot[1024:]
