"""ORACLE — TEST INFRASTRUCTURE ONLY.

Plain CPU references for symmetric sparse MTTKRP (SySTeC, arXiv 2406.09266).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` leg may import this package.  It shares
no code with the CUDA path (``paper_2406_09266_b200``) and never imports it.

* :func:`mttkrp` / :func:`mttkrp_rows` — the expansion oracle (plain C,
  ``mttkrp_oracle.c``): every stored canonical entry is expanded to its
  distinct permutations and the naive non-symmetric MTTKRP runs in fp64
  (north_star; PAPER.md:859-865 for the MTTKRP definition
  for "as many assignments as unique permutations").  Also returns S, the sum
  of absolute terms used to normalise the parity error.
* :func:`mttkrp_general` — the naive kernel on a general (non-symmetric) COO
  tensor, for the non-symmetric GPU baseline.
* :func:`minplus_sym2` — one Bellman-Ford (min, +) relaxation over a
  symmetric matrix.
* :func:`ttm_sym3` — naive TTM over the expanded order-3 tensor (NEXT-4).
* :mod:`oracle.symmetric_ref` — the per-position multiplicity-coefficient
  formula, written independently in fp64 numpy (pin P4 of SURVEY.md §8(c)).

Pins: see tests/test_oracle_pins.py (P1-P10).  No function here is "parity
unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mttkrp_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile the plain-C oracle with gcc (no GPU code involved)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-pthread",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _bind(lib):
    i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
    lib.oracle_mttkrp.argtypes = [i32, i64, i64, vp, vp, vp, i32, vp, vp, i32, i64]
    lib.oracle_mttkrp.restype = i32
    lib.oracle_count_expanded.argtypes = [i32, i64, vp]
    lib.oracle_count_expanded.restype = i64
    return lib


def load_variant(path: str):
    """A separately compiled oracle (the mutation tests build deliberately
    broken variants with -DORACLE_MUTATION=k to show the pins catch them)."""
    return _bind(ctypes.CDLL(path))


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        i64, i32, vp = ctypes.c_int64, ctypes.c_int, ctypes.c_void_p
        lib.oracle_mttkrp.argtypes = [i32, i64, i64, vp, vp, vp, i32, vp, vp, i32, i64]
        lib.oracle_mttkrp.restype = i32
        lib.oracle_mttkrp_rows.argtypes = [i32, i64, i64, vp, vp, vp, i32, i64, vp, vp, vp, i32]
        lib.oracle_mttkrp_rows.restype = i32
        lib.oracle_mttkrp_general.argtypes = [i32, i64, i64, vp, vp, vp, i32, vp, vp]
        lib.oracle_mttkrp_general.restype = i32
        lib.oracle_minplus_sym2.argtypes = [i64, i64, vp, vp, vp, vp]
        lib.oracle_minplus_sym2.restype = i32
        lib.oracle_ttm_sym3.argtypes = [i64, i64, vp, vp, vp, i32, vp]
        lib.oracle_ttm_sym3.restype = i32
        lib.oracle_count_expanded.argtypes = [i32, i64, vp]
        lib.oracle_count_expanded.restype = i64
        lib.oracle_mttkrp_symmetric.argtypes = [i32, i64, i64, vp, vp, vp, i32, vp]
        lib.oracle_mttkrp_symmetric.restype = i32
        _lib = lib
    return _lib


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _prep(order, idx, vals, B):
    idx = np.ascontiguousarray(idx, dtype=np.int32).reshape(-1, order)
    vals = np.ascontiguousarray(vals, dtype=np.float32).reshape(-1)
    B = np.ascontiguousarray(B, dtype=np.float32)
    if vals.shape[0] != idx.shape[0]:
        raise ValueError("idx and vals disagree on nnz")
    if B.ndim != 2:
        raise ValueError("B must be [dim][R]")
    return idx, vals, B


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def mttkrp(order: int, dim: int, idx, vals, B, threads: int | None = None,
           mem_budget_bytes: int = 0, lib=None):
    """Expansion oracle.  Returns (C, S), fp64 [dim][R]."""
    idx, vals, B = _prep(order, idx, vals, B)
    if B.shape[0] != dim:
        raise ValueError("B must have dim rows")
    R = B.shape[1]
    C = np.empty((dim, R), np.float64)
    S = np.empty((dim, R), np.float64)
    T = threads if threads else default_threads()
    rc = (lib or _load()).oracle_mttkrp(order, dim, idx.shape[0], _ptr(idx), _ptr(vals), _ptr(B), R,
                                        _ptr(C), _ptr(S), T, mem_budget_bytes)
    if rc == 3:
        raise IndexError("index outside [0, dim)")
    if rc != 0:
        raise RuntimeError(f"oracle_mttkrp failed with status {rc}")
    return C, S


def mttkrp_symmetric(order: int, dim: int, idx, vals, B):
    """The symmetric method (coefficient per run-first position) in plain C,
    one thread, fp64: pin P4 against the expansion and the one-core CPU
    analogue of the paper's experiment.  Returns C, fp64 [dim][R]."""
    idx, vals, B = _prep(order, idx, vals, B)
    if B.shape[0] != dim:
        raise ValueError("B must have dim rows")
    C = np.empty((dim, B.shape[1]), np.float64)
    rc = _load().oracle_mttkrp_symmetric(order, dim, idx.shape[0], _ptr(idx), _ptr(vals), _ptr(B), B.shape[1],
                                         _ptr(C))
    if rc == 3:
        raise IndexError("index outside [0, dim)")
    if rc != 0:
        raise RuntimeError(f"oracle_mttkrp_symmetric failed with status {rc}")
    return C


def mttkrp_rows(order: int, dim: int, idx, vals, B, rows, threads: int | None = None):
    """Expansion oracle restricted to output rows ``rows``: (C, S) [len(rows)][R]."""
    idx, vals, B = _prep(order, idx, vals, B)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    R = B.shape[1]
    C = np.empty((rows.shape[0], R), np.float64)
    S = np.empty((rows.shape[0], R), np.float64)
    T = threads if threads else default_threads()
    rc = _load().oracle_mttkrp_rows(order, dim, idx.shape[0], _ptr(idx), _ptr(vals), _ptr(B), R,
                                    rows.shape[0], _ptr(rows), _ptr(C), _ptr(S), T)
    if rc == 3:
        raise IndexError("index outside [0, dim)")
    if rc != 0:
        raise RuntimeError(f"oracle_mttkrp_rows failed with status {rc}")
    return C, S


def mttkrp_general(order: int, dim: int, idx, vals, B):
    """Naive non-symmetric MTTKRP on a general COO tensor (tuples as given):
    C[idx_e[0], r] += v_e prod_{t>=1} B[idx_e[t], r].  Returns (C, S) fp64."""
    idx, vals, B = _prep(order, idx, vals, B)
    R = B.shape[1]
    C = np.empty((dim, R), np.float64)
    S = np.empty((dim, R), np.float64)
    rc = _load().oracle_mttkrp_general(order, dim, idx.shape[0], _ptr(idx), _ptr(vals), _ptr(B), R,
                                       _ptr(C), _ptr(S))
    if rc == 3:
        raise IndexError("index outside [0, dim)")
    if rc != 0:
        raise RuntimeError(f"oracle_mttkrp_general failed with status {rc}")
    return C, S


def minplus_sym2(dim: int, idx, vals, d):
    """One (min,+) relaxation over a symmetric matrix given by its stored
    entries (either orientation): y = min(d, min_j A[i,j] + d[j]), fp32 adds."""
    idx = np.ascontiguousarray(idx, dtype=np.int32).reshape(-1, 2)
    vals = np.ascontiguousarray(vals, dtype=np.float32)
    d = np.ascontiguousarray(d, dtype=np.float32)
    y = np.empty(dim, np.float32)
    rc = _load().oracle_minplus_sym2(dim, idx.shape[0], _ptr(idx), _ptr(vals), _ptr(d), _ptr(y))
    if rc == 3:
        raise IndexError("index outside [0, dim)")
    if rc != 0:
        raise RuntimeError(f"oracle_minplus_sym2 failed with status {rc}")
    return y


def ttm_sym3(dim: int, idx, vals, B):
    """Naive TTM over the expanded order-3 tensor: full C [dim][dim][R] fp64
    with C[j][l][r] = sum_k A[k,j,l] B[k,r]."""
    idx, vals, B = _prep(3, idx, vals, B)
    R = B.shape[1]
    C = np.empty((dim, dim, R), np.float64)
    rc = _load().oracle_ttm_sym3(dim, idx.shape[0], _ptr(idx), _ptr(vals), _ptr(B), R, _ptr(C))
    if rc == 3:
        raise IndexError("index outside [0, dim)")
    if rc != 0:
        raise RuntimeError(f"oracle_ttm_sym3 failed with status {rc}")
    return C


def count_expanded(order: int, idx, lib=None) -> int:
    """Σ over entries of the number of distinct permutations (expanded nnz)."""
    idx = np.ascontiguousarray(idx, dtype=np.int32).reshape(-1, order)
    return int((lib or _load()).oracle_count_expanded(order, idx.shape[0], _ptr(idx)))
