"""B200-native symmetric sparse MTTKRP — the hot path of SySTeC (arXiv 2406.09266).

The computation lives in ``libsystec.so`` (hand-written sm_100a CUDA behind the
C ABI of ``include/systec.h``); this package is the thin ctypes binding with
the same names.  See DESIGN.md.
"""
from .systec import (EXPORTS, LIB_PATH, Plan, SystecError, expand_symmetric, load, mttkrp, mttkrp_host,
                     plan_create, plan_create_general, testing_cpd_pass)

__all__ = ["EXPORTS", "LIB_PATH", "Plan", "SystecError", "expand_symmetric", "load", "mttkrp", "mttkrp_host",
           "plan_create", "plan_create_general", "testing_cpd_pass"]
