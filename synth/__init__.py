"""Seeded synthetic workloads shared by the oracle side and the CUDA side.

This package holds NO arithmetic of the method (no permutation expansion, no
multiplicity coefficients, no MTTKRP).  It only draws canonical-triangle COO
tensors and dense factor matrices with the shapes of BASELINE.json's configs.
"""
from .workloads import (CONFIGS, Workload, generate, key_bits, scramble,
                        integer_workload, small_random)

__all__ = ["CONFIGS", "Workload", "generate", "key_bits", "scramble",
           "integer_workload", "small_random"]
