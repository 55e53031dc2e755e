"""B200-native (sm_100a) engine for the hot path of arXiv 2311.09275:
replica-parallel Metropolis sweeps with parallel tempering over sparse Ising couplings.

The compute path is libising.so (hand-written CUDA, C ABI in include/ising.h);
`ising` is its thin ctypes binding and `driver` the run schedule (Engine, run_pt).
"""
from . import ising  # noqa: F401
from .driver import Engine, run_pt, shard  # noqa: F401

__all__ = ["ising", "Engine", "run_pt", "shard"]
