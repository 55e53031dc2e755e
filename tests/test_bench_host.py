"""Host-side logic of bench.py (no GPU): which kernel a workload's line is attributed to, and the
algorithmic bytes its roofline uses."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
import synth  # noqa: E402


def _c5(sweeps=0):
    cfg = bench.workload_params("c5", sweeps)
    inst = {"kind": "csr", "w": np.zeros(4, np.float32)}
    return cfg, inst


def test_c5_kernel_attribution(monkeypatch):
    """C5 sweeps >= 4 per call on the packed rows unless ISING_I8_PACKED=0; a call of < 4 sweeps
    on the int8 rows unless ISING_I8_PACKED=1 (the library's rule, include/ising.h ising_sweep)."""
    cfg, inst = _c5()
    R = cfg["K"] * cfg["C"]
    monkeypatch.delenv("ISING_I8_PACKED", raising=False)
    assert bench.kernel_name(None, inst, cfg, cfg["K"], R, False) == "k_csr_packed"
    monkeypatch.setenv("ISING_I8_PACKED", "0")
    assert bench.kernel_name(None, inst, cfg, cfg["K"], R, False) == "k_csr_i8_ring"
    cfg3, _ = _c5(3)
    monkeypatch.delenv("ISING_I8_PACKED", raising=False)
    assert bench.kernel_name(None, inst, cfg3, cfg["K"], R, False) == "k_csr_i8_ring"
    monkeypatch.setenv("ISING_I8_PACKED", "1")
    assert bench.kernel_name(None, inst, cfg3, cfg["K"], R, False) == "k_csr_packed"
    # R not a multiple of 256: neither packed nor ring
    assert bench.kernel_name(None, inst, cfg, cfg["K"], 128, False) == "k_csr_i8_phase"


def test_packed_algorithmic_bytes():
    """196 bytes per 256 attempts: own row read + written (2 x 32), three neighbour rows (3 x 32),
    the table entry (4 columns + 4 weights + original id = 36) -- C5 is 3-regular."""
    cfg = synth.CONFIGS["c5"]
    assert cfg["K"] * cfg["C"] == 256
    own, nbr, table = 2 * 256 // 8, 3 * 256 // 8, 16 + 16 + 4
    assert own + nbr + table == 196
