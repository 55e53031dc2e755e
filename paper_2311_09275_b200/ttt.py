"""Time-to-target arithmetic of PAPER.md §II.B and the copies-as-trials harness (SURVEY §8(f)
NEXT-2).

Eq.(1)  r   = max(1.0, log(1 - 0.99) / log(1 - P_s))
Eq.(2)  TTT = t_trial * r
sweeps-to-target = sweeps per run * r
quality = solution value / best-known value
BLS projection (Appendix I footnote 4): total time = average time per success x
successes; time per run = total / runs; projected TTT = time per run x r(P_s).

The harness treats the C copies of a PT run as the trials ("Each batch of 100 trials",
P:59): every copy is an independent ladder with its own best-so-far (ising_copy_best); a trial
succeeds when its best cut reaches the target.  All copies run concurrently on the GPU, so the
batch time T is both the latency of one trial and, divided by the number of trials, the
amortised time per trial; TTT is reported for both.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np


def repetitions(p_s: float, confidence: float = 0.99) -> float:
    """Eq.(1): repetitions needed to reach the target with `confidence`."""
    if p_s <= 0.0:
        return math.inf
    if p_s >= 1.0:
        return 1.0
    return max(1.0, math.log(1.0 - confidence) / math.log(1.0 - p_s))


def time_to_target(t_trial: float, p_s: float, confidence: float = 0.99) -> float:
    """Eq.(2)."""
    return t_trial * repetitions(p_s, confidence)


def sweeps_to_target(sweeps_per_run: float, p_s: float, confidence: float = 0.99) -> float:
    """Sweeps per run multiplied by the number of runs from Eq.(1)."""
    return sweeps_per_run * repetitions(p_s, confidence)


def quality(value: float, best_known: float) -> float:
    return value / best_known


def speedup(ttt_ref: float, ttt_new: float) -> float:
    return ttt_ref / ttt_new


def bls_projection(avg_time_per_success: float, p_s: float, runs: int = 20):
    """Appendix I footnote 4: (projected time per run, projected TTT)."""
    successes = p_s * runs
    per_run = avg_time_per_success * successes / runs
    return per_run, time_to_target(per_run, p_s)


def round_sig(x: float, digits: int = 3) -> float:
    """Round to `digits` significant figures, halves away from zero (as printed tables do)."""
    from decimal import ROUND_HALF_UP, Decimal
    if x == 0 or not math.isfinite(x):
        return x
    e = int(math.floor(math.log10(abs(x)))) - digits + 1
    q = Decimal(1).scaleb(e)
    return float(Decimal(repr(x)).quantize(q, rounding=ROUND_HALF_UP))


@dataclass
class TrialStats:
    trials: int
    successes: int
    target_cut: float
    sweeps_per_run: int
    batch_seconds: float
    best_cuts: np.ndarray = field(repr=False)
    p_s: float = 0.0
    r: float = math.inf
    sweeps_to_target: float = math.inf
    ttt_latency: float = math.inf
    ttt_amortised: float = math.inf

    def __post_init__(self):
        self.p_s = self.successes / self.trials
        self.r = repetitions(self.p_s)
        self.sweeps_to_target = self.sweeps_per_run * self.r
        self.ttt_latency = self.batch_seconds * self.r
        self.ttt_amortised = self.batch_seconds / self.trials * self.r


def trial_outcomes(best_E, W, target_cut):
    """Per-trial best cuts (W - E)/2 and successes (cut >= target)."""
    cuts = (W - np.asarray(best_E, dtype=np.float64)) / 2.0
    return cuts, int(np.count_nonzero(cuts >= target_cut))


def run_trials(engine, sweeps: int, k_ex: int, target_cut: float, W: float) -> TrialStats:
    """Run one batch (all copies of `engine` are trials) and compute P_s, r, STT and TTT."""
    from .driver import run_pt
    try:
        import torch
        sync = torch.cuda.synchronize if torch.cuda.is_available() else (lambda: None)
    except ImportError:  # pragma: no cover
        sync = lambda: None  # noqa: E731
    sync()
    t0 = time.perf_counter()
    run_pt(engine, sweeps, k_ex)
    E, _, _ = engine.copy_best()
    sync()
    dt = time.perf_counter() - t0
    cuts, ok = trial_outcomes(E, W, target_cut)
    return TrialStats(trials=len(cuts), successes=ok, target_cut=target_cut, sweeps_per_run=sweeps,
                      batch_seconds=dt, best_cuts=cuts)
