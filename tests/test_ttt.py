"""Pins of the Eq.(1)/(2) arithmetic against the values PAPER.md prints (Tables I, II, IV)."""
import math
import os

import numpy as np
import pytest

from paper_2311_09275_b200 import ttt

GOLD = os.path.join(os.path.dirname(__file__), "golden", "paper_tables_ttt.txt")


def table(name):
    rows, cur = [], None
    for line in open(GOLD):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        if line.startswith("["):
            cur = line.strip("[]")
            continue
        if cur == name:
            rows.append(line.split())
    return rows


def test_eq1_special_values():
    assert ttt.repetitions(0.99) == 1.0          # max(1, 1) ("required here to be at least 1.0")
    assert ttt.repetitions(1.0) == 1.0
    assert ttt.repetitions(0.0) == math.inf
    assert abs(ttt.repetitions(0.10) - 43.709) < 1e-3
    assert abs(ttt.repetitions(0.05) - 89.781) < 1e-3


def test_table1_sweeps_to_target_and_speedup():
    rows = table("table1")
    assert len(rows) == 7
    for name, sbm, spr, ps, stt, cosm, spd in rows:
        got = ttt.sweeps_to_target(float(spr), float(ps))
        assert ttt.round_sig(got, 3) == float(stt), (name, got)
        assert ttt.round_sig(ttt.speedup(float(sbm), float(cosm)), 3) == float(spd), name


def test_table2_sweeps_to_target():
    for name, spr, ps, stt in table("table2"):
        got = ttt.sweeps_to_target(float(spr), float(ps))
        assert ttt.round_sig(got, 3) == float(stt), (name, got)


def test_table4_bls_projection():
    for name, avg, ps, per_run, proj, cosm, spd in table("table4"):
        pr, tt = ttt.bls_projection(float(avg), float(ps))
        assert abs(pr - float(per_run)) < 1e-6, name
        assert round(tt) == int(proj), (name, tt)
        # the printed speedup divides the printed (rounded) projected TTT
        assert ttt.round_sig(ttt.speedup(float(proj), float(cosm)), 3) == float(spd), name


def test_trial_outcomes_and_stats():
    W = 10.0
    E = np.array([-10, -8, -6, -10])   # cuts 10, 9, 8, 10
    cuts, ok = ttt.trial_outcomes(E, W, 9.0)
    assert list(cuts) == [10, 9, 8, 10] and ok == 3
    st = ttt.TrialStats(trials=4, successes=ok, target_cut=9.0, sweeps_per_run=100,
                        batch_seconds=2.0, best_cuts=cuts)
    assert st.p_s == 0.75
    assert abs(st.r - math.log(0.01) / math.log(0.25)) < 1e-12
    assert abs(st.ttt_amortised - 0.5 * st.r) < 1e-12
