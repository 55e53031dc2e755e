"""Paper-style time-to-target table (§II.B Eq.(1)/(2), Table I columns) for the
synthetic G65-shaped torus (C2 instance) on one B200, with the copies of a PT run as trials
(paper_2311_09275_b200/ttt.py).

The instance is a seeded stand-in, so its best-known cut is unknown: the target is the best
cut found by a long reference run (64 copies x REF sweeps); each budget then runs one batch
of 64 independent trials (fresh seeds) and reports P_s, r (Eq. 1), sweeps-to-target and TTT
(Eq. 2) as batch latency x r and as amortised time per trial x r, for targets at fractions of
that best cut (the paper's "quality").

    python tools/ttt_table.py [--ref 50000] [--budgets 1000,2000,5000,10000] [--out FILE]
"""
import argparse
import json
import sys
import time

import numpy as np
import torch

sys.path.insert(0, "/root/repo")
import synth  # noqa: E402
from paper_2311_09275_b200 import Engine, run_pt, ttt  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ref", type=int, default=50000)
    ap.add_argument("--budgets", default="5000,20000,50000,100000,200000")
    ap.add_argument("--quality", default="1.0,0.999,0.998",
                    help="targets as fractions of the reference run's best cut")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    cfg = synth.CONFIGS["c2"]
    inst = synth.make_instance(cfg)
    K, C, kex = cfg["K"], cfg["C"], cfg["k_ex"]
    betas = synth.beta_ladder(K)
    W = float(inst["J_right"].sum() + inst["J_down"].sum())
    eng = Engine(inst, K, C, betas, seed=synth.PHILOX_KEY + 1000, layout="bits")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rec = run_pt(eng, a.ref, kex)
    torch.cuda.synchronize()
    ref_s = time.perf_counter() - t0
    target = (W - rec["E"]) / 2.0
    rows = []
    for i, b in enumerate(int(x) for x in a.budgets.split(",")):
        e = Engine(inst, K, C, betas, seed=synth.PHILOX_KEY + 3000 + i, layout="bits")
        st = ttt.run_trials(e, b, kex, target, W)
        for q in (float(x) for x in a.quality.split(",")):
            tq = np.ceil(q * target)
            ok = int(np.count_nonzero(st.best_cuts >= tq))
            p = ok / st.trials
            r = ttt.repetitions(p)
            rows.append({"quality": q, "target_cut": float(tq), "sweeps_per_trial": b, "trials": st.trials,
                         "successes": ok, "P_s": p, "r": r, "sweeps_to_target": b * r,
                         "batch_s": st.batch_seconds, "ttt_latency_s": st.batch_seconds * r,
                         "ttt_amortised_s": st.batch_seconds / st.trials * r,
                         "best_cut_median": float(np.median(st.best_cuts)),
                         "best_cut_max": float(st.best_cuts.max())})
        e.close()
    out = {"instance": "C2 synthetic 80x100 +-1 torus (G65 shape), seed 65", "replicas_per_trial": K,
           "exchange_every": kex, "target": {"cut": target, "energy": rec["E"],
                                             "source": f"best of a {a.ref}-sweep run of 64 copies ({ref_s:.2f} s)"},
           "rows": rows}
    s = json.dumps(out, indent=1)
    print(s)
    if a.out:
        open(a.out, "w").write(s + "\n")


if __name__ == "__main__":
    main()
