"""Block-size invariance diagnostic of the torus kernel (energies/spins for several CTA sizes
against the oracle).  python tools/diag_blocksize.py"""
import sys; sys.path.insert(0, '.')
import numpy as np, synth, oracle
from paper_2311_09275_b200 import Engine, run_pt
Jr, Jd = synth.torus_pm1(16, 12, 5)
inst = dict(kind="grid", Lx=16, Ly=12, J_right=Jr, J_down=Jd, n=192)
betas = synth.beta_ladder(32)
o = oracle.Oracle(inst, 32, betas, 7, 0, 4, rng=oracle.RNG_PLANE).run(25, 5)
for fused in (False, True):
    for thr in (32, 64, 96, 128, 256, 512):
        eng = Engine(inst, 32, 4, betas, seed=7, layout="bits", block_threads=thr)
        run_pt(eng, 25, 5, fused=fused)
        print("fused", fused, "thr", thr, np.array_equal(eng.energies(), o.Ei), flush=True)
