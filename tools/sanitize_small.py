"""Small runs of every kernel for compute-sanitizer (one tool per gpurun call):
bits grid (per-round and fused PT), bits CSR, int8 integer and float, ICM, anneal."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import synth
from paper_2311_09275_b200 import Engine, run_pt

Jr, Jd = synth.torus_pm1(8, 6, 3)
grid = dict(kind="grid", Lx=8, Ly=6, J_right=Jr, J_down=Jd, n=48)
e = Engine(grid, 64, 2, synth.beta_ladder(64), seed=1, layout="bits")
run_pt(e, 20, 5, fused=False); run_pt(e, 20, 5, fused=True); e.icm(0); e.energies(); e.best(spins=True); e.close()
u, v = synth.gnm(300, 320, 4)
rp, col, w = synth.edges_to_csr(300, u, v, np.ones(u.size, np.int32))
csr = dict(kind="csr", n=300, row_ptr=rp, col=col, w=w.astype(np.int32))
e = Engine(csr, 32, 2, synth.beta_ladder(32), seed=1, layout="bits", colour="sl")
run_pt(e, 20, 5, fused=True); e.energies(); e.close()
e = Engine(csr, 16, 2, synth.beta_ladder(16), seed=1, layout="i8")
run_pt(e, 10, 5); e.energies(); e.close()
u, v = synth.random_regular(400, 3, 5)
rp, col, w = synth.edges_to_csr(400, u, v, synth.gaussian_f32(u.size, 6))
fl = dict(kind="csr", n=400, row_ptr=rp, col=col, w=w.astype(np.float32))
e = Engine(fl, 256, 1, synth.beta_ladder(256), seed=1, layout="i8", colour="sl")
e.sweep(6); e.energies(); e.close()
e = Engine(grid, 32, 2, synth.beta_ladder(32), seed=2, layout="bits")
sched = np.tile(synth.beta_ladder(32), (8, 1))
e.anneal(sched); e.energies(); e.close()
print("sanitize-run ok")
