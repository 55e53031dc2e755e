"""Host-side cost of the public create/destroy path (bench e2e): python tools/create_timing.py [workload]"""
import sys
import time

import torch

sys.path.insert(0, "/root/repo")
import synth  # noqa: E402
from paper_2311_09275_b200 import Engine  # noqa: E402

w = sys.argv[1] if len(sys.argv) > 1 else "c2"
cfg = synth.CONFIGS[w]
inst = synth.make_instance(cfg)
betas = synth.beta_ladder(cfg["K"])
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    e = Engine(inst, cfg["K"], cfg["C"], betas, seed=synth.PHILOX_KEY, layout=cfg["layout"],
               colour=cfg.get("colouring"))
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    rec = e.best(spins=False) if False else None
    E = e.energies()
    t2 = time.perf_counter()
    e.close()
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    print(f"{w} create {1e3 * (t1 - t0):.2f} ms  energies {1e3 * (t2 - t1):.2f} ms  destroy {1e3 * (t3 - t2):.2f} ms")
