"""C5 on one GPU with the smallest-last vs the ascending greedy colouring: create time and
attempts/s of 100 sweeps (R12b).  python tools/c5_colouring_ab.py"""
import time, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
import synth
from paper_2311_09275_b200 import Engine
cfg = synth.CONFIGS["c5"]; inst = synth.make_instance(cfg)
for col in ("sl", None, "sl", None):
    t = time.time()
    eng = Engine(inst, cfg["K"], cfg["C"], synth.beta_ladder(cfg["K"]), seed=synth.PHILOX_KEY, layout="i8", colour=col)
    torch.cuda.synchronize(); tc = time.time() - t
    eng.sweep(5); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); eng.sweep(100); b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    print(col, "ncol", eng.info.n_colours, "create %.2fs" % tc, "attempts/s %.4g" % (inst["n"] * 256 * 100 / (ms * 1e-3)), flush=True)
    eng.close()
