"""Greedy-colour class sizes of the C5 instance (same rule as the library: ascending id,
smallest colour unused by coloured neighbours).  Tooling only (profiles/inst_per_attempt)."""
import sys, os
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
inst = synth.make_instance(synth.CONFIGS["c5"])
rp, col = inst["row_ptr"], inst["col"]
n = inst["n"]
colour = np.full(n, -1, np.int64)
for i in range(n):
    used = set(colour[col[rp[i]:rp[i + 1]]].tolist())
    c = 0
    while c in used:
        c += 1
    colour[i] = c
print(np.bincount(colour).tolist())
