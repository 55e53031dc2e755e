"""Class sizes of the C5 instance under the library's Jones-Plassmann colouring (the bench's
colouring), computed on the GPU through ising_colour_jp.  Tooling only: it converts an ncu
capture of one colour-class launch into per-attempt figures (profiles/inst_per_attempt.json)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2311_09275_b200 import ising as L  # noqa: E402

inst = synth.make_instance(synth.CONFIGS["c5"])
colour, nc = L.ising_colour_jp(inst["n"], inst["row_ptr"], inst["col"])
print({"n_colours": int(nc), "class_sizes": np.bincount(colour).tolist()})
