#!/usr/bin/env python
"""Measured memory roof of the C5 access pattern.

Builds tools/gather_peak.cu, runs its two variants (cp.async ring skeleton, plain loads) over
a few depths / occupancies on the GPU and writes the best one to profiles/gather_peak.json:

  attempts_per_s  -- rows x 256 replicas per sweep / time, with no arithmetic per attempt;
  gbs             -- the pattern's bytes (5.14 per attempt) per second.

bench.py reports the C5 line's value against it ("pattern_frac") next to the HBM fraction
against MEASURED_PEAKS.json.  Run under gpurun:

    python tools/gather_peak.py --out profiles/gather_peak.json
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "gather_peak.cu")
BIN = os.path.join(HERE, "gather_peak")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CONFIGS = [("ring", 4, 3), ("ring", 6, 2), ("ring", 8, 2), ("ldg", 2, 8), ("ldg", 4, 4), ("ldg", 4, 8),
           ("ldg", 8, 4)]


def build():
    if os.path.exists(BIN) and os.path.getmtime(BIN) >= os.path.getmtime(SRC):
        return
    subprocess.run([NVCC, "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-o", BIN, SRC],
                   check=True)


def clocks():
    q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,clocks.mem,clocks_throttle_reasons.active",
                        "--format=csv,noheader,nounits"], capture_output=True, text=True)
    return q.stdout.strip()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(os.path.dirname(HERE), "profiles", "gather_peak.json"))
    ap.add_argument("--sweeps", type=int, default=20)
    a = ap.parse_args()
    build()
    runs = []
    for v, d, c in CONFIGS:
        r = subprocess.run([BIN, v, str(d), str(c), str(a.sweeps)], capture_output=True, text=True, timeout=300)
        if r.returncode != 0:
            print(v, d, c, "failed:", r.stderr.strip())
            continue
        rec = json.loads(r.stdout.strip().splitlines()[-1])
        rec["clocks_after"] = clocks()
        runs.append(rec)
        print(json.dumps(rec))
    best = max(runs, key=lambda x: x["attempts_per_s"])
    out = {"source": "tools/gather_peak.cu: the C5 access pattern (4e6 rows x 256 B, C5 class sizes, 3 random "
                     "neighbour rows in other classes, 36 B of table per vertex, own row read + written) with "
                     "no arithmetic per attempt",
           "attempts_per_s": best["attempts_per_s"], "gbs": best["gbs"],
           "bytes_per_attempt": best["bytes_per_attempt"], "best": best, "runs": runs}
    with open(a.out, "w") as f:
        json.dump(out, f, indent=1)
    print("best", best["variant"], best["depth"], best["ctas_per_sm"], "%.4g attempts/s" % best["attempts_per_s"])


if __name__ == "__main__":
    main()
