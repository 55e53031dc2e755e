#!/usr/bin/env python
"""Measured issue roof for the ALU-bound bit-packed kernels.

Builds tools/alu_peak.cu, counts the SASS instructions of its timed loop (per mode), runs it
on the GPU over a few occupancies and writes profiles/alu_peak.json:

  warp_inst_per_sm_cycle   -- best issue rate of the PLANE instruction mix (mode 1), per SM
                              per cycle (4 = one warp instruction per scheduler per cycle);
  warp_inst_per_s          -- the same at the clock measured in-kernel during that run.

bench.py multiplies warp_inst_per_sm_cycle by 148 SMs and the SM clock it samples during its
own timed region, so the roof is taken "at the same clock".  Run under gpurun:

    python tools/alu_peak.py --out profiles/alu_peak.json
"""
from __future__ import annotations

import argparse
import csv
import json
import os
import re
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "alu_peak.cu")
BIN = os.path.join(HERE, "alu_peak")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


def build():
    if os.path.exists(BIN) and os.path.getmtime(BIN) >= os.path.getmtime(SRC):
        return
    subprocess.run([NVCC, "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
                    "-o", BIN, SRC], check=True)


def loop_counts():
    """{mode: (instructions in the loop body, opcode histogram)} from cuobjdump -sass."""
    sass = subprocess.run(["cuobjdump", "-sass", BIN], capture_output=True, text=True, check=True).stdout
    out = {}
    fun, lines = None, []
    for ln in sass.splitlines() + ["Function : END"]:
        m = re.search(r"Function : (\S+)", ln)
        if m:
            if fun is not None:
                mode = 1 if "ILi1E" in fun else 0
                out[mode] = _loop(lines)
            fun, lines = m.group(1), []
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            lines.append((int(m.group(1), 16), m.group(2).strip()))
    return out


def _loop(lines):
    # the timed loop ends in the only backward branch with a lower target address
    for addr, ins in lines:
        m = re.match(r"(?:@!?U?P\d+\s+)?BRA(?:\.U)?\s+(?:!?U?P\d+,\s*)?0x([0-9a-f]+)", ins)
        if m and int(m.group(1), 16) < addr:
            lo = int(m.group(1), 16)
            body = [i for a, i in lines if lo <= a <= addr]
            hist = {}
            for i in body:
                op = re.sub(r"^@!?U?P\d+\s+", "", i).split()[0]
                hist[op] = hist.get(op, 0) + 1
            return len(body), hist
    raise RuntimeError("no loop found")


def run(mode, threads, per_sm, iters):
    r = subprocess.run([BIN, str(mode), str(threads), str(per_sm), str(iters)], capture_output=True,
                       text=True, timeout=300)
    if r.returncode != 0:
        raise RuntimeError(r.stderr)
    return json.loads(r.stdout.strip().splitlines()[-1])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--iters", type=int, default=20000)
    ap.add_argument("--ncu", action="store_true", help="also count the loop's pipe instructions with ncu")
    args = ap.parse_args()
    build()
    counts = loop_counts()
    res = {"source": "tools/alu_peak.cu (Philox4x32-10 rounds 2-9 of the PLANE contract, hoisted as in "
                     "bits_core.cuh, + the 8-plane LOP3 comparison; no memory traffic)",
           "loop_instructions": {str(m): {"count": c, "opcodes": h} for m, (c, h) in counts.items()},
           "runs": []}
    nsm = 148
    for mode in (0, 1):
        for threads, per_sm in ((1024, 2), (512, 2), (512, 1), (256, 4)):
            r = run(mode, threads, per_sm, args.iters)
            warps = r["grid"] * threads // 32
            inst = warps * r["iters"] * counts[mode][0]  # warp instructions per launch (loop only)
            r["warp_inst_per_s"] = inst / (r["ms_per_launch"] * 1e-3)
            r["warp_inst_per_sm_cycle"] = r["warp_inst_per_s"] / (nsm * r["sm_mhz_in_kernel"] * 1e6)
            res["runs"].append(r)
            print(json.dumps(r), flush=True)
    best = max((r for r in res["runs"] if r["mode"] == 1), key=lambda r: r["warp_inst_per_sm_cycle"])
    best0 = max((r for r in res["runs"] if r["mode"] == 0), key=lambda r: r["warp_inst_per_sm_cycle"])
    res["warp_inst_per_sm_cycle"] = best["warp_inst_per_sm_cycle"]
    res["warp_inst_per_s"] = best["warp_inst_per_s"]
    res["sm_mhz"] = best["sm_mhz_in_kernel"]
    res["philox_only_warp_inst_per_sm_cycle"] = best0["warp_inst_per_sm_cycle"]
    res["note"] = ("roof = best mode-1 (PLANE mix) run; per SM cycle so bench.py can scale it by the clock of "
                   "its own timed region; 4.0 would be one warp instruction per scheduler per cycle")
    if args.ncu:  # pipe counts of the best mode-1 / mode-0 configurations (plain runs exited 0 above)
        M = ("sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,smsp__inst_executed.sum,"
             "sm__cycles_elapsed.avg,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,"
             "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active")
        for key, r in (("plane", best), ("philox", best0)):
            cmd = [BIN, str(r["mode"]), str(r["threads"]), str(r["ctas_per_sm"]), "2000"]
            out = subprocess.run(["ncu", "--metrics", M, "--clock-control", "none", "-c", "1", "--csv"] + cmd,
                                 capture_output=True, text=True, timeout=600).stdout
            vals = {}
            for row in csv.reader(out.splitlines()):
                if len(row) > 14 and row[0] != "ID":
                    vals[row[12]] = float(row[14].replace(",", ""))
            pipe = vals["sm__inst_executed_pipe_alu.sum"] + vals["sm__inst_executed_pipe_fma.sum"]
            res[f"ncu_{key}"] = vals
            res[f"{key}_alu_fma_pipe_inst_per_sm_cycle"] = pipe / (nsm * vals["sm__cycles_elapsed.avg"])
        res["pipe_inst_per_sm_cycle"] = res["plane_alu_fma_pipe_inst_per_sm_cycle"]
        res["pipe_note"] = ("ALU + FMA pipe warp instructions per SM cycle of the PLANE mix (ncu "
                            "sm__inst_executed_pipe_alu + _fma over 148 x sm__cycles_elapsed): the measured "
                            "integer roof; LOP3 (ALU pipe) and IMAD.WIDE (FMA-heavy pipe) do not overlap on "
                            "sm_100a beyond ~0.5 warp instruction per scheduler per cycle combined")
    try:
        res["clocks"] = subprocess.run(
            ["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,clocks_event_reasons.active",
             "--format=csv,noheader"], capture_output=True, text=True, timeout=10).stdout.strip()
    except Exception:
        pass
    print(json.dumps({k: v for k, v in res.items() if k != "runs"}), flush=True)
    if args.out:
        with open(args.out, "w") as f:
            json.dump(res, f, indent=1)


if __name__ == "__main__":
    sys.exit(main())
