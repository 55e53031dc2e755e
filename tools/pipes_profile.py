#!/usr/bin/env python
"""Per-attempt instruction mix of the dominant kernel of each workload (run under gpurun).

For every workload: one plain bench.py run (must exit 0), then the same command under
`ncu --metrics <pipe metrics>` for one launch of the workload's kernel.  The counts are divided
by the attempts of that launch (n x replicas x sweeps of the launch) and written to
gpurun_out/pipes_<workload>.json; tools/pipes_profile.py --merge folds them into
profiles/inst_per_attempt.json, which bench.py's roofline entry reads:

  alu_fma_pipe_inst_per_attempt -- warp instructions on the ALU + FMA pipes (the integer roof
                                   measured by tools/alu_peak.cu is in those units);
  warp_inst_per_attempt         -- all warp instructions (smsp__inst_executed.sum);
  dram_bytes_per_launch         -- dram__bytes_read.sum + dram__bytes_write.sum.

    python tools/pipes_profile.py c2 c4b ...      # on the GPU box
    python tools/pipes_profile.py --merge          # here, after gpurun brought the JSON back
"""
from __future__ import annotations

import csv
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = ["smsp__inst_executed.sum", "sm__inst_executed_pipe_alu.sum", "sm__inst_executed_pipe_fma.sum",
           "sm__inst_executed_pipe_lsu.sum", "sm__inst_executed_pipe_uniform.sum",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__cycles_elapsed.avg",
           "sm__cycles_active.avg", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"]

# workload -> (bench args, kernel regex, launches to skip, attempts of the profiled launch)
SWEEPS = 100


def plan(w):
    import synth
    cfg = synth.CONFIGS[w.split(":")[0]]
    n = cfg["Lx"] * cfg["Ly"] if cfg["kind"] == "grid" else cfg["n"]
    base = ["--steps", "1", "--warmup", "1", "--no-cpu", "--no-e2e", "--no-c5", "--no-projection"]
    if w == "c1":
        return ["--workload", "c1"] + base, "k_i8_cluster", 1, n * cfg["K"] * cfg["C"] * cfg["sweeps"]
    if w == "c4b:share16":
        return (["--workload", "c4b", "--copies", "16", "--sweeps", str(SWEEPS)] + base, "k_grid_bands", 1,
                n * cfg["K"] * 16 * SWEEPS)
    if w in ("c4b:full", "c4a:full"):  # the bench's own launch: the whole 50,000-sweep schedule
        ww = w.split(":")[0]
        return (["--workload", ww] + base, "k_grid_sched", 0, n * cfg["K"] * cfg["C"] * cfg["sweeps"])
    if w == "c4b:clusters":  # the cluster launch the persistent one replaced (ISING_GRID_SCHED=0)
        return (["--workload", "c4b", "--sweeps", str(SWEEPS)] + base, "k_grid_bits", 1,
                n * cfg["K"] * cfg["C"] * SWEEPS)
    if w == "c5:packed":  # one whole sweep (the 4 colour-class launches) of the packed-row kernel
        return (["--workload", "c5", "--sweeps", "4"] + base, "k_csr_packed", 16, n * cfg["K"] * cfg["C"], 4)
    kern = {"c2": "k_grid_bits", "c3": "k_csr_bits", "c4a": "k_grid_sched", "c4b": "k_grid_sched"}[w]
    return (["--workload", w, "--sweeps", str(SWEEPS)] + base, kern, 1, n * cfg["K"] * cfg["C"] * SWEEPS)


def run(w):
    pl = plan(w)
    args, kern, skip, attempts = pl[:4]
    count = pl[4] if len(pl) > 4 else 1
    tag = w.replace(":", "_")
    cmd = [sys.executable, "bench.py"] + args
    env = dict(os.environ)
    if w == "c4b:clusters":
        env["ISING_GRID_SCHED"] = "0"
    plain = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, env=env)
    if plain.returncode != 0:
        print(w, "plain run failed:", plain.stderr[-2000:])
        return
    csvp = os.path.join(ROOT, "gpurun_out", f"pipes_{tag}.csv")
    # (the band split's cooperative launch, c4b:share16, fails under ncu in kernel and in
    # application replay alike: its copy barriers spin on global memory)
    prof = subprocess.run(["ncu", "--metrics", ",".join(METRICS), "--clock-control", "none", "-k",
                           f"regex:{kern}", "-s", str(skip), "-c", str(count), "--csv"] + cmd, cwd=ROOT,
                          capture_output=True, text=True, timeout=1800, env=env)
    with open(csvp, "w") as f:
        f.write(prof.stdout + prof.stderr)
    vals = {}
    for r in csv.reader(prof.stdout.splitlines()):
        if len(r) > 14 and r[0] != "ID":
            try:  # summed over the profiled launches
                vals[r[12]] = vals.get(r[12], 0.0) + float(r[14].replace(",", ""))
            except ValueError:
                pass
    for k in list(vals):  # rates are averaged over the profiled launches, counts summed
        if "pct" in k or k.endswith(".avg"):
            vals[k] /= count
    if "smsp__inst_executed.sum" not in vals:
        print(w, "no ncu data; see", csvp)
        return
    out = {"workload": w, "kernel": kern, "attempts_per_launch": attempts,
           "warp_inst_per_attempt": vals["smsp__inst_executed.sum"] / attempts,
           "alu_fma_pipe_inst_per_attempt": (vals["sm__inst_executed_pipe_alu.sum"] +
                                             vals["sm__inst_executed_pipe_fma.sum"]) / attempts,
           "dram_bytes_per_launch": vals.get("dram__bytes_read.sum", 0) + vals.get("dram__bytes_write.sum", 0),
           "ncu": vals, "command": " ".join(cmd)}
    with open(os.path.join(ROOT, "gpurun_out", f"pipes_{tag}.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: v for k, v in out.items() if k != "ncu"}))


def merge():
    path = os.path.join(ROOT, "profiles", "inst_per_attempt.json")
    db = json.load(open(path))
    # the bench's full launch (":full") wins over a short profiled launch of the same kernel
    files = sorted(glob.glob(os.path.join(ROOT, "gpurun_out", "pipes_*.json")), key=lambda f: "_full" in f)
    for f in files:
        d = json.load(open(f))
        key = {"c5:packed": "c5_packed", "c4b:share16": "c4b_bands", "c4b": "c4b_sched", "c4a": "c4a_sched",
               "c4b:clusters": "c4b", "c4b:full": "c4b_sched", "c4a:full": "c4a_sched"}.get(d["workload"], d["workload"])
        e = db.setdefault(key, {})
        e.update({"kernel": d["kernel"], "layout": "bits" if d["kernel"] not in ("k_i8_cluster", "k_csr_packed") else "i8",
                  "warp_inst_per_attempt": d["warp_inst_per_attempt"],
                  "alu_fma_pipe_inst_per_attempt": d["alu_fma_pipe_inst_per_attempt"],
                  "dram_bytes_per_launch": d["dram_bytes_per_launch"],
                  "issue_active_pct": d["ncu"].get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                  "alu_pipe_pct": d["ncu"].get("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"),
                  "fmaheavy_pipe_pct": d["ncu"].get("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active"),
                  "pipes_source": f"profiles/r02/{os.path.basename(f)} (ncu --metrics, one launch of "
                                  f"{d['attempts_per_launch']:.4g} attempts: {d['command']})"})
    with open(path, "w") as f:
        json.dump(db, f, indent=1)
    print("merged into", path)


if __name__ == "__main__":
    if "--merge" in sys.argv:
        merge()
    else:
        for w in sys.argv[1:]:
            run(w)
