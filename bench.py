#!/usr/bin/env python
"""Benchmark of the hot path: replica-parallel Metropolis sweeps + parallel tempering.

Metric (BASELINE.json): spin-flip attempts/s (attempts = n x replicas x sweeps, every
site of every replica counted once per sweep) at N GPUs, plus the
fraction of the roofline of the dominant kernel.

Default workload (BASELINE.json configs[3], the config the metric "attempts/s at 1/2/4/8
B200" is quoted on, and the largest single-GPU one): the 100x200 +-1 torus (G81 shape,
PAPER.md:35 Table I), 128 temperatures x 128 copies = 16,384 replicas, beta 0.1-3.0
geometric, 50,000 sweeps with a replica exchange every 10 sweeps, bit-packed spins.  One
step = that whole schedule (5,000 rounds of 10 sweeps + best check + exchange) on inputs
already resident on the GPU.  Strong scaling: the 128 copies are split over the N ranks
(one process per GPU), exchanges are local to a copy, and one NCCL all-gather of the
per-rank best records per step feeds the library's merge (ising_merge_best).

The same JSON line carries:
  * "c5": the HBM-bound stress config (BASELINE.json configs[4]: random 3-regular graph,
    4e6 vertices, N(0,1) float32 couplings, 256 replicas per GPU, 1,000 sweeps) measured in
    the same run (value, roofline against measured HBM, clocks, e2e);
  * "scaling_projection" (N=1 only): one GPU's share of the N = 2/4/8 job (64/32/16 copies)
    timed on this GPU, i.e. the strong-scaling efficiency the kernels allow;
  * "north_star_mode" (N=1 only): driver.run_pt(gather=True)'s per-round path (sweep launch,
    16-byte record export, record all-gather, global best + exchange) over 2,000 C4b sweeps,
    next to the fused schedule's rate;
  * "roofline" of the dominant kernel against the MEASURED issue roof of its instruction mix
    (tools/alu_peak.cu -> profiles/alu_peak.json) at the clock sampled in the timed region.
Other workloads: --workload c1|c2|c3|c4a|c5 (c2/c3 weak scaling: a 64-copy shard per rank);
--copies overrides the copy count (c4b --copies 16 = one rank's share of the 8-GPU job).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|c3|c4a|c4b|c1|c5]
    python bench.py --impl reference ...   # the CPU oracle on the host cores
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
PROFILE_FILE = os.path.join(ROOT, "profiles", "inst_per_attempt.json")

STRONG = ("c4a", "c4b")  # fixed total replicas sharded over the GPUs (BASELINE.json configs[3])

WORKLOADS = {
    "c1": "16x16 +-1 torus, 64 temps x 1 copy, 1000 sweeps, exchange every 10, int8 spins",
    "c2": "80x100 +-1 torus (G65 shape), 64 temps x 64 copies = 4096 replicas, beta 0.1-3.0 "
          "geometric, 10000 sweeps, exchange every 10, bit-packed spins",
    "c3": "G(10000, 9999) unweighted MaxCut (J=+1, G70 shape), greedy colouring, 64 temps x 64 "
          "copies, 10000 sweeps, exchange every 10, bit-packed spins",
    "c4a": "100x140 +-1 torus (G77 shape), 128 temps x 128 copies, exchange every 10, bit-packed",
    "c4b": "100x200 +-1 torus (G81 shape), 128 temps x 128 copies, exchange every 10, bit-packed",
    "c5": "random 3-regular, 4e6 vertices, N(0,1) float32 couplings, 256 replicas/GPU, 1000 "
          "sweeps, int8 spins",
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="c4b", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sweeps", type=int, default=0, help="override sweeps per step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--copies", type=int, default=0,
                    help="copies override: per rank (weak-scaling workloads) or in total (c4a/c4b); "
                         "e.g. --workload c4b --copies 16 measures one rank's share at 8 GPUs")
    ap.add_argument("--threads", type=int, default=0, help="CTA size override")
    ap.add_argument("--no-c5", action="store_true", help="skip the nested C5 (HBM-bound) record")
    ap.add_argument("--no-c5-int8", action="store_true",
                    help="skip the nested C5 record on the int8 rows (ISING_I8_PACKED=0)")
    ap.add_argument("--no-projection", action="store_true",
                    help="skip the one-GPU share runs of the strong-scaling workload (N = 2, 4, 8)")
    return ap.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def workload_params(name, sweeps_override):
    cfg = dict(synth.CONFIGS[name])
    if sweeps_override:
        cfg["sweeps"] = sweeps_override
    return cfg


def json_line(d):
    print(json.dumps(d), flush=True)


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if not self.proc:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        note = None
        if not out.strip():  # timed region shorter than nvidia-smi's start-up + period
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=10).stdout
                note = "timed region shorter than the sampling period: one query right after it"
            except Exception:
                out = ""
        sm, mx, reasons = [], [], set()
        for line in out.strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
            except ValueError:
                continue
            for name, v in zip(("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                "sw_power_cap"), f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        if not sm:
            return None
        r = {"sm_mhz": float(np.median(sm)), "sm_max_mhz": float(max(mx)),
             "samples": len(sm), "reasons": sorted(reasons)}
        if note:
            r["note"] = note
        return r


# ------------------------------------------------------------------ reference (oracle) arm
def cpu_oracle_sample(cfg, target_s=12.0):
    """The CPU oracle as it stands, one thread per copy on the host cores, on a bounded
    sample of the workload: `threads` copies x S sweeps (S sized for ~target_s)."""
    import oracle
    inst = synth.make_instance(cfg)
    K = cfg["K"]
    betas = synth.beta_ladder(K)
    cores = os.cpu_count() or 1
    threads = max(1, min(cores, cfg["C"], 16))
    if cfg["C"] == 1 and cfg["K"] > 64:  # one copy: threads take disjoint replica pairs instead
        threads = max(1, min(cores, 16, cfg["K"] // 2))
    n = inst["n"]
    kex = cfg["k_ex"] if cfg["k_ex"] > 0 else 0
    rng = oracle.RNG_PLANE if cfg["layout"] == "bits" else oracle.RNG_WORD
    colour = None  # the workload's colouring, computed by the oracle's own implementation
    if cfg.get("colouring") == "sl":
        colour, _ = oracle.greedy_colour_sl(n, inst["row_ptr"], inst["col"])
    elif cfg.get("colouring") == "jp":
        colour, _ = oracle.greedy_colour_jp(n, inst["row_ptr"], inst["col"])
    # calibrate on one copy x 2 sweeps
    t0 = time.perf_counter()
    if cfg["C"] == 1 and cfg["K"] > 64:
        o = oracle.Oracle(inst, K, betas, synth.PHILOX_KEY, 0, 1, rng=rng, colour=colour, slots=(0, 4))
        o.sweeps(1)
        per = (time.perf_counter() - t0) / (4 * n)
    else:
        o = oracle.Oracle(inst, K, betas, synth.PHILOX_KEY, 0, 1, rng=rng, colour=colour)
        o.sweeps(2)
        per = (time.perf_counter() - t0) / (2 * K * n)
    if cfg["C"] == 1 and cfg["K"] > 64:
        # replica sample (no exchange): `threads` slots per thread-run
        import threading
        reps = threads * 2
        sweeps = max(1, int(target_s * threads / (per * n * reps)))
        res = []

        def work(q):
            oo = oracle.Oracle(inst, K, betas, synth.PHILOX_KEY, 0, 1, rng=rng, colour=colour,
                               slots=(2 * q, 2 * q + 2))
            oo.sweeps(sweeps)
            res.append(oo)
        t0 = time.perf_counter()
        ts = [threading.Thread(target=work, args=(q,)) for q in range(threads)]
        [t.start() for t in ts]
        [t.join() for t in ts]
        dt = time.perf_counter() - t0
        attempts = n * reps * sweeps
        sample = f"{reps} replicas x {sweeps} sweeps of the {cfg['kind']} instance (no exchange)"
    else:
        sweeps = max(kex or 1, int(target_s * threads / (per * n * K * threads)))
        if kex:
            sweeps = max(kex, (sweeps // kex) * kex)
        t0 = time.perf_counter()
        oracle.run_sharded(inst, K, betas, synth.PHILOX_KEY, 0, threads, sweeps, kex, rng=rng,
                           threads=threads, colour=colour)
        dt = time.perf_counter() - t0
        attempts = n * K * threads * sweeps
        sample = f"{threads} copies x {K} temps x {sweeps} sweeps (exchange every {kex})"
    return {"value": attempts / dt, "unit": "attempts/s", "cores": threads, "kind": "oracle",
            "sample": sample, "seconds": round(dt, 2), "host_cores_available": cores}


def run_reference(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return
    cfg = workload_params(args.workload, args.sweeps)
    vals = []
    for s in range(args.warmup + args.steps):
        r = cpu_oracle_sample(cfg, target_s=4.0)
        if s >= args.warmup:
            vals.append(r)
    v = float(np.median([r["value"] for r in vals]))
    cb = dict(vals[-1])
    cb["value"] = v
    json_line({
        "impl": "reference", "metric": "spin-flip attempts/s", "value": v, "unit": "attempts/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": float(np.median([r["seconds"] for r in vals]) * 1e3),
        "higher_is_better": True, "scaling": "strong" if args.workload in STRONG else "weak",
        "vs_baseline": None,
        "dtype": "int8 spins / int64 energies (scalar C)", "data": "synthetic",
        "config": {"workload": args.workload, "description": WORKLOADS[args.workload],
                   "note": "CPU oracle on host cores, bounded sample per step"},
        "cpu_baseline": cb,
        "e2e": {"value": v, "unit": "attempts/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    })


# ------------------------------------------------------------------ our arm
ALU_PEAK_FILE = os.path.join(ROOT, "profiles", "alu_peak.json")
GATHER_PEAK_FILE = os.path.join(ROOT, "profiles", "gather_peak.json")


def kernel_name(eng, inst, cfg, K, R, fused_one_launch):
    if inst["kind"] == "grid" and cfg["layout"] == "bits":
        if eng.info.fused_pt == 3:
            return "k_grid_sched"
        return "k_grid_bands" if eng.info.bands > 1 else "k_grid_bits"
    if cfg["layout"] == "bits":
        return "k_csr_bits"
    if inst.get("w") is not None and inst["w"].dtype == np.float32 and R % 256 == 0:
        # the library sweeps a packed-row working copy when a call has >= 4 sweeps
        # (ISING_I8_PACKED=0|1 overrides)
        mode = os.environ.get("ISING_I8_PACKED")
        calls = cfg["sweeps"] if cfg["k_ex"] <= 0 else cfg["k_ex"]
        return "k_csr_packed" if mode == "1" or (mode != "0" and calls >= 4) else "k_csr_i8_ring"
    if fused_one_launch:
        return "k_i8_cluster" if K <= 64 else "k_i8_small"
    return "k_csr_i8_phase"


def roofline_entry(kernel_ms, attempts_per_launch, layout, clocks, ipa_key):
    """Roofline of the dominant kernel.

    int8 per-lane sweeps (C5) are HBM bound: achieved = algorithmic bytes per attempt (DESIGN.md
    §5.4: 2 own + 3 neighbour + 0.11 CSR = 5.11 B) x attempts per launch / live CUDA-event launch
    time, against MEASURED_PEAKS.json hbm_gbs.

    Bit-packed sweeps (C1-C4) keep their state on chip and are bound by the integer pipes (Philox
    IMAD.WIDE on the FMA pipe, LOP3 on the ALU pipe): achieved = ALU + FMA pipe warp instructions
    per launch (ncu sm__inst_executed_pipe_alu + _fma per attempt, profiles/inst_per_attempt.json,
    times the live attempts per launch) / live launch time; peak = the MEASURED ALU + FMA pipe rate
    of the PLANE instruction mix (tools/alu_peak.cu -> profiles/alu_peak.json, per SM cycle) x 148
    SMs x the SM clock sampled during this run's timed region (SURVEY.md §8(d) "ALU fraction ... at
    the same clock").  Falls back to all-instruction issue rates if those counts are missing."""
    peaks = json.load(open(PEAKS_FILE)) if os.path.exists(PEAKS_FILE) else {}
    ipa = None
    if os.path.exists(PROFILE_FILE):
        ipa = json.load(open(PROFILE_FILE)).get(ipa_key)
    if layout == "i8":
        bpa = ipa.get("alg_bytes_per_attempt", 5.11) if ipa else 5.11
        ach = attempts_per_launch * bpa / (kernel_ms * 1e-3) / 1e9
        peak = peaks.get("hbm_gbs", 6551.4)
        out = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
               "traffic": (ipa or {}).get("dram_bytes_per_attempt") and
               ipa["dram_bytes_per_attempt"] * attempts_per_launch,
               "alg_bytes_per_attempt": bpa,
               "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)"}
        if os.path.exists(GATHER_PEAK_FILE):
            # the same access pattern without arithmetic (tools/gather_peak.cu): what this kernel's
            # memory traffic alone can reach on a B200 (~23% of its gathers hit L2)
            gp = json.load(open(GATHER_PEAK_FILE))
            rate = attempts_per_launch / (kernel_ms * 1e-3)
            out["pattern_roof"] = {"attempts_per_s": gp["attempts_per_s"], "frac": rate / gp["attempts_per_s"],
                                   "source": "profiles/gather_peak.json (tools/gather_peak.cu, best of "
                                             f"{len(gp.get('runs', []))} configurations)"}
        return out
    mhz_max = peaks.get("sm_max_mhz", 1965.0)
    mhz = (clocks or {}).get("sm_mhz") or mhz_max
    alu = json.load(open(ALU_PEAK_FILE)) if os.path.exists(ALU_PEAK_FILE) else None
    traffic_launch = None
    if ipa:
        if ipa.get("dram_bytes_per_launch") is not None:  # on-chip state: a fixed load/store per launch
            traffic_launch = ipa["dram_bytes_per_launch"]
        elif ipa.get("dram_bytes_per_attempt") is not None:
            traffic_launch = ipa["dram_bytes_per_attempt"] * attempts_per_launch
    if ipa and ipa.get("alu_fma_pipe_inst_per_attempt") and alu and alu.get("pipe_inst_per_sm_cycle"):
        # the integer roof: ALU + FMA pipe warp instructions (LOP3 / IMAD.WIDE), measured
        peak = alu["pipe_inst_per_sm_cycle"] * 148 * mhz * 1e6 / 1e9
        ach = attempts_per_launch * ipa["alu_fma_pipe_inst_per_attempt"] / (kernel_ms * 1e-3) / 1e9
        out = {"bound": "alu", "achieved": ach, "peak": peak, "unit": "G ALU+FMA-pipe warp-inst/s",
               "frac": ach / peak, "traffic": traffic_launch,
               "peak_source": (f"measured: tools/alu_peak.cu PLANE mix, {alu['pipe_inst_per_sm_cycle']:.3f} ALU+FMA "
                               f"pipe warp-inst per SM cycle (ncu, profiles/alu_peak.json) x 148 SMs x {mhz:.0f} "
                               "MHz sampled in this timed region"),
               "alu_fma_pipe_inst_per_attempt": ipa["alu_fma_pipe_inst_per_attempt"],
               "inst_per_attempt_source": ipa.get("pipes_source") or ipa.get("source")}
        if ipa.get("warp_inst_per_attempt"):
            out["issue_frac_of_4_per_cycle"] = (attempts_per_launch * ipa["warp_inst_per_attempt"] /
                                                (kernel_ms * 1e-3) / (148 * 4 * mhz * 1e6))
        return out
    if alu:
        peak = alu["warp_inst_per_sm_cycle"] * 148 * mhz * 1e6 / 1e9
        src = (f"measured: tools/alu_peak.cu PLANE mix {alu['warp_inst_per_sm_cycle']:.3f} warp-inst per SM "
               f"cycle (profiles/alu_peak.json) x 148 SMs x {mhz:.0f} MHz sampled in this timed region")
    else:
        peak = 148 * 4 * mhz * 1e6 / 1e9
        src = f"derived: 148 SMs x 4 issue/cycle x {mhz:.0f} MHz (no alu_peak.json yet)"
    if not ipa:
        return {"bound": "alu", "achieved": None, "peak": peak, "unit": "Ginst/s", "frac": None,
                "traffic": None, "peak_source": src,
                "note": "no ncu instruction count for this kernel (the band split's cooperative launch "
                        "fails under ncu replay)" if ipa_key.endswith("_bands") else
                        "no ncu instruction count committed yet"}
    ach = attempts_per_launch * ipa["warp_inst_per_attempt"] / (kernel_ms * 1e-3) / 1e9
    return {"bound": "alu", "achieved": ach, "peak": peak, "unit": "Ginst/s", "frac": ach / peak,
            "traffic": traffic_launch, "peak_source": src,
            "warp_inst_per_attempt": ipa["warp_inst_per_attempt"],
            "inst_per_attempt_source": ipa.get("source")}


def measure(args, workload, world, rank, local, steps, warmup, e2e_steps, copies=0, sweeps=0,
            cpu=True, quiet_cfg=False):
    """Time `steps` steps of `workload` (one step = the whole schedule: all sweeps, exchanges and
    best checks) after `warmup` untimed ones; returns this workload's JSON record (all ranks
    compute it, rank 0 prints).  e2e_steps > 0 also times the public API from host arrays."""
    import torch
    import torch.distributed as dist

    from paper_2311_09275_b200.driver import Engine, merge_best_over_ranks

    cfg = workload_params(workload, sweeps)
    inst = synth.make_instance(cfg)
    K, C = cfg["K"], cfg["C"]
    if copies:
        C = copies
    betas = synth.beta_ladder(K)
    strong = workload in STRONG
    if strong:  # BASELINE configs[3]: the 128 copies (16,384 replicas) are sharded over the ranks
        if C % world:
            raise SystemExit(f"{workload}: {C} copies do not split over {world} ranks")
        Cg = C
        c_lo, c_hi = rank * C // world, (rank + 1) * C // world
    else:  # weak scaling: every rank runs a C-copy shard with distinct global ids
        Cg = C * world
        c_lo, c_hi = rank * C, (rank + 1) * C
    stream = torch.cuda.current_stream(local)
    mk = dict(seed=synth.PHILOX_KEY, copy_begin=c_lo, copy_end=c_hi, layout=cfg["layout"], device=local,
              block_threads=args.threads, stream=stream.cuda_stream, colour=cfg.get("colouring"))
    eng = Engine(inst, K, Cg, betas, **mk)
    n, R = inst["n"], eng.R
    sweeps_, kex = cfg["sweeps"], cfg["k_ex"]
    rounds = sweeps_ // kex if kex > 0 else 0
    rem = sweeps_ - rounds * kex if kex > 0 else sweeps_
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=torch.device("cuda", local))

    # bit-packed kernels run all rounds in one launch (unless a band-split handle's clusters would
    # not all be resident: then ising_run takes per-round launches, counted as such); small int8
    # instances with integer weights (C1) also run all rounds in one launch
    fused = kex > 0 and (cfg["layout"] == "bits" or bool(eng.info.fused_pt))
    fused_one_launch = fused and bool(eng.info.fused_pt)

    def timed(kev, fn, *a):
        if kev is None:
            return fn(*a)
        ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
        ev[0].record(stream)
        fn(*a)
        ev[1].record(stream)
        kev.append(ev)

    def packed_extra(ns):
        """k_pack_rows + k_unpack_rows around a packed-row sweep call."""
        if inst.get("w") is None or inst["w"].dtype != np.float32 or R % 256 or cfg["layout"] != "i8":
            return 0
        mode = os.environ.get("ISING_I8_PACKED")
        return 2 if mode == "1" or (mode != "0" and ns >= 4) else 0

    def schedule(e, kev=None):
        """One pass of the whole hot path over the workload; returns our kernel launches."""
        launches = 0
        if fused:
            timed(kev, e.run, rounds, kex)
            launches += 2 if fused_one_launch else 3 * rounds
        else:
            for _ in range(rounds):
                timed(kev, e.sweep, kex)
                e.exchange()
                launches += (1 if cfg["layout"] == "bits" else kex * e.info.n_colours + 2 + packed_extra(kex)) + 2
        if rem:
            timed(kev, e.sweep, rem)
            e.check_best()
            launches += (1 if cfg["layout"] == "bits" else rem * e.info.n_colours + 2 + packed_extra(rem)) + 1
        return launches

    def step(kev=None):
        launches = schedule(eng, kev)
        rec = eng.best(spins=False)
        if world > 1:
            rec = merge_best_over_ranks(rec, None, engine=eng)
        return launches, rec

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    total_ms, kernel_ms, nk, launches = 0.0, 0.0, 0, 0
    step_ms = []  # this rank's per-step device times (the spread behind the mean)
    rec = None
    clocks.start()
    for _ in range(steps):
        flush.zero_()  # L2 flush between timed steps (outside the timed events)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        kev = []
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        nl, rec = step(kev)
        b.record(stream)
        torch.cuda.synchronize()
        launches += nl
        step_ms.append(a.elapsed_time(b))
        total_ms += step_ms[-1]
        kernel_ms += sum(x.elapsed_time(y) for x, y in kev)
        nk += len(kev)
    clk = clocks.stop()
    t = torch.tensor([total_ms], dtype=torch.float64, device=torch.device("cuda", local))
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = n * K * Cg * sweeps_ * steps / (total_ms * 1e-3)  # all ranks' attempts
    avg_launch_ms = kernel_ms / max(nk, 1)
    per_launch_attempts = n * R * (rounds * kex if fused else (kex if kex > 0 else sweeps_))
    kname = kernel_name(eng, inst, cfg, K, R, fused_one_launch)
    # instruction counts per attempt are kernel-specific
    ipa_key = workload + {"k_grid_bands": "_bands", "k_grid_sched": "_sched", "k_csr_packed": "_packed"}.get(kname, "")
    roof = roofline_entry(avg_launch_ms, per_launch_attempts,
                          "bits" if cfg["layout"] == "bits" or fused_one_launch or kname == "k_csr_packed"
                          else cfg["layout"], clk, ipa_key)
    if kname == "k_csr_packed":
        # the packed rows move 196 algorithmic bytes per 256 attempts (own row read +
        # written 64, three neighbour rows 96, table entry 36): against HBM for reference; the
        # kernel is bound by the integer pipes (the roofline above)
        pk_bpa = 196 / 256
        roof["hbm"] = {"alg_bytes_per_attempt": pk_bpa,
                       "achieved_gbs": per_launch_attempts * pk_bpa / (avg_launch_ms * 1e-3) / 1e9,
                       "frac": per_launch_attempts * pk_bpa / (avg_launch_ms * 1e-3) / 1e9 /
                       json.load(open(PEAKS_FILE)).get("hbm_gbs", 6551.4) if os.path.exists(PEAKS_FILE) else None}
    roof["kernel"] = kname
    if kname in ("k_i8_small", "k_i8_cluster"):
        per = K // 8 if kname == "k_i8_cluster" else 1
        roof["note"] = (f"{per} CTA(s) per copy: {eng.R // K} copies use {per * (eng.R // K)} of the GPU's "
                        "SMs; frac is against the whole-GPU issue peak")
    roof["kernel_share_of_step"] = kernel_ms / max(sum(step_ms), 1e-9)
    roof["avg_launch_ms"] = avg_launch_ms
    roof["attempts_per_launch"] = per_launch_attempts

    # ---- end to end through the public API with host buffers, every step
    e2e = None
    if e2e_steps > 0:
        # the step's inputs in pinned host memory (page-locked once, outside the timed region)
        def pinned(a):
            t = torch.from_numpy(np.ascontiguousarray(a)).pin_memory()
            return t.numpy()
        inst_h = {k: (pinned(v) if isinstance(v, np.ndarray) else v) for k, v in inst.items()}
        e2e_ms = 0.0
        ew = min(warmup, 3)
        for s in range(ew + e2e_steps):  # untimed warm-up steps, then timed ones
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            e = Engine(inst_h, K, Cg, betas, **{**mk, "seed": synth.PHILOX_KEY + s})
            schedule(e)
            e.best(spins=True)
            e.energies()
            b.record(stream)
            torch.cuda.synchronize()
            e.close()
            if s >= ew:
                e2e_ms += a.elapsed_time(b)
        if inst["kind"] == "grid":
            h2d = 2 * n + 8 * K
        else:
            h2d = 8 * (n + 1) + inst["col"].nbytes + inst["w"].nbytes + 8 * K
        d2h = 8 * R + n + 32
        t = torch.tensor([e2e_ms], dtype=torch.float64, device=torch.device("cuda", local))
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ev = n * K * Cg * sweeps_ * e2e_steps / (float(t.item()) * 1e-3)
        e2e = {"value": ev, "unit": "attempts/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "steps": e2e_steps, "frac_of_device_value": ev / value,
               "includes": "create from pinned host arrays (validate, colour, tables, upload, init) + full "
                           "schedule + best configuration / energies readback"}
    eng.close()
    del flush

    cpu_rec = None
    if rank == 0 and world == 1 and cpu:
        cpu_rec = cpu_oracle_sample(cfg, target_s=12.0 if not quiet_cfg else 8.0)

    peaks = json.load(open(PEAKS_FILE)) if os.path.exists(PEAKS_FILE) else {}
    bpa = 0.25 if cfg["layout"] == "bits" else (196 / 256 if kname == "k_csr_packed" else 5.11)
    return {
        "metric": "spin-flip attempts/s", "value": value, "unit": "attempts/s",
        "n_gpus": world, "steps": steps, "warmup": warmup, "ms_per_step": total_ms / steps,
        "step_ms_rank0": {"median": float(np.median(step_ms)), "min": min(step_ms), "max": max(step_ms)},
        "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
        "dtype": "u32" if cfg["layout"] == "bits" else ("f32" if cfg["kind"] == "regular" else "int32"),
        "data": "synthetic",
        "config": {"workload": workload, "description": WORKLOADS[workload],
                   "n": n, "replicas_per_gpu": R, "sweeps_per_step": sweeps_, "exchange_every": kex,
                   "copies_total": Cg, "copies_per_gpu": c_hi - c_lo,
                   "parallelism": f"copies sharded over {world} GPU(s), "
                                  + ("strong scaling (fixed total)" if strong else "weak scaling"),
                   "l2": ("flushed between timed steps (256 MB write); the state is SMEM/L2-resident "
                          "by design" if cfg["layout"] == "bits" or n * R < (64 << 20) else
                          "flushed between timed steps (256 MB write); spins (%.2f GB) exceed L2"
                          % (n * R / 1e9))},
        "roofline": roof,
        "hbm_frac": value / world * bpa / 1e9 / peaks.get("hbm_gbs", 6551.4),
        "cpu_baseline": cpu_rec,
        "e2e": e2e,
        "gpu_launches": launches,
        "clocks": clk,
        "best": {k: rec[k] for k in ("E", "slot", "sweep")} if rec else None,
    }


def scaling_projection(args, main_value, local):
    """One GPU's share of the strong-scaling job at N = 2, 4, 8 (copies 64 / 32 / 16 of C4b's 128),
    each timed on this GPU over 5,000 sweeps: projected N-GPU value = N x share rate, efficiency =
    share rate / 1-GPU rate.  The N-GPU run adds one NCCL all-gather of 24-byte best records per
    step (driver.merge_best_over_ranks), microseconds against seconds of sweeps."""
    out = {}
    cfg = workload_params(args.workload, 0)
    for N in (2, 4, 8):
        r = measure(args, args.workload, 1, 0, local, steps=2, warmup=1, e2e_steps=0,
                    copies=cfg["C"] // N, sweeps=5000, cpu=False, quiet_cfg=True)
        out[str(N)] = {"copies_per_gpu": cfg["C"] // N, "share_rate": r["value"],
                       "projected_value": N * r["value"], "projected_efficiency": r["value"] / main_value,
                       "kernel": r["roofline"]["kernel"], "sweeps": 5000}
    return out


def north_star_mode(args, main_value, local, sweeps=2000):
    """The record-gather mode of driver.run_pt(gather=True) (BASELINE.json north_star: an all-gather
    of the per-replica records at every tempering exchange) on this GPU's C4b handle: per round one
    sweep launch (k_ex sweeps), ising_exchange_begin (16-byte records), the all-gather -- at one
    rank a device copy of the records, the data NCCL would move -- and ising_exchange_end (global
    best over the gathered records, exchange decisions, swaps).  Timed with CUDA events over
    `sweeps` sweeps; reported next to the fused single-launch rate of the main line."""
    import torch

    from paper_2311_09275_b200.driver import Engine

    cfg = workload_params(args.workload, sweeps)
    inst = synth.make_instance(cfg)
    K, C, kex = cfg["K"], cfg["C"], cfg["k_ex"]
    stream = torch.cuda.current_stream(local)
    eng = Engine(inst, K, C, synth.beta_ladder(K), seed=synth.PHILOX_KEY, layout=cfg["layout"], device=local,
                 block_threads=args.threads, stream=stream.cuda_stream)
    send, recv = eng.record_buffers(1)
    rounds = sweeps // kex

    def step():
        for _ in range(rounds):
            eng.sweep(kex)
            eng.exchange_begin(send)
            recv.copy_(send)
            eng.exchange_end(recv)

    step()
    torch.cuda.synchronize()
    ms = []
    for _ in range(2):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        step()
        b.record(stream)
        torch.cuda.synchronize()
        ms.append(a.elapsed_time(b))
    eng.close()
    value = inst["n"] * K * C * rounds * kex / (min(ms) * 1e-3)
    return {"value": value, "unit": "attempts/s", "sweeps": rounds * kex, "rounds": rounds,
            "launches_per_round": "1 sweep launch + exchange_begin + record copy + exchange_end",
            "frac_of_fused_value": value / main_value,
            "note": "driver.run_pt(gather=True) device work at one rank; the default line runs the "
                    "fused schedule (local exchanges, one best-record all-gather per step), which "
                    "gives the same final best record (min over ranks of the per-rank first-reached "
                    "minima, DESIGN.md §7)"}


def run_ours(args):
    import torch
    import torch.distributed as dist

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    e2e_steps = 0 if args.no_e2e else min(args.steps, 5)
    line = measure(args, args.workload, world, rank, local, args.steps, args.warmup, e2e_steps,
                   copies=args.copies, sweeps=args.sweeps, cpu=not args.no_cpu)
    if args.workload in STRONG and world == 1 and not args.copies and not args.no_projection:
        line["scaling_projection"] = scaling_projection(args, line["value"], local)
        try:  # context record; never allowed to break the main line
            line["north_star_mode"] = north_star_mode(args, line["value"], local)
        except Exception as exc:  # pragma: no cover
            line["north_star_mode"] = {"error": repr(exc)[:200]}
    if args.workload != "c5" and not args.no_c5:
        # the HBM-bound config (BASELINE.json configs[4], the north star's 60%-of-HBM target),
        # measured in the same run: 256 replicas per GPU, weak scaling
        c5 = measure(args, "c5", world, rank, local, min(args.steps, 5), min(args.warmup, 3),
                     0 if args.no_e2e else min(args.steps, 3), cpu=not args.no_cpu, quiet_cfg=True)
        line["c5"] = {k: c5[k] for k in ("value", "unit", "ms_per_step", "step_ms_rank0", "steps", "warmup",
                                         "scaling", "dtype", "config", "roofline", "hbm_frac", "e2e",
                                         "gpu_launches", "clocks", "cpu_baseline", "best")}
        if c5["roofline"].get("kernel") == "k_csr_packed" and not args.no_c5_int8:
            # the same workload on the int8 rows themselves (the HBM-bound kernel):
            # the memory-roofline record of BASELINE.json's 60%-of-HBM target
            prev = os.environ.get("ISING_I8_PACKED")
            os.environ["ISING_I8_PACKED"] = "0"
            try:
                c5b = measure(args, "c5", world, rank, local, min(args.steps, 3), min(args.warmup, 3), 0,
                              cpu=False, quiet_cfg=True)
            finally:
                if prev is None:
                    os.environ.pop("ISING_I8_PACKED", None)
                else:
                    os.environ["ISING_I8_PACKED"] = prev
            line["c5"]["int8_rows"] = {k: c5b[k] for k in ("value", "unit", "ms_per_step", "steps", "roofline",
                                                            "hbm_frac", "clocks", "best")}
    if rank == 0:
        json_line(line)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
