#!/usr/bin/env python
"""Benchmark of the hot path: replica-parallel Metropolis sweeps + parallel tempering.

Metric (BASELINE.json): spin-flip attempts/s (attempts = n x replicas x sweeps, every
site of every replica counted once per sweep) at N GPUs, plus the
fraction of the roofline of the dominant kernel.

Workload at N=1 (BASELINE.json configs[1], the metric's config): 80x100 +-1 torus
(G65 shape, Table I), 64 temperatures x 64 copies = 4096 replicas, beta
0.1-3.0 geometric, 10,000 sweeps with a replica exchange every 10 sweeps, bit-packed
spins.  One step = that whole schedule (1,000 rounds of 10 sweeps + best check +
exchange) on inputs already resident on the GPU.  N>1: weak scaling -- every rank
runs its own 64-copy shard (distinct global copy ids), local exchanges, and one NCCL
all-gather of the per-rank best records per step.  C4 (--workload c4a|c4b) is strong
scaling as BASELINE.json configs[3] states: 128 copies = 16,384 replicas in total, split
over the N ranks (--copies overrides the copy count, e.g. --workload c4b --copies 16 runs
one rank's share of the 8-GPU job on one GPU).

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
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--sweeps", type=int, default=0, help="override sweeps per step")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--copies", type=int, default=0,
                    help="copies override: per rank (weak-scaling workloads) or in total (c4a/c4b); "
                         "e.g. --workload c4b --copies 16 measures one rank's share at 8 GPUs")
    ap.add_argument("--threads", type=int, default=0, help="CTA size override")
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
    n = inst["n"]
    kex = cfg["k_ex"] if cfg["k_ex"] > 0 else 0
    rng = oracle.RNG_PLANE if cfg["layout"] == "bits" else oracle.RNG_WORD
    colour = None  # the workload's colouring, computed by the oracle's own implementation
    if cfg.get("colouring") == "sl":
        colour, _ = oracle.greedy_colour_sl(n, inst["row_ptr"], inst["col"])
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
def roofline_entry(kernel_ms, attempts_per_launch, layout, clocks, workload="c2"):
    """Roofline of the dominant kernel.  Bit-packed sweeps are issue (ALU) bound: achieved
    = warp instructions per launch (ncu-measured per attempt, profiles/inst_per_attempt.json,
    times the live attempts per launch) / live CUDA-event launch time; peak = 148 SMs x 4
    schedulers x 1 warp-instruction/cycle x max SM clock."""
    peaks = json.load(open(PEAKS_FILE)) if os.path.exists(PEAKS_FILE) else {}
    mhz = peaks.get("sm_max_mhz", 1965.0)
    ipa = None
    if os.path.exists(PROFILE_FILE):
        ipa = json.load(open(PROFILE_FILE)).get(workload)
    if layout == "i8":
        # int8 per-lane sweeps: HBM bound; algorithmic bytes per attempt stated in DESIGN.md
        bpa = ipa.get("alg_bytes_per_attempt", 5.11) if ipa else 5.11
        ach = attempts_per_launch * bpa / (kernel_ms * 1e-3) / 1e9
        peak = peaks.get("hbm_gbs", 6551.4)
        return {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                "traffic": (ipa or {}).get("dram_bytes_per_attempt") and
                ipa["dram_bytes_per_attempt"] * attempts_per_launch,
                "peak_source": "measured (MEASURED_PEAKS.json hbm_gbs)"}
    peak = 148 * 4 * mhz * 1e6 / 1e9  # Ginst/s (warp instructions)
    if not ipa:
        return {"bound": "alu", "achieved": None, "peak": peak, "unit": "Ginst/s", "frac": None,
                "traffic": None, "note": "no ncu instruction count committed yet"}
    ach = attempts_per_launch * ipa["warp_inst_per_attempt"] / (kernel_ms * 1e-3) / 1e9
    traffic = ipa.get("dram_bytes_per_attempt")
    if ipa.get("dram_bytes_per_launch") is not None:  # on-chip state: a fixed load/store per launch
        traffic_launch = ipa["dram_bytes_per_launch"]
    else:
        traffic_launch = traffic * attempts_per_launch if traffic is not None else None
    return {"bound": "alu", "achieved": ach, "peak": peak, "unit": "Ginst/s", "frac": ach / peak,
            "traffic": traffic_launch,
            "peak_source": f"derived: 148 SMs x 4 issue/cycle x {mhz:.0f} MHz (MEASURED_PEAKS sm_max_mhz)",
            "inst_per_attempt_source": ipa.get("source")}


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2311_09275_b200 import Engine
    from paper_2311_09275_b200.driver import merge_best_over_ranks

    world, rank, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    cfg = workload_params(args.workload, args.sweeps)
    inst = synth.make_instance(cfg)
    K, C = cfg["K"], cfg["C"]
    if args.copies:
        C = args.copies
    betas = synth.beta_ladder(K)
    strong = args.workload in STRONG
    if strong:  # BASELINE configs[3]: the 128 copies (16,384 replicas) are sharded over the ranks
        if C % world:
            raise SystemExit(f"{args.workload}: {C} copies do not split over {world} ranks")
        Cg = C
        c_lo, c_hi = rank * C // world, (rank + 1) * C // world
    else:  # weak scaling: every rank runs a C-copy shard with distinct global ids
        Cg = C * world
        c_lo, c_hi = rank * C, (rank + 1) * C
    stream = torch.cuda.current_stream()
    eng = Engine(inst, K, Cg, betas, seed=synth.PHILOX_KEY, copy_begin=c_lo,
                 copy_end=c_hi, layout=cfg["layout"], device=local,
                 block_threads=args.threads, stream=stream.cuda_stream, colour=cfg.get("colouring"))
    n, R = inst["n"], eng.R
    sweeps, kex = cfg["sweeps"], cfg["k_ex"]
    rounds = sweeps // kex if kex > 0 else 0
    rem = sweeps - rounds * kex if kex > 0 else sweeps
    attempts_step = n * R * sweeps  # this rank's attempts per step
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")

    # bit-packed kernels run all rounds in one launch (unless a band-split handle's clusters
    # would not all be resident: then ising_run takes per-round launches, counted as such)
    # (small int8 instances with integer weights, C1, also run all rounds in one launch)
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

    def step(kev=None):
        """One pass of the whole hot path over the workload; returns (our launches, best)."""
        launches = 0
        if fused:
            # all rounds in ONE k_grid_bits launch (clusters exchange through DSMEM) + merge
            timed(kev, eng.run, rounds, kex)
            launches += 2 if fused_one_launch else 3 * rounds
        else:
            for _ in range(rounds):
                timed(kev, eng.sweep, kex)
                eng.exchange()
                launches += (1 if cfg["layout"] == "bits" else kex * eng.info.n_colours + 2) + 2
        if rem:
            timed(kev, eng.sweep, rem)
            eng.check_best()
            launches += (1 if cfg["layout"] == "bits" else rem * eng.info.n_colours + 2) + 1
        rec = eng.best(spins=False)
        if world > 1:
            rec = merge_best_over_ranks(rec, None)
        return launches, rec

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    total_ms, kernel_ms, nk, launches = 0.0, 0.0, 0, 0
    step_ms = []  # this rank's per-step device times (the spread behind the mean)
    clocks.start()
    for _ in range(args.steps):
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
    t = torch.tensor([total_ms], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    value = n * K * Cg * sweeps * args.steps / (total_ms * 1e-3)  # all ranks' attempts
    ms_step = total_ms / args.steps
    avg_launch_ms = kernel_ms / max(nk, 1)
    per_launch_attempts = n * R * (rounds * kex if fused else (kex if kex > 0 else sweeps))
    # instruction counts per attempt are kernel-specific: the band-split kernel has its own entry
    ipa_key = args.workload + ("_bands" if eng.info.bands > 1 else "")
    roof = roofline_entry(avg_launch_ms, per_launch_attempts,
                          "bits" if fused_one_launch else cfg["layout"], clk, ipa_key)
    roof["kernel"] = ("k_grid_bands" if eng.info.bands > 1 else "k_grid_bits") \
        if (inst["kind"] == "grid" and cfg["layout"] == "bits") else \
        ("k_csr_bits" if cfg["layout"] == "bits" else
         ("k_csr_i8_ring" if inst.get("w") is not None and inst["w"].dtype == np.float32 and R % 256 == 0
          else (("k_i8_cluster" if K <= 64 else "k_i8_small") if fused_one_launch else "k_csr_i8_phase")))
    if roof["kernel"] in ("k_i8_small", "k_i8_cluster"):
        per = K // 8 if roof["kernel"] == "k_i8_cluster" else 1
        roof["note"] = (f"{per} CTA(s) per copy: {eng.R // K} copies use {per * (eng.R // K)} of the GPU's "
                        "SMs; frac is against the whole-GPU issue peak")
    roof["kernel_share_of_step"] = kernel_ms / max(total_ms * (1 if world == 1 else 1), 1e-9)
    roof["avg_launch_ms"] = avg_launch_ms

    # ---- end to end through the public API with host buffers, every step
    e2e = None
    if not args.no_e2e:
        e2e_ms = 0.0
        h2d = d2h = 0
        Jr = torch.from_numpy(inst["J_right"]).pin_memory() if inst["kind"] == "grid" else None
        for s in range(args.warmup + args.steps):  # W untimed warm-up steps, then K timed
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            e = Engine(inst, K, Cg, betas, seed=synth.PHILOX_KEY + s, copy_begin=c_lo,
                       copy_end=c_hi, layout=cfg["layout"], device=local,
                       block_threads=args.threads, stream=stream.cuda_stream,
                       colour=cfg.get("colouring"))
            if fused:
                e.run(rounds, kex)
            else:
                for _ in range(rounds):
                    e.sweep(kex)
                    e.exchange()
            if rem:
                e.sweep(rem)
                e.check_best()
            rec = e.best(spins=True)
            E = e.energies()
            b.record(stream)
            torch.cuda.synchronize()
            e.close()
            if s >= args.warmup:
                e2e_ms += a.elapsed_time(b)
        if inst["kind"] == "grid":
            h2d = 2 * n + 8 * K
        else:
            h2d = 8 * (n + 1) + inst["col"].nbytes + inst["w"].nbytes + 8 * K
        d2h = 8 * R + n + 32
        t = torch.tensor([e2e_ms], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e = {"value": n * K * Cg * sweeps * args.steps / (float(t.item()) * 1e-3),
               "unit": "attempts/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "includes": "create (validate, tables, upload, init) + full schedule + best/energy readback"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_oracle_sample(cfg)

    if rank == 0:
        peaks = json.load(open(PEAKS_FILE)) if os.path.exists(PEAKS_FILE) else {}
        bpa = 0.25 if cfg["layout"] == "bits" else 5.11
        json_line({
            "metric": "spin-flip attempts/s", "value": value, "unit": "attempts/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "step_ms_rank0": {"median": float(np.median(step_ms)), "min": min(step_ms), "max": max(step_ms)},
            "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": "u32" if cfg["layout"] == "bits" else ("f32" if cfg["kind"] == "regular" else "int32"),
            "data": "synthetic",
            "config": {"workload": args.workload, "description": WORKLOADS[args.workload],
                       "n": n, "replicas_per_gpu": R, "sweeps_per_step": sweeps, "exchange_every": kex,
                       "copies_total": Cg, "copies_per_gpu": c_hi - c_lo,
                       "parallelism": f"copies sharded over {world} GPU(s), "
                                      + ("strong scaling (fixed total)" if strong else "weak scaling"),
                       "l2": ("flushed between timed steps (256 MB write); the state is SMEM/L2-resident "
                              "by design" if cfg["layout"] == "bits" or n * R < (64 << 20) else
                              "flushed between timed steps (256 MB write); spins (%.2f GB) exceed L2"
                              % (n * R / 1e9))},
            "roofline": roof,
            "hbm_frac": value / world * bpa / 1e9 / peaks.get("hbm_gbs", 6551.4),
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk,
            "best": {k: rec[k] for k in ("E", "slot", "sweep")},
        })
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
