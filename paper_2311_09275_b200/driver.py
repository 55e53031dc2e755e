"""Run schedule of the hot path on top of libising.

`Engine` owns one libising handle (one copy shard on one GPU).  `run_pt` drives
the parallel-tempering schedule -- rounds of `k_ex` Metropolis sweeps, each
followed by a best-so-far check and a replica exchange, plus a final check
("exchanges replicas across temperatures"; P:59 sweeps as the unit
of work; SPEC.md S:261-264/S:327 best-so-far, first reached wins).

Multi-GPU: one process per GPU, copies sharded contiguously over ranks (copies
are independent PT ladders).  Exchange decisions only need a
copy's own energies, so they are local.  Two modes:
  * gather=True  -- north-star mode: each exchange all-gathers the 16-byte
    per-slot records (energy, global slot) over NCCL; every rank then applies the
    same global best-so-far rule (exchange_end);
  * gather=False -- each rank keeps its local best; one all-gather of the
    per-rank best records at the end, merged by (E, sweep, slot).
Both give the same record as a single process holding all copies (tests).
"""
from __future__ import annotations

import numpy as np

from . import ising as L


class Engine:
    """One libising handle.  inst: dict from synth.make_instance (grid or csr).  colour (csr):
    None = the library's ascending-id greedy colouring, "sl" = smallest-last greedy
    (ising_greedy_colour_sl, host), "jp" = greedy in Jones-Plassmann priority order (computed
    by the library on the GPU), or an explicit int32 array (validated by the library)."""

    def __init__(self, inst: dict, K: int, C: int, betas, seed: int, copy_begin: int = 0,
                 copy_end: int | None = None, layout: str = "bits", device: int = 0,
                 colour=None, block_threads: int = 0, stream=None):
        kw = dict(seed=seed, n_temps=K, n_copies=C, betas=betas, copy_begin=copy_begin,
                  copy_end=C if copy_end is None else copy_end, layout=layout, device=device,
                  block_threads=block_threads, stream=stream)
        if inst["kind"] == "grid":
            self.h = L.ising_create_grid(inst["Lx"], inst["Ly"], inst["J_right"], inst["J_down"], **kw)
        else:
            if isinstance(colour, str):
                if colour == "sl":  # the library's smallest-last greedy colouring (host)
                    colour, _ = L.ising_greedy_colour_sl(inst["n"], inst["row_ptr"], inst["col"])
                elif colour == "jp":  # greedy in Jones-Plassmann order, computed on the GPU in create
                    kw["colouring"] = L.ISING_COLOUR_JP
                    colour = None
                else:
                    raise ValueError(f"unknown colouring {colour!r}")
            self.h = L.ising_create_csr(inst["n"], inst["row_ptr"], inst["col"], inst["w"],
                                        colour=colour, **kw)
        self.info = L.ising_info(self.h)
        self.device = device
        self.K, self.C = K, C
        self.R = int(self.info.n_slots)
        self.slot0 = int(self.info.slot_begin)
        self.is_float = self.info.wtype == L.ISING_W_F32

    # ---- hot path
    def sweep(self, n: int):
        L.ising_sweep(self.h, n)

    def exchange(self):
        L.ising_exchange(self.h)

    def anneal(self, schedule):
        """Simulated annealing: sweep s uses schedule[s, k] for temperature index k."""
        L.ising_anneal(self.h, schedule)

    def icm(self, k_min: int):
        """Houdayer cluster move on copy pairs at temperatures k >= k_min."""
        L.ising_icm(self.h, k_min)

    def run(self, n_rounds: int, k_ex: int):
        """n_rounds x (k_ex sweeps + exchange); one fused launch on bit-packed tori."""
        L.ising_run(self.h, n_rounds, k_ex)

    def exchange_begin(self, send):
        L.ising_exchange_begin(self.h, send.data_ptr())

    def exchange_end(self, recv):
        L.ising_exchange_end(self.h, recv.data_ptr(), recv.shape[0])

    def check_best(self, recv=None):
        if recv is None:
            L.ising_check_best(self.h)
        else:
            L.ising_check_best(self.h, recv.data_ptr(), recv.shape[0])

    def record_buffers(self, world: int):
        import torch
        dev = torch.device("cuda", self.device)
        send = torch.empty((self.R, 2), dtype=torch.int64, device=dev)
        recv = torch.empty((self.R * world, 2), dtype=torch.int64, device=dev)
        return send, recv

    # ---- readback
    def energies(self):
        return L.ising_energy(self.h)

    def cuts(self):
        return L.ising_cut(self.h)

    def best(self, spins: bool = True):
        try:
            return L.ising_best(self.h, spins=spins)
        except L.IsingError as e:
            if e.code == L.ISING_E_STATE and spins:
                return L.ising_best(self.h, spins=False)
            raise

    def merge_best(self, recs):
        """Global best over gathered ising_best_record rows (int64 tensor [n, 3]: energy bits,
        sweep, slot) by the library's device merge."""
        import torch
        d = recs.to(torch.device("cuda", self.device)).contiguous()
        r = L.ising_merge_best(self.h, d.data_ptr(), d.shape[0])
        return r

    def copy_best(self):
        """Per-copy best-so-far (E[C_local], slot[C_local], sweep[C_local])."""
        return L.ising_copy_best(self.h)

    def spins(self, slot: int):
        return L.ising_get_spins(self.h, slot)

    def set_spins(self, slot: int, s):
        L.ising_set_spins(self.h, slot, s)

    def walkers(self):
        return L.ising_get_walkers(self.h)

    def sync(self):
        L.ising_sync(self.h)

    # ---- checkpoint / resume (include/ising.h ising_state_*)
    def save_state(self) -> bytes:
        """Complete dynamic state (spins, energies, walkers, counters, best records)."""
        return L.ising_state_save(self.h)

    def load_state(self, blob: bytes):
        """Resume from save_state of an Engine built from the same instance and arguments."""
        L.ising_state_load(self.h, blob)

    def close(self):
        if getattr(self, "h", None):
            L.ising_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def geometric_schedule(betas, sweeps: int, start: float, end: float):
    """Annealing schedule: every slot's beta_k scaled by a geometric ramp from `start` to
    `end` over the sweeps ("T multiplied by the geometric factor each
    sweep")."""
    betas = np.asarray(betas, np.float64)
    if sweeps == 1:
        return (betas * end)[None, :]
    s = np.arange(sweeps, dtype=np.float64) / (sweeps - 1)
    ramp = start * np.power(end / start, s)
    return ramp[:, None] * betas[None, :]


def shard(C: int, world: int, rank: int):
    """Contiguous copy shard of `rank` (copies split as evenly as possible)."""
    return (C * rank) // world, (C * (rank + 1)) // world


def best_key(rec):
    return (rec["E"], rec["sweep"], rec["slot"])


def all_gather(recv, send, group=None):
    """all_gather_into_tensor where the backend has it (NCCL), list all_gather otherwise."""
    import torch
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        torch.cuda.nvtx.range_push("record_all_gather")  # NVTX, next to the library's ranges
        dist.all_gather_into_tensor(recv, send, group=group)
        torch.cuda.nvtx.range_pop()
        return
    world = dist.get_world_size(group)
    host = send.device.type != "cpu"  # gloo: gather host copies of device records
    src = send.cpu() if host else send
    bufs = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(bufs, src, group=group)
    recv.copy_(torch.cat(bufs, dim=0))


def run_pt(engine, sweeps: int, k_ex: int, group=None, gather: bool = True, fused: bool = True,
           icm_k_min: int | None = None):
    """PT schedule: rounds of k_ex sweeps + (best check, exchange); final check.

    k_ex <= 0 -> plain Metropolis (no exchange), one best check at the end.
    fused: local exchanges go through Engine.run (one launch for all rounds where the
    kernel supports it); the record gather of north-star mode needs per-round calls.
    Returns the global best record {E, slot, sweep} (same on every rank)."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    multi = world > 1
    done = 0
    if multi and gather:
        send, recv = engine.record_buffers(world)
    if k_ex > 0 and fused and icm_k_min is None and not (multi and gather) and hasattr(engine, "run"):
        rounds = sweeps // k_ex
        if rounds:
            engine.run(rounds, k_ex)
            done = rounds * k_ex
    if k_ex > 0:
        while done + k_ex <= sweeps:
            engine.sweep(k_ex)
            done += k_ex
            if multi and gather:
                engine.exchange_begin(send)
                all_gather(recv, send, group)
                engine.exchange_end(recv)
            else:
                engine.exchange()
            if icm_k_min is not None:  # Houdayer/ICM after each exchange
                engine.icm(icm_k_min)
    if done < sweeps or k_ex <= 0:
        engine.sweep(sweeps - done)
        if multi and gather:
            engine.exchange_begin(send)
            all_gather(recv, send, group)
            engine.check_best(recv)
        else:
            engine.check_best()
    rec = engine.best(spins=False)
    if multi and not gather:
        rec = merge_best_over_ranks(rec, group, engine)
    return {k: rec[k] for k in ("E", "slot", "sweep")}


def merge_best_over_ranks(rec, group, engine):
    """Global best over the ranks' local best records: one all-gather of a 24-byte
    ising_best_record per rank (energy, sweep, slot), merged by the library on the device
    (ising_merge_best: lexicographic (E, sweep, slot), S:327 first reached)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", engine.device) if backend == "nccl" else torch.device("cpu")
    E = rec["E"]
    e_bits = int(np.array([E], np.float64).view(np.int64)[0]) if isinstance(E, float) else int(E)
    mine = torch.tensor([[e_bits, rec["sweep"], rec["slot"]]], dtype=torch.int64, device=dev)
    allr = torch.empty((world, 3), dtype=torch.int64, device=dev)
    all_gather(allr, mine, group)
    return engine.merge_best(allr)
