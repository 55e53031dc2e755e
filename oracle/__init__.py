"""CPU oracle for the replica-parallel Metropolis + parallel-tempering hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  The product
library (paper_2311_09275_b200) never imports it and shares no code with it
(the C source is oracle/oracle.c, transcribed from DESIGN.md §3 on its own).

The C file holds the per-attempt arithmetic; this wrapper holds the run
schedule of SURVEY.md §8(c) (sweeps, best-so-far check, exchange) in plain
Python/numpy.  Citations: PAPER.md P:53 (PT), P:59 (sweeps), SPEC.md S:261-264,
S:327 (best-so-far, first reached wins).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

RNG_PLANE, RNG_WORD = 0, 1


def build(force: bool = False) -> str:
    """Compile oracle.c (plain C, -O2, no FP contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
                               "-fPIC", "-shared", "-o", _LIB, _SRC, "-lm"])
    return _LIB


class _Run(C.Structure):
    _fields_ = [("n", C.c_int32), ("rp", C.c_void_p), ("col", C.c_void_p), ("wi", C.c_void_p),
                ("wf", C.c_void_p), ("colour", C.c_void_p), ("ncol", C.c_int32),
                ("seed", C.c_uint64), ("K", C.c_int32), ("copy_begin", C.c_int32),
                ("copy_end", C.c_int32), ("beta", C.c_void_p), ("rng", C.c_int32),
                ("slot_lo", C.c_int64), ("slot_hi", C.c_int64)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            vp = C.c_void_p
            L.or_philox4x32_10.argtypes = [vp, vp, vp]
            L.or_p64.argtypes = [C.c_double]
            L.or_p64.restype = C.c_uint64
            L.or_threshold_int.argtypes = [C.c_double, C.c_int64]
            L.or_threshold_int.restype = C.c_uint64
            L.or_threshold_exch.argtypes = [C.c_double, C.c_double, C.c_int64]
            L.or_threshold_exch.restype = C.c_uint64
            L.or_cexp32.argtypes = [C.c_float]
            L.or_cexp32.restype = C.c_float
            L.or_threshold_f32.argtypes = [C.c_double, C.c_float]
            L.or_threshold_f32.restype = C.c_uint64
            L.or_grid_to_csr.argtypes = [C.c_int32, C.c_int32, vp, vp, vp, vp, vp, vp]
            L.or_greedy_colour.argtypes = [C.c_int32, vp, vp, vp]
            L.or_greedy_colour.restype = C.c_int32
            L.or_greedy_colour_sl.argtypes = [C.c_int32, vp, vp, vp]
            L.or_greedy_colour_sl.restype = C.c_int32
            L.or_greedy_colour_jp.argtypes = [C.c_int32, vp, vp, vp, vp]
            L.or_greedy_colour_jp.restype = C.c_int32
            L.or_init.argtypes = [C.POINTER(_Run), vp]
            L.or_energy.argtypes = [C.POINTER(_Run), vp, vp, vp]
            L.or_sweeps.argtypes = [C.POINTER(_Run), vp, vp, C.c_uint32, C.c_int32]
            L.or_sweeps.restype = C.c_int64
            L.or_exchange.argtypes = [C.POINTER(_Run), vp, vp, vp, C.c_uint32]
            L.or_exchange.restype = C.c_int64
            L.or_icm.argtypes = [C.POINTER(_Run), vp, vp, C.c_uint32, C.c_int32]
            L.or_icm.restype = C.c_int64
            _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


# ------------------------------------------------------------------ primitives
def philox(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, np.uint32)
    k = np.ascontiguousarray(key, np.uint32)
    out = np.zeros(4, np.uint32)
    lib().or_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def p64(x: float) -> int:
    return int(lib().or_p64(float(x)))


def threshold_int(beta: float, dE: int) -> int:
    return int(lib().or_threshold_int(float(beta), int(dE)))


def threshold_exch(beta_lo: float, beta_hi: float, d: int) -> int:
    return int(lib().or_threshold_exch(float(beta_lo), float(beta_hi), int(d)))


def cexp32(x: float) -> float:
    return float(lib().or_cexp32(float(x)))


def threshold_f32(beta: float, dE: float) -> int:
    return int(lib().or_threshold_f32(float(beta), float(np.float32(dE))))


def grid_to_csr(Lx, Ly, J_right, J_down):
    n = Lx * Ly
    rp = np.zeros(n + 1, np.int64)
    col = np.zeros(4 * n, np.int32)
    w = np.zeros(4 * n, np.int32)
    colour = np.zeros(n, np.int32)
    Jr = np.ascontiguousarray(J_right, np.int8)
    Jd = np.ascontiguousarray(J_down, np.int8)
    lib().or_grid_to_csr(Lx, Ly, _p(Jr), _p(Jd), _p(rp), _p(col), _p(w), _p(colour))
    return rp, col, w, colour


def greedy_colour(n, row_ptr, col):
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cc = np.ascontiguousarray(col, np.int32)
    out = np.zeros(n, np.int32)
    ncol = lib().or_greedy_colour(n, _p(rp), _p(cc), _p(out))
    return out, int(ncol)


def greedy_colour_sl(n, row_ptr, col):
    """Smallest-last greedy colouring (R12b), the oracle's own implementation."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cc = np.ascontiguousarray(col, np.int32)
    out = np.zeros(n, np.int32)
    ncol = lib().or_greedy_colour_sl(n, _p(rp), _p(cc), _p(out))
    return out, int(ncol)


def greedy_colour_jp(n, row_ptr, col, with_priority=False):
    """Greedy colouring in Jones-Plassmann priority order (R12c), sequentially:
    decreasing Philox priority, ties by lower id, smallest free colour."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cc = np.ascontiguousarray(col, np.int32)
    out = np.zeros(n, np.int32)
    pr = np.zeros(n, np.uint32)
    ncol = lib().or_greedy_colour_jp(n, _p(rp), _p(cc), _p(out), _p(pr))
    return (out, int(ncol), pr) if with_priority else (out, int(ncol))


# ------------------------------------------------------------------ the run
@dataclass
class Best:
    E: float = float("inf")
    slot: int = -1
    sweep: int = -1
    walker: int = -1
    spins: np.ndarray | None = None

    def key(self):
        return (self.E, self.sweep, self.slot)


@dataclass
class Oracle:
    """One PT run over global copies [copy_begin, copy_end) of a K-temperature ladder.

    inst: dict with kind 'grid' (Lx, Ly, J_right, J_down) or 'csr' (n, row_ptr, col,
    w int32 / float32).  colour: None -> checkerboard (grid) / greedy (csr).
    """
    inst: dict
    K: int
    betas: np.ndarray
    seed: int
    copy_begin: int = 0
    copy_end: int = 1
    rng: int = RNG_PLANE
    colour: np.ndarray | None = None
    slots: tuple | None = None  # (lo, hi) global slot subset (no exchange), else whole copies
    t: int = 0
    e: int = 0
    f: int = 0  # Houdayer/ICM steps done
    best: Best = field(default_factory=Best)
    copy_best: list = field(default_factory=list)  # per local copy: Best (trials)

    def __post_init__(self):
        inst = self.inst
        if inst["kind"] == "grid":
            rp, col, w, chk = grid_to_csr(inst["Lx"], inst["Ly"], inst["J_right"], inst["J_down"])
            self.n = inst["Lx"] * inst["Ly"]
            self.wi, self.wf = w, None
            if self.colour is None:
                self.colour = chk
        else:
            self.n = int(inst["n"])
            rp = np.ascontiguousarray(inst["row_ptr"], np.int64)
            col = np.ascontiguousarray(inst["col"], np.int32)
            w = np.asarray(inst["w"])
            if w.dtype == np.float32:
                self.wi, self.wf = None, np.ascontiguousarray(w, np.float32)
            else:
                self.wi, self.wf = np.ascontiguousarray(w, np.int32), None
            if self.colour is None:
                self.colour, _ = greedy_colour(self.n, rp, col)
        self.rp, self.col = rp, col
        self.colour = np.ascontiguousarray(self.colour, np.int32)
        self.ncol = int(self.colour.max()) + 1
        self.betas = np.ascontiguousarray(self.betas, np.float64)
        assert self.betas.size == self.K
        if self.slots is not None:
            self.slot0, self.R = int(self.slots[0]), int(self.slots[1] - self.slots[0])
        else:
            self.R = (self.copy_end - self.copy_begin) * self.K
            self.slot0 = self.copy_begin * self.K
        self.s = np.zeros((self.R, self.n), np.int8)
        self.Ei = np.zeros(self.R, np.int64)
        self.walker = np.arange(self.slot0, self.slot0 + self.R, dtype=np.int64)
        self._run = _Run(self.n, _p(self.rp).value, _p(self.col).value,
                         _p(self.wi).value if self.wi is not None else None,
                         _p(self.wf).value if self.wf is not None else None,
                         _p(self.colour).value, self.ncol, self.seed & (2**64 - 1), self.K,
                         self.copy_begin, self.copy_end, _p(self.betas).value, self.rng,
                         self.slots[0] if self.slots else 0, self.slots[1] if self.slots else 0)
        lib().or_init(C.byref(self._run), _p(self.s))
        self.Ei[:] = self.energy_scratch() if self.wi is not None else 0

    @property
    def is_float(self):
        return self.wf is not None

    def energy_scratch(self) -> np.ndarray:
        Ei = np.zeros(self.R, np.int64)
        Ef = np.zeros(self.R, np.float64)
        lib().or_energy(C.byref(self._run), _p(self.s), _p(Ei), _p(Ef))
        return Ef if self.is_float else Ei

    def energies(self) -> np.ndarray:
        return self.energy_scratch() if self.is_float else self.Ei.copy()

    def sweeps(self, nsweeps: int) -> int:
        acc = lib().or_sweeps(C.byref(self._run), _p(self.s),
                              _p(self.Ei) if not self.is_float else None, self.t, nsweeps)
        self.t += nsweeps
        return int(acc)

    def check_best(self):
        """Best-so-far check (strict <, ascending slot), globally and
        per copy (each copy is one independent trial)."""
        E = self.energies()
        r = int(np.argmin(E))
        if E[r] < self.best.E:
            self.best = Best(E=E[r].item(), slot=self.slot0 + r, sweep=self.t,
                             walker=int(self.walker[r]), spins=self.s[r].copy())
        if self.slots is None:
            if not self.copy_best:
                self.copy_best = [Best() for _ in range(self.copy_end - self.copy_begin)]
            for c in range(self.copy_end - self.copy_begin):
                Ec = E[c * self.K:(c + 1) * self.K]
                k = int(np.argmin(Ec))
                if Ec[k] < self.copy_best[c].E:
                    self.copy_best[c] = Best(E=Ec[k].item(), slot=self.slot0 + c * self.K + k,
                                             sweep=self.t)

    def exchange(self) -> int:
        if self.is_float:
            raise ValueError("exchange requires integer weights")
        if self.slots is not None:
            raise ValueError("slot subsets cannot exchange")
        acc = 0
        if self.K >= 2:
            acc = lib().or_exchange(C.byref(self._run), _p(self.s), _p(self.Ei), _p(self.walker),
                                    self.e)
        self.e += 1
        return int(acc)

    def anneal(self, schedule) -> int:
        """Simulated annealing: sweep s uses schedule[s, k] for temperature index k
        (SPEC.md S:276-284); then a best-so-far check."""
        sched = np.ascontiguousarray(schedule, np.float64)
        acc = 0
        keep = self.betas
        try:
            for s in range(sched.shape[0]):
                self.betas = np.ascontiguousarray(sched[s])
                self._run.beta = _p(self.betas).value
                acc += self.sweeps(1)
        finally:
            self.betas = keep
            self._run.beta = _p(self.betas).value
        self.check_best()
        return acc

    def icm(self, k_min: int) -> int:
        """Houdayer cluster move f on copy pairs (2p, 2p+1) at temperatures k >= k_min."""
        n = lib().or_icm(C.byref(self._run), _p(self.s), _p(self.Ei) if not self.is_float else None,
                         self.f, k_min)
        if n < 0:
            raise ValueError("ICM needs a pair-aligned copy range")
        self.f += 1
        return int(n)

    def run(self, sweeps: int, k_ex: int, icm_k_min: int | None = None):
        """rounds of k_ex sweeps, best check, exchange [, ICM]; final check."""
        if k_ex <= 0:
            self.sweeps(sweeps)
            self.check_best()
            return self
        done = 0
        while done + k_ex <= sweeps:
            self.sweeps(k_ex)
            done += k_ex
            self.check_best()
            self.exchange()
            if icm_k_min is not None:
                self.icm(icm_k_min)
        if done < sweeps:
            self.sweeps(sweeps - done)
            self.check_best()
        return self


def merge_best(bests):
    """Global best from per-shard bests: lexicographic (E, sweep, slot)."""
    cands = [b for b in bests if b.slot >= 0]
    return min(cands, key=lambda b: b.key()) if cands else Best()


def run_sharded(inst, K, betas, seed, copy_begin, copy_end, sweeps, k_ex, rng=RNG_PLANE,
                threads=1, colour=None):
    """Run copies [copy_begin, copy_end) split over `threads` host threads (copies are
    independent PT ladders).  Returns (list of Oracle shards, merged Best)."""
    ncopy = copy_end - copy_begin
    threads = max(1, min(threads, ncopy))
    bounds = [copy_begin + (ncopy * q) // threads for q in range(threads + 1)]
    shards = [None] * threads

    def work(q):
        o = Oracle(inst, K, betas, seed, bounds[q], bounds[q + 1], rng, colour)
        o.run(sweeps, k_ex)
        shards[q] = o

    ts = [threading.Thread(target=work, args=(q,)) for q in range(threads)]
    for th in ts:
        th.start()
    for th in ts:
        th.join()
    return shards, merge_best([o.best for o in shards])
