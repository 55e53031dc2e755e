"""Thin ctypes binding of libising.so (include/ising.h), same names as the C ABI.

Argument marshalling only: every step of the hot path runs in the library's CUDA
kernels.  There is no CPU fallback -- if the shared library or a GPU is missing,
the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import build as _build

ISING_OK, ISING_E_ARG, ISING_E_GRAPH, ISING_E_UNSUPPORTED = 0, -1, -2, -3
ISING_E_CUDA, ISING_E_OOM, ISING_E_STATE = -4, -5, -6
ISING_W_I32, ISING_W_F32 = 0, 1
ISING_SPINS_BITS, ISING_SPINS_I8 = 0, 1
ISING_RNG_PLANE, ISING_RNG_WORD = 0, 1
ISING_COLOUR_GREEDY, ISING_COLOUR_JP = 0, 1

LAYOUTS = {"bits": ISING_SPINS_BITS, "i8": ISING_SPINS_I8}

EXPORTED = [
    "ising_create_grid", "ising_create_csr", "ising_sweep", "ising_run", "ising_anneal", "ising_energy", "ising_cut",
    "ising_exchange", "ising_icm", "ising_exchange_begin", "ising_exchange_end", "ising_check_best",
    "ising_best", "ising_merge_best", "ising_copy_best", "ising_get_spins", "ising_set_spins", "ising_get_walkers", "ising_info",
    "ising_sync", "ising_last_error", "ising_destroy", "ising_greedy_colour", "ising_greedy_colour_sl", "ising_colour_jp", "ising_threshold",
    "ising_version", "ising_debug_philox", "ising_debug_exp_bound",
    "ising_state_size", "ising_state_save", "ising_state_load",
]


class IsingError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libising error {code}: {msg}")
        self.code = code


class RunDesc(C.Structure):
    _fields_ = [("seed", C.c_uint64), ("n_temps", C.c_int32), ("n_copies", C.c_int32),
                ("copy_begin", C.c_int32), ("copy_end", C.c_int32), ("betas", C.c_void_p),
                ("layout", C.c_int32), ("rng", C.c_int32), ("device", C.c_int32),
                ("block_threads", C.c_int32), ("stream", C.c_void_p), ("colouring", C.c_int32)]


class Record(C.Structure):
    _fields_ = [("energy", C.c_int64), ("slot", C.c_int64)]


class Info(C.Structure):
    _fields_ = [("n", C.c_int32), ("n_colours", C.c_int32), ("n_edges", C.c_int64),
                ("n_temps", C.c_int32), ("n_copies", C.c_int32), ("copy_begin", C.c_int32),
                ("copy_end", C.c_int32), ("slot_begin", C.c_int64), ("n_slots", C.c_int64),
                ("layout", C.c_int32), ("rng", C.c_int32), ("wtype", C.c_int32),
                ("kernel", C.c_int32), ("sweeps_done", C.c_int64), ("exchanges_done", C.c_int64),
                ("W_int", C.c_int64), ("W_f64", C.c_double), ("bands", C.c_int32), ("fused_pt", C.c_int32)]


_lib = None


def lib(build_if_missing: bool = True):
    """Load libising.so from the package tree (built in-tree by __graft_entry__.build())."""
    global _lib
    if _lib is not None:
        return _lib
    path = _build.LIB
    if _build.needs_build():  # missing, or older than a source file: never load a stale binary
        if not build_if_missing:
            raise ImportError(f"libising.so missing or older than its sources: {path}")
        _build.build()
    L = C.CDLL(path)
    vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
    sig = {
        "ising_create_grid": ([i32, i32, vp, vp, C.POINTER(RunDesc), C.POINTER(vp)], C.c_int),
        "ising_create_csr": ([i32, vp, vp, vp, i32, vp, C.POINTER(RunDesc), C.POINTER(vp)], C.c_int),
        "ising_sweep": ([vp, i32], C.c_int),
        "ising_run": ([vp, i32, i32], C.c_int),
        "ising_anneal": ([vp, i32, vp], C.c_int),
        "ising_energy": ([vp, vp], C.c_int),
        "ising_cut": ([vp, vp], C.c_int),
        "ising_exchange": ([vp], C.c_int),
        "ising_icm": ([vp, i32], C.c_int),
        "ising_exchange_begin": ([vp, vp], C.c_int),
        "ising_exchange_end": ([vp, vp, i64], C.c_int),
        "ising_check_best": ([vp, vp, i64], C.c_int),
        "ising_best": ([vp, vp, C.POINTER(i64), C.POINTER(i64), vp], C.c_int),
        "ising_merge_best": ([vp, vp, i64, vp, C.POINTER(i64), C.POINTER(i64)], C.c_int),
        "ising_get_spins": ([vp, i64, vp], C.c_int),
        "ising_copy_best": ([vp, vp, vp, vp], C.c_int),
        "ising_set_spins": ([vp, i64, vp], C.c_int),
        "ising_get_walkers": ([vp, vp], C.c_int),
        "ising_info": ([vp, C.POINTER(Info)], C.c_int),
        "ising_state_size": ([vp, C.POINTER(i64)], C.c_int),
        "ising_state_save": ([vp, vp, i64], C.c_int),
        "ising_state_load": ([vp, vp, i64], C.c_int),
        "ising_sync": ([vp], C.c_int),
        "ising_last_error": ([], C.c_char_p),
        "ising_destroy": ([vp], None),
        "ising_greedy_colour": ([i32, vp, vp, vp], C.c_int),
        "ising_greedy_colour_sl": ([i32, vp, vp, vp], C.c_int),
        "ising_colour_jp": ([i32, i32, vp, vp, vp], C.c_int),
        "ising_threshold": ([C.c_double, i64], C.c_uint64),
        "ising_version": ([], C.c_char_p),
        "ising_debug_philox": ([i32, vp, i32, vp, vp], C.c_int),
        "ising_debug_exp_bound": ([i32, vp, i32, C.POINTER(C.c_float), C.POINTER(C.c_float)], C.c_int),
    }
    for name, (args, res) in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = res
    _lib = L
    return L


def _check(rc: int):
    if rc != ISING_OK:
        raise IsingError(rc, lib().ising_last_error().decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _current_stream(stream, device=0):
    """The caller's stream, else torch's current stream OF THE HANDLE'S DEVICE (not of torch's
    current device: a handle on device d must enqueue on a stream of d)."""
    if stream is not None:
        return stream
    try:
        import torch
        if torch.cuda.is_available():
            return torch.cuda.current_stream(device).cuda_stream
    except Exception:  # pragma: no cover - torch absent
        pass
    return None


def _desc(seed, n_temps, n_copies, betas, copy_begin=0, copy_end=None, layout="bits", device=0,
          block_threads=0, stream=None, colouring=ISING_COLOUR_GREEDY):
    betas = np.ascontiguousarray(betas, np.float64)
    lay = LAYOUTS[layout] if isinstance(layout, str) else int(layout)
    d = RunDesc(seed=seed & (2**64 - 1), n_temps=n_temps, n_copies=n_copies,
                copy_begin=copy_begin, copy_end=n_copies if copy_end is None else copy_end,
                betas=betas.ctypes.data, layout=lay,
                rng=ISING_RNG_PLANE if lay == ISING_SPINS_BITS else ISING_RNG_WORD,
                device=device, block_threads=block_threads, stream=_current_stream(stream, device),
                colouring=colouring)
    return d, betas


# ------------------------------------------------------------------ ABI wrappers
def ising_create_grid(Lx, Ly, J_right, J_down, **desc_kw):
    d, _keep = _desc(**desc_kw)
    Jr = np.ascontiguousarray(J_right, np.int8)
    Jd = np.ascontiguousarray(J_down, np.int8)
    h = C.c_void_p()
    _check(lib().ising_create_grid(int(Lx), int(Ly), _ptr(Jr), _ptr(Jd), C.byref(d), C.byref(h)))
    return h


def ising_create_csr(n, row_ptr, col, w, colour=None, **desc_kw):
    d, _keep = _desc(**desc_kw)
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cc = np.ascontiguousarray(col, np.int32)
    w = np.asarray(w)
    if w.dtype == np.float32:
        ww, wt = np.ascontiguousarray(w, np.float32), ISING_W_F32
    else:
        ww, wt = np.ascontiguousarray(w, np.int32), ISING_W_I32
    colp = _ptr(np.ascontiguousarray(colour, np.int32)) if colour is not None else None
    keep = np.ascontiguousarray(colour, np.int32) if colour is not None else None
    if keep is not None:
        colp = _ptr(keep)
    h = C.c_void_p()
    _check(lib().ising_create_csr(int(n), _ptr(rp), _ptr(cc), _ptr(ww), wt, colp, C.byref(d),
                                  C.byref(h)))
    return h


def ising_info(h) -> Info:
    info = Info()
    _check(lib().ising_info(h, C.byref(info)))
    return info


def ising_sweep(h, n_sweeps: int):
    _check(lib().ising_sweep(h, int(n_sweeps)))


def ising_run(h, n_rounds: int, k_ex: int):
    _check(lib().ising_run(h, int(n_rounds), int(k_ex)))


def ising_anneal(h, schedule):
    """schedule: (n_sweeps, K) inverse temperatures."""
    s = np.ascontiguousarray(schedule, np.float64)
    _check(lib().ising_anneal(h, int(s.shape[0]), _ptr(s)))


def ising_energy(h) -> np.ndarray:
    info = ising_info(h)
    out = np.zeros(info.n_slots, np.float64 if info.wtype == ISING_W_F32 else np.int64)
    _check(lib().ising_energy(h, _ptr(out)))
    return out


def ising_cut(h) -> np.ndarray:
    info = ising_info(h)
    out = np.zeros(info.n_slots, np.float64 if info.wtype == ISING_W_F32 else np.int64)
    _check(lib().ising_cut(h, _ptr(out)))
    return out


def ising_exchange(h):
    _check(lib().ising_exchange(h))


def ising_icm(h, k_min: int):
    _check(lib().ising_icm(h, int(k_min)))


def ising_exchange_begin(h, dev_send_ptr: int):
    _check(lib().ising_exchange_begin(h, C.c_void_p(dev_send_ptr)))


def ising_exchange_end(h, dev_recv_ptr: int, n_records: int):
    _check(lib().ising_exchange_end(h, C.c_void_p(dev_recv_ptr), int(n_records)))


def ising_check_best(h, dev_recv_ptr: int | None = None, n_records: int = 0):
    _check(lib().ising_check_best(h, C.c_void_p(dev_recv_ptr) if dev_recv_ptr else None,
                                  int(n_records)))


def ising_best(h, spins: bool = True):
    info = ising_info(h)
    e = np.zeros(1, np.float64 if info.wtype == ISING_W_F32 else np.int64)
    slot, sweep = C.c_int64(), C.c_int64()
    sp = np.zeros(info.n, np.int8) if spins else None
    _check(lib().ising_best(h, _ptr(e), C.byref(slot), C.byref(sweep),
                            _ptr(sp) if sp is not None else None))
    return dict(E=e[0].item(), slot=slot.value, sweep=sweep.value, spins=sp)


def ising_merge_best(h, dev_recs_ptr: int, n: int):
    """Global best over n gathered ising_best_record (device memory, 24 bytes each)."""
    info = ising_info(h)
    e = np.zeros(1, np.float64 if info.wtype == ISING_W_F32 else np.int64)
    slot, sweep = C.c_int64(), C.c_int64()
    _check(lib().ising_merge_best(h, C.c_void_p(dev_recs_ptr), int(n), _ptr(e), C.byref(slot), C.byref(sweep)))
    return dict(E=e[0].item(), slot=slot.value, sweep=sweep.value)


def ising_copy_best(h):
    info = ising_info(h)
    nc = info.copy_end - info.copy_begin
    e = np.zeros(nc, np.float64 if info.wtype == ISING_W_F32 else np.int64)
    slot = np.zeros(nc, np.int64)
    sweep = np.zeros(nc, np.int64)
    _check(lib().ising_copy_best(h, _ptr(e), _ptr(slot), _ptr(sweep)))
    return e, slot, sweep


def ising_get_spins(h, slot: int) -> np.ndarray:
    info = ising_info(h)
    out = np.zeros(info.n, np.int8)
    _check(lib().ising_get_spins(h, int(slot), _ptr(out)))
    return out


def ising_set_spins(h, slot: int, spins):
    s = np.ascontiguousarray(spins, np.int8)
    _check(lib().ising_set_spins(h, int(slot), _ptr(s)))


def ising_get_walkers(h) -> np.ndarray:
    info = ising_info(h)
    out = np.zeros(info.n_slots, np.int64)
    _check(lib().ising_get_walkers(h, _ptr(out)))
    return out


def ising_state_size(h) -> int:
    n = C.c_int64(0)
    _check(lib().ising_state_size(h, C.byref(n)))
    return n.value


def ising_state_save(h) -> bytes:
    """Checkpoint blob of the handle's complete dynamic state (include/ising.h)."""
    buf = np.zeros(ising_state_size(h), np.uint8)
    _check(lib().ising_state_save(h, _ptr(buf), buf.size))
    return buf.tobytes()


def ising_state_load(h, blob: bytes):
    """Restore a blob written by ising_state_save on a handle of the same instance/desc."""
    buf = np.frombuffer(bytes(blob), np.uint8).copy()
    _check(lib().ising_state_load(h, _ptr(buf), buf.size))


def ising_sync(h):
    _check(lib().ising_sync(h))


def ising_destroy(h):
    if h:
        lib().ising_destroy(h)


def ising_last_error() -> str:
    return lib().ising_last_error().decode()


def ising_version() -> str:
    return lib().ising_version().decode()


def ising_greedy_colour(n, row_ptr, col):
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cc = np.ascontiguousarray(col, np.int32)
    out = np.zeros(n, np.int32)
    rc = lib().ising_greedy_colour(int(n), _ptr(rp), _ptr(cc), _ptr(out))
    if rc < 0:
        _check(rc)
    return out, rc


def ising_greedy_colour_sl(n, row_ptr, col):
    """Smallest-last greedy colouring (include/ising.h); returns (colour, n_colours)."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cc = np.ascontiguousarray(col, np.int32)
    out = np.zeros(n, np.int32)
    rc = lib().ising_greedy_colour_sl(int(n), _ptr(rp), _ptr(cc), _ptr(out))
    if rc < 0:
        _check(rc)
    return out, rc


def ising_colour_jp(n, row_ptr, col, device: int = 0):
    """Greedy colouring in Jones-Plassmann priority order, computed on the GPU (include/ising.h);
    returns (colour, n_colours)."""
    rp = np.ascontiguousarray(row_ptr, np.int64)
    cc = np.ascontiguousarray(col, np.int32)
    out = np.zeros(n, np.int32)
    rc = lib().ising_colour_jp(int(device), int(n), _ptr(rp), _ptr(cc), _ptr(out))
    if rc < 0:
        _check(rc)
    return out, rc


def ising_threshold(beta: float, dE: int) -> int:
    return int(lib().ising_threshold(float(beta), int(dE)))


def ising_debug_philox(tuples, device: int = 0):
    a = np.ascontiguousarray(tuples, np.uint32).reshape(-1, 6)
    n = a.shape[0]
    o1 = np.zeros((n, 4), np.uint32)
    o2 = np.zeros((n, 4), np.uint32)
    _check(lib().ising_debug_philox(device, _ptr(a), n, _ptr(o1), _ptr(o2)))
    return o1, o2


def ising_debug_exp_bound(beta2, device: int = 0):
    """(worst relative error where c >= 1/2, max estimate where c < 1/2) of the I8 kernels'
    fast float decision over every float field value, for each slope 2*beta in beta2."""
    b = np.ascontiguousarray(beta2, np.float32)
    worst, small = C.c_float(), C.c_float()
    _check(lib().ising_debug_exp_bound(device, _ptr(b), b.size, C.byref(worst), C.byref(small)))
    return worst.value, small.value
