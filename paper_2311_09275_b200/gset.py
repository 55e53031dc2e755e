"""Gset file I/O, hexadecimal solution codec and cut certification.

Gset format (the instance files of the benchmark named in PAPER.md P:21-35): a first line
"n m", then m lines "u v w" with 1-based vertex ids.  The instance files themselves are not
in this container; the parser is exercised on files this module writes.

Solution bitstrings (Appendix II/III): "expanding the hexadecimal string
to binary values representing variables 1 to n from left to right" -- each hex digit gives 4
bits, most significant first (SURVEY §8(c) reading #24).  Bit 1 <-> spin -1 (the cut
is invariant under the global flip, so either mapping certifies the same value).

certify() evaluates the cut of a configuration twice: on the host from its definition
(sum of w over edges whose endpoints differ) and on the GPU through the library
(ising_set_spins + ising_cut), and reports both.
"""
from __future__ import annotations

import numpy as np


def parse_gset(text: str):
    """-> (n, u, v, w) with 0-based endpoints and int32 weights."""
    toks = text.split()
    n, m = int(toks[0]), int(toks[1])
    a = np.array(toks[2:2 + 3 * m], dtype=np.int64).reshape(m, 3)
    if a.shape[0] != m:
        raise ValueError("truncated Gset file")
    u, v, w = a[:, 0] - 1, a[:, 1] - 1, a[:, 2].astype(np.int32)
    if np.any((u < 0) | (u >= n) | (v < 0) | (v >= n)):
        raise ValueError("vertex id out of range")
    return n, u, v, w


def write_gset(n: int, u, v, w) -> str:
    lines = [f"{n} {len(u)}"]
    lines += [f"{a + 1} {b + 1} {c}" for a, b, c in zip(np.asarray(u), np.asarray(v), np.asarray(w))]
    return "\n".join(lines) + "\n"


def decode_hex(hexstr: str, n: int) -> np.ndarray:
    """Hex digits (whitespace ignored) -> n bits, MSB first; only final-digit padding allowed."""
    s = "".join(hexstr.split())
    if any(ch not in "0123456789abcdefABCDEF" for ch in s):
        raise ValueError("non-hex character")
    if 4 * len(s) < n:
        raise ValueError(f"{len(s)} hex digits give {4 * len(s)} bits < n = {n}")
    if 4 * len(s) - n >= 4:
        raise ValueError("more hex digits than n needs")
    vals = np.array([int(ch, 16) for ch in s], dtype=np.uint8)
    bits = ((vals[:, None] >> np.arange(3, -1, -1)[None, :]) & 1).reshape(-1)
    return bits[:n].astype(np.uint8)


def encode_hex(bits) -> str:
    b = np.asarray(bits, dtype=np.uint8)
    pad = (-b.size) % 4
    b = np.concatenate([b, np.zeros(pad, np.uint8)]).reshape(-1, 4)
    vals = (b * np.array([8, 4, 2, 1], np.uint8)).sum(axis=1)
    return "".join("0123456789ABCDEF"[x] for x in vals)


def bits_to_spins(bits) -> np.ndarray:
    return (1 - 2 * np.asarray(bits, dtype=np.int8)).astype(np.int8)


def cut_of(u, v, w, spins) -> int:
    s = np.asarray(spins)
    return int(np.sum(np.where(s[u] != s[v], w, 0)))


def certify(n, u, v, w, spins, claimed=None, device: int = 0):
    """Cut of `spins` on the instance: host definition and GPU library value."""
    from synth import edges_to_csr
    from . import ising as L
    rp, col, ww = edges_to_csr(n, u, v, w)
    host = cut_of(u, v, w, spins)
    betas = np.linspace(0.1, 3.0, 8)
    h = L.ising_create_csr(n, rp, col, ww.astype(np.int32), seed=1, n_temps=8, n_copies=1,
                           betas=betas, layout="i8", device=device)
    try:
        L.ising_set_spins(h, 0, spins)
        gpu = int(L.ising_cut(h)[0])
    finally:
        L.ising_destroy(h)
    return dict(cut=host, cut_gpu=gpu, matches_claim=None if claimed is None else host == claimed)
