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
    """-> (n, u, v, w) with 0-based endpoints and int32 weights.  Rejects (ValueError, naming
    the edge line -- line 1 is the header) a header that is not two integers, a token count
    other than 2 + 3m (truncated or trailing data), ids out of range, self-loops and
    duplicate undirected edges (S:43-60, S:29-35 instance invariants)."""
    toks = text.split()
    if len(toks) < 2:
        raise ValueError("Gset header 'n m' missing")
    n, m = int(toks[0]), int(toks[1])
    if n < 1 or m < 0:
        raise ValueError(f"bad Gset header: n={n} m={m}")
    if len(toks) != 2 + 3 * m:
        raise ValueError(f"Gset file has {len(toks) - 2} edge tokens, expected 3*m = {3 * m} "
                         f"({'truncated' if len(toks) < 2 + 3 * m else 'trailing data'})")
    a = np.array(toks[2:], dtype=np.int64).reshape(m, 3)
    u, v, w = a[:, 0] - 1, a[:, 1] - 1, a[:, 2]
    bad = np.flatnonzero((u < 0) | (u >= n) | (v < 0) | (v >= n))
    if bad.size:
        raise ValueError(f"vertex id out of range on line {bad[0] + 2}")
    loop = np.flatnonzero(u == v)
    if loop.size:
        raise ValueError(f"self-loop on line {loop[0] + 2}")
    key = np.minimum(u, v) * n + np.maximum(u, v)
    order = np.argsort(key, kind="stable")
    dup = np.flatnonzero(key[order][1:] == key[order][:-1])
    if dup.size:
        raise ValueError(f"duplicate edge on line {int(np.min(order[dup + 1])) + 2}")
    if np.any(np.abs(w) >= 2**31):
        raise ValueError("weight outside int32")
    return n, u, v, w.astype(np.int32)


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
