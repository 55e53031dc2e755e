"""Seeded synthetic input generators shared by the oracle and the CUDA path.

This module holds NONE of the method's arithmetic (no fields, energies,
thresholds, RNG contracts or sweeps).  It only produces problem instances and
run parameters shaped like the paper's workloads:

* +-1 toroidal square grids stand in for the Gset spin-glass instances
  G65/G66/G67/G72/G77/G81 ("random +-1 weights and a toroidal square grid",
  PAPER.md:23, Table I);
* an unweighted sparse random graph G(n, m) stands in for G70 ("Unweighted
  MaxCut on sparse random graph", 10,000 vertices / 9,999 edges);
* a random 3-regular graph with N(0,1) float32 couplings is the scale probe
  ("assess scalability beyond 20,000 variables"; BASELINE.json
  configs[4]).

The Gset files themselves are not in this container, so
nothing here reproduces them; the shapes, sizes and value distributions do.

All randomness is SplitMix64 (Steele, Lea & Flood 2014) evaluated with numpy
uint64 arithmetic, so instances are bit-identical across numpy versions.
"""
from __future__ import annotations

import numpy as np

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int, offset: int = 0) -> np.ndarray:
    """Outputs offset..offset+count-1 of the SplitMix64 stream seeded with `seed`."""
    with np.errstate(over="ignore"):
        k = np.arange(offset + 1, offset + count + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + k * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def _below(z: np.ndarray, n: int) -> np.ndarray:
    """Map uniform uint64 to [0, n) by the high 32 bits (Lemire multiply)."""
    return ((z >> np.uint64(32)) * np.uint64(n) >> np.uint64(32)).astype(np.int64)


def _sub_seed(seed: int, tag: int) -> int:
    return int(splitmix64(seed ^ (tag * 0x632BE59BD9B4E019 & 0xFFFFFFFFFFFFFFFF), 1)[0])


# --------------------------------------------------------------------------- grids
def torus_pm1(Lx: int, Ly: int, seed: int):
    """+-1 equiprobable couplings on an Lx x Ly torus.

    Site i = x + Lx*y.  J_right[i] couples (x,y)-((x+1)%Lx,y); J_down[i] couples
    (x,y)-(x,(y+1)%Ly) (SURVEY.md §8 Conv "Grid").  Returns two int8 arrays.
    """
    n = Lx * Ly
    z = splitmix64(seed, 2 * n)
    bit = (z >> np.uint64(63)).astype(np.int8)
    J = (1 - 2 * bit).astype(np.int8)
    return J[:n].copy(), J[n:].copy()


def torus_edges(Lx: int, Ly: int, J_right: np.ndarray, J_down: np.ndarray):
    """The torus as an undirected edge list (u, v, w) in site order (harness only)."""
    n = Lx * Ly
    i = np.arange(n, dtype=np.int64)
    x, y = i % Lx, i // Lx
    right = ((x + 1) % Lx) + Lx * y
    down = x + Lx * ((y + 1) % Ly)
    u = np.concatenate([i, i])
    v = np.concatenate([right, down])
    w = np.concatenate([J_right, J_down]).astype(np.int32)
    return u, v, w


def checkerboard(Lx: int, Ly: int) -> np.ndarray:
    i = np.arange(Lx * Ly, dtype=np.int64)
    return (((i % Lx) + (i // Lx)) & 1).astype(np.int32)


# --------------------------------------------------------------------------- graphs
def gnm(n: int, m: int, seed: int):
    """Uniform simple graph with n vertices and m edges (rejection of self-loops and
    repeated pairs while drawing uniform pairs in sequence; BASELINE.json configs[2]).
    Returns canonical (u < v) edge arrays sorted lexicographically."""
    if m > n * (n - 1) // 2:
        raise ValueError("too many edges")
    got_u = np.empty(0, np.int64)
    got_v = np.empty(0, np.int64)
    offset = 0
    keys_seen = np.empty(0, np.int64)
    while got_u.size < m:
        batch = max(1024, int(1.3 * (m - got_u.size)) + 64)
        z = splitmix64(seed, 2 * batch, offset)
        offset += 2 * batch
        a = _below(z[0::2], n)
        b = _below(z[1::2], n)
        ok = a != b
        a, b = a[ok], b[ok]
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        key = lo * n + hi
        allkeys = np.concatenate([keys_seen, key])
        _, first = np.unique(allkeys, return_index=True)
        first = np.sort(first)
        first = first[first >= keys_seen.size] - keys_seen.size
        need = m - got_u.size
        first = first[:need]
        got_u = np.concatenate([got_u, lo[first]])
        got_v = np.concatenate([got_v, hi[first]])
        keys_seen = np.concatenate([keys_seen, key[first]])
    order = np.lexsort((got_v, got_u))
    return got_u[order], got_v[order]


def random_regular(n: int, d: int, seed: int, max_tries: int = 200):
    """Uniform simple d-regular graph by the pairing (configuration) model with
    rejection until simple (BASELINE.json configs[4]).  Canonical sorted edges."""
    if (n * d) % 2:
        raise ValueError("n*d must be even")
    stubs = np.repeat(np.arange(n, dtype=np.int64), d)
    for attempt in range(max_tries):
        z = splitmix64(_sub_seed(seed, attempt + 1), stubs.size)
        perm = np.argsort(z, kind="stable")
        p = stubs[perm].reshape(-1, 2)
        a, b = p[:, 0], p[:, 1]
        if np.any(a == b):
            continue
        lo, hi = np.minimum(a, b), np.maximum(a, b)
        key = lo * n + hi
        key.sort()
        if np.any(key[1:] == key[:-1]):
            continue
        return key // n, key % n
    raise RuntimeError("no simple pairing found")


def gaussian_f32(count: int, seed: int) -> np.ndarray:
    """N(0,1) samples by Box-Muller in float64 from SplitMix64, rounded to float32
    (one sample per pair of uniforms, cosine branch)."""
    z = splitmix64(seed, 2 * count)
    u1 = ((z[0::2] >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53  # (0, 1]
    u2 = (z[1::2] >> np.uint64(11)).astype(np.float64) * 2.0 ** -53          # [0, 1)
    g = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
    return g.astype(np.float32)


def edges_to_csr(n: int, u: np.ndarray, v: np.ndarray, w: np.ndarray):
    """Symmetric CSR (row_ptr int64[n+1], col int32[2m], w[2m]); each row sorted by
    neighbour id.  The row order is the caller's order of record (float fold order)."""
    u = np.asarray(u, np.int64)
    v = np.asarray(v, np.int64)
    src = np.concatenate([u, v])
    dst = np.concatenate([v, u])
    ww = np.concatenate([w, w])
    order = np.lexsort((dst, src))
    src, dst, ww = src[order], dst[order], ww[order]
    row_ptr = np.zeros(n + 1, np.int64)
    np.add.at(row_ptr, src + 1, 1)
    row_ptr = np.cumsum(row_ptr)
    return row_ptr, dst.astype(np.int32), ww


def torus_csr(Lx: int, Ly: int, J_right: np.ndarray, J_down: np.ndarray):
    u, v, w = torus_edges(Lx, Ly, J_right, J_down)
    return edges_to_csr(Lx * Ly, u, v, w)


# --------------------------------------------------------------------------- run params
def beta_ladder(K: int, lo: float = 0.1, hi: float = 3.0) -> np.ndarray:
    """Geometric inverse-temperature ladder beta_k = lo*(hi/lo)^(k/(K-1)) (BASELINE.json
    configs: 'geometric beta ladder 0.1-3.0'; SURVEY.md §8(c) reading #7)."""
    if K == 1:
        return np.array([lo], np.float64)
    k = np.arange(K, dtype=np.float64)
    return lo * np.power(hi / lo, k / (K - 1))


# --------------------------------------------------------------------------- presets
PHILOX_KEY = 2311  # SURVEY.md §8(d) proposed seeds

CONFIGS = {
    # BASELINE.json configs[0]: 16x16 torus, 64 replicas, 1000 sweeps, int8 spins
    "c1": dict(kind="grid", Lx=16, Ly=16, seed=1616, K=64, C=1, sweeps=1000, k_ex=10,
               layout="i8"),
    # configs[1]: 80x100 torus, 64 temps x 64 copies, 10000 sweeps, exchange /10, packed
    "c2": dict(kind="grid", Lx=80, Ly=100, seed=65, K=64, C=64, sweeps=10000, k_ex=10,
               layout="bits"),
    # configs[2]: G(1e4, 9999), J=+1, greedy colouring, 4096 replicas, 10000 sweeps
    "c3": dict(kind="gnm", n=10000, m=9999, seed=70, K=64, C=64, sweeps=10000, k_ex=10,
               layout="bits", colouring="sl"),
    # configs[3]: 100x140 / 100x200 tori, 128 temps x 128 copies, 50000 sweeps
    "c4a": dict(kind="grid", Lx=100, Ly=140, seed=77, K=128, C=128, sweeps=50000, k_ex=10,
                layout="bits"),
    "c4b": dict(kind="grid", Lx=100, Ly=200, seed=81, K=128, C=128, sweeps=50000, k_ex=10,
                layout="bits"),
    # configs[4]: random 3-regular 4e6 vertices, N(0,1) f32, 256 replicas/GPU, 1000 sweeps
    "c5": dict(kind="regular", n=4_000_000, d=3, seed=3, K=256, C=1, sweeps=1000, k_ex=0,
               layout="i8", colouring="jp"),
}


def make_instance(cfg: dict):
    """Materialise a preset: returns dict with either grid (Lx, Ly, J_right, J_down)
    or CSR (n, row_ptr, col, w) arrays."""
    kind = cfg["kind"]
    if kind == "grid":
        Jr, Jd = torus_pm1(cfg["Lx"], cfg["Ly"], cfg["seed"])
        return dict(kind="grid", Lx=cfg["Lx"], Ly=cfg["Ly"], J_right=Jr, J_down=Jd,
                    n=cfg["Lx"] * cfg["Ly"])
    if kind == "gnm":
        u, v = gnm(cfg["n"], cfg["m"], cfg["seed"])
        w = np.ones(u.size, np.int32)
        rp, col, ww = edges_to_csr(cfg["n"], u, v, w)
        return dict(kind="csr", n=cfg["n"], row_ptr=rp, col=col, w=ww.astype(np.int32))
    if kind == "regular":
        u, v = random_regular(cfg["n"], cfg["d"], cfg["seed"])
        w = gaussian_f32(u.size, _sub_seed(cfg["seed"], 0xC0FFEE))
        rp, col, ww = edges_to_csr(cfg["n"], u, v, w)
        return dict(kind="csr", n=cfg["n"], row_ptr=rp, col=col, w=ww.astype(np.float32))
    raise ValueError(kind)
