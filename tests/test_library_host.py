"""Host-side checks of libising.so that need no GPU: the library loads, exports every
symbol include/ising.h declares, its host tables/colouring agree with the oracle's
independent implementation, and create() validates inputs before touching a device."""
import os
import re

import numpy as np
import pytest

import oracle
import synth
from paper_2311_09275_b200 import ising as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "ising.h")).read()
    return sorted(set(re.findall(r"ISING_API[^;(]*?\b(ising_\w+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    lib = L.lib()
    names = header_functions()
    assert len(names) >= 20
    for nm in names:
        assert hasattr(lib, nm), nm
    assert set(names) == set(L.EXPORTED)
    assert "sm_100a" in L.ising_version()


def test_threshold_table_matches_oracle():
    for beta in synth.beta_ladder(64)[::5]:
        for dE in (2, 4, 6, 8, 10, 20):
            assert L.ising_threshold(beta, dE) == oracle.threshold_int(beta, dE)


def test_greedy_colouring_matches_oracle():
    u, v = synth.gnm(3000, 2999, 70)
    rp, col, _ = synth.edges_to_csr(3000, u, v, np.ones(u.size, np.int32))
    a, na = L.ising_greedy_colour(3000, rp, col)
    b, nb = oracle.greedy_colour(3000, rp, col)
    assert na == nb and np.array_equal(a, b)


def test_smallest_last_colouring_matches_oracle():
    for n, m, seed in ((3000, 2999, 70), (2000, 3000, 3)):
        u, v = synth.gnm(n, m, seed)
        rp, col, _ = synth.edges_to_csr(n, u, v, np.ones(u.size, np.int32))
        a, na = L.ising_greedy_colour_sl(n, rp, col)
        b, nb = oracle.greedy_colour_sl(n, rp, col)
        assert na == nb and np.array_equal(a, b)
    u, v = synth.random_regular(3000, 3, 9)
    rp, col, _ = synth.edges_to_csr(3000, u, v, np.ones(u.size, np.int32))
    a, na = L.ising_greedy_colour_sl(3000, rp, col)
    b, nb = oracle.greedy_colour_sl(3000, rp, col)
    assert na == nb and np.array_equal(a, b)
    # bitmap buckets with degrees beyond one byte (the 32-bit remaining-degree array): a hub of
    # 400 leaves inside a sparse random graph on 3000 vertices
    n = 3000
    x, y = synth.gnm(n, 3000, 12)
    keep = (x != 0) & (y != 0)
    u = np.concatenate([np.zeros(400, np.int64), x[keep]])
    v = np.concatenate([np.arange(1, 401, dtype=np.int64), y[keep]])
    pairs = {(min(a_, b_), max(a_, b_)) for a_, b_ in zip(u.tolist(), v.tolist())}
    u = np.array([p[0] for p in sorted(pairs)], np.int64)
    v = np.array([p[1] for p in sorted(pairs)], np.int64)
    rp, col, _ = synth.edges_to_csr(n, u, v, np.ones(u.size, np.int32))
    assert int(np.diff(rp).max()) >= 255
    a, na = L.ising_greedy_colour_sl(n, rp, col)
    b, nb = oracle.greedy_colour_sl(n, rp, col)
    assert na == nb and np.array_equal(a, b)
    # the library's bitmap buckets give way to its heap when (max degree + 1) x n / 64
    # words exceed 2^25: a star on 2^16 vertices plus a sparse random part takes that path
    n = 1 << 16
    hub = np.zeros(n - 1, np.int64)
    leaves = np.arange(1, n, dtype=np.int64)
    x, y = synth.gnm(n - 1, 4000, 11)
    u = np.concatenate([hub, x + 1])
    v = np.concatenate([leaves, y + 1])
    rp, col, _ = synth.edges_to_csr(n, u, v, np.ones(u.size, np.int32))
    a, na = L.ising_greedy_colour_sl(n, rp, col)
    b, nb = oracle.greedy_colour_sl(n, rp, col)
    assert na == nb and np.array_equal(a, b)


def _desc(**kw):
    d = dict(seed=1, n_temps=32, n_copies=1, betas=synth.beta_ladder(32), layout="bits", device=0)
    d.update(kw)
    return d


def _code(fn, *a, **kw):
    with pytest.raises(L.IsingError) as ei:
        fn(*a, **kw)
    return ei.value.code, str(ei.value)


def test_create_validation_errors():
    Jr, Jd = synth.torus_pm1(8, 8, 1)
    assert _code(L.ising_create_grid, 7, 8, Jr, Jd, **_desc())[0] == L.ISING_E_ARG
    assert _code(L.ising_create_grid, 2, 8, Jr[:16], Jd[:16], **_desc())[0] == L.ISING_E_ARG
    bad = Jr.copy(); bad[5] = 0
    c, msg = _code(L.ising_create_grid, 8, 8, bad, Jd, **_desc())
    assert c == L.ISING_E_GRAPH and "J_right[5]" in msg
    assert _code(L.ising_create_grid, 8, 8, Jr, Jd, **_desc(n_temps=48, betas=synth.beta_ladder(48)))[0] == L.ISING_E_ARG
    b = synth.beta_ladder(32); b[3] = b[2]
    assert _code(L.ising_create_grid, 8, 8, Jr, Jd, **_desc(betas=b))[0] == L.ISING_E_ARG
    assert _code(L.ising_create_grid, 8, 8, Jr, Jd, **_desc(copy_begin=1, copy_end=1))[0] == L.ISING_E_ARG
    # CSR invariants
    rp = np.array([0, 1, 2], np.int64)
    assert _code(L.ising_create_csr, 2, rp, np.array([0, 0], np.int32), np.array([1, 1], np.int32), **_desc())[0] == L.ISING_E_GRAPH  # self-loop
    assert _code(L.ising_create_csr, 2, rp, np.array([1, 0], np.int32), np.array([1, -1], np.int32), **_desc())[0] == L.ISING_E_GRAPH  # asymmetric w
    assert _code(L.ising_create_csr, 2, rp, np.array([1, 5], np.int32), np.array([1, 1], np.int32), **_desc())[0] == L.ISING_E_GRAPH  # range
    rp3 = np.array([0, 2, 3, 4], np.int64)
    assert _code(L.ising_create_csr, 3, rp3, np.array([1, 1, 0, 0], np.int32), np.ones(4, np.int32), **_desc())[0] == L.ISING_E_GRAPH  # duplicate
    # the row checks run on host threads over vertex ranges: the error reported is still the
    # lowest failing vertex's, row checks before symmetry, entries in row order
    nb = 1 << 18
    ring_u = np.arange(nb, dtype=np.int64)
    rpb, colb, wb = synth.edges_to_csr(nb, ring_u, (ring_u + 1) % nb, np.ones(nb, np.int32))
    colb = colb.copy(); wb = wb.copy()
    colb[rpb[250000]] = 250000               # self-loop, late chunk
    colb[rpb[150000] + 1] = colb[rpb[150000]]  # duplicate, earlier chunk
    wb[rpb[7]] = -1                           # asymmetric weight, first chunk (symmetry pass)
    c, msg = _code(L.ising_create_csr, nb, rpb, colb, wb, **_desc())
    assert c == L.ISING_E_GRAPH and msg.endswith("duplicate edge 150000-" + str(colb[rpb[150000]])), msg
    colb[rpb[150000] + 1] = 150001 if colb[rpb[150000]] == 149999 else 149999
    c, msg = _code(L.ising_create_csr, nb, rpb, colb, wb, **_desc())
    assert c == L.ISING_E_GRAPH and msg.endswith("self-loop at vertex 250000"), msg
    colb[rpb[250000]] = 249999 if colb[rpb[250000] + 1] == 250001 else 250001
    c, msg = _code(L.ising_create_csr, nb, rpb, colb, wb, **_desc())
    assert c == L.ISING_E_GRAPH and msg.endswith("asymmetric coupling 6-7"), msg  # 6 meets it first
    # a long row (> 64 entries, sorted-set duplicate check) with its duplicate at the end
    hub_rp = np.array([0, 70] + [70 + k + 1 for k in range(70)], np.int64)
    hub_col = np.concatenate([np.arange(1, 71), np.zeros(70)]).astype(np.int32)
    hub_col[69] = 5
    c, msg = _code(L.ising_create_csr, 71, hub_rp, hub_col, np.ones(140, np.int32), **_desc())
    assert c == L.ISING_E_GRAPH and msg.endswith("duplicate edge 0-5"), msg
    # improper colouring
    c, msg = _code(L.ising_create_csr, 2, rp, np.array([1, 0], np.int32), np.array([1, 1], np.int32),
                   colour=np.array([0, 0], np.int32), **_desc())
    assert c == L.ISING_E_GRAPH and "colour" in msg
    # weights other than +-1 are not supported by the bit-packed kernels
    assert _code(L.ising_create_csr, 2, rp, np.array([1, 0], np.int32), np.array([2, 2], np.int32), **_desc())[0] == L.ISING_E_UNSUPPORTED
    # I8 needs K % 4 == 0; BITS needs K % 32 == 0
    assert _code(L.ising_create_csr, 2, rp, np.array([1, 0], np.int32), np.array([2, 2], np.int32),
                 **_desc(layout="i8", n_temps=6, betas=synth.beta_ladder(6)))[0] == L.ISING_E_ARG


def test_no_cpu_fallback_without_gpu():
    """A valid create on a box without a usable GPU fails loudly (no CPU path)."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("GPU present")
    except ImportError:
        pass
    Jr, Jd = synth.torus_pm1(8, 8, 1)
    c, msg = _code(L.ising_create_grid, 8, 8, Jr, Jd, **_desc())
    assert c in (L.ISING_E_CUDA, L.ISING_E_OOM)


def test_grid_band_override_is_validated(monkeypatch):
    """ISING_GRID_BANDS (torus band split) accepts only 1 or 2, and 2 only
    where the fused PT clusters stay within 8 CTAs (n_temps <= 128); checked before any
    device work, so it fails the same way with or without a GPU."""
    Jr, Jd = synth.torus_pm1(8, 8, 1)
    monkeypatch.setenv("ISING_GRID_BANDS", "3")
    c, msg = _code(L.ising_create_grid, 8, 8, Jr, Jd, **_desc())
    assert c == L.ISING_E_ARG and "ISING_GRID_BANDS" in msg
    monkeypatch.setenv("ISING_GRID_BANDS", "2")
    c, msg = _code(L.ising_create_grid, 8, 8, Jr, Jd, **_desc(n_temps=256, betas=synth.beta_ladder(256)))
    assert c == L.ISING_E_UNSUPPORTED and "ISING_GRID_BANDS" in msg


def test_colour_jp_argument_errors_without_gpu():
    """ising_colour_jp validates its CSR before any device work (include/ising.h)."""
    rp = np.array([0, 1, 2], np.int64)
    c, _ = _code(L.ising_colour_jp, 2, rp, np.array([1, 5], np.int32))
    assert c == L.ISING_E_GRAPH
    c, _ = _code(L.ising_colour_jp, 2, np.array([1, 1, 2], np.int64), np.array([1, 0], np.int32))
    assert c == L.ISING_E_GRAPH


def test_desc_colouring_is_validated():
    """An unknown ising_run_desc.colouring is an argument error, checked before device work."""
    rp = np.array([0, 1, 2], np.int64)
    c, msg = _code(L.ising_create_csr, 2, rp, np.array([1, 0], np.int32), np.array([1, 1], np.int32),
                   **_desc(layout="i8", n_temps=8, betas=synth.beta_ladder(8), colouring=7))
    assert c == L.ISING_E_ARG and "colouring" in msg
