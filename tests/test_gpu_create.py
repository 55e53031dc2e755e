"""The device-side create path of the int8 layout (k_create.cu) on a B200.

* The Jones-Plassmann colouring computed on the GPU equals the oracle's sequential greedy in
  priority order (R12c) vertex for vertex, incl. a hub of degree > 64 (the path
  that does not fit a 64-bit colour mask) and the C5-shaped 3-regular graph.
* Every CSR / colouring error of the device checks equals the host checks' (the bit-packed
  layout validates on the host): same status, same message, same lowest failing vertex.
* The internal (colour-sorted) order and the per-replica readback / overwrite through it:
  set_spins / get_spins round trips and energies from the oracle's definition.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no GPU", allow_module_level=True)

from paper_2311_09275_b200 import Engine, ising as L, run_pt  # noqa: E402

KEY = synth.PHILOX_KEY


def _graphs():
    u, v = synth.gnm(2000, 5000, 11)
    yield "gnm", 2000, u, v
    u, v = synth.random_regular(200000, 3, 3)
    yield "regular", 200000, u, v
    # a hub joined to 150 leaves plus a sparse random part: degree 150 > 64
    hu = np.zeros(150, np.int64)
    hv = np.arange(1, 151, dtype=np.int64)
    gu, gv = synth.gnm(400, 900, 12)
    yield "hub", 551, np.concatenate([hu, gu + 151]), np.concatenate([hv, gv + 151])
    yield "empty", 50, np.zeros(0, np.int64), np.zeros(0, np.int64)


@pytest.mark.parametrize("kind,n,u,v", list(_graphs()), ids=lambda x: x if isinstance(x, str) else "")
def test_jp_colouring_equals_oracle(kind, n, u, v):
    rp, col, _ = synth.edges_to_csr(n, u, v, np.ones(u.size, np.int32))
    mine, nm = L.ising_colour_jp(n, rp, col)
    ref, nr = oracle.greedy_colour_jp(n, rp, col)
    assert nm == nr and np.array_equal(mine, ref)


def _desc(layout, **kw):
    d = dict(seed=1, n_temps=32, n_copies=1, betas=synth.beta_ladder(32), layout=layout, device=0)
    d.update(kw)
    return d


def _err(fn, *a, **kw):
    with pytest.raises(L.IsingError) as ei:
        fn(*a, **kw)
    return ei.value.code, str(ei.value)


def _both(n, rp, col, w, colour=None):
    """(code, message) of the host checks (BITS) and of the device checks (I8)."""
    return (_err(L.ising_create_csr, n, rp, col, w, colour=colour, **_desc("bits")),
            _err(L.ising_create_csr, n, rp, col, w, colour=colour, **_desc("i8")))


def test_device_checks_equal_host_checks():
    rp = np.array([0, 1, 2], np.int64)
    cases = [(2, rp, np.array([0, 0], np.int32), np.array([1, 1], np.int32), None),     # self-loop
             (2, rp, np.array([1, 0], np.int32), np.array([1, -1], np.int32), None),    # asymmetric w
             (2, rp, np.array([1, 5], np.int32), np.array([1, 1], np.int32), None),     # range
             (3, np.array([0, 2, 3, 4], np.int64), np.array([1, 1, 0, 0], np.int32), np.ones(4, np.int32), None),
             (2, rp, np.array([1, 0], np.int32), np.array([1, 1], np.int32), np.array([0, 0], np.int32)),
             (2, rp, np.array([1, 0], np.int32), np.array([1, 1], np.int32), np.array([0, 70000], np.int32)),
             (3, np.array([0, 1, 2, 2], np.int64), np.array([1, 0], np.int32), np.ones(2, np.int32),
              np.array([0, 2, 0], np.int32))]                                            # colour gap
    # lowest failing vertex across a large graph, row checks before symmetry
    nb = 1 << 18
    ring = np.arange(nb, dtype=np.int64)
    rpb, colb, wb = synth.edges_to_csr(nb, ring, (ring + 1) % nb, np.ones(nb, np.int32))
    colb = colb.copy(); wb = wb.copy()
    colb[rpb[250000]] = 250000
    colb[rpb[150000] + 1] = colb[rpb[150000]]
    wb[rpb[7]] = -1
    cases.append((nb, rpb, colb.copy(), wb.copy(), None))
    colb[rpb[150000] + 1] = 150001 if colb[rpb[150000]] == 149999 else 149999
    cases.append((nb, rpb, colb.copy(), wb.copy(), None))
    colb[rpb[250000]] = 249999 if colb[rpb[250000] + 1] == 250001 else 250001
    cases.append((nb, rpb, colb.copy(), wb.copy(), None))
    hub_rp = np.array([0, 70] + [70 + k + 1 for k in range(70)], np.int64)
    hub_col = np.concatenate([np.arange(1, 71), np.zeros(70)]).astype(np.int32)
    hub_col[69] = 5
    cases.append((71, hub_rp, hub_col, np.ones(140, np.int32), None))
    for n, r, c, w, colour in cases:
        host, dev = _both(n, r, c, w, colour)
        assert host == dev, (host, dev)
        assert host[0] == L.ISING_E_GRAPH


def test_device_checks_int8_only_errors():
    """Errors only the int8 layout can meet: non-finite float weights, |w| sums >= 2^30."""
    rp = np.array([0, 1, 2], np.int64)
    c, msg = _err(L.ising_create_csr, 2, rp, np.array([1, 0], np.int32), np.array([np.inf, np.inf], np.float32),
                  **_desc("i8"))
    assert c == L.ISING_E_GRAPH and msg.endswith("non-finite weight at entry 0"), msg
    rp3 = np.array([0, 2, 3, 4], np.int64)
    big = np.array([1 << 29, 1 << 29, 1 << 29, 1 << 29], np.int32)
    c, msg = _err(L.ising_create_csr, 3, rp3, np.array([1, 2, 0, 0], np.int32), big, **_desc("i8"))
    assert c == L.ISING_E_GRAPH and msg.endswith("sum of |w| at vertex 0 >= 2^30"), msg


@pytest.mark.parametrize("colouring", [None, "jp", "explicit"])
def test_int8_internal_order_readback(colouring):
    """Slots read back in original vertex order through the device permutation: set_spins /
    get_spins round trip, energies equal the definition for the written configuration, and a
    run equals the oracle under the same colouring."""
    n, K, C = 700, 32, 8
    u, v = synth.random_regular(n, 3, 9)
    w = synth.gaussian_f32(u.size, 10)
    rp, col, ww = synth.edges_to_csr(n, u, v, w)
    inst = dict(kind="csr", n=n, row_ptr=rp, col=col, w=ww.astype(np.float32))
    betas = synth.beta_ladder(K)
    if colouring == "explicit":
        colour, _ = oracle.greedy_colour_sl(n, rp, col)
        eng = Engine(inst, K, C, betas, seed=KEY, layout="i8", colour=colour)
    else:
        eng = Engine(inst, K, C, betas, seed=KEY, layout="i8", colour=colouring)
        colour = (oracle.greedy_colour_jp if colouring == "jp" else oracle.greedy_colour)(n, rp, col)[0]
    assert eng.info.n_colours == colour.max() + 1
    run_pt(eng, 6, 0)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_WORD, colour=colour).run(6, 0)
    for r in range(0, K * C, 17):
        assert np.array_equal(eng.spins(r), o.s[r])
    s = np.where(synth.splitmix64(5, n) >> np.uint64(63), -1, 1).astype(np.int8)
    eng.set_spins(77, s)
    assert np.array_equal(eng.spins(77), s)
    o.s[77 - o.slot0] = s
    assert abs(eng.energies()[77] - o.energy_scratch()[77]) <= 1e-5 * abs(o.energy_scratch()[77])
