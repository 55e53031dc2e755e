"""GPU-vs-oracle parity through the C ABI (needs a B200).

Integer weights: bit-exact spins, energies, walker ids and best records.
Float weights (C5 shape): identical spins (both sides take every accept decision
with the float32 contract of DESIGN.md §3.5) and energies within 1e-5 relative
(BASELINE.json north_star).  Full-size configs are checked on sampled copies /
replicas in the same launch configuration bench.py times.
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


def grid(Lx, Ly, seed):
    Jr, Jd = synth.torus_pm1(Lx, Ly, seed)
    return dict(kind="grid", Lx=Lx, Ly=Ly, J_right=Jr, J_down=Jd, n=Lx * Ly)


def csr_pm1(n, m, seed, signed=False):
    u, v = synth.gnm(n, m, seed)
    if signed:
        w = np.where(synth.splitmix64(seed + 1, u.size) >> np.uint64(63), -1, 1).astype(np.int32)
    else:
        w = np.ones(u.size, np.int32)
    rp, col, ww = synth.edges_to_csr(n, u, v, w)
    return dict(kind="csr", n=n, row_ptr=rp, col=col, w=ww.astype(np.int32))


def compare_copies(eng, o, check_best=True):
    E = eng.energies()
    W = eng.walkers()
    lo = o.slot0 - eng.slot0
    assert np.array_equal(E[lo:lo + o.R], o.energies())
    if not o.is_float:
        assert np.array_equal(W[lo:lo + o.R], o.walker)
    for r in range(o.R):
        assert np.array_equal(eng.spins(o.slot0 + r), o.s[r]), f"slot {o.slot0 + r}"
    if check_best:
        b = eng.best(spins=True)
        assert (b["E"], b["slot"], b["sweep"]) == (o.best.E, o.best.slot, o.best.sweep)
        assert np.array_equal(b["spins"], o.best.spins)


def test_philox_matches_curand_and_oracle():
    z = synth.splitmix64(99, 6 * 2000).astype(np.uint64)
    tuples = (z & np.uint64(0xFFFFFFFF)).astype(np.uint32).reshape(-1, 6)
    mine, cur = L.ising_debug_philox(tuples)
    assert np.array_equal(mine, cur)  # library routine curand_Philox4x32_10 pins the device Philox
    for t in tuples[:64]:
        assert np.array_equal(oracle.philox(t[:4], t[4:]), mine[tuples.tolist().index(t.tolist())])


@pytest.fixture(params=[1, 2], ids=["bands1", "bands2"])
def bands(request, monkeypatch):
    """Torus kernel row bands per word group: 1 = one CTA per group,
    2 = a CTA pair exchanging halo rows through DSMEM.  Read by ising_create_grid."""
    monkeypatch.setenv("ISING_GRID_BANDS", str(request.param))
    return request.param


@pytest.mark.parametrize("Lx,Ly,K,C,sweeps,kex,threads", [
    (4, 4, 32, 1, 50, 10, 0),
    (16, 16, 64, 2, 100, 10, 0),
    (6, 4, 32, 3, 33, 7, 0),       # ragged: 12 sites per colour, odd copies, tail rounds
    (10, 8, 96, 2, 40, 5, 64),     # K = 96 (3 words per copy), small CTA
    (12, 20, 128, 1, 30, 10, 256),  # 4 words per copy
    (48, 52, 32, 2, 30, 10, 320),   # 1 column-less warp takes the 4 leftover rows (as C2's 16th warp)
])
def test_grid_bits_parity(Lx, Ly, K, C, sweeps, kex, threads, bands):
    inst = grid(Lx, Ly, 1000 + Lx * Ly)
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="bits", block_threads=threads)
    run_pt(eng, sweeps, kex, fused=False)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_PLANE).run(sweeps, kex)
    compare_copies(eng, o)


@pytest.mark.parametrize("Lx,Ly,K,C,sweeps,kex", [
    (16, 16, 64, 2, 100, 10),    # clusters of 2 CTAs
    (6, 4, 32, 3, 33, 7),        # cluster of 1, tail sweeps after the fused rounds
    (10, 8, 96, 2, 40, 5),       # clusters of 3 (cross-word pairs at both ends of word 1)
    (12, 20, 256, 1, 60, 3),     # cluster of 8
])
def test_fused_pt_launch_parity(Lx, Ly, K, C, sweeps, kex, bands):
    """ising_run (one launch, cluster exchange through DSMEM) == oracle, bit for bit."""
    if bands == 2 and K > 128:
        pytest.skip("band split needs clusters of <= 8 CTAs (n_temps <= 128)")
    inst = grid(Lx, Ly, 77 + Lx * Ly)
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    rec = run_pt(eng, sweeps, kex, fused=True)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_PLANE).run(sweeps, kex)
    compare_copies(eng, o)
    assert (rec["E"], rec["slot"], rec["sweep"]) == (o.best.E, o.best.slot, o.best.sweep)
    # split into two fused calls + per-round calls: same state
    eng2 = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    eng2.run(2, kex)
    for _ in range(sweeps // kex - 2):
        eng2.sweep(kex)
        eng2.exchange()
    if sweeps % kex:
        eng2.sweep(sweeps % kex)
        eng2.check_best()
    assert np.array_equal(eng2.energies(), eng.energies())
    assert np.array_equal(eng2.walkers(), eng.walkers())
    b1, b2 = eng.best(), eng2.best()
    assert (b1["E"], b1["slot"], b1["sweep"]) == (b2["E"], b2["slot"], b2["sweep"])


def test_grid_bits_block_size_invariance():
    inst = grid(16, 12, 5)
    betas = synth.beta_ladder(32)
    outs = []
    for thr in (32, 128, 512):
        eng = Engine(inst, 32, 4, betas, seed=7, layout="bits", block_threads=thr)
        run_pt(eng, 25, 5)
        outs.append((eng.energies(), [eng.spins(r) for r in range(0, 128, 13)]))
    for e, s in outs[1:]:
        assert np.array_equal(e, outs[0][0])
        assert all(np.array_equal(a, b) for a, b in zip(s, outs[0][1]))


@pytest.mark.parametrize("seed", [404, 405, 406, 407])
def test_grid_bits_finds_bruteforce_ground_state_4x4(seed):
    inst = grid(4, 4, seed)
    betas = synth.beta_ladder(64)
    o = oracle.Oracle(inst, 1, np.array([1.0]), 0)
    u, v, w = [], [], []
    for i in range(16):
        for e in range(o.rp[i], o.rp[i + 1]):
            if o.col[e] > i:
                u.append(i); v.append(o.col[e]); w.append(o.wi[e])
    states = 1 - 2 * ((np.arange(2**16)[:, None] >> np.arange(16)[None, :]) & 1)
    Emin = np.sum(np.array(w) * states[:, u] * states[:, v], axis=1).min()
    eng = Engine(inst, 64, 1, betas, seed=KEY)
    rec = run_pt(eng, 200, 10)
    assert rec["E"] == Emin


def test_c2_full_size_sampled_copies():
    cfg = synth.CONFIGS["c2"]
    inst = synth.make_instance(cfg)
    betas = synth.beta_ladder(cfg["K"])
    eng = Engine(inst, cfg["K"], cfg["C"], betas, seed=KEY, layout="bits")
    run_pt(eng, 20, cfg["k_ex"])
    for c0 in (0, 37, 63):
        o = oracle.Oracle(inst, cfg["K"], betas, KEY, c0, c0 + 1, rng=oracle.RNG_PLANE).run(20, 10)
        compare_copies(eng, o, check_best=False)


def test_c4b_eight_gpu_share_band_split():
    """One rank's share of C4b at 8 GPUs (16 copies = 64 word groups): the default picks the
    band split (128 CTAs); sampled copies equal the oracle bit for bit, fused PT launch."""
    cfg = synth.CONFIGS["c4b"]
    inst = synth.make_instance(cfg)
    betas = synth.beta_ladder(cfg["K"])
    eng = Engine(inst, cfg["K"], 16, betas, seed=KEY, layout="bits")
    run_pt(eng, 20, cfg["k_ex"])
    for c0 in (0, 9, 15):
        o = oracle.Oracle(inst, cfg["K"], betas, KEY, c0, c0 + 1, rng=oracle.RNG_PLANE).run(20, 10)
        compare_copies(eng, o, check_best=False)


def test_band_split_multicluster_pt_parity(monkeypatch):
    """36 copies of K = 64 on a 100x100 torus (one CTA per SM): 72 word groups -> band split
    (144 CTAs); the copies' clusters of 4 CTAs do not all fit at once (33 on a B200), so
    ising_run uses ONE cooperative launch whose copies span 2 clusters (band pairs) meeting at
    global-memory copy barriers (ising_info.fused_pt == 2).  Sampled copies equal the oracle
    and every copy equals the single-band fused launch, bit for bit."""
    inst = grid(100, 100, 2024)
    K, C, sweeps, kex = 64, 36, 20, 10
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    assert eng.info.bands == 2 and eng.info.fused_pt == 2
    run_pt(eng, sweeps, kex)
    for c0 in (0, 17, 35):
        o = oracle.Oracle(inst, K, betas, KEY, c0, c0 + 1, rng=oracle.RNG_PLANE).run(sweeps, kex)
        compare_copies(eng, o, check_best=False)
    monkeypatch.setenv("ISING_GRID_BANDS", "1")
    one = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    run_pt(one, sweeps, kex)
    assert np.array_equal(one.energies(), eng.energies())
    assert np.array_equal(one.walkers(), eng.walkers())
    for x, y in zip(one.copy_best(), eng.copy_best()):
        assert np.array_equal(x, y)
    b1, b2 = one.best(), eng.best()
    assert (b1["E"], b1["slot"], b1["sweep"]) == (b2["E"], b2["slot"], b2["sweep"])
    assert np.array_equal(b1["spins"], b2["spins"])


def test_grid_kernel_equals_csr_kernel_on_torus():
    inst = grid(12, 8, 3)
    rp, col, w = synth.torus_csr(12, 8, inst["J_right"], inst["J_down"])
    cinst = dict(kind="csr", n=96, row_ptr=rp, col=col, w=w.astype(np.int32))
    betas = synth.beta_ladder(64)
    a = Engine(inst, 64, 2, betas, seed=11)
    b = Engine(cinst, 64, 2, betas, seed=11, colour=synth.checkerboard(12, 8))
    run_pt(a, 30, 10)
    run_pt(b, 30, 10)
    assert b.info.kernel == 1 and a.info.kernel == 0
    assert np.array_equal(a.energies(), b.energies())
    assert np.array_equal(a.walkers(), b.walkers())
    for r in range(0, 128, 5):
        assert np.array_equal(a.spins(r), b.spins(r))


@pytest.mark.parametrize("n,m,K,C,signed", [(300, 299, 32, 2, False), (500, 900, 64, 1, True),
                                           (64, 0, 32, 1, False), (40, 150, 32, 2, True)])
def test_csr_bits_parity(n, m, K, C, signed):
    inst = csr_pm1(n, m, 17 + n, signed)
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    run_pt(eng, 40, 10, fused=False)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_PLANE).run(40, 10)
    compare_copies(eng, o)


@pytest.mark.parametrize("n,m,K,C,sweeps,kex,signed", [(300, 299, 64, 2, 50, 10, True),
                                                       (200, 700, 96, 1, 31, 5, False),
                                                       (64, 0, 32, 2, 20, 10, False)])
def test_csr_bits_fused_pt_parity(n, m, K, C, sweeps, kex, signed):
    inst = csr_pm1(n, m, 5 + n, signed)
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    run_pt(eng, sweeps, kex, fused=True)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_PLANE).run(sweeps, kex)
    compare_copies(eng, o)


def test_c3_full_size_sampled_copies():
    cfg = synth.CONFIGS["c3"]
    inst = synth.make_instance(cfg)
    betas = synth.beta_ladder(cfg["K"])
    eng = Engine(inst, cfg["K"], cfg["C"], betas, seed=KEY, layout="bits", colour=cfg["colouring"])
    assert eng.info.n_colours == 3  # smallest-last greedy on G(1e4, 9999)
    run_pt(eng, 20, 10, fused=True)
    col, _ = (oracle.greedy_colour_jp if cfg["colouring"] == "jp" else oracle.greedy_colour_sl)(
        inst["n"], inst["row_ptr"], inst["col"])
    for c0 in (0, 50):
        o = oracle.Oracle(inst, cfg["K"], betas, KEY, c0, c0 + 1, rng=oracle.RNG_PLANE, colour=col).run(20, 10)
        compare_copies(eng, o, check_best=False)


def test_c1_int8_full_parity():
    cfg = synth.CONFIGS["c1"]
    inst = synth.make_instance(cfg)
    betas = synth.beta_ladder(cfg["K"])
    eng = Engine(inst, cfg["K"], cfg["C"], betas, seed=KEY, layout="i8")
    run_pt(eng, cfg["sweeps"], cfg["k_ex"])
    o = oracle.Oracle(inst, cfg["K"], betas, KEY, 0, cfg["C"], rng=oracle.RNG_WORD).run(cfg["sweeps"], cfg["k_ex"])
    compare_copies(eng, o)


def test_int8_general_integer_weights_parity():
    u, v = synth.gnm(200, 500, 8)
    w = (synth._below(synth.splitmix64(8, u.size), 7) - 3).astype(np.int32)
    w[w == 0] = 5
    rp, col, ww = synth.edges_to_csr(200, u, v, w)
    inst = dict(kind="csr", n=200, row_ptr=rp, col=col, w=ww.astype(np.int32))
    betas = synth.beta_ladder(16)
    eng = Engine(inst, 16, 3, betas, seed=KEY, layout="i8")
    run_pt(eng, 60, 6)
    o = oracle.Oracle(inst, 16, betas, KEY, 0, 3, rng=oracle.RNG_WORD).run(60, 6)
    compare_copies(eng, o)


@pytest.mark.parametrize("n,m,K,C,sweeps,kex", [(300, 700, 128, 2, 47, 10), (96, 200, 8, 5, 30, 3)])
def test_int8_fused_small_pt_parity(n, m, K, C, sweeps, kex):
    """k_i8_small (one launch for all rounds, one CTA per copy) == per-round launches == oracle:
    spins, energies, walkers, best record and per-copy best, with a tail of sweeps."""
    u, v = synth.gnm(n, m, n + m)
    w = (synth._below(synth.splitmix64(n, u.size), 5) - 2).astype(np.int32)
    w[w == 0] = 3
    rp, col, ww = synth.edges_to_csr(n, u, v, w)
    inst = dict(kind="csr", n=n, row_ptr=rp, col=col, w=ww.astype(np.int32))
    betas = synth.beta_ladder(K)
    a = Engine(inst, K, C, betas, seed=KEY, layout="i8")
    assert a.info.fused_pt == 1
    run_pt(a, sweeps, kex, fused=True)
    b = Engine(inst, K, C, betas, seed=KEY, layout="i8")
    run_pt(b, sweeps, kex, fused=False)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_WORD).run(sweeps, kex)
    compare_copies(a, o)
    compare_copies(b, o)
    for x, y in zip(a.copy_best(), b.copy_best()):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("n,drop,K,C,sweeps,kex", [
    (256, 7, 32, 2, 43, 5),   # <= 4 classes of <= 128 vertices, degree <= 3 with pads: register path
    (220, 0, 64, 1, 30, 10),  # 3-regular, 8 CTAs per copy: register path at the C1 cluster size
    (600, 0, 16, 2, 20, 4),   # a class of > 128 vertices: the CSR path of the same kernel
])
def test_int8_cluster_register_path_parity(n, drop, K, C, sweeps, kex):
    """k_i8_cluster's register path (each thread's class vertices, rows and weights in registers,
    4 replicas per thread, branch-free threshold lookups) and its CSR path == per-round launches
    == oracle on non-torus graphs with padded rows, integer weights in [-3, 3] \\ {0}."""
    u, v = synth.random_regular(n, 3, 90 + n)
    if drop:
        keep = np.arange(u.size) % drop != 0
        u, v = u[keep], v[keep]
    w = (synth._below(synth.splitmix64(91 + n, u.size), 7) - 3).astype(np.int32)
    w[w == 0] = 2
    rp, col, ww = synth.edges_to_csr(n, u, v, w)
    inst = dict(kind="csr", n=n, row_ptr=rp, col=col, w=ww.astype(np.int32))
    betas = synth.beta_ladder(K)
    a = Engine(inst, K, C, betas, seed=KEY, layout="i8")
    assert a.info.fused_pt == 1
    run_pt(a, sweeps, kex, fused=True)
    b = Engine(inst, K, C, betas, seed=KEY, layout="i8")
    run_pt(b, sweeps, kex, fused=False)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_WORD).run(sweeps, kex)
    compare_copies(a, o)
    compare_copies(b, o)
    for x, y in zip(a.copy_best(), b.copy_best()):
        assert np.array_equal(x, y)


def _regular_inst(n, seed):
    u, v = synth.random_regular(n, 3, seed)
    w = synth.gaussian_f32(u.size, seed + 5)
    rp, col, ww = synth.edges_to_csr(n, u, v, w)
    return dict(kind="csr", n=n, row_ptr=rp, col=col, w=ww.astype(np.float32))


def test_exp_bracket_bound():
    """The I8 kernels decide float-weight attempts from the 16-bit hi word with a 2^-16
    relative margin around the estimate ex2.approx(RN(2 beta log2e) sh + 16); exact-decision
    safety needs it within half the margin of the contract exponential wherever c >= 1/2 and
    below 1 elsewhere, for EVERY float field value sh (exhaustive) and every ladder used by
    the float tests and the C5 bench."""
    b2 = np.unique(np.concatenate([2.0 * synth.beta_ladder(k).astype(np.float32) for k in (8, 16, 256)]))
    worst, small = L.ising_debug_exp_bound(b2.astype(np.float32))
    assert worst < 2.0 ** -17, worst
    assert small < 1.0, small


def test_float_int8_parity_small():
    inst = _regular_inst(3000, 21)
    betas = synth.beta_ladder(16)
    eng = Engine(inst, 16, 2, betas, seed=KEY, layout="i8")
    run_pt(eng, 25, 0)
    o = oracle.Oracle(inst, 16, betas, KEY, 0, 2, rng=oracle.RNG_WORD).run(25, 0)
    for r in range(o.R):
        assert np.array_equal(eng.spins(r), o.s[r])
    E, Eo = eng.energies(), o.energies()
    assert np.allclose(E, Eo, rtol=1e-5, atol=0)
    b = eng.best(spins=True)
    assert b["slot"] == o.best.slot and abs(b["E"] - o.best.E) <= 1e-5 * abs(o.best.E)


@pytest.mark.parametrize("n,d,drop,K,C,sweeps", [
    (3000, 3, 0, 32, 8, 12),      # R = 256: one replica slice per warp, DEG 3 (C5 shape)
    (2000, 4, 10, 64, 8, 8),      # R = 512: two slices, DEG 4 with pads (every 10th edge dropped)
    (38, 3, 0, 16, 16, 20),       # fewer vertices per class than warps: 1-vertex chunks
])
@pytest.mark.parametrize("colouring", ["sl", "jp"])
def test_float_int8_ring_parity(n, d, drop, K, C, sweeps, colouring):
    """cp.async ring kernel (float weights, padded table, R % 256 == 0): identical spins and
    energies within 1e-5 relative of the oracle, over ragged chunks and table widths."""
    u, v = synth.random_regular(n, d, 40 + n)
    if drop:
        keep = np.arange(u.size) % drop != 0
        u, v = u[keep], v[keep]
    w = synth.gaussian_f32(u.size, 41 + n)
    rp, col, ww = synth.edges_to_csr(n, u, v, w)
    inst = dict(kind="csr", n=n, row_ptr=rp, col=col, w=ww.astype(np.float32))
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="i8", colour=colouring)
    run_pt(eng, sweeps, 0)
    colour, _ = (oracle.greedy_colour_jp if colouring == "jp" else oracle.greedy_colour_sl)(n, rp, col)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_WORD, colour=colour).run(sweeps, 0)
    for r in range(o.R):
        assert np.array_equal(eng.spins(r), o.s[r]), f"slot {r}"
    assert np.allclose(eng.energies(), o.energies(), rtol=1e-5, atol=0)


@pytest.mark.parametrize("wset", [
    [-1.0, 0.0, 1.0],                      # integer-valued: s h = 0 ties on every third term pattern
    [0.0, -0.0, 0.5, -0.5, 1e-3, -1e-3, 1e-38, -1e-38, 1e-41, -1e-41, 3.0, -3.0],  # zeros, tiny, subnormal
])
def test_float_int8_degenerate_weights(wset):
    """Float-weight ring kernel on degenerate couplings: exact zeros of both signs, ties s h = 0
    (the estimate e = 2^16 leaves hi16 = 65535 to the exact path), subnormal and tiny terms in
    the left fold.  Spins identical to the oracle; energies within 1e-5 of the scale sum |w|."""
    n, K, C, sweeps = 2000, 32, 8, 20
    u, v = synth.random_regular(n, 3, 60)
    pick = (synth.splitmix64(61, u.size) % np.uint64(len(wset))).astype(np.int64)
    w = np.asarray(wset, np.float32)[pick]
    rp, col, ww = synth.edges_to_csr(n, u, v, w)
    inst = dict(kind="csr", n=n, row_ptr=rp, col=col, w=ww.astype(np.float32))
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="i8", colour="jp")
    run_pt(eng, sweeps, 0)
    colour, _ = oracle.greedy_colour_jp(n, rp, col)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_WORD, colour=colour).run(sweeps, 0)
    for r in range(o.R):
        assert np.array_equal(eng.spins(r), o.s[r]), f"slot {r}"
    scale = float(np.abs(w.astype(np.float64)).sum())
    assert np.allclose(eng.energies(), o.energies(), rtol=1e-5, atol=1e-5 * scale)


@pytest.mark.parametrize("n,d,drop,K,C,sweeps", [
    (3000, 3, 0, 32, 8, 12),      # R = 256, DEG 3 (C5 shape)
    (2000, 4, 10, 64, 8, 8),      # R = 512: two slices per vertex, DEG 4 with pads
    (1500, 2, 0, 32, 8, 10),      # DEG 2 (a random 2-regular graph: cycles)
    (38, 3, 0, 16, 16, 20),       # fewer vertices per class than warps
])
@pytest.mark.parametrize("colouring", ["sl", "jp"])
def test_float_packed_rows_parity(monkeypatch, n, d, drop, K, C, sweeps, colouring):
    """Packed-row sweeps (k_csr_packed) forced on: identical spins to the
    oracle and to the int8 ring kernel (forced off), energies within 1e-5 relative."""
    u, v = synth.random_regular(n, d, 40 + n)
    if drop:
        keep = np.arange(u.size) % drop != 0
        u, v = u[keep], v[keep]
    w = synth.gaussian_f32(u.size, 41 + n)
    rp, col, ww = synth.edges_to_csr(n, u, v, w)
    inst = dict(kind="csr", n=n, row_ptr=rp, col=col, w=ww.astype(np.float32))
    betas = synth.beta_ladder(K)
    out = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("ISING_I8_PACKED", mode)
        eng = Engine(inst, K, C, betas, seed=KEY, layout="i8", colour=colouring)
        run_pt(eng, sweeps, 0)
        out[mode] = ([eng.spins(r) for r in range(eng.R)], eng.energies())
        eng.close()
    colour, _ = (oracle.greedy_colour_jp if colouring == "jp" else oracle.greedy_colour_sl)(n, rp, col)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_WORD, colour=colour).run(sweeps, 0)
    for r in range(o.R):
        assert np.array_equal(out["1"][0][r], o.s[r]), f"slot {r}"
        assert np.array_equal(out["0"][0][r], o.s[r]), f"slot {r} (int8 ring)"
    assert np.allclose(out["1"][1], o.energies(), rtol=1e-5, atol=0)
    assert np.array_equal(out["1"][1], out["0"][1])  # same spins, same energy kernel


def test_float_packed_rows_call_pattern(monkeypatch):
    """Packed rows over mixed call patterns on one handle: single-sweep calls (pack / unpack
    around every sweep), a long call, spins written between calls, and an annealing schedule
    (per-sweep betas) -- identical to the int8 kernels throughout."""
    n, K, C = 2500, 32, 8
    inst = _regular_inst(n, 77)
    betas = synth.beta_ladder(K)
    sched = np.stack([betas * (0.5 + 0.1 * s) for s in range(6)]).astype(np.float64)
    res = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("ISING_I8_PACKED", mode)
        eng = Engine(inst, K, C, betas, seed=KEY, layout="i8", colour="jp")
        for _ in range(3):
            eng.sweep(1)
        eng.sweep(9)
        s0 = eng.spins(5)
        s0[: n // 2] *= -1
        eng.set_spins(5, s0)
        eng.sweep(5)
        eng.anneal(sched)
        res[mode] = ([eng.spins(r) for r in range(eng.R)], eng.energies())
        eng.close()
    for r in range(K * C):
        assert np.array_equal(res["1"][0][r], res["0"][0][r]), f"slot {r}"
    assert np.array_equal(res["1"][1], res["0"][1])


def test_float_packed_rows_sharded_handles(monkeypatch):
    """Packed rows on copy shards (slot0 = 256: the Philox counter words of the second shard's
    lanes start at 32): two 8-copy handles equal one 16-copy handle slot for slot."""
    monkeypatch.setenv("ISING_I8_PACKED", "1")
    n, K, C, sweeps = 1800, 32, 16, 9
    inst = _regular_inst(n, 91)
    betas = synth.beta_ladder(K)
    full = Engine(inst, K, C, betas, seed=KEY, layout="i8", colour="jp")
    full.sweep(sweeps)
    Ef = full.energies()
    for lo, hi in ((0, 8), (8, 16)):
        part = Engine(inst, K, C, betas, seed=KEY, layout="i8", colour="jp", copy_begin=lo, copy_end=hi)
        part.sweep(sweeps)
        Ep = part.energies()
        for r in range(part.R):
            assert np.array_equal(part.spins(lo * K + r), full.spins(lo * K + r)), f"slot {lo * K + r}"
        assert np.array_equal(Ep, Ef[lo * K:hi * K])
        part.close()


@pytest.mark.parametrize("wset", [
    [-1.0, 0.0, 1.0],
    [0.0, -0.0, 0.5, -0.5, 1e-3, -1e-3, 1e-38, -1e-38, 1e-41, -1e-41, 3.0, -3.0],
])
def test_float_packed_rows_degenerate_weights(monkeypatch, wset):
    """The packed-row kernel on degenerate couplings (signed zeros, s h = 0 ties through the
    exact path, tiny and subnormal terms): spins identical to the oracle."""
    monkeypatch.setenv("ISING_I8_PACKED", "1")
    n, K, C, sweeps = 2000, 32, 8, 20
    u, v = synth.random_regular(n, 3, 60)
    pick = (synth.splitmix64(61, u.size) % np.uint64(len(wset))).astype(np.int64)
    w = np.asarray(wset, np.float32)[pick]
    rp, col, ww = synth.edges_to_csr(n, u, v, w)
    inst = dict(kind="csr", n=n, row_ptr=rp, col=col, w=ww.astype(np.float32))
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="i8", colour="jp")
    run_pt(eng, sweeps, 0)
    colour, _ = oracle.greedy_colour_jp(n, rp, col)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_WORD, colour=colour).run(sweeps, 0)
    for r in range(o.R):
        assert np.array_equal(eng.spins(r), o.s[r]), f"slot {r}"
    scale = float(np.abs(w.astype(np.float64)).sum())
    assert np.allclose(eng.energies(), o.energies(), rtol=1e-5, atol=1e-5 * scale)


@pytest.mark.parametrize("packed", ["1", "0"])
def test_c5_full_size_sampled_replicas(monkeypatch, packed):
    monkeypatch.setenv("ISING_I8_PACKED", packed)
    cfg = synth.CONFIGS["c5"]
    inst = synth.make_instance(cfg)
    betas = synth.beta_ladder(cfg["K"])
    eng = Engine(inst, cfg["K"], cfg["C"], betas, seed=KEY, layout="i8", colour=cfg["colouring"])
    assert eng.info.n_colours >= 3
    sweeps = 4
    eng.sweep(sweeps)
    E = eng.energies()
    col, _ = (oracle.greedy_colour_jp if cfg["colouring"] == "jp" else oracle.greedy_colour_sl)(
        inst["n"], inst["row_ptr"], inst["col"])
    for lo in (0, 255):
        o = oracle.Oracle(inst, cfg["K"], betas, KEY, 0, 1, rng=oracle.RNG_WORD, colour=col,
                          slots=(lo, lo + 1))
        o.sweeps(sweeps)
        assert np.array_equal(eng.spins(lo), o.s[0])
        assert abs(E[lo] - o.energies()[0]) <= 1e-5 * abs(o.energies()[0])


def test_sharded_handles_equal_single_handle():
    inst = grid(16, 16, 77)
    betas = synth.beta_ladder(64)
    full = Engine(inst, 64, 4, betas, seed=5)
    rec_full = run_pt(full, 30, 10)
    parts = [Engine(inst, 64, 4, betas, seed=5, copy_begin=a, copy_end=b) for a, b in ((0, 1), (1, 3), (3, 4))]
    recs = [run_pt(p, 30, 10) for p in parts]
    Ef = full.energies()
    assert np.array_equal(np.concatenate([p.energies() for p in parts]), Ef)
    assert np.array_equal(np.concatenate([p.walkers() for p in parts]), full.walkers())
    for p in parts:
        for r in range(p.slot0, p.slot0 + p.R, 7):
            assert np.array_equal(p.spins(r), full.spins(r))
    best = min(recs, key=lambda r: (r["E"], r["sweep"], r["slot"]))
    assert best == rec_full


def test_exchange_records_and_global_best():
    inst = grid(8, 8, 2)
    betas = synth.beta_ladder(32)
    eng = Engine(inst, 32, 3, betas, seed=3)
    eng.sweep(5)
    send, recv = eng.record_buffers(1)
    eng.exchange_begin(send)
    torch.cuda.synchronize()
    rec = send.cpu().numpy()
    assert np.array_equal(rec[:, 0], eng.energies())
    assert np.array_equal(rec[:, 1], np.arange(96))
    # records of a "remote" shard with a lower energy win the global best; no snapshot here
    fake = torch.tensor([[-10**6, 500]], dtype=torch.int64, device="cuda")
    eng.check_best(torch.cat([send, fake]))
    b = eng.best(spins=False)
    assert b["E"] == -10**6 and b["slot"] == 500
    with pytest.raises(L.IsingError):
        L.ising_best(eng.h, spins=True)


def test_set_spins_and_cut_identity():
    inst = grid(8, 6, 9)
    betas = synth.beta_ladder(32)
    for layout in ("bits", "i8"):
        eng = Engine(inst, 32, 1, betas, seed=3, layout=layout)
        W = int(inst["J_right"].sum() + inst["J_down"].sum())
        eng.set_spins(5, np.ones(48, np.int8))
        E = eng.energies()
        assert E[5] == W
        cut = eng.cuts()
        assert np.array_equal(cut, (W - E) // 2)
        s = eng.spins(9)
        eng.set_spins(9, -s)  # global flip invariance
        assert eng.energies()[9] == E[9]


@pytest.mark.parametrize("fused,layout", [(True, "bits"), (False, "bits"), (False, "i8")])
def test_copy_best_parity(fused, layout):
    """Per-copy best-so-far (copies = trials of the NEXT-2 harness) equals the oracle's."""
    inst = grid(16, 16, 9)
    K, C = (64, 4) if layout == "bits" else (8, 5)
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout=layout)
    run_pt(eng, 60, 10, fused=fused)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C,
                      rng=oracle.RNG_PLANE if layout == "bits" else oracle.RNG_WORD).run(60, 10)
    E, slot, sweep = eng.copy_best()
    assert list(E) == [b.E for b in o.copy_best]
    assert list(slot) == [b.slot for b in o.copy_best]
    assert list(sweep) == [b.sweep for b in o.copy_best]


def test_trial_harness_reaches_ground_state_4x4():
    from paper_2311_09275_b200 import ttt
    inst = grid(4, 4, 405)
    u, v, w = synth.torus_edges(4, 4, inst["J_right"], inst["J_down"])
    states = 1 - 2 * ((np.arange(2**16)[:, None] >> np.arange(16)[None, :]) & 1)
    Emin = int(np.sum(w * states[:, u] * states[:, v], axis=1).min())
    W = int(w.sum())
    eng = Engine(inst, 64, 16, synth.beta_ladder(64), seed=KEY)
    st = ttt.run_trials(eng, 200, 10, target_cut=(W - Emin) / 2, W=W)
    assert st.trials == 16 and st.p_s == 1.0 and st.r == 1.0 and st.sweeps_to_target == 200
    assert np.all(st.best_cuts == (W - Emin) / 2)


@pytest.mark.parametrize("kind,K,C,kmin", [("grid", 64, 4, 32), ("grid", 96, 2, 0), ("csr", 32, 2, 0),
                                           ("csr", 64, 4, 40)])
def test_icm_parity(kind, K, C, kmin):
    """Houdayer cluster moves (NEXT-1): GPU == oracle bit for bit, every round."""
    inst = grid(10, 8, 31) if kind == "grid" else csr_pm1(120, 200, 9, signed=True)
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    run_pt(eng, 40, 10, icm_k_min=kmin)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_PLANE).run(40, 10, icm_k_min=kmin)
    compare_copies(eng, o)


def test_icm_c2_sampled_pair_and_errors():
    cfg = synth.CONFIGS["c2"]
    inst = synth.make_instance(cfg)
    betas = synth.beta_ladder(64)
    eng = Engine(inst, 64, 64, betas, seed=KEY, layout="bits")
    run_pt(eng, 20, 10, icm_k_min=32)
    o = oracle.Oracle(inst, 64, betas, KEY, 10, 12, rng=oracle.RNG_PLANE).run(20, 10, icm_k_min=32)
    compare_copies(eng, o, check_best=False)
    odd = Engine(grid(8, 8, 1), 32, 3, synth.beta_ladder(32), seed=1, copy_begin=1, copy_end=3)
    with pytest.raises(L.IsingError):
        odd.icm(0)
    i8 = Engine(grid(8, 8, 1), 8, 2, synth.beta_ladder(8), seed=1, layout="i8")
    with pytest.raises(L.IsingError):
        i8.icm(0)


@pytest.mark.parametrize("kind,layout,K,C", [("grid", "bits", 64, 2), ("csr", "bits", 32, 2),
                                             ("grid", "i8", 8, 3), ("float", "i8", 8, 2)])
def test_anneal_parity(kind, layout, K, C):
    """Simulated annealing (NEXT-3): GPU == oracle, per-sweep schedules."""
    from paper_2311_09275_b200.driver import geometric_schedule
    if kind == "grid":
        inst = grid(10, 8, 12)
    elif kind == "csr":
        inst = csr_pm1(150, 260, 4, signed=True)
    else:
        inst = _regular_inst(400, 8)
    betas = synth.beta_ladder(K)
    sched = geometric_schedule(betas, 30, 0.2, 2.5)
    eng = Engine(inst, K, C, betas, seed=KEY, layout=layout)
    eng.anneal(sched)
    rng = oracle.RNG_PLANE if layout == "bits" else oracle.RNG_WORD
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=rng)
    o.anneal(sched)
    for r in range(K * C):
        assert np.array_equal(eng.spins(r), o.s[r]), r
    if kind == "float":
        assert np.allclose(eng.energies(), o.energies(), rtol=1e-5, atol=0)
    else:
        assert np.array_equal(eng.energies(), o.energies())
        b = eng.best(spins=False)
        assert (b["E"], b["slot"], b["sweep"]) == (o.best.E, o.best.slot, o.best.sweep)


def test_certify_cut_on_gpu_matches_definition():
    from paper_2311_09275_b200 import gset
    u, v = synth.gnm(500, 1200, 3)
    w = (synth._below(synth.splitmix64(4, u.size), 5) - 2).astype(np.int32)
    w[w == 0] = 1
    bits = gset.decode_hex(gset.encode_hex((synth.splitmix64(5, 500) >> np.uint64(63)).astype(np.uint8)), 500)
    s = gset.bits_to_spins(bits)
    rep = gset.certify(500, u, v, w, s, claimed=gset.cut_of(u, v, w, s))
    assert rep["cut"] == rep["cut_gpu"] and rep["matches_claim"]


def _state_tuple(eng):
    n_copies = eng.R // eng.K
    return (eng.energies(), eng.walkers(), [eng.spins(eng.slot0 + r) for r in range(eng.R)],
            eng.best(spins=True), eng.copy_best(), (eng.info.n_slots, n_copies),
            (L.ising_info(eng.h).sweeps_done, L.ising_info(eng.h).exchanges_done))


def _assert_same_state(a, b):
    for x, y in zip(a[0:2], b[0:2]):
        assert np.array_equal(x, y)
    assert all(np.array_equal(x, y) for x, y in zip(a[2], b[2]))
    assert {k: a[3][k] for k in ("E", "slot", "sweep")} == {k: b[3][k] for k in ("E", "slot", "sweep")}
    assert np.array_equal(a[3]["spins"], b[3]["spins"])
    for x, y in zip(a[4], b[4]):
        assert np.array_equal(x, y)
    assert a[5:] == b[5:]


@pytest.mark.parametrize("kind,layout,K,C,kex,icm", [
    ("grid", "bits", 64, 2, 10, None),   # fused PT launch (ising_run)
    ("grid", "bits", 64, 4, 5, 32),      # per-round exchange + Houdayer moves (counter f)
    ("csr", "bits", 32, 2, 10, None),
    ("csr", "i8", 16, 2, 10, None),
])
def test_checkpoint_resume_parity(kind, layout, K, C, kex, icm):
    """SURVEY §5 checkpoint/resume: a fresh handle that loads a checkpoint continues bit for bit
    as the saving handle, and both equal the oracle's uninterrupted run."""
    inst = grid(16, 12, 31) if kind == "grid" else csr_pm1(400, 500, 32, signed=True)
    betas = synth.beta_ladder(K)
    kw = dict(seed=KEY, layout=layout)
    a = Engine(inst, K, C, betas, **kw)
    run_pt(a, 30, kex, icm_k_min=icm)
    blob = a.save_state()
    assert len(blob) == L.ising_state_size(a.h)
    run_pt(a, 40, kex, icm_k_min=icm)
    b = Engine(inst, K, C, betas, **kw)
    b.load_state(blob)
    run_pt(b, 40, kex, icm_k_min=icm)
    sa, sb = _state_tuple(a), _state_tuple(b)
    _assert_same_state(sa, sb)
    if icm is None:
        rng = oracle.RNG_PLANE if layout == "bits" else oracle.RNG_WORD
        o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=rng).run(70, kex)
        compare_copies(b, o)


def test_checkpoint_rejects_other_handles():
    inst = grid(8, 8, 33)
    betas = synth.beta_ladder(32)
    a = Engine(inst, 32, 2, betas, seed=KEY)
    blob = a.save_state()
    for other in (Engine(inst, 32, 2, betas, seed=KEY + 1),          # seed
                  Engine(inst, 32, 2, betas * 1.01, seed=KEY),       # ladder
                  Engine(grid(8, 8, 34), 32, 2, betas, seed=KEY),    # couplings
                  Engine(inst, 32, 2, betas, seed=KEY, copy_begin=1)):  # shard
        with pytest.raises(L.IsingError) as e:
            other.load_state(blob)
        assert e.value.code == L.ISING_E_STATE
    with pytest.raises(L.IsingError) as e:
        a.load_state(blob[:-1])
    assert e.value.code == L.ISING_E_ARG
    with pytest.raises(L.IsingError) as e:
        a.load_state(b"x" * len(blob))
    assert e.value.code == L.ISING_E_STATE


def _code_of(fn, *a):
    with pytest.raises(L.IsingError) as e:
        fn(*a)
    return e.value.code


def test_api_error_paths_on_live_handles():
    """include/ising.h error contract on live handles: wrong call order, slots outside the
    shard, bad values, and operations a layout / weight type does not support."""
    inst = grid(8, 8, 9)
    betas = synth.beta_ladder(32)
    eng = Engine(inst, 32, 4, betas, seed=KEY, copy_begin=1, copy_end=3, layout="bits")
    assert _code_of(L.ising_best, eng.h) == L.ISING_E_STATE               # no best check yet
    assert _code_of(L.ising_get_spins, eng.h, 0) == L.ISING_E_STATE       # slot of copy 0: not held
    assert _code_of(L.ising_get_spins, eng.h, 3 * 32) == L.ISING_E_STATE  # past the shard
    bad = np.ones(64, np.int8)
    bad[7] = 0
    assert _code_of(L.ising_set_spins, eng.h, 32, bad) == L.ISING_E_ARG
    assert _code_of(L.ising_sweep, eng.h, -1) == L.ISING_E_ARG
    assert _code_of(L.ising_run, eng.h, 1, 0) == L.ISING_E_ARG
    assert _code_of(L.ising_anneal, eng.h, -np.ones((2, 32))) == L.ISING_E_ARG
    assert _code_of(L.ising_icm, eng.h, 0) == L.ISING_E_UNSUPPORTED      # shard [1, 3) splits pairs
    eng.sweep(3)
    eng.check_best()
    b = eng.best(spins=True)
    assert 32 <= b["slot"] < 96 and b["spins"].shape == (64,)
    # float weights: no replica exchange (R15), no cluster moves on the int8 layout
    finst = _regular_inst(200, 4)
    f = Engine(finst, 8, 2, synth.beta_ladder(8), seed=KEY, layout="i8")
    assert _code_of(L.ising_exchange, f.h) == L.ISING_E_UNSUPPORTED
    assert _code_of(L.ising_run, f.h, 1, 10) == L.ISING_E_UNSUPPORTED
    assert _code_of(L.ising_icm, f.h, 0) == L.ISING_E_UNSUPPORTED
    assert "unsupported" in L.ising_last_error().lower() or L.ising_last_error() != ""
