"""GPU-vs-oracle parity on the configurations and launches bench.py times (needs a B200).

* C4a / C4b (BASELINE.json configs[3]): all 128 copies (16,384 replicas) on one GPU in the
  launch the bench times -- the persistent ticket-scheduled kernel (k_grid_sched, one CTA per
  SM taking (word group, round) tasks) and the cluster launch it replaced (k_grid_bits, clusters
  of 4 CTAs in ~4 waves) -- sampled copies from every wave, >= 100 sweeps (10 exchanges), bit for
  bit: spins of every slot of the copy, energies, walker ids and the per-copy best record.
* C2 (configs[1]) and C3 (configs[2]): 2 whole copies x 2,000 sweeps of the full 64-copy fused
  launch.
* C5 (configs[4]): 8 replicas of the full 4e6-vertex instance x 50 sweeps, and 16 replicas x 200
  sweeps in one call (the bench's packed-row kernel): identical spins, energies within 1e-5
  relative.
* k_grid_sched on small tori (forced with ISING_GRID_SCHED=1): every slot against the oracle and
  against the cluster launch, incl. swaps that cross words and tail sweeps after the rounds.
PAPER.md P:53 (PT exchanges replicas across temperatures), P:59 (sweeps as the unit of work).
"""
import threading

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no GPU", allow_module_level=True)

from paper_2311_09275_b200 import Engine, run_pt  # noqa: E402

KEY = synth.PHILOX_KEY


def grid(Lx, Ly, seed):
    Jr, Jd = synth.torus_pm1(Lx, Ly, seed)
    return dict(kind="grid", Lx=Lx, Ly=Ly, J_right=Jr, J_down=Jd, n=Lx * Ly)


def oracle_copies(inst, K, betas, copies, sweeps, kex, rng=oracle.RNG_PLANE, colour=None):
    """One oracle per sampled copy, run on host threads (the C oracle releases the GIL)."""
    out = {}

    def work(c0):
        out[c0] = oracle.Oracle(inst, K, betas, KEY, c0, c0 + 1, rng=rng, colour=colour).run(sweeps, kex)

    ts = [threading.Thread(target=work, args=(c,)) for c in copies]
    [t.start() for t in ts]
    [t.join() for t in ts]
    return out


def check_copy(eng, o, cb):
    """Every slot of oracle copy o (spins, energies, walkers) and its per-copy best record."""
    E, W = eng.energies(), eng.walkers()
    lo = o.slot0 - eng.slot0
    assert np.array_equal(E[lo:lo + o.R], o.energies())
    assert np.array_equal(W[lo:lo + o.R], o.walker)
    for r in range(o.R):
        assert np.array_equal(eng.spins(o.slot0 + r), o.s[r]), f"slot {o.slot0 + r}"
    c = o.copy_begin - eng.slot0 // eng.K
    ob = o.copy_best[0]
    assert (cb[0][c], cb[1][c], cb[2][c]) == (ob.E, ob.slot, ob.sweep)


@pytest.mark.parametrize("workload,sched,sweeps", [("c4b", "1", 1000), ("c4a", "1", 300), ("c4b", "0", 100),
                                                    ("c4a", "0", 100)],
                         ids=["c4b-sched", "c4a-sched", "c4b-clusters", "c4a-clusters"])
def test_c4_full_launch_sampled_copies(workload, sched, sweeps, monkeypatch):
    """The bench's C4 launch at 1 GPU: 128 copies x 128 temperatures, exchange every 10 --
    1,000 sweeps (100 exchanges) on C4b's persistent launch, the bench's kernel; copies 0, 41,
    86, 127 (first/middle/last waves of the cluster launch, tasks handed out across the whole
    grid by the persistent launch) equal the oracle bit for bit."""
    monkeypatch.setenv("ISING_GRID_SCHED", sched)
    cfg = synth.CONFIGS[workload]
    inst = synth.make_instance(cfg)
    K, C = cfg["K"], cfg["C"]
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    assert eng.info.fused_pt == (3 if sched == "1" else 1)
    run_pt(eng, sweeps, cfg["k_ex"])
    cb = eng.copy_best()
    for c0, o in oracle_copies(inst, K, betas, (0, 41, 86, 127), sweeps, cfg["k_ex"]).items():
        check_copy(eng, o, cb)


def test_c4b_sched_equals_cluster_launch_all_copies(monkeypatch):
    """All 16,384 slots: the persistent launch equals the cluster launch (energies, walkers,
    per-copy best, global best record and configuration), 200 sweeps."""
    cfg = synth.CONFIGS["c4b"]
    inst = synth.make_instance(cfg)
    K, C = cfg["K"], cfg["C"]
    betas = synth.beta_ladder(K)
    engs = []
    for sched in ("1", "0"):
        monkeypatch.setenv("ISING_GRID_SCHED", sched)
        e = Engine(inst, K, C, betas, seed=KEY, layout="bits")
        run_pt(e, 200, cfg["k_ex"])
        engs.append(e)
    a, b = engs
    assert a.info.fused_pt == 3 and b.info.fused_pt == 1
    assert np.array_equal(a.energies(), b.energies())
    assert np.array_equal(a.walkers(), b.walkers())
    for x, y in zip(a.copy_best(), b.copy_best()):
        assert np.array_equal(x, y)
    ba, bb = a.best(), b.best()
    assert (ba["E"], ba["slot"], ba["sweep"]) == (bb["E"], bb["slot"], bb["sweep"])
    assert np.array_equal(ba["spins"], bb["spins"])
    for r in range(0, K * C, 997):
        assert np.array_equal(a.spins(r), b.spins(r))


def test_c2_two_whole_copies_2000_sweeps():
    """C2's fused launch (64 copies) over 2,000 sweeps (200 exchanges): copies 5 and 58 equal
    the oracle bit for bit, including walker ids and per-copy best."""
    cfg = synth.CONFIGS["c2"]
    inst = synth.make_instance(cfg)
    K, C = cfg["K"], cfg["C"]
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    run_pt(eng, 2000, cfg["k_ex"])
    cb = eng.copy_best()
    for c0, o in oracle_copies(inst, K, betas, (5, 58), 2000, cfg["k_ex"]).items():
        check_copy(eng, o, cb)


def test_c3_two_whole_copies_2000_sweeps():
    """C3's fused launch (G(1e4, 9999), smallest-last colouring, 64 copies) over 2,000 sweeps:
    copies 3 and 60 equal the oracle bit for bit, including walker ids and per-copy best."""
    cfg = synth.CONFIGS["c3"]
    inst = synth.make_instance(cfg)
    K, C = cfg["K"], cfg["C"]
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="bits", colour=cfg["colouring"])
    run_pt(eng, 2000, cfg["k_ex"])
    cb = eng.copy_best()
    col, _ = oracle.greedy_colour_sl(inst["n"], inst["row_ptr"], inst["col"])
    for c0, o in oracle_copies(inst, K, betas, (3, 60), 2000, cfg["k_ex"], colour=col).items():
        check_copy(eng, o, cb)


def test_c5_full_size_eight_replicas_50_sweeps():
    """C5 at full size (4e6 vertices, 256 replicas, the cp.async ring kernel): 8 replicas
    spread over the 256 x 50 sweeps -- identical spins, energies within 1e-5 relative."""
    cfg = synth.CONFIGS["c5"]
    inst = synth.make_instance(cfg)
    K = cfg["K"]
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, cfg["C"], betas, seed=KEY, layout="i8", colour=cfg["colouring"])
    sweeps = 50
    eng.sweep(sweeps)
    E = eng.energies()
    col, _ = (oracle.greedy_colour_jp if cfg["colouring"] == "jp" else oracle.greedy_colour_sl)(
        inst["n"], inst["row_ptr"], inst["col"])
    slots = (0, 37, 64, 101, 128, 170, 211, 255)
    res = {}

    def work(lo):
        o = oracle.Oracle(inst, K, betas, KEY, 0, 1, rng=oracle.RNG_WORD, colour=col, slots=(lo, lo + 1))
        o.sweeps(sweeps)
        res[lo] = (o.s[0].copy(), o.energies()[0])

    ts = [threading.Thread(target=work, args=(lo,)) for lo in slots]
    [t.start() for t in ts]
    [t.join() for t in ts]
    for lo in slots:
        s, e = res[lo]
        assert np.array_equal(eng.spins(lo), s), f"slot {lo}"
        assert abs(E[lo] - e) <= 1e-5 * abs(e)


def test_c5_packed_rows_16_replicas_200_sweeps():
    """C5 at full size on the bench's kernel (the packed-row working copy: one ising_sweep call of
    200 sweeps) against the oracle for 16 replicas spread over the 256 (every lane group of a
    warp, both halves of a Philox call): identical spins, energies within 1e-5 relative."""
    cfg = synth.CONFIGS["c5"]
    inst = synth.make_instance(cfg)
    K = cfg["K"]
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, cfg["C"], betas, seed=KEY, layout="i8", colour=cfg["colouring"])
    sweeps = 200
    eng.sweep(sweeps)
    E = eng.energies()
    col, _ = oracle.greedy_colour_jp(inst["n"], inst["row_ptr"], inst["col"])
    slots = (1, 14, 30, 47, 62, 77, 91, 108, 126, 143, 157, 172, 190, 205, 222, 254)
    res = {}

    def work(lo):
        o = oracle.Oracle(inst, K, betas, KEY, 0, 1, rng=oracle.RNG_WORD, colour=col, slots=(lo, lo + 1))
        o.sweeps(sweeps)
        res[lo] = (o.s[0].copy(), o.energies()[0])

    ts = [threading.Thread(target=work, args=(lo,)) for lo in slots]
    [t.start() for t in ts]
    [t.join() for t in ts]
    for lo in slots:
        s, e = res[lo]
        assert np.array_equal(eng.spins(lo), s), f"slot {lo}"
        assert abs(E[lo] - e) <= 1e-5 * abs(e)


@pytest.mark.parametrize("Lx,Ly,K,C,sweeps,kex", [
    (16, 16, 64, 2, 100, 10),    # 4 groups
    (6, 4, 32, 3, 33, 7),        # one word per copy, tail sweeps after the rounds
    (10, 8, 96, 2, 40, 5),       # 3 words per copy: cross-word pairs at both ends of word 1
    (12, 20, 256, 1, 60, 3),     # 8 words per copy
    (8, 8, 128, 41, 30, 10),     # 164 groups > 148 SMs: tasks of two rounds in flight
    (80, 100, 32, 2, 30, 10),    # C2 geometry: leftover rows spill onto the column-less warps
])
def test_sched_fused_pt_parity(Lx, Ly, K, C, sweeps, kex, monkeypatch):
    """k_grid_sched (forced) == oracle for every slot, and == the cluster launch."""
    monkeypatch.setenv("ISING_GRID_SCHED", "1")
    monkeypatch.setenv("ISING_GRID_BANDS", "1")  # the persistent launch is the single-band kernel
    inst = grid(Lx, Ly, 91 + Lx * Ly)
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    assert eng.info.fused_pt == 3
    rec = run_pt(eng, sweeps, kex, fused=True)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_PLANE).run(sweeps, kex)
    assert np.array_equal(eng.energies(), o.energies())
    assert np.array_equal(eng.walkers(), o.walker)
    for r in range(K * C):
        assert np.array_equal(eng.spins(r), o.s[r]), f"slot {r}"
    assert (rec["E"], rec["slot"], rec["sweep"]) == (o.best.E, o.best.slot, o.best.sweep)
    b = eng.best(spins=True)
    assert np.array_equal(b["spins"], o.best.spins)
    cb = eng.copy_best()
    for c in range(C):
        assert (cb[0][c], cb[1][c], cb[2][c]) == (o.copy_best[c].E, o.copy_best[c].slot, o.copy_best[c].sweep)
    monkeypatch.setenv("ISING_GRID_SCHED", "0")
    ref = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    run_pt(ref, sweeps, kex, fused=True)
    assert np.array_equal(ref.energies(), eng.energies())
    assert np.array_equal(ref.walkers(), eng.walkers())


@pytest.mark.parametrize("Lx,Ly,K,C,sweeps,kex", [
    (16, 16, 64, 2, 40, 10),     # 4 groups, per-round sweep calls of 10 (2 chunks of 5)
    (6, 4, 32, 3, 21, 4),        # one word per copy; a tail call of 1 sweep (odd: k_grid_bits)
    (8, 8, 128, 41, 24, 6),      # 164 groups > 148 SMs: chunks of a group on different CTAs
    (80, 100, 32, 2, 20, 10),    # C2 geometry (leftover-row spill)
])
def test_sched_plain_sweeps_parity(Lx, Ly, K, C, sweeps, kex, monkeypatch):
    """Plain sweep calls on k_grid_sched (tasks = (group, half of the call's sweeps), the per-round
    path of run_pt(gather=True)): every slot, walker and the best record equal the oracle's and
    the k_grid_bits sweeps' (ISING_GRID_SCHED=0)."""
    monkeypatch.setenv("ISING_GRID_BANDS", "1")
    inst = grid(Lx, Ly, 191 + Lx * Ly)
    betas = synth.beta_ladder(K)
    res = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("ISING_GRID_SCHED", mode)
        eng = Engine(inst, K, C, betas, seed=KEY, layout="bits")
        assert (eng.info.fused_pt == 3) == (mode == "1")
        rec = run_pt(eng, sweeps, kex, fused=False)
        res[mode] = (eng.energies(), eng.walkers(), [eng.spins(r) for r in range(K * C)], rec)
        eng.close()
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_PLANE).run(sweeps, kex)
    for mode in ("1", "0"):
        E, W, S, rec = res[mode]
        assert np.array_equal(E, o.energies()), mode
        assert np.array_equal(W, o.walker), mode
        for r in range(K * C):
            assert np.array_equal(S[r], o.s[r]), f"{mode}: slot {r}"
        assert (rec["E"], rec["slot"], rec["sweep"]) == (o.best.E, o.best.slot, o.best.sweep)


def test_c4b_north_star_mode_sched_sweeps(monkeypatch):
    """C4b's per-round path (sweep calls of 10 on the persistent kernel, record export, gathered
    records, exchange) over 100 sweeps equals the fused schedule on every slot of 3 sampled
    copies and in the best record."""
    cfg = synth.CONFIGS["c4b"]
    inst = synth.make_instance(cfg)
    K, C, kex = cfg["K"], cfg["C"], cfg["k_ex"]
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    assert eng.info.fused_pt == 3
    send, recv = eng.record_buffers(1)
    for _ in range(10):
        eng.sweep(kex)
        eng.exchange_begin(send)
        recv.copy_(send)
        eng.exchange_end(recv)
    ref = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    ref.run(10, kex)
    assert np.array_equal(eng.energies(), ref.energies())
    assert np.array_equal(eng.walkers(), ref.walkers())
    for c in (0, 63, 127):
        for r in range(c * K, (c + 1) * K, 5):
            assert np.array_equal(eng.spins(r), ref.spins(r)), f"slot {r}"
    b, rb = eng.best(spins=False), ref.best(spins=False)
    assert (b["E"], b["slot"], b["sweep"]) == (rb["E"], rb["slot"], rb["sweep"])


def test_sched_split_runs_and_state_roundtrip(monkeypatch):
    """Two ising_run calls (the second continuing t and e) and a checkpoint of the persistent
    launch's state, resumed on a fresh handle, equal one oracle run."""
    monkeypatch.setenv("ISING_GRID_SCHED", "1")
    monkeypatch.setenv("ISING_GRID_BANDS", "1")
    inst = grid(12, 10, 5)
    K, C = 64, 5
    betas = synth.beta_ladder(K)
    eng = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    eng.run(3, 10)
    blob = eng.save_state()
    eng.run(2, 10)
    o = oracle.Oracle(inst, K, betas, KEY, 0, C, rng=oracle.RNG_PLANE).run(50, 10)
    assert np.array_equal(eng.energies(), o.energies())
    assert np.array_equal(eng.walkers(), o.walker)
    again = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    again.load_state(blob)
    again.run(2, 10)
    assert np.array_equal(again.energies(), o.energies())
    for r in range(0, K * C, 7):
        assert np.array_equal(again.spins(r), o.s[r])


def test_merge_best_records_on_device():
    """ising_merge_best == the lexicographic (E, sweep, slot) minimum, int and float
    energies, records without a slot ignored."""
    inst = grid(4, 4, 404)
    eng = Engine(inst, 32, 1, synth.beta_ladder(32), seed=KEY, layout="bits")
    rows = np.array([[-10, 50, 7], [-12, 90, 3], [-12, 40, 9], [-12, 40, 2], [-99, 1, -1]], np.int64)
    r = eng.merge_best(torch.from_numpy(rows))
    assert (r["E"], r["sweep"], r["slot"]) == (-12, 40, 2)
    rng = np.random.default_rng(3)
    big = np.stack([rng.integers(-40, 0, 3000), rng.integers(0, 5, 3000), rng.permutation(3000)], 1).astype(np.int64)
    want = min(tuple(x) for x in big.tolist())
    r = eng.merge_best(torch.from_numpy(big))
    assert (r["E"], r["sweep"], r["slot"]) == want
    # float energies (double bits): a float handle
    u, v = synth.random_regular(64, 3, 1)
    rp, col, w = synth.edges_to_csr(64, u, v, synth.gaussian_f32(u.size, 2))
    feng = Engine(dict(kind="csr", n=64, row_ptr=rp, col=col, w=w.astype(np.float32)), 8, 1,
                  synth.beta_ladder(8), seed=KEY, layout="i8")
    fr = np.array([[-1.5, 3, 4], [-2.25, 9, 1], [-2.25, 9, 0], [-0.5, 0, 2]], np.float64)
    recs = np.stack([fr[:, 0].view(np.int64), fr[:, 1].astype(np.int64), fr[:, 2].astype(np.int64)], 1)
    r = feng.merge_best(torch.from_numpy(np.ascontiguousarray(recs)))
    assert (r["E"], r["sweep"], r["slot"]) == (-2.25, 9, 0)


def test_c4b_gpu_count_invariance_with_each_shares_kernel():
    """The strong-scaling shares of C4b -- 2 / 4 / 8 GPUs hold 64 / 32 / 16 copies, run by the
    persistent launch / the cluster launch / the band-split cooperative launch -- reproduce the
    1-GPU run (persistent launch over all 128 copies) bit for bit: energies, walkers and
    per-copy best of every slot, 200 sweeps (every RNG counter uses global ids)."""
    cfg = synth.CONFIGS["c4b"]
    inst = synth.make_instance(cfg)
    K, C = cfg["K"], cfg["C"]
    betas = synth.beta_ladder(K)
    full = Engine(inst, K, C, betas, seed=KEY, layout="bits")
    run_pt(full, 200, cfg["k_ex"])
    E, W = full.energies(), full.walkers()
    cb = full.copy_best()
    for N, kernel_fused in ((2, 3), (4, 1), (8, 2)):
        share = C // N
        for rank in (0, N - 1):
            a, b = rank * share, (rank + 1) * share
            eng = Engine(inst, K, C, betas, seed=KEY, copy_begin=a, copy_end=b, layout="bits")
            assert eng.info.fused_pt == kernel_fused, (N, eng.info.fused_pt)
            run_pt(eng, 200, cfg["k_ex"])
            assert np.array_equal(eng.energies(), E[a * K:b * K]), N
            assert np.array_equal(eng.walkers(), W[a * K:b * K]), N
            for x, y in zip(eng.copy_best(), cb):
                assert np.array_equal(x, y[a:b]), N
