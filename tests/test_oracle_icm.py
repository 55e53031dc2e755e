"""Pins of the oracle's Houdayer / isoenergetic cluster move (PAPER.md
P:53, refs [20][21]; SPEC.md S:294-302, S:325 for the invariants)."""
import numpy as np
import pytest
from scipy import stats
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import connected_components

import oracle
import synth


def grid(Lx, Ly, seed):
    Jr, Jd = synth.torus_pm1(Lx, Ly, seed)
    return dict(kind="grid", Lx=Lx, Ly=Ly, J_right=Jr, J_down=Jd)


def test_icm_conserves_pair_energy_and_overlap():
    inst = grid(8, 8, 3)
    K, C = 8, 4
    o = oracle.Oracle(inst, K, synth.beta_ladder(K), 9, 0, C)
    o.sweeps(5)
    moved = 0
    for _ in range(40):
        before = o.s.copy()
        E0 = o.Ei.copy().reshape(C, K)
        moved += o.icm(k_min=3)
        E1 = o.Ei.reshape(C, K)
        assert np.array_equal(E0[0::2] + E0[1::2], E1[0::2] + E1[1::2])  # S:302 isoenergetic
        assert np.array_equal(o.Ei, o.energy_scratch())
        s0, s1 = before.reshape(C, K, -1), o.s.reshape(C, K, -1)
        # overlap invariant; temperatures below k_min untouched
        assert np.array_equal(s0[0::2] != s0[1::2], s1[0::2] != s1[1::2])
        assert np.array_equal(s0[:, :3], s1[:, :3])
        o.sweeps(1)
    assert moved > 0


def test_icm_identical_replicas_is_noop_and_opposite_flips_component():
    inst = grid(6, 6, 4)
    o = oracle.Oracle(inst, 4, synth.beta_ladder(4), 1, 0, 2)
    o.s[4:8] = o.s[0:4]                       # copy 1 == copy 0
    o.Ei[:] = o.energy_scratch()
    snap = o.s.copy()
    assert o.icm(0) == 0 and np.array_equal(o.s, snap)
    o.s[4:8] = -o.s[0:4]                      # copy 1 == -copy 0: cluster = whole torus
    o.Ei[:] = o.energy_scratch()
    snap = o.s.copy()
    assert o.icm(0) == 4
    assert np.array_equal(o.s[0:4], -snap[0:4]) and np.array_equal(o.s[4:8], -snap[4:8])


def test_icm_flips_exactly_one_component_of_the_overlap_graph():
    inst = grid(10, 8, 7)
    o = oracle.Oracle(inst, 2, synth.beta_ladder(2), 5, 0, 2)
    n = o.n
    A = csr_matrix((np.ones(o.col.size), o.col, o.rp), shape=(n, n))
    for _ in range(20):
        o.sweeps(3)
        before = o.s.copy()
        o.icm(0)
        for k in range(2):
            a0, b0 = before[k], before[2 + k]
            F = np.flatnonzero(o.s[k] != a0)
            if F.size == 0:
                continue
            X = np.flatnonzero(a0 != b0)
            sub = A[X][:, X]
            ncomp, lab = connected_components(sub, directed=False)
            comp_of = dict(zip(X.tolist(), lab.tolist()))
            labs = {comp_of[i] for i in F.tolist()}
            assert len(labs) == 1                      # one component ...
            lab0 = labs.pop()
            comp = {i for i in X.tolist() if comp_of[i] == lab0}
            assert comp == set(F.tolist())             # ... and all of it
            assert np.array_equal(np.flatnonzero(o.s[2 + k] != b0), F)


def test_pt_with_icm_samples_boltzmann():
    """Detailed balance: sweeps + Houdayer moves keep each temperature Boltzmann."""
    u = np.array([0, 1, 2, 2, 3, 0]); v = np.array([1, 2, 0, 3, 4, 4])
    w = np.array([1, -1, 1, -1, 1, -1])
    rp, col, ww = synth.edges_to_csr(5, u, v, w)
    inst = dict(kind="csr", n=5, row_ptr=rp, col=col, w=ww.astype(np.int32))
    betas = np.array([0.5, 1.0])
    C = 256
    o = oracle.Oracle(inst, 2, betas, 77, 0, C)
    pw = 1 << np.arange(5)
    hist = np.zeros((2, 32))
    o.sweeps(10)
    for rnd in range(60):
        o.sweeps(2)
        o.icm(0)
        if rnd >= 5:
            idx = ((o.s < 0).astype(np.int64) @ pw)
            for k in range(2):
                hist[k] += np.bincount(idx[k::2], minlength=32)
    states = 1 - 2 * ((np.arange(32)[:, None] >> np.arange(5)[None, :]) & 1)
    Es = np.sum(w * states[:, u] * states[:, v], axis=1)
    for k, b in enumerate(betas):
        p = np.exp(-b * (Es - Es.min())); p /= p.sum()
        chi2 = np.sum((hist[k] - p * hist[k].sum()) ** 2 / (p * hist[k].sum()))
        assert stats.chi2.sf(chi2, 31) > 1e-4, (k, chi2)
