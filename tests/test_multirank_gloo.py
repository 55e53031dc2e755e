"""N>1 path of the driver on CPU: world_size 2 over gloo.

The run schedule (driver.run_pt), the per-exchange record all-gather (north-star
mode) and the end-of-run best merge are exercised with 2 ranks, each simulating a
contiguous copy shard.  The per-rank engine here is a test-only adapter around the
CPU oracle (it implements the Engine interface; the product Engine needs a GPU).
Both modes must give the same best record as one process holding all copies."""
import os
import socket
import tempfile

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth
from paper_2311_09275_b200.driver import run_pt, shard


class OracleEngine:
    """Engine interface backed by the CPU oracle (tests only)."""

    def __init__(self, inst, K, C, betas, seed, copy_begin, copy_end):
        self.o = oracle.Oracle(inst, K, betas, seed, copy_begin, copy_end)
        self.R, self.slot0 = self.o.R, self.o.slot0
        self.gbest = None

    def sweep(self, n):
        self.o.sweeps(n)

    def exchange(self):
        self.o.check_best()
        self.o.exchange()

    def record_buffers(self, world):
        return torch.zeros((self.R, 2), dtype=torch.int64), torch.zeros((self.R * world, 2), dtype=torch.int64)

    def exchange_begin(self, send):
        send[:, 0] = torch.from_numpy(self.o.Ei)
        send[:, 1] = torch.arange(self.slot0, self.slot0 + self.R)

    def _global_best(self, recv):
        rows = recv.numpy()
        i = np.lexsort((rows[:, 1], rows[:, 0]))[0]
        E, slot = int(rows[i, 0]), int(rows[i, 1])
        if self.gbest is None or E < self.gbest["E"]:
            self.gbest = dict(E=E, slot=slot, sweep=self.o.t)

    def exchange_end(self, recv):
        self._global_best(recv)
        self.o.exchange()

    def check_best(self, recv=None):
        if recv is None:
            self.o.check_best()
        else:
            self._global_best(recv)

    def merge_best(self, recs):
        """ising_merge_best's rule on the host: lexicographic (E, sweep, slot) over the ranks'
        records (test-side; the product Engine merges on the device)."""
        rows = [tuple(int(x) for x in r) for r in recs.numpy() if r[2] >= 0]
        E, sweep, slot = min(rows)
        return dict(E=E, slot=slot, sweep=sweep)

    def best(self, spins=True):
        if self.gbest is not None:
            return dict(self.gbest)
        b = self.o.best
        return dict(E=b.E, slot=b.slot, sweep=b.sweep)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out, gather, sweeps, kex):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    inst = synth.make_instance(dict(kind="grid", Lx=8, Ly=8, seed=31))
    K, C = 16, 6
    a, b = shard(C, world, rank)
    eng = OracleEngine(inst, K, C, synth.beta_ladder(K), 99, a, b)
    rec = run_pt(eng, sweeps, kex, group=None, gather=gather)
    np.save(os.path.join(out, f"E{rank}.npy"), eng.o.Ei)
    np.save(os.path.join(out, f"rec{rank}.npy"), np.array([rec["E"], rec["slot"], rec["sweep"]]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("gather", [True, False])
@pytest.mark.parametrize("sweeps,kex", [(40, 10), (33, 10)])
def test_two_rank_run_equals_single_process(gather, sweeps, kex):
    world = 2
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_worker, args=(world, _free_port(), out, gather, sweeps, kex), nprocs=world, join=True)
        recs = [np.load(os.path.join(out, f"rec{r}.npy")) for r in range(world)]
        E = np.concatenate([np.load(os.path.join(out, f"E{r}.npy")) for r in range(world)])
    inst = synth.make_instance(dict(kind="grid", Lx=8, Ly=8, seed=31))
    ref = oracle.Oracle(inst, 16, synth.beta_ladder(16), 99, 0, 6).run(sweeps, kex)
    assert np.array_equal(E, ref.Ei)
    for r in recs:  # every rank reports the same global record
        assert (r[0], r[1], r[2]) == (ref.best.E, ref.best.slot, ref.best.sweep)
