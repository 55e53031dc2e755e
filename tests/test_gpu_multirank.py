"""N>1 path with the REAL library on one GPU: two processes (ranks), each holding its own
libising handle for a contiguous copy shard on cuda:0, exchanging through gloo (SURVEY.md
§8(e)).  The ranks' kernels never wait on one another -- the only coupling is the host-side
collective of the 16-byte per-slot records (north-star mode, gather=True: one all-gather per
exchange; gather=False: local best + one merge per run) -- so this is the multi-rank code
path of driver.run_pt + ising_exchange_begin/end, not a stand-in for more GPUs.
Both modes must reproduce the single-process oracle run bit for bit."""
import os
import socket
import tempfile

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no GPU", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

KEY = synth.PHILOX_KEY
K, C = 32, 4


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inst(kind):
    if kind == "grid":
        return synth.make_instance(dict(kind="grid", Lx=12, Ly=10, seed=55))
    u, v = synth.gnm(300, 420, 56)
    w = np.where(synth.splitmix64(57, u.size) >> np.uint64(63), -1, 1).astype(np.int32)
    rp, col, ww = synth.edges_to_csr(300, u, v, w)
    return dict(kind="csr", n=300, row_ptr=rp, col=col, w=ww.astype(np.int32))


def _worker(rank, world, port, out, kind, layout, gather, sweeps, kex):
    from paper_2311_09275_b200 import Engine
    from paper_2311_09275_b200.driver import run_pt, shard
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    a, b = shard(C, world, rank)
    eng = Engine(_inst(kind), K, C, synth.beta_ladder(K), seed=KEY, copy_begin=a, copy_end=b, layout=layout)
    rec = run_pt(eng, sweeps, kex, group=None, gather=gather)
    np.save(os.path.join(out, f"E{rank}.npy"), eng.energies())
    np.save(os.path.join(out, f"W{rank}.npy"), eng.walkers())
    np.save(os.path.join(out, f"rec{rank}.npy"), np.array([rec["E"], rec["slot"], rec["sweep"]]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,layout", [("grid", "bits"), ("csr", "i8")])
@pytest.mark.parametrize("gather", [True, False])
def test_two_ranks_on_library_equal_oracle(kind, layout, gather):
    world, sweeps, kex = 2, 35, 10
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_worker, args=(world, _free_port(), out, kind, layout, gather, sweeps, kex), nprocs=world,
                 join=True)
        E = np.concatenate([np.load(os.path.join(out, f"E{r}.npy")) for r in range(world)])
        W = np.concatenate([np.load(os.path.join(out, f"W{r}.npy")) for r in range(world)])
        recs = [np.load(os.path.join(out, f"rec{r}.npy")) for r in range(world)]
    rng = oracle.RNG_PLANE if layout == "bits" else oracle.RNG_WORD
    ref = oracle.Oracle(_inst(kind), K, synth.beta_ladder(K), KEY, 0, C, rng=rng).run(sweeps, kex)
    assert np.array_equal(E, ref.energies())
    assert np.array_equal(W, ref.walker)
    for r in recs:  # every rank reports the same global record
        assert (r[0], r[1], r[2]) == (ref.best.E, ref.best.slot, ref.best.sweep)


def _nccl_worker(rank, world, port, out):
    from paper_2311_09275_b200 import Engine
    from paper_2311_09275_b200.driver import all_gather
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", 0))
    inst = _inst("grid")
    eng = Engine(inst, K, C, synth.beta_ladder(K), seed=KEY, layout="bits")
    send, recv = eng.record_buffers(world)
    for _ in range(4):  # north-star round: sweeps, NCCL all-gather of the records, exchange
        eng.sweep(10)
        eng.exchange_begin(send)
        all_gather(recv, send, None)
        eng.exchange_end(recv)
    torch.cuda.synchronize()
    np.save(os.path.join(out, "E.npy"), eng.energies())
    np.save(os.path.join(out, "W.npy"), eng.walkers())
    from paper_2311_09275_b200.driver import merge_best_over_ranks
    b = merge_best_over_ranks(eng.best(spins=False), None, eng)  # the bench's per-step NCCL merge
    np.save(os.path.join(out, "rec.npy"), np.array([b["E"], b["slot"], b["sweep"]]))
    dist.destroy_process_group()


def test_nccl_record_gather_single_rank():
    """The NCCL branch of the record all-gather (all_gather_into_tensor on device buffers)
    feeding ising_exchange_end, and the NCCL best-record merge bench.py uses per step, on one
    rank: equal to the oracle's local exchanges."""
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_nccl_worker, args=(1, _free_port(), out), nprocs=1, join=True)
        E = np.load(os.path.join(out, "E.npy"))
        W = np.load(os.path.join(out, "W.npy"))
        rec = np.load(os.path.join(out, "rec.npy"))
    ref = oracle.Oracle(_inst("grid"), K, synth.beta_ladder(K), KEY, 0, C, rng=oracle.RNG_PLANE).run(40, 10)
    assert np.array_equal(E, ref.energies())
    assert np.array_equal(W, ref.walker)
    assert (rec[0], rec[1], rec[2]) == (ref.best.E, ref.best.slot, ref.best.sweep)


def _nccl2_worker(rank, world, port, out, gather, workload_kind):
    """One process per GPU (cuda:rank), NCCL, each rank a contiguous copy shard."""
    from paper_2311_09275_b200 import Engine
    from paper_2311_09275_b200.driver import run_pt, shard
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    a, b = shard(C, world, rank)
    eng = Engine(_inst(workload_kind), K, C, synth.beta_ladder(K), seed=KEY, copy_begin=a, copy_end=b,
                 layout="bits", device=rank)
    rec = run_pt(eng, 35, 10, group=None, gather=gather)
    np.save(os.path.join(out, f"E{rank}.npy"), eng.energies())
    np.save(os.path.join(out, f"W{rank}.npy"), eng.walkers())
    np.save(os.path.join(out, f"rec{rank}.npy"), np.array([rec["E"], rec["slot"], rec["sweep"]]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs (one process per GPU over NCCL)")
@pytest.mark.parametrize("gather", [True, False])
@pytest.mark.parametrize("kind", ["grid", "csr"])
def test_two_gpus_nccl_equal_oracle(gather, kind):
    """The N>1 path on hardware: 2 ranks on 2 GPUs over NCCL (record all-gather per exchange,
    or local bests merged by ising_merge_best), equal to the single-process oracle run."""
    world = 2
    with tempfile.TemporaryDirectory() as out:
        mp.spawn(_nccl2_worker, args=(world, _free_port(), out, gather, kind), nprocs=world, join=True)
        E = np.concatenate([np.load(os.path.join(out, f"E{r}.npy")) for r in range(world)])
        W = np.concatenate([np.load(os.path.join(out, f"W{r}.npy")) for r in range(world)])
        recs = [np.load(os.path.join(out, f"rec{r}.npy")) for r in range(world)]
    ref = oracle.Oracle(_inst(kind), K, synth.beta_ladder(K), KEY, 0, C, rng=oracle.RNG_PLANE).run(35, 10)
    assert np.array_equal(E, ref.energies())
    assert np.array_equal(W, ref.walker)
    for r in recs:
        assert (r[0], r[1], r[2]) == (ref.best.E, ref.best.slot, ref.best.sweep)
