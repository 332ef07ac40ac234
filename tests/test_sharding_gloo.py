"""World-size-2 gloo run of the multi-rank path on CPU: each rank solves its
cfg4 shard with the serial emulation of the device solver, the step time is
max-reduced, results are gathered, and the union equals a single-rank run."""

import os
import sys

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as tmp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from emu.emu_binding import EmuEngine
    from paper_2503_06922_b200 import scenarios, shard
    per = 3
    start, stop = shard.shard_range(rank, world, per, scenarios.CFG4_TOTAL)
    w = scenarios.cfg4(per, start=start)
    H = EmuEngine(**w.engine_kwargs()).solve(w.x0, w.tensions, w.applied, w.tol, w.max_frames)
    t = shard.max_over_ranks(float(rank + 1), dist)
    coords, frames, status = shard.gather_results([H["coords"], H["frames"], H["status"]], dist)
    if rank == 0:
        np.savez(out_path, coords=coords, frames=frames, status=status, tmax=t)
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_shards_equal_single_rank(tmp_path):
    from emu.emu_binding import EmuEngine
    from paper_2503_06922_b200 import scenarios
    out = str(tmp_path / "r.npz")
    port = 29500 + os.getpid() % 1000
    tmp.spawn(_worker, args=(2, port, out), nprocs=2, join=True)
    r = np.load(out)
    assert float(r["tmax"]) == 2.0
    w = scenarios.cfg4(6)
    H = EmuEngine(**w.engine_kwargs()).solve(w.x0, w.tensions, w.applied, w.tol, w.max_frames)
    assert np.array_equal(r["frames"], H["frames"])
    assert np.array_equal(r["status"], H["status"])
    assert np.array_equal(r["coords"], H["coords"])


def test_shard_range():
    from paper_2503_06922_b200.shard import shard_range
    assert shard_range(0, 8, 8192, 65536) == (0, 8192)
    assert shard_range(7, 8, 8192, 65536) == (57344, 65536)
    with pytest.raises(ValueError):
        shard_range(2, 2, 1, 10)


def _queue_worker(rank, world, port, out_path):
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2503_06922_b200 import shard
    store = dist.distributed_c10d._get_default_store()
    total = 1000
    mine = np.full(total, -1, np.int64)
    q = shard.ChunkQueue(store, "t0", total, 64)
    while True:
        r = q.next()
        if r is None:
            break
        mine[r[0]:r[1]] = rank
    owners = shard.all_max([mine], dist)[0]
    claimed = shard.gather_results([np.array([(mine >= 0).sum()])], dist)[0]
    if rank == 0:
        np.savez(out_path, owners=owners, claimed=claimed)
    dist.barrier()
    dist.destroy_process_group()


def test_dynamic_chunk_queue_covers_the_table_once(tmp_path):
    """ChunkQueue over the gloo store: every scenario claimed by exactly one rank."""
    out = str(tmp_path / "q.npz")
    port = 30500 + os.getpid() % 1000
    tmp.spawn(_queue_worker, args=(2, port, out), nprocs=2, join=True)
    r = np.load(out)
    assert (r["owners"] >= 0).all()
    assert int(r["claimed"].sum()) == 1000
