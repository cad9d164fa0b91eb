"""World-size-2 gloo test of the multi-GPU host logic (sharding + top-K gather).

Each rank docks its shard with the CPU oracle standing in for its GPU, then
the ranks all-gather the top-K tables; the merged table must equal a
single-process run over all ligands, bit for bit.
"""
import os
import socket
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, scaling, out_dir):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    from oracle import oracle_py as O
    from paper_1901_06363_b200 import Knobs, synth_ligands, synth_pocket
    from paper_1901_06363_b200.sharding import gather_topk, shard_ids

    dist.init_process_group("gloo", rank=rank, world_size=world)
    pocket = synth_pocket(6.0, 5.0, 4.0, 1.0)
    knobs = Knobs.baseline(90, 60, 1, 4)
    n = 3 if scaling == "weak" else 5
    ids = shard_ids(rank, world, n, scaling)
    batch = synth_ligands(77, ids, 12, 20, centre=pocket.mean(axis=0))
    res = O.dock_batch(batch, pocket, knobs, nthreads=1, keep_poses=False)
    merged = gather_topk(res, world, device="cpu")
    if rank == 0:
        np.savez(Path(out_dir) / f"merged_{scaling}.npz", **merged)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_sharded_gather_equals_single_process(tmp_path, scaling):
    import torch.multiprocessing as mp
    from oracle import oracle_py as O
    from paper_1901_06363_b200 import Knobs, synth_ligands, synth_pocket
    from paper_1901_06363_b200.sharding import shard_ids

    world = 2
    mp.spawn(_worker, args=(world, _free_port(), scaling, str(tmp_path)), nprocs=world, join=True)
    merged = np.load(tmp_path / f"merged_{scaling}.npz")
    pocket = synth_pocket(6.0, 5.0, 4.0, 1.0)
    n = 3 if scaling == "weak" else 5
    ids = [i for r in range(world) for i in shard_ids(r, world, n, scaling)]
    assert ids == list(range(len(ids)))
    batch = synth_ligands(77, ids, 12, 20, centre=pocket.mean(axis=0))
    want = O.dock_batch(batch, pocket, Knobs.baseline(90, 60, 1, 4), nthreads=2, keep_poses=False)
    from paper_1901_06363_b200.sharding import LIGAND_FIELDS, SLOT_FIELDS
    for f, dt in {**SLOT_FIELDS, **LIGAND_FIELDS}.items():
        assert merged[f].dtype == dt, f  # native dtypes, no float64 packing
        assert np.array_equal(merged[f], getattr(want, f)), f


def _gather_worker(rank, world, port, out_dir):
    sys.path.insert(0, str(ROOT))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    from paper_1901_06363_b200.sharding import DeviceGather

    dist.init_process_group("gloo", rank=rank, world_size=world)
    L, K = 3, 4
    tables = {"final_score": torch.full((L, K), float(rank) + 0.5, dtype=torch.float64),
              "orientation": torch.full((L, K), rank, dtype=torch.int32),
              "seed_rank": torch.arange(L * K, dtype=torch.int32).reshape(L, K),
              "evaluations": torch.full((L, K), 10 * rank, dtype=torch.int64),
              "rigid_score": torch.full((L, K), float(rank) + 0.25, dtype=torch.float64),
              "feasibility_checks": torch.full((L, K), 7 * rank + 2**40, dtype=torch.int64),
              "k_eff": torch.full((L,), K - rank, dtype=torch.int32),
              "poses_scored": torch.full((L,), 2**41 + rank, dtype=torch.int64),
              "status": torch.full((L,), rank, dtype=torch.int32)}
    out = DeviceGather(tables, world)()
    if rank == 0:
        np.savez(Path(out_dir) / "gather.npz",
                 **{f: torch.stack(out[f]).numpy() for f in DeviceGather.FIELDS})
    dist.barrier()
    dist.destroy_process_group()


def test_device_gather_all_gathers_every_field(tmp_path):
    """The per-step top-K gather bench.py runs over NCCL, here over gloo."""
    import torch.multiprocessing as mp
    world = 2
    mp.spawn(_gather_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    z = np.load(tmp_path / "gather.npz")
    for r in range(world):
        assert (z["final_score"][r] == r + 0.5).all()
        assert (z["orientation"][r] == r).all()
        assert (z["evaluations"][r] == 10 * r).all()
        assert np.array_equal(z["seed_rank"][r], np.arange(12).reshape(3, 4))
        assert (z["rigid_score"][r] == r + 0.25).all()
        assert (z["feasibility_checks"][r] == 7 * r + 2**40).all()
        assert (z["k_eff"][r] == 4 - r).all() and (z["status"][r] == r).all()
        assert (z["poses_scored"][r] == 2**41 + r).all() and z["poses_scored"].dtype == np.int64


def test_shard_ids_cover_exactly():
    from paper_1901_06363_b200.sharding import shard_ids
    for world in (1, 2, 3, 8):
        got = [i for r in range(world) for i in shard_ids(r, world, 10, "strong")]
        assert got == list(range(10))
        got = [i for r in range(world) for i in shard_ids(r, world, 4, "weak")]
        assert got == list(range(4 * world))
