"""Multi-GPU plumbing: ligand sharding and the per-ligand top-K gather.

Every (ligand, pocket) dock is independent, so the only
exchange is gathering results at the end.  One process
per GPU; `torch.distributed` carries the gather (NCCL on GPUs, gloo on CPU
for the tests).  (One process driving several GPUs is the C-ABI's
gd_multi_* instead: no collective at all, each device's chunks land in the
caller's arrays.)
"""
from __future__ import annotations

import numpy as np

# Every per-slot ([L, K]) and per-ligand ([L]) field of gd_result except the
# poses, with its native dtype.
SLOT_FIELDS = {"final_score": np.float64, "orientation": np.int32, "seed_rank": np.int32,
               "evaluations": np.int64, "rigid_score": np.float64, "feasibility_checks": np.int64}
LIGAND_FIELDS = {"k_eff": np.int32, "poses_scored": np.int64, "status": np.int32}


def shard_ids(rank: int, world: int, n: int, scaling: str = "weak") -> range:
    """Ligand ids of `rank`: weak = every rank docks its own n ligands;
    strong = n ligands split into contiguous, near-equal shards."""
    if scaling == "weak":
        return range(rank * n, (rank + 1) * n)
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


class DeviceGather:
    """Per-step top-K gather straight from each rank's device-resident result
    table (Docker.device_results()): one NCCL all-gather per field, native
    dtypes, over NVLink/NVSwitch, no host round trip.  Weak scaling: equal
    shard shapes."""

    FIELDS = tuple(SLOT_FIELDS) + tuple(LIGAND_FIELDS)

    def __init__(self, tables: dict, world: int):
        import torch
        self.world = world
        self.tables = tables
        self.out = {f: [torch.empty_like(tables[f]) for _ in range(world)] for f in self.FIELDS}

    def __call__(self):
        import torch.distributed as dist
        for f in self.FIELDS:
            dist.all_gather(self.out[f], self.tables[f])
        return self.out


def gather_topk(result, world: int, device=None) -> dict:
    """All-gather every rank's result (all SLOT_FIELDS [L, K] and
    LIGAND_FIELDS [L], native dtypes) and return them concatenated in rank
    order, i.e. ligand-id order for contiguous shards.  Shards may differ in
    length (padded to the longest for the collective)."""
    import torch
    import torch.distributed as dist

    dev = device or ("cuda" if torch.cuda.is_available() and dist.get_backend() == "nccl" else "cpu")
    L, K = result.final_score.shape
    sizes = torch.tensor([L], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes)
    n = [int(s.item()) for s in all_sizes]
    Lmax = max(n)
    merged = {}
    for f, dt in {**SLOT_FIELDS, **LIGAND_FIELDS}.items():
        a = np.asarray(getattr(result, f), dtype=dt)
        pad = np.zeros((Lmax,) + a.shape[1:], dtype=dt)
        pad[:L] = a
        t = torch.from_numpy(pad).to(dev)
        outs = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(outs, t)  # NCCL over NVLink on GPUs; gloo on CPU
        merged[f] = np.concatenate([outs[r].cpu().numpy()[: n[r]] for r in range(world)], axis=0)
    return merged
