"""Multi-GPU plumbing: ligand sharding and the per-ligand top-K gather.

Every (ligand, pocket) dock is independent, so the only
exchange is gathering results at the end.  One process
per GPU; `torch.distributed` carries the gather (NCCL on GPUs, gloo on CPU
for the tests).
"""
from __future__ import annotations

import numpy as np


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
    table (Docker.device_results()): one NCCL all-gather per field over
    NVLink/NVSwitch, no host round trip.  Weak scaling: equal shard shapes."""

    FIELDS = ("final_score", "orientation", "seed_rank", "evaluations")

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


def gather_topk(result, world: int, device=None):
    """All-gather every rank's [L, K] top-K table (final score, orientation,
    seed rank, evaluations) and return them concatenated in rank order, i.e.
    ligand-id order for contiguous shards.  Shards may differ in length."""
    import torch
    import torch.distributed as dist

    dev = device or ("cuda" if torch.cuda.is_available() and dist.get_backend() == "nccl" else "cpu")
    L, K = result.final_score.shape
    sizes = torch.tensor([L], dtype=torch.int64, device=dev)
    all_sizes = [torch.zeros_like(sizes) for _ in range(world)]
    dist.all_gather(all_sizes, sizes)
    Lmax = int(max(s.item() for s in all_sizes))
    pack = np.zeros((Lmax, K, 4), dtype=np.float64)
    pack[:L, :, 0] = result.final_score
    pack[:L, :, 1] = result.orientation
    pack[:L, :, 2] = result.seed_rank
    pack[:L, :, 3] = result.evaluations
    t = torch.from_numpy(pack).to(dev)
    outs = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(outs, t)  # NCCL all-gather over NVLink on GPUs; gloo on CPU
    parts = [outs[r].cpu().numpy()[: int(all_sizes[r].item())] for r in range(world)]
    cat = np.concatenate(parts, axis=0)
    return {"final_score": cat[..., 0], "orientation": cat[..., 1].astype(np.int32),
            "seed_rank": cat[..., 2].astype(np.int32), "evaluations": cat[..., 3].astype(np.int64)}
