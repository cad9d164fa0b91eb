"""Device-resident kernel times for quick A/B on the box (not the bench line).

    python tools/quick_bench.py [--configs 1 2] [--reps 5] [--count]
Prints, per config: median rigid / flex / total ms over reps (L2 flushed
before each), ligands/s, and with --count the flex/rigid work counters.
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import torch  # noqa: E402

from paper_1901_06363_b200 import Docker, workloads as W  # noqa: E402
from paper_1901_06363_b200.native import GD_FLAG_COUNT_WORK  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", type=int, nargs="+", default=[1, 2])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--count", action="store_true")
    ap.add_argument("--exact", action="store_true", help="GD_FLAG_EXACT_FP64: no fp32 screens")
    a = ap.parse_args()
    d = Docker(0)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for c in a.configs:
        w = W.config(c)
        pocket = w.pocket()
        batch = w.ligands()
        d.set_pocket(pocket)
        d.upload(batch)
        from paper_1901_06363_b200 import Knobs
        from paper_1901_06363_b200 import native as _nat
        GD_FLAG_EXACT_FP64 = getattr(_nat, "GD_FLAG_EXACT_FP64", 0)
        knobs = Knobs(**{**w.knobs.__dict__, "flags": GD_FLAG_EXACT_FP64 if a.exact else 0})
        rows = []
        for r in range(a.reps + 2):
            flush.random_()
            torch.cuda.synchronize()
            d.dock_resident(knobs)
            t = d.timing()
            if r >= 2:
                rows.append((t["rigid_ms"], t["flex_ms"], t["total_ms"]))
        med = [statistics.median(x[i] for x in rows) for i in range(3)]
        out = {"config": c, "rigid_ms": med[0], "flex_ms": med[1], "total_ms": med[2],
               "ligands_per_s": batch.n_ligands / (med[2] * 1e-3)}
        try:
            info = d.pocket_info()
            out["index_mb"] = info["index_bytes"] / 1e6
            out["levels"] = [(x["voxel"], round(x["record_bytes"] / 1e6, 1), round(x["list_bytes"] / 1e6, 1))
                             for x in info["levels"]]
        except Exception:  # older trees (A/B) lack gd_pocket_index_stats
            pass
        if a.count:
            k = Knobs(**{**knobs.__dict__, "flags": knobs.flags | GD_FLAG_COUNT_WORK})
            d.dock_resident(k)
            out["work"] = d.work_counters()
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
