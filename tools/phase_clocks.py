"""Attribute the flex kernel's warp time to its phases (config 1).

Run on the GPU box from the repo root; rebuilds the library with
-DGD_PHASE_CLOCKS=1 (the clocks cost registers, so the numbers are shares,
not timings) and restores the normal build afterwards.

    python tools/phase_clocks.py [--config 1] [--ligands 10000]
"""
import argparse
import os
import subprocess
import sys

sys.path.insert(0, os.getcwd())
PHASES = ["chain start", "step setup", "bump prefilter", "term pre-fill", "bump checks",
          "queries", "folds", "decisions", "commit"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=1)
    ap.add_argument("--ligands", type=int, default=10000)
    a = ap.parse_args()
    env = dict(os.environ, GD_DEFS="-DGD_PHASE_CLOCKS=1")
    subprocess.run([sys.executable, "paper_1901_06363_b200/build.py", "--force"], env=env, check=True,
                   stdout=subprocess.DEVNULL)
    try:
        from paper_1901_06363_b200 import Docker, Knobs, workloads as W
        from paper_1901_06363_b200.native import GD_FLAG_COUNT_WORK
        w = W.config(a.config)
        pocket = w.pocket()
        batch = w.ligands(range(a.ligands), pocket.mean(axis=0))
        d = Docker(0)
        d.set_pocket(pocket)
        d.upload(batch)
        d.dock_resident(Knobs(**{**w.knobs.__dict__, "flags": GD_FLAG_COUNT_WORK}))
        ck = d.phase_clocks()[: len(PHASES)]
        tot = sum(ck) or 1
        for name, c in zip(PHASES, ck):
            print(f"{name:16s} {c / tot * 100:5.1f}%  {c:.3e} cycles")
    finally:
        subprocess.run([sys.executable, "paper_1901_06363_b200/build.py", "--force"], check=True,
                       stdout=subprocess.DEVNULL)


if __name__ == "__main__":
    main()
