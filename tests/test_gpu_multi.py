"""The in-process multi-device dispatcher (gd_multi_*) and the pocket cache.

This box has one GPU, so the multi-device path runs with two and three
contexts on device 0: every context has its own host thread, streams and
staged pocket, exactly as on an 8-GPU node, and the chunk cursor hands out
the same cost-weighted chunks.  The result must equal the single-context
gd_dock_batch bit for bit (docks are independent, so the device count
cannot change a result), with every chunk's results at its global offsets.
"""
import numpy as np
import pytest

from paper_1901_06363_b200 import Knobs, MultiDocker, workloads as W
from gd_test_helpers import assert_same_result

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("devices", [[0, 0], [0, 0, 0]])
def test_multi_context_equals_single_context(docker, devices):
    w = W.config(1)
    pocket = w.pocket()
    batch = w.ligands(range(3000))
    docker.set_pocket(pocket)
    want = docker.dock(batch, w.knobs, keep_poses=True)
    m = MultiDocker(devices)
    try:
        assert m.size == len(devices)
        m.set_pocket(pocket)
        got = m.dock(batch, w.knobs, keep_poses=True)
        assert_same_result(got, want, ctx=f"{len(devices)} contexts: ")
        st = m.stats()
        assert sum(s["ligands"] for s in st) == batch.n_ligands
        assert all(s["chunks"] >= 1 for s in st), st
    finally:
        m.close()


def test_multi_context_c2_knobs_and_skipped_ligands(docker):
    """K = 100 through the rank-merge top-K, plus an invalid ligand (a
    self-bond) in the middle of a chunk: it is skipped at its global slot."""
    from paper_1901_06363_b200 import LigandBatch
    w = W.config(2)
    pocket = w.pocket()
    good = w.ligands(range(600))
    parts = [good.ligand(l) for l in range(600)]
    x, r, b, ro = parts[317]
    b = b.copy()
    b[0] = [0, 0]  # self-bond: Ligand validation fails
    parts[317] = (x, r, b, ro)
    batch = LigandBatch.from_parts(parts)
    docker.set_pocket(pocket)
    want = docker.dock(batch, w.knobs)
    assert want.status[317] == 1 and (np.delete(want.status, 317) == 0).all()
    assert "self-bond" in docker.ligand_error(317)
    m = MultiDocker([0, 0])
    try:
        m.set_pocket(pocket)
        got = m.dock(batch, w.knobs)
        assert_same_result(got, want, poses=False)
        assert m.ligand_error(317) == docker.ligand_error(317)
        assert m.ligand_error(316) == ""
        assert sum(st["ligands"] for st in m.stats()) == 600
    finally:
        m.close()


def test_pocket_cache_restages_without_rebuild(docker):
    """Alternating pockets re-stages cached indexes (no rebuild): same
    results and index statistics, and a re-stage is much faster than a
    build."""
    import time
    w = W.config(3)
    pa, pb = W.pocket_of(w, 0), W.pocket_of(w, 1)
    ba = w.ligands(range(64), pa.mean(axis=0))
    bb = w.ligands(range(64), pb.mean(axis=0))
    docker.set_pocket(pa)
    ra = docker.dock(ba, w.knobs)
    ia = docker.pocket_info()
    docker.set_pocket(pb)
    rb = docker.dock(bb, w.knobs)
    t0 = time.perf_counter()
    for _ in range(10):
        docker.set_pocket(pa)
        docker.set_pocket(pb)
    restage = (time.perf_counter() - t0) / 20
    docker.set_pocket(pa)
    assert docker.pocket_info()["n_candidates"] == ia["n_candidates"]
    assert_same_result(docker.dock(ba, w.knobs), ra, poses=False)
    docker.set_pocket(pb)
    assert_same_result(docker.dock(bb, w.knobs), rb, poses=False)
    # A moved pocket is a different pocket (compared by coordinates).
    docker.set_pocket(pa + 1e-9)
    assert docker.pocket_info()["centre"][0] != ia["centre"][0]
    assert restage < 2e-3, restage
