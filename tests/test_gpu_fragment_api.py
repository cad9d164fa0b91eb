"""GPU parity of the fine-grained drop-in entry points against the
reference itself (oracle/_ref):

* gd_optimize_fragment_batch  <- optimize_fragment_flat / _refined
  (kernel.hpp:125-198): FragmentSearchResult, SearchCounters and the
  committed pose, with and without the refined search's entry score;
* gd_rotate_fragment_batch    <- rotate_fragment (geometry.hpp:161-193),
  integer and non-integer angles, angle 0, and the degenerate axis;
* gd_check_bumps_batch        <- check_bumps (geometry.hpp:199-213).

Every (ligand, fragment) item is one ligand of one batched call; the
fragment comes from the reference's own find_rotamers + grow_fragments.
Bar: bit-exact.
"""
import numpy as np
import pytest

from paper_1901_06363_b200 import LigandBatch, workloads as W
from gd_test_helpers import bump_probe, chain, peak_rig

pytestmark = pytest.mark.gpu


def _O():
    from oracle import oracle_py as O
    if not O.have_ref():
        pytest.skip("oracle/_ref (the compiled reference) is not built")
    return O


def _items(ligs):
    """(ligand parts, f, membership, axis, anchor) for every fragment of `ligs`."""
    O = _O()
    out = []
    for (x, r, b, ro) in ligs:
        g = O.ref_ligand_graph(x, r, b, ro)
        assert g is not None
        rb, mem = g
        for f in range(len(mem)):
            a, c = sorted(b[rb[f // 2]])
            axis, anchor = (a, c) if f % 2 == 0 else (c, a)
            out.append(((x, r, b, ro), f, mem[f], axis, anchor))
    return out


def _batch(items, poses=None):
    parts = []
    for k, (p, *_rest) in enumerate(items):
        x, r, b, ro = p
        parts.append((x if poses is None else poses[k], r, b, ro))
    batch = LigandBatch.from_parts(parts)
    mem = np.concatenate([it[2] for it in items]).astype(np.uint8)
    ax = np.array([it[3] for it in items], np.int32)
    an = np.array([it[4] for it in items], np.int32)
    return batch, mem, ax, an


def _c1_ligands(k):
    w = W.config(1)
    b = w.ligands(range(k))
    return [b.ligand(l) for l in range(k)], w.pocket()


@pytest.mark.parametrize("step,refined", [(30, False), (10, False), (90, False), (360, False),
                                          (1, True), (5, True), (30, True)])
def test_optimize_fragment_matches_reference(docker, step, refined):
    O = _O()
    ligs, pocket = _c1_ligands(12)
    rig, rig_pocket = peak_rig()
    items = _items(ligs)[:60]
    docker.set_pocket(pocket)
    batch, mem, ax, an = _batch(items)
    got = docker.optimize_fragment(batch, mem, ax, an, step, refined)
    assert (got["status"] == 0).all()
    for k, (p, f, *_r) in enumerate(items):
        x, r, b, ro = p
        a, s, ev, ck, pose = O.ref_optimize_fragment(x, r, b, ro, pocket, f, step, refined)
        assert got["best_angle"][k] == a, k
        assert got["best_score"][k] == s, k
        assert got["evaluations"][k] == ev and got["feasibility_checks"][k] == ck, k
        a0, a1 = batch.atom_offsets[k], batch.atom_offsets[k + 1]
        assert np.array_equal(got["pose"][a0:a1], pose.reshape(-1, 3)), k
    # The PeakRig known answer (test_kernel.cpp:75-97): the peak at 90 degrees.
    docker.set_pocket(rig_pocket)
    items = _items([rig.args])[:1]
    batch, mem, ax, an = _batch(items)
    got = docker.optimize_fragment(batch, mem, ax, an, step, refined)
    a, s, ev, ck, pose = O.ref_optimize_fragment(*rig.args, rig_pocket, 0, step, refined)
    assert (got["best_angle"][0], got["best_score"][0]) == (a, s)
    assert (got["evaluations"][0], got["feasibility_checks"][0]) == (ev, ck)


def test_refined_entry_score_is_honoured(docker):
    """optimize_fragment_refined's optional entry score decides the final
    entry comparison (kernel.hpp:192-194) but not angle-0 candidates."""
    O = _O()
    ligs, pocket = _c1_ligands(6)
    items = _items(ligs)[:20]
    docker.set_pocket(pocket)
    batch, mem, ax, an = _batch(items)
    for scale in (0.5, 1e6):
        base = docker.optimize_fragment(batch, mem, ax, an, 2, True)
        entry = np.array([O.overlap_score(batch.ligand(k)[0], pocket) for k in range(len(items))])
        entry = entry * scale
        got = docker.optimize_fragment(batch, mem, ax, an, 2, True, entry_score=entry)
        for k, (p, f, *_r) in enumerate(items):
            x, r, b, ro = p
            a, s, ev, ck, pose = O.ref_optimize_fragment(x, r, b, ro, pocket, f, 2, True,
                                                         entry_score=entry[k])
            assert (got["best_angle"][k], got["best_score"][k]) == (a, s), (scale, k)
            assert (got["evaluations"][k], got["feasibility_checks"][k]) == (ev, ck)
        if scale > 1:
            assert (got["best_angle"] == 0).all()
        assert base["best_score"].shape == got["best_score"].shape


@pytest.mark.parametrize("angle", [0.0, 1.0, 30.0, 37.25, -12.5, 90.0, 179.999, 725.0])
def test_rotate_fragment_and_check_bumps_match_reference(docker, angle):
    O = _O()
    ligs, _ = _c1_ligands(16)
    probe = [bump_probe(sep, 1.0).args for sep in (0.5, 1.4, 2.0, 3.5)]
    items = _items(ligs + probe)
    batch, mem, ax, an = _batch(items)
    pose, status = docker.rotate_fragment(batch, mem, ax, an, np.full(len(items), angle))
    assert (status == 0).all()
    rot_batch, *_ = _batch(items, poses=[pose[batch.atom_offsets[k]:batch.atom_offsets[k + 1]]
                                         for k in range(len(items))])
    feas, status = docker.check_bumps(rot_batch, mem, ax, an)
    assert (status == 0).all()
    n_bump = 0
    for k, (p, f, *_r) in enumerate(items):
        x, r, b, ro = p
        want, ok = O.rotate_fragment(x, r, b, ro, x, f, angle, impl="ref")
        a0, a1 = batch.atom_offsets[k], batch.atom_offsets[k + 1]
        assert np.array_equal(pose[a0:a1], want.reshape(-1, 3)), (angle, k)
        assert feas[k] == ok, (angle, k)
        n_bump += not ok
    if angle == 0.0:
        assert np.array_equal(pose, batch.xyz)  # exact identity


def test_degenerate_axis_is_reported(docker):
    """Two bonded atoms at the same position: "rotate_fragment: degenerate
    rotation axis" (geometry.hpp:168), for a rotation even at angle 0 (the
    reference checks the axis first) and for a fragment search."""
    lig = chain([[0, 0, 0], [0, 0, 0], [1.5, 0, 0], [3.0, 0, 0]])
    items = _items([lig.args])
    batch, mem, ax, an = _batch(items[:1])
    _, status = docker.rotate_fragment(batch, mem, ax, an, [0.0])
    assert status[0] == 3
    docker.set_pocket(np.zeros((1, 3)))
    got = docker.optimize_fragment(batch, mem, ax, an, 30)
    assert got["status"][0] == 3
    feas, status = docker.check_bumps(batch, mem, ax, an)  # no axis needed
    assert status[0] == 0 and feas[0]


def test_fragment_api_errors(docker):
    from paper_1901_06363_b200 import GeoDockError
    lig = chain([[0, 0, 0], [1.5, 0, 0], [3.0, 0, 0]])
    items = _items([lig.args])
    batch, mem, ax, an = _batch(items[:1])
    docker.set_pocket(np.zeros((1, 3)))
    with pytest.raises(GeoDockError, match="optimize_fragment_flat: step must divide 360"):
        docker.optimize_fragment(batch, mem, ax, an, 7)
    with pytest.raises(GeoDockError, match="optimize_fragment_refined: step must divide 360"):
        docker.optimize_fragment(batch, mem, ax, an, 0, refined=True)
    with pytest.raises(GeoDockError, match="out of range"):
        docker.rotate_fragment(batch, mem, [5], an, [10.0])
