"""GPU rotation profiles (gd_rotation_profiles) against the reference.

Bar: bit-exact.  Every profile entry is a reference overlap_score / check_bumps
decision, so scores, validity, relative sizes, fragment numbering and
per-ligand status must equal the reference's rotation_profile
(analysis.hpp:37-56) run through oracle/_ref, or the C oracle where the
reference is not built.
"""
import numpy as np
import pytest

from paper_1901_06363_b200 import Knobs, LigandBatch, workloads as W
from paper_1901_06363_b200.analysis import analyze_ligands, detect_peaks

pytestmark = pytest.mark.gpu


def _oracle():
    from oracle import oracle_py
    return oracle_py


def _want(batch, pocket):
    O = _oracle()
    if O.have_ref():
        return O.rotation_profiles(batch, pocket, "ref", nthreads=O.threads())
    return O.rotation_profiles(batch, pocket, "oracle")


def _check(docker, batch, pocket):
    docker.set_pocket(pocket)
    got = docker.rotation_profiles(batch)
    want = _want(batch, pocket)
    names = ["scores", "valid", "relative_size", "frag_offsets", "status"]
    for name, x, y in zip(names, (got.scores, got.valid, got.relative_size, got.frag_offsets,
                                  got.status), want):
        assert np.array_equal(x, y), name
    return got


def test_profiles_reference_datasets(docker):
    O = _oracle()
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    for count, seed in ((6, 1234), (8, 4096), (4, 88)):
        pocket, batch = O.ref_generate_synthetic(count, seed)
        got = _check(docker, batch, pocket)
        assert got.valid.any() and not got.valid.all()


def test_profiles_config1_ligands(docker):
    w = W.config(1)
    pocket = w.pocket()
    got = _check(docker, w.ligands(range(20), pocket.mean(axis=0)), pocket)
    assert len(got.scores) > 20


def test_profiles_multiword_ligands_and_rough_pocket(docker):
    O = _oracle()
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    pocket, batch = O.ref_generate_synthetic(3, 2718, 65, 153, 8, 30, 400, 10.0)
    assert batch.sizes.max() > 64
    _check(docker, batch, pocket)
    w = W.config(3)
    rough = W.pocket_of(w, 5)
    _check(docker, w.ligands(range(6), rough.mean(axis=0)), rough)


def test_profiles_edge_ligands(docker):
    """A rigid ligand (no fragments), an invalid one (skipped, status 1) and a
    two-atom-fragment ligand that cannot bump (test_analysis.cpp:26-37)."""
    from gd_test_helpers import Lig
    parts = [
        Lig([[0, 0, 0], [0, 0, 1.5]], [(0, 1, False)]),
        Lig([[0, 0, 0], [1.5, 0, 0], [9, 9, 9]], [(0, 1, True)]),  # disconnected
        Lig([[0, 0, 0], [0, 0, 1.4], [1.2, 0, 1.4]], [(0, 1, True), (1, 2, False)]),
    ]
    batch = LigandBatch.from_parts([p.args for p in parts])
    got = _check(docker, batch, np.array([[0.0, 0.0, 1.0]]))
    assert got.frag_offsets.tolist() == [0, 0, 0, 2]
    assert got.status.tolist() == [0, 1, 0]
    assert got.valid.all()


def test_analyze_ligands_matches_reference_composition(docker):
    """analyze_ligand (analysis.hpp:177-215): dock from the given pose, then
    profile every fragment from the final pose; compared row by row with the
    reference's match_probes_shape + rotation_profile + detect_peaks."""
    O = _oracle()
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    pocket, batch = O.ref_generate_synthetic(5, 31337)
    knobs = Knobs(3, 90, 0.0, 1, False)
    docker.set_pocket(pocket)
    got = analyze_ligands(docker, batch, knobs)
    dock = O.dock_batch(batch, pocket, knobs, nthreads=O.threads(), impl="ref")
    final = LigandBatch(batch.atom_offsets, dock.final_pose.reshape(-1, 3), batch.radii,
                        batch.bond_offsets, batch.bonds, batch.rotatable)
    scores, valid, rel, offs, status = O.rotation_profiles(final, pocket, "ref")
    for l, la in enumerate(got):
        assert la is not None and la.score == dock.final_score[l, 0] > 0.0
        assert np.array_equal(la.final_pose, final.xyz[batch.atom_offsets[l]:batch.atom_offsets[l + 1]])
        rows = []
        for f in range(offs[l], offs[l + 1]):
            want = O.ref_detect_peaks(scores[f], valid[f])
            if want is not None:
                rows.append((f - offs[l], rel[f], want))
        assert len(rows) == len(la.fragments) == len(la.stats)
        for (fl, r, (delta, bw, peaks)), row, st in zip(rows, la.fragments, la.stats):
            assert (row.rotamer_index, row.side) == (fl // 2, "left" if fl % 2 == 0 else "right")
            assert row.relative_size == r and 0.0 < r < 1.0
            assert (row.delta_overlap, row.best_peak_width, row.peak_count) == (delta, bw, len(peaks))
            assert row.delta_normalized == delta / la.score
            assert [(p.start_angle, p.width, p.height_ratio) for p in st.peaks] == peaks
