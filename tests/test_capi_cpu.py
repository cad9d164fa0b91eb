"""The C-ABI library on the CPU: it loads, exports every symbol
include/geodock_b200.h declares, and its host-only helpers match the
reference (no compute calls need a GPU here)."""
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "geodock_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(gd_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1901_06363_b200 import native
    lib = native.lib()
    names = declared_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
        assert name in native.SIGNATURES, f"{name} missing from the ctypes binding"


def test_version_and_create_without_gpu():
    import torch
    from paper_1901_06363_b200 import native
    assert b"sm_100a" in native.lib().gd_version()
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(native.GeoDockError) as e:
        native.Docker(0)
    assert e.value.code == native.GD_ERR_CUDA


def test_optimal_tile_size_matches_reference():
    from oracle import oracle_py as O
    from paper_1901_06363_b200 import optimal_tile_size
    assert optimal_tile_size(1) == 18 and optimal_tile_size(4) == 36 and optimal_tile_size(360) == 360
    z = np.load(ROOT / "tests" / "golden" / "reference_kernel.npz")
    assert [optimal_tile_size(s) for s in range(1, 361)] == z["tile_sizes"].tolist()
    assert optimal_tile_size(0) == -1
    assert all(optimal_tile_size(s) == O.oracle().gdo_optimal_tile_size(s) for s in range(1, 361))


@pytest.mark.parametrize("knobs,msg", [
    ((1, 45, 0.0, 3, False), None),
    ((7, 45, 0.0, 3, False), "high-precision step must be a divisor of 360"),
    ((10, 5, 0.0, 3, False), "low-precision step must be >= high-precision step"),
    ((1, 45, 1.5, 3, False), "threshold must be in [0,1]"),
    ((1, 45, 0.0, 0, False), "repetitions must be >= 1"),
    ((0, 45, 0.0, 3, False), "high-precision step must be a divisor of 360"),
    ((1, 7, 0.0, 3, False), "low-precision step must be a divisor of 360"),
])
def test_validate_knobs_messages(knobs, msg):
    """KnobConfig::validate (kernel.hpp:28-38), same checks and messages."""
    from paper_1901_06363_b200 import GeoDockError, Knobs
    k = Knobs(*knobs)
    if msg is None:
        k.validate()
    else:
        with pytest.raises(GeoDockError, match=re.escape(msg)):
            k.validate()


def test_batch_knob_validation():
    from paper_1901_06363_b200 import GeoDockError, Knobs
    with pytest.raises(GeoDockError, match="rigid step"):
        Knobs(30, 45, 0.0, 1, False, 7, 30).validate()
    with pytest.raises(GeoDockError, match="top_k"):
        Knobs(30, 45, 0.0, 1, False, 30, 0).validate()
    Knobs.baseline(10, 10, 3, 100).validate()


def test_orientations_match_oracle():
    """E2 built by the product equals the oracle's independent build."""
    from oracle import oracle_py as O
    from paper_1901_06363_b200 import orientations
    for step in (45, 30, 20, 15, 10, 90, 120, 180, 360):
        a, Ra = orientations(step)
        b, Rb = O.orientations(step)
        assert np.array_equal(a, b) and np.array_equal(Ra, Rb), step


def test_synthetic_generator_rules():
    """BASELINE generator: 1.5 A bonds, 109.5+-5 deg angles, valence <= 4,
    radii U(1.2,1.9), R rotatable bonds, centroid on the centre, determinism."""
    from paper_1901_06363_b200 import synth_ligands, workloads as W
    w = W.config(1)
    centre = np.array([0.5, -0.25, 1.0])
    b = w.ligands(range(40), centre)
    again = w.ligands(range(40), centre)
    assert np.array_equal(b.xyz, again.xyz) and np.array_equal(b.bonds, again.bonds)
    assert ((b.sizes >= 20) & (b.sizes <= 60)).all()
    for l in range(b.n_ligands):
        x, r, bd, ro = b.ligand(l)
        n = len(x)
        assert len(bd) == n - 1
        assert ((r >= 1.2) & (r <= 1.9)).all()
        np.testing.assert_allclose(np.linalg.norm(x[bd[:, 0]] - x[bd[:, 1]], axis=1), 1.5, atol=1e-9)
        deg = np.bincount(bd.ravel(), minlength=n)
        assert deg.max() <= 4
        assert ro.sum() <= min(12, n // 4)
        assert all(deg[a] >= 2 and deg[c] >= 2 for (a, c), rr in zip(bd, ro) if rr)
        np.testing.assert_allclose(x.mean(axis=0), centre, atol=1e-9)
        nbrs = [[] for _ in range(n)]
        for a, c in bd:
            nbrs[a].append(c)
            nbrs[c].append(a)
        for a in range(n):
            for i in range(len(nbrs[a])):
                for j in range(i + 1, len(nbrs[a])):
                    u, v = x[nbrs[a][i]] - x[a], x[nbrs[a][j]] - x[a]
                    ang = np.degrees(np.arccos(np.dot(u, v) / (np.linalg.norm(u) * np.linalg.norm(v))))
                    if len(nbrs[a]) == 2:  # a chain atom: the sampled bond angle
                        assert 104.4 < ang < 114.6
    c0 = W.config(0).ligands()
    assert c0.sizes.tolist() == [32] and int(c0.rotatable.sum()) == 6


def test_pocket_counts():
    from paper_1901_06363_b200 import synth_pocket, workloads as W
    assert len(W.config(0).pocket()) == 1983
    assert len(W.config(1).pocket()) == 3991
    assert len(synth_pocket(8, 6, 5, 1.0)) == 983
    assert len(synth_pocket(10, 8, 6, 1.0)) == 1989
    rough = synth_pocket(10, 8, 6, 1.0, 0.2, 5)
    assert 0.8 * 1989 <= len(rough) <= 1989


def test_ligand_graph_matches_reference():
    """gd_ligand_graph (native find_rotamers + grow_fragments) against the
    reference's own functions, on the reference generator's ligands (with
    rings) and on invalid ligands."""
    from oracle import oracle_py as O
    from paper_1901_06363_b200.native import GeoDockError, ligand_graph
    if not O.have_ref():
        pytest.skip("oracle/_ref not built")
    pocket, batch = O.ref_generate_synthetic(40, 77, 6, 60, 0, 12)
    for l in range(batch.n_ligands):
        args = batch.ligand(l)
        want = O.ref_ligand_graph(*args)
        got = ligand_graph(*args)
        assert np.array_equal(got[0], want[0]) and np.array_equal(got[1], want[1])
    bad = (np.zeros((3, 3)), np.ones(3), np.array([[0, 0]]), np.array([1]))
    assert O.ref_ligand_graph(*bad) is None
    with pytest.raises(GeoDockError, match="self-bond"):
        ligand_graph(*bad)


def test_standalone_synth_library_matches_product():
    """bench.py's reference arm builds its inputs with oracle/libgd_synth.so
    (the same csrc/synth.cpp built alone); they equal the product's."""
    import subprocess
    import sys
    code = """
import sys, numpy as np
sys.path.insert(0, {root!r})
from oracle import oracle_py as O
from paper_1901_06363_b200 import native, workloads as W
w = W.config(1)
a = (w.pocket(), w.ligands(range(40)))
native.set_synth_library(O.HERE / "libgd_synth.so")
b = (w.pocket(), w.ligands(range(40)))
assert np.array_equal(a[0], b[0])
for f in ("atom_offsets", "xyz", "radii", "bond_offsets", "bonds", "rotatable"):
    assert np.array_equal(getattr(a[1], f), getattr(b[1], f)), f
print("ok")
""".format(root=str(ROOT))
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True)
    assert out.stdout.strip() == "ok", out.stderr
