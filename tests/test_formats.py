"""PQR / MSMS ingestion on hand-made fixtures."""
import numpy as np
import pytest

import bipb_inputs as g

TET_VERT = """# MSMS solvent excluded surface vertices
#vertex #sphere density probe_r
4 4 1.0 1.5
 1.0  1.0  1.0   0.577  0.577  0.577 0 1 2
-1.0 -1.0  1.0  -0.577 -0.577  0.577 0 2 2
-1.0  1.0 -1.0  -0.577  0.577 -0.577 0 3 2
 1.0 -1.0 -1.0   0.577 -0.577 -0.577 0 4 2
"""
# windings deliberately mixed: orientation must come from the vertex normals
TET_FACE = """# MSMS solvent excluded surface faces
#faces #sphere density probe_r
4 4 1.0 1.5
1 2 3 1 1
1 4 2 1 1
1 3 4 1 1
2 3 4 1 1
"""


def test_pqr():
    txt = "REMARK x\nATOM 1 C RES 1 0.0 0.0 0.0 1.0 1.5\nHETATM 2 O HOH 2 1.0 2.0 3.0 -0.834 1.52\nEND\n"
    q = g.parse_pqr(txt)
    assert q.shape == (2, 4) and np.allclose(q[1], [1.0, 2.0, 3.0, -0.834])
    with pytest.raises(ValueError):
        g.parse_pqr("ATOM 1 C RES 1 0.0 0.0 abc 1.0 1.5\n")
    with pytest.raises(ValueError):
        g.parse_pqr("REMARK nothing\n")


def test_msms_tetrahedron_orientation_and_euler():
    V, VN, F = g.parse_msms(TET_VERT, TET_FACE)
    assert V.shape == (4, 3) and F.shape == (4, 3) and F.min() == 0
    e = np.unique(np.sort(np.concatenate([F[:, [0, 1]], F[:, [1, 2]], F[:, [2, 0]]]), axis=1), axis=0)
    assert len(V) + len(F) - len(e) == 2  # Euler
    c, n, a, dropped = g.elements_from_msms(V, VN, F)
    assert dropped == 0 and np.all(a > 0)
    assert np.all(np.einsum("ij,ij->i", n, c) > 0)  # outward despite mixed windings
    with pytest.raises(ValueError):
        g.parse_msms(TET_VERT, TET_FACE.replace("2 3 4 1 1", "2 3 5 1 1"))


def test_msms_round_trip_and_sliver_drop():
    v, f = g.icosphere(2, 4.0)
    vn = v / np.linalg.norm(v, axis=1)[:, None]
    V, VN, F = g.parse_msms(*g.write_msms(v, vn, f))
    assert np.array_equal(V, v) and np.array_equal(F, f)
    c, n, a, dropped = g.elements_from_msms(V, VN, F)
    c0, n0, a0 = g.elements(v, f)
    assert dropped == 0 and np.allclose(c, c0) and np.allclose(n, n0) and np.allclose(a, a0)
    # a zero-area sliver face is dropped
    F2 = np.concatenate([F, [[0, 0, 1]]])
    *_, dropped = g.elements_from_msms(V, VN, F2)
    assert dropped == 1
