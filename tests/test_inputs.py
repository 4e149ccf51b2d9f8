"""Input generator (bipb_inputs): Euler formula, icosphere counts, areas,
orientation, seeded reproducibility."""
import numpy as np
import pytest

import bipb_inputs as g


@pytest.mark.parametrize("L", range(0, 6))
def test_icosphere_topology(L):
    v, f = g.unit_icosphere(L)
    assert f.shape[0] == 20 * 4 ** L
    assert v.shape[0] == 10 * 4 ** L + 2
    e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]])
    e.sort(axis=1)
    ne = np.unique(e, axis=0).shape[0]
    assert ne == 30 * 4 ** L
    assert v.shape[0] + f.shape[0] - ne == 2  # Euler N_v + N - N_e = 2
    np.testing.assert_allclose(np.linalg.norm(v, axis=1), 1.0, rtol=0, atol=1e-15)


def test_elements_geometry():
    prev = 0.0
    for L in range(1, 7):
        p = g.sphere_problem(L, 4.0, np.zeros((0, 4)))
        tot = p.areas.sum()
        assert prev < tot < 4 * np.pi * 16  # inscribed polyhedron, monotone in level
        prev = tot
        np.testing.assert_allclose(np.linalg.norm(p.normals, axis=1), 1.0, atol=1e-14)
        assert np.all(np.einsum("ij,ij->i", p.normals, p.centroids) > 0)  # outward
        assert np.all(p.areas > 0)
    assert tot == pytest.approx(4 * np.pi * 16, rel=2e-4)
    # unit right triangle, CCW in z=0: area 0.5, normal +z
    c, n, a = g.elements(np.array([[0.0, 0, 0], [1, 0, 0], [0, 1, 0]]), np.array([[0, 1, 2]]),
                         center=(0.2, 0.2, -1.0))
    assert a[0] == 0.5 and np.allclose(n[0], [0, 0, 1]) and np.allclose(c[0], [1 / 3, 1 / 3, 0])


def test_configs_shapes_and_seeds():
    p1 = g.config("C1")
    assert p1.n == 5120 and p1.nc == 1 and p1.areas.sum() == pytest.approx(50.205, abs=1e-3)
    p2 = g.config("C2")
    assert p2.n == 20480 and p2.nc == 50
    assert np.all(np.linalg.norm(p2.charges[:, :3], axis=1) <= 3.0)
    assert np.all(np.abs(p2.charges[:, 3]) <= 1.0)
    assert g.config("C2").sha256() == p2.sha256()  # seeded, reproducible
    p3 = g.config("C3")
    assert p3.n == 81920 and p3.nc == 2000
    assert p3.areas.sum() == pytest.approx(4332.1, abs=0.1)
    q = p3.charges[:, :3] / np.array([21.0, 15.0, 11.0])
    assert np.all(np.linalg.norm(q, axis=1) <= 1.0)


def test_helix_charges():
    h = g.helix_charges()
    assert h.shape == (9, 4)
    np.testing.assert_allclose(h[:, 3], np.arange(1, 10) * 0.1)
    assert np.all(np.linalg.norm(h[:, :3], axis=1) < 4.0)
