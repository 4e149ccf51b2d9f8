"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no Green's functions, kernels, sums or
solvers).  It only builds the *inputs* the paper's pipeline feeds to its kernels
(Table 1 steps 2-4): triangle centroids, unit outward
normals and areas (the paper gets them from MSMS; we triangulate analytic
spheres/ellipsoids instead) and point charges (x, y, z, Q).

Element precompute follows SPEC.md S:76-84 / SURVEY.md R6: centroid = mean of the three
vertices, area W = |e1 x e2| / 2, normal = (e1 x e2)/|e1 x e2| oriented outward.

Configs C1..C5 are BASELINE.json `configs` (recipes in SURVEY.md §8(d) and DESIGN.md
"Input recipe").  Random numbers come from numpy PCG64 `default_rng(seed)`.
"""
from __future__ import annotations

import hashlib
from dataclasses import dataclass, field

import numpy as np

# Physics shared by every BASELINE config (reading R10).
EPS1 = 1.0
EPS2 = 80.0
KAPPA = 0.1257


def _icosahedron():
    t = (1.0 + 5.0 ** 0.5) / 2.0
    v = np.array(
        [[-1, t, 0], [1, t, 0], [-1, -t, 0], [1, -t, 0],
         [0, -1, t], [0, 1, t], [0, -1, -t], [0, 1, -t],
         [t, 0, -1], [t, 0, 1], [-t, 0, -1], [-t, 0, 1]], dtype=np.float64)
    f = np.array(
        [[0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
         [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
         [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
         [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return v, f


def unit_icosphere(level: int):
    """Unit icosphere: icosahedron subdivided `level` times (each triangle -> 4 via edge
    midpoints), vertices projected to the unit sphere.
    Returns (vertices [V,3] float64, faces [F,3] int64) with F = 20*4^level,
    V = 10*4^level + 2, counter-clockwise (outward) winding."""
    if level < 0:
        raise ValueError("level must be >= 0")
    v, f = _icosahedron()
    for _ in range(level):
        nv = v.shape[0]
        e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]], axis=0)
        e.sort(axis=1)
        key = e[:, 0] * (nv + 1) + e[:, 1]
        uniq, inv = np.unique(key, return_inverse=True)
        a, b = uniq // (nv + 1), uniq % (nv + 1)
        mid = v[a] + v[b]
        mid /= np.linalg.norm(mid, axis=1, keepdims=True)
        v = np.concatenate([v, mid], axis=0)
        nf = f.shape[0]
        m01 = nv + inv[:nf]
        m12 = nv + inv[nf:2 * nf]
        m20 = nv + inv[2 * nf:]
        f = np.concatenate([
            np.stack([f[:, 0], m01, m20], 1),
            np.stack([f[:, 1], m12, m01], 1),
            np.stack([f[:, 2], m20, m12], 1),
            np.stack([m01, m12, m20], 1)], axis=0)
    return v, f


def elements(vertices: np.ndarray, faces: np.ndarray, center=(0.0, 0.0, 0.0)):
    """Per-element centroid, unit normal and area.
    Normals are oriented away from `center` (valid for star-shaped closed surfaces)."""
    p0, p1, p2 = vertices[faces[:, 0]], vertices[faces[:, 1]], vertices[faces[:, 2]]
    cen = (p0 + p1 + p2) / 3.0
    cr = np.cross(p1 - p0, p2 - p0)
    nrm2 = np.linalg.norm(cr, axis=1)
    area = 0.5 * nrm2
    nrm = cr / nrm2[:, None]
    flip = np.einsum("ij,ij->i", nrm, cen - np.asarray(center)[None, :]) < 0
    nrm[flip] *= -1.0
    return np.ascontiguousarray(cen), np.ascontiguousarray(nrm), np.ascontiguousarray(area)


def icosphere(level: int, radius: float, center=(0.0, 0.0, 0.0)):
    v, f = unit_icosphere(level)
    v = v * radius + np.asarray(center, dtype=np.float64)[None, :]
    return v, f


def ellipsoid(level: int, axes):
    v, f = unit_icosphere(level)
    return v * np.asarray(axes, dtype=np.float64)[None, :], f


def charges_in_ball(n: int, rmax: float, seed: int, axes=None):
    """n charges uniform in the ball |y| <= rmax (or in the ellipsoid with semi-axes
    `axes`), Q ~ U(-1, 1).  Returns [n,4] float64 rows (x, y, z, Q)."""
    rng = np.random.default_rng(seed)
    d = rng.normal(size=(n, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    r = rng.random(n) ** (1.0 / 3.0)
    pos = d * r[:, None]
    if axes is None:
        pos *= rmax
    else:
        pos *= np.asarray(axes, dtype=np.float64)[None, :]
    q = rng.uniform(-1.0, 1.0, n)
    return np.ascontiguousarray(np.concatenate([pos, q[:, None]], axis=1))


def helix_charges():
    """PAPER.md §3.2 (Table 2 caption P:432): nine charges 0.1..0.9 e_c on
    r(t) = <3/(4pi) cos t, 3/(4pi) sin t, t/pi>, read as t = 0, pi/4, ..., 2pi
    (the printed step pi/2 yields five points, not nine)."""
    t = np.arange(9) * (np.pi / 4.0)
    pos = np.stack([3.0 / (4 * np.pi) * np.cos(t), 3.0 / (4 * np.pi) * np.sin(t), t / np.pi], 1)
    q = 0.1 * np.arange(1, 10)
    return np.ascontiguousarray(np.concatenate([pos, q[:, None]], axis=1))


@dataclass
class Problem:
    name: str
    centroids: np.ndarray  # [N,3]
    normals: np.ndarray    # [N,3]
    areas: np.ndarray      # [N]
    charges: np.ndarray    # [Nc,4] x,y,z,Q
    eps1: float = EPS1
    eps2: float = EPS2
    kappa: float = KAPPA
    meta: dict = field(default_factory=dict)

    @property
    def n(self) -> int:
        return int(self.centroids.shape[0])

    @property
    def nc(self) -> int:
        return int(self.charges.shape[0])

    def sha256(self) -> str:
        h = hashlib.sha256()
        for a in (self.centroids, self.normals, self.areas, self.charges):
            h.update(np.ascontiguousarray(a, dtype="<f8").tobytes())
        h.update(np.array([self.eps1, self.eps2, self.kappa], dtype="<f8").tobytes())
        return h.hexdigest()


def sphere_problem(level, radius, charges, name="sphere", center=(0.0, 0.0, 0.0),
                   eps1=EPS1, eps2=EPS2, kappa=KAPPA):
    v, f = icosphere(level, radius, center)
    c, nrm, a = elements(v, f, center)
    return Problem(name, c, nrm, a, np.ascontiguousarray(charges, dtype=np.float64),
                   eps1, eps2, kappa, {"level": level, "radius": radius})


def config(name: str) -> Problem:
    """BASELINE.json configs."""
    if name == "C1":  # Born ion: icosphere L4, R=2, Q=+1 at the centre
        return sphere_problem(4, 2.0, np.array([[0.0, 0.0, 0.0, 1.0]]), "C1_born_L4")
    if name == "C2":  # Kirkwood sphere L5, R=4, 50 charges in r<=3, seed 2
        return sphere_problem(5, 4.0, charges_in_ball(50, 3.0, 2), "C2_kirkwood_L5")
    if name == "C3":  # ellipsoid from L6 scaled (24,18,14), 2000 charges in (21,15,11), seed 3
        v, f = ellipsoid(6, (24.0, 18.0, 14.0))
        c, nrm, a = elements(v, f)
        q = charges_in_ball(2000, 1.0, 3, axes=(21.0, 15.0, 11.0))
        return Problem("C3_ellipsoid_L6", c, nrm, a, q, meta={"level": 6, "axes": (24, 18, 14)})
    if name == "C4":  # icosphere L7, R=20, 5000 charges in r<=18, seed 4
        return sphere_problem(7, 20.0, charges_in_ball(5000, 18.0, 4), "C4_icosphere_L7")
    if name == "C5":  # icosphere L8, R=20, 10000 charges in r<=18, seed 5
        return sphere_problem(8, 20.0, charges_in_ball(10000, 18.0, 5), "C5_icosphere_L8")
    raise KeyError(name)


def random_vector(n2: int, seed: int, smooth_centroids=None):
    """Seeded operand u for matvec parity: U(-1,1) entries, or a smooth field
    f = cos(0.3x) + sin(0.2y) + 0.1z evaluated at the centroids when given (u = [f, f/2])."""
    if smooth_centroids is not None:
        c = smooth_centroids
        f = np.cos(c[:, 0] * 0.3) + np.sin(0.2 * c[:, 1]) + 0.1 * c[:, 2]
        return np.ascontiguousarray(np.concatenate([f, 0.5 * f]))
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n2)


# ---------------------------------------------------------------- molecular input formats
# SURVEY.md §8(f) item 4 / SPEC.md S:49-84: the paper reads PDB/CHARMM22 charges and MSMS
# triangulations.  These parsers ingest the text formats so real
# molecular surfaces can be fed to bipb_setup; no molecular data ships with the repo.

def parse_pqr(text: str) -> np.ndarray:
    """PQR: records starting ATOM/HETATM; the last five whitespace-separated numeric fields
    are x y z charge radius.  Returns [nc, 4] (x, y, z, Q) float64."""
    rows = []
    for ln, line in enumerate(text.splitlines(), 1):
        if not (line.startswith("ATOM") or line.startswith("HETATM")):
            continue
        tok = line.split()
        try:
            x, y, z, q, r = (float(t) for t in tok[-5:])
        except ValueError as e:
            raise ValueError(f"PQR line {ln}: malformed numeric field") from e
        rows.append((x, y, z, q))
    if not rows:
        raise ValueError("PQR: no ATOM/HETATM records")
    return np.ascontiguousarray(np.array(rows, dtype=np.float64))


def _data_lines(text: str):
    lines = [l for l in text.splitlines() if l.strip()]
    i = 0
    while i < len(lines) and lines[i].lstrip().startswith("#"):
        i += 1
    return lines[i:]


def parse_msms(vert_text: str, face_text: str):
    """MSMS .vert/.face: after '#' comment lines and one counts line, vert
    records begin 'x y z nx ny nz', face records begin 'i j k' (1-based).  Returns
    (vertices [V,3], vertex_normals [V,3], faces [F,3] 0-based)."""
    vl = _data_lines(vert_text)
    fl = _data_lines(face_text)
    nv = int(vl[0].split()[0])
    nf = int(fl[0].split()[0])
    V, VN = np.empty((nv, 3)), np.empty((nv, 3))
    for k, l in enumerate(vl[1:1 + nv]):
        t = l.split()
        if len(t) < 6:
            raise ValueError(f"MSMS vert record {k + 1}: fewer than 6 fields")
        V[k] = [float(a) for a in t[:3]]
        VN[k] = [float(a) for a in t[3:6]]
    Fc = np.empty((nf, 3), dtype=np.int64)
    for k, l in enumerate(fl[1:1 + nf]):
        Fc[k] = [int(a) for a in l.split()[:3]]
    if Fc.min() < 1 or Fc.max() > nv:
        raise ValueError("MSMS face index out of range (indices are 1-based)")
    return V, VN, Fc - 1


def write_msms(vertices, vertex_normals, faces):
    """Inverse of parse_msms (1-based faces), for fixtures and round trips."""
    vt = ["# MSMS solvent excluded surface vertices", f"{len(vertices)} 0 0 0"]
    vt += [" ".join(f"{a:.17g}" for a in (*v, *n)) + " 0 0 1" for v, n in zip(vertices, vertex_normals)]
    ft = ["# MSMS solvent excluded surface faces", f"{len(faces)} 0 0 0"]
    ft += [f"{a + 1} {b + 1} {c + 1} 1 1" for a, b, c in faces]
    return "\n".join(vt) + "\n", "\n".join(ft) + "\n"


def elements_from_msms(vertices, vertex_normals, faces, min_area=1e-12):
    """Element precompute for an ingested mesh: centroid, unit normal from the
    winding, flipped if it disagrees with the mean vertex normal; faces with area < min_area
    are dropped.  Returns (centroids, normals, areas, n_dropped)."""
    p0, p1, p2 = vertices[faces[:, 0]], vertices[faces[:, 1]], vertices[faces[:, 2]]
    cr = np.cross(p1 - p0, p2 - p0)
    nrm2 = np.linalg.norm(cr, axis=1)
    area = 0.5 * nrm2
    keep = area >= min_area
    cen = (p0 + p1 + p2)[keep] / 3.0
    nrm = cr[keep] / nrm2[keep, None]
    vn = (vertex_normals[faces[:, 0]] + vertex_normals[faces[:, 1]] + vertex_normals[faces[:, 2]])[keep]
    flip = np.einsum("ij,ij->i", nrm, vn) < 0
    nrm[flip] *= -1.0
    return (np.ascontiguousarray(cen), np.ascontiguousarray(nrm), np.ascontiguousarray(area[keep]),
            int((~keep).sum()))
