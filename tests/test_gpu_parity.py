"""GPU parity: the CUDA path (through the C ABI, via the thin binding) against the CPU oracle
on the same seeded inputs.  Tolerances are north_star's (BASELINE.json): matvec rel-L2 <= 1e-11
(overall and per block), source <= 1e-12, energy <= 1e-8 relative at GMRES tol 1e-10,
iterations within +-1."""
import json
import os

import numpy as np
import pytest

import bipb_inputs as g
import oracle
from oracle.kirkwood import kirkwood_energy

pytestmark = pytest.mark.gpu

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def bp():
    import torch
    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_1301_5885_b200 as bp
    return bp


def _ctx(bp, p):
    return bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa)


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def _ragged(L, R, keep, seed, charges, kappa=g.KAPPA):
    """Icosphere with a random subset of elements kept (N not a multiple of any tile)."""
    p = g.sphere_problem(L, R, charges, kappa=kappa)
    idx = np.sort(np.random.default_rng(seed).choice(p.n, keep, replace=False))
    return g.Problem(f"ragged{keep}", np.ascontiguousarray(p.centroids[idx]), np.ascontiguousarray(p.normals[idx]),
                     np.ascontiguousarray(p.areas[idx]), p.charges, p.eps1, p.eps2, kappa)


CASES = [
    ("L2", lambda k: g.sphere_problem(2, 4.0, g.helix_charges(), kappa=k)),
    ("L3", lambda k: g.sphere_problem(3, 4.0, g.charges_in_ball(20, 3.0, 7), kappa=k)),
    ("C1", lambda k: g.sphere_problem(4, 2.0, np.array([[0.0, 0, 0, 1.0]]), kappa=k)),
    ("ragged4999", lambda k: _ragged(4, 4.0, 4999, 1, g.charges_in_ball(37, 3.0, 8), k)),
    ("ellipsoidL4", lambda k: g.Problem("ell", *g.elements(*g.ellipsoid(4, (24.0, 18.0, 14.0))),
                                       g.charges_in_ball(300, 1.0, 3, axes=(21.0, 15.0, 11.0)), kappa=k)),
]


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("kappa", [g.KAPPA, 0.0])
@pytest.mark.parametrize("name,make", CASES)
def test_matvec_parity(bp, name, make, kappa, kind):
    p = make(kappa)
    ctx = _ctx(bp, p)
    ctx.set_matvec_kernel(kind)
    for u in (g.random_vector(2 * p.n, 11), g.random_vector(2 * p.n, 0, smooth_centroids=p.centroids)):
        y = bp.bipb_matvec(ctx, u)
        ref = oracle.matvec(p, u)
        n = p.n
        assert _rel(y, ref) <= 1e-11
        assert _rel(y[:n], ref[:n]) <= 1e-11 and _rel(y[n:], ref[n:]) <= 1e-11
        # element-wise (relative to the row scale of each block)
        assert np.max(np.abs(y[:n] - ref[:n])) <= 1e-11 * np.max(np.abs(ref[:n]))
        assert np.max(np.abs(y[n:] - ref[n:])) <= 1e-11 * np.max(np.abs(ref[n:]))
    ctx.close()


@pytest.mark.parametrize("name,make", CASES)
def test_source_and_energy_parity(bp, name, make):
    p = make(g.KAPPA)
    ctx = _ctx(bp, p)
    b = bp.bipb_source(ctx)
    bo = oracle.source(p)
    assert _rel(b[:p.n], bo[:p.n]) <= 1e-12 and _rel(b[p.n:], bo[p.n:]) <= 1e-12
    x = g.random_vector(2 * p.n, 5)
    phi = np.zeros(p.nc)
    e = bp.bipb_energy(ctx, x, phi)
    phio = oracle.reaction_potential(p, x)
    assert _rel(phi, phio) <= 1e-12
    assert e == pytest.approx(oracle.energy(p, x), rel=1e-11)
    ctx.close()


@pytest.mark.parametrize("nc", [1, 511, 512, 513, 20000])
def test_energy_launch_shapes(bp, nc):
    """The energy launch's chunk rule (whole waves of resident CTAs, 4 charges per thread, r02) over
    charge counts that give one partial / one full / one-plus-one charge tile and many tiles (N_c =
    20,000 > N): per-charge phi_reac and E_sol against the oracle, and the source b."""
    p = g.sphere_problem(4, 4.0, g.charges_in_ball(nc, 3.0, 40 + nc))
    ctx = _ctx(bp, p)
    b = bp.bipb_source(ctx)
    bo = oracle.source(p)
    assert _rel(b[:p.n], bo[:p.n]) <= 1e-12 and _rel(b[p.n:], bo[p.n:]) <= 1e-12
    x = g.random_vector(2 * p.n, 6)
    phi = np.zeros(p.nc)
    e = bp.bipb_energy(ctx, x, phi)
    ctx.close()
    phio = oracle.reaction_potential(p, x)
    assert _rel(phi, phio) <= 1e-12
    assert np.max(np.abs(phi - phio)) <= 1e-12 * np.max(np.abs(phio))
    assert e == pytest.approx(oracle.energy(p, x), rel=1e-11)


@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("m", [10, 20])
@pytest.mark.parametrize("name,make", CASES[:4])
def test_solve_parity_small(bp, name, make, m, kind):
    p = make(g.KAPPA)
    ref = oracle.solve(p, restart=m, tol=1e-10)
    ctx = _ctx(bp, p)
    ctx.set_matvec_kernel(kind)
    x = np.zeros(2 * p.n)
    bp.bipb_source(ctx)
    st, rep = bp.bipb_gmres_solve(ctx, x, None, m, 1e-10, 500, check_true=True)
    e = bp.bipb_energy(ctx, x)
    assert st == bp.OK and rep["converged"]
    assert abs(rep["iterations"] - ref["report"]["iterations"]) <= 1
    assert e == pytest.approx(ref["energy"], rel=1e-8)
    assert rep["rel_res_true"] <= 1e-9
    assert _rel(x, ref["x"]) <= 1e-8
    ctx.close()


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4"])
def test_solve_parity_golden(bp, cfg):
    """Full-size BASELINE configs against stored oracle solves (tests/make_oracle_golden.py)."""
    path = os.path.join(GOLD, f"oracle_{cfg}.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated")
    gold = json.load(open(path))
    p = g.config(cfg)
    assert p.sha256() == gold["sha256"]
    ctx = _ctx(bp, p)
    b = bp.bipb_source(ctx)
    for m, ref in gold["solves"].items():
        rows = np.array(ref["rows"])
        np.testing.assert_allclose(b[rows], ref["b_phi"], rtol=1e-12, atol=1e-14 * ref["b_norm"])
        np.testing.assert_allclose(b[rows + p.n], ref["b_dphi"], rtol=1e-12, atol=1e-14 * ref["b_norm"])
        x = np.zeros(2 * p.n)
        st, rep = bp.bipb_gmres_solve(ctx, x, None, int(m), gold["tol"], 500, check_true=True)
        e = bp.bipb_energy(ctx, x)
        assert st == bp.OK
        assert abs(rep["iterations"] - ref["iterations"]) <= 1
        assert e == pytest.approx(ref["energy"], rel=1e-8)
        np.testing.assert_allclose(x[rows], ref["x_phi"], rtol=1e-7, atol=1e-9 * ref["x_norm"])
        np.testing.assert_allclose(x[rows + p.n], ref["x_dphi"], rtol=1e-7, atol=1e-9 * ref["x_norm"])
    ctx.close()


@pytest.mark.parametrize("n_keep", [44799, 44800, 44801])
def test_symmetric_block_edges_b640(bp, n_keep):
    """Block edges of the bench's block shape B = 640 (chosen once there are >= 2,048 block pairs,
    N >~ 40k): N = 70*640 - 1, 70*640, 70*640 + 1 (partial last block, nb even / odd).  >= 2,048
    sampled rows including every 640-row block edge against the oracle (per block), the whole
    product against the independently pinned row kernel."""
    p = _ragged(6, 20.0, n_keep, 12, g.charges_in_ball(10, 15.0, 6))
    ctx = _ctx(bp, p)
    assert ctx.matvec_kernel == 1 and ctx.sum_mode == 1
    u = g.random_vector(2 * p.n, 7)
    y1 = bp.bipb_matvec(ctx, u)
    ctx.set_matvec_kernel(0)
    y0 = bp.bipb_matvec(ctx, u)
    ctx.close()
    assert _rel(y1, y0) <= 1e-13
    edges = np.arange(0, p.n + 1, 640)
    rows = np.unique(np.clip(np.concatenate([edges - 1, edges, np.linspace(0, p.n - 1, 2100).astype(np.int64)]),
                             0, p.n - 1))
    assert rows.size >= 2048
    yi, yin = oracle.matvec_rows(p, u, rows)
    for got, want in ((y1[rows], yi), (y1[rows + p.n], yin)):
        assert _rel(got, want) <= 1e-11
        assert np.max(np.abs(got - want)) <= 1e-11 * np.max(np.abs(want))


def test_full_size_c4_sampled(bp):
    """C4 (N = 327,680, the bench workload): sampled rows of the matvec and source, sampled
    charges of phi_reac against the oracle; the solved energy against the Kirkwood series
    (a property that holds at any size: BEM -> Kirkwood with discretisation error ~1e-3)."""
    p = g.config("C4")
    ctx = _ctx(bp, p)
    # 2,048 sampled rows plus the 640-row block edges near both ends
    rows = np.unique(np.concatenate([np.linspace(0, p.n - 1, 2048).astype(np.int64),
                                     [0, 1, 639, 640, 641, 1279, 1280, p.n - 641, p.n - 640, p.n - 1]]))
    assert rows.size >= 2048
    u = g.random_vector(2 * p.n, 21)
    y = bp.bipb_matvec(ctx, u)
    yi, yin = oracle.matvec_rows(p, u, rows)
    for got, want in ((y[rows], yi), (y[rows + p.n], yin)):  # per block: rel-L2 and element-wise
        assert _rel(got, want) <= 1e-11
        assert np.max(np.abs(got - want)) <= 1e-11 * np.max(np.abs(want))
    b = bp.bipb_source(ctx)
    sub = g.Problem("sub", p.centroids[rows], p.normals[rows], p.areas[rows], p.charges, p.eps1, p.eps2, p.kappa)
    bo = oracle.source(sub)
    for got, want in ((b[rows], bo[:rows.size]), (b[rows + p.n], bo[rows.size:])):  # per block (north_star 1e-12)
        assert _rel(got, want) <= 1e-12
        np.testing.assert_allclose(got, want, rtol=1e-12, atol=1e-13 * np.abs(want).max())
    ks = np.linspace(0, p.nc - 1, 16).astype(np.int64)
    phi = np.zeros(p.nc)
    bp.bipb_energy(ctx, u, phi)
    subq = g.Problem("subq", p.centroids, p.normals, p.areas, np.ascontiguousarray(p.charges[ks]), p.eps1, p.eps2,
                     p.kappa)
    np.testing.assert_allclose(phi[ks], oracle.reaction_potential(subq, u), rtol=1e-11,
                               atol=1e-13 * np.abs(phi).max())
    x = np.zeros(2 * p.n)
    st, rep = bp.bipb_gmres_solve(ctx, x, None, 20, 1e-10, 500, check_true=True)
    e = bp.bipb_energy(ctx, x)
    kpath = os.path.join(GOLD, "kirkwood.json")
    ek = json.load(open(kpath))["C4"]["energy"] if os.path.exists(kpath) else \
        kirkwood_energy(p.charges, 20.0, p.eps1, p.eps2, p.kappa)[0]
    assert st == bp.OK and rep["rel_res_true"] <= 1e-9
    assert abs(e / ek - 1) < 5e-3
    assert 10 <= rep["iterations"] <= 60
    # the GPU solution checked against the oracle's own equations (sampled rows of b - A x) and
    # its full N_c x N energy sum (Eq. (14); 1.6e9 pairs, seconds on the host)
    axi, axin = oracle.matvec_rows(p, x, rows)
    bnorm = np.linalg.norm(b)
    assert np.max(np.abs(bo[:rows.size] - axi)) <= 2e-9 * bnorm
    assert np.max(np.abs(bo[rows.size:] - axin)) <= 2e-9 * bnorm
    assert e == pytest.approx(oracle.energy(p, x), rel=1e-11)
    ctx.close()


def test_degenerate_and_errors(bp):
    # N = 1: sums are empty -> y = (1/2 (1+eps) u1, 1/2 (1+1/eps) u2)
    p = g.Problem("n1", np.array([[1.0, 0, 0]]), np.array([[1.0, 0, 0]]), np.array([0.3]), np.zeros((0, 4)))
    ctx = _ctx(bp, p)
    y = bp.bipb_matvec(ctx, np.array([2.0, 3.0]))
    assert y[0] == 0.5 * 81.0 * 2.0 and y[1] == pytest.approx(0.5 * (1 + 1 / 80.0) * 3.0, rel=1e-15)
    # N_c = 0: b = 0, x = 0, E = 0 (R17)
    b = bp.bipb_source(ctx)
    assert np.all(b == 0)
    x = np.ones(2)
    st, rep = bp.bipb_gmres_solve(ctx, x)
    assert st == bp.OK and np.all(x == 0) and rep["iterations"] == 0
    assert bp.bipb_energy(ctx, x) == 0.0
    ctx.close()
    # N = 2 against the oracle
    q = g.Problem("n2", np.array([[1.0, 0, 0], [0.0, 1.3, 0.2]]), np.array([[1.0, 0, 0], [0, 1.0, 0]]),
                  np.array([0.3, 0.2]), np.array([[0.1, 0.1, 0.1, 1.0]]))
    ctx = _ctx(bp, q)
    u = np.array([0.3, -1.0, 2.0, 0.7])
    assert _rel(bp.bipb_matvec(ctx, u), oracle.matvec(q, u)) <= 1e-14
    ctx.close()
    c1 = g.config("C1")
    bad = c1.areas.copy()
    bad[3] = 0.0
    with pytest.raises(bp.BipbError) as ei:
        bp.bipb_setup(c1.centroids, c1.normals, bad, c1.charges, 1, 80, 0.1)
    assert ei.value.status == bp.ERR_INPUT
    nb = c1.normals.copy()
    nb[0] *= 1.01
    with pytest.raises(bp.BipbError) as ei:
        bp.bipb_setup(c1.centroids, nb, c1.areas, c1.charges, 1, 80, 0.1)
    assert ei.value.status == bp.ERR_INPUT
    ch = np.array([[*c1.centroids[17], 1.0]])
    with pytest.raises(bp.BipbError) as ei:
        bp.bipb_setup(c1.centroids, c1.normals, c1.areas, ch, 1, 80, 0.1)
    assert ei.value.status == bp.ERR_SINGULAR
    # max_iters reached -> NOT_CONVERGED with x filled
    ctx = _ctx(bp, c1)
    bp.bipb_source(ctx)
    x = np.zeros(2 * c1.n)
    st, rep = bp.bipb_gmres_solve(ctx, x, None, 5, 1e-14, 7)
    assert st == bp.NOT_CONVERGED and rep["iterations"] == 7 and np.linalg.norm(x) > 0
    ctx.close()


def test_device_pointers_and_determinism(bp):
    import torch
    p = g.sphere_problem(3, 4.0, g.helix_charges())
    dev = torch.device("cuda:0")
    T = lambda a: torch.from_numpy(np.ascontiguousarray(a)).to(dev)
    ctx = bp.bipb_setup(T(p.centroids), T(p.normals), T(p.areas), T(p.charges), 1.0, 80.0, g.KAPPA,
                        stream=torch.cuda.current_stream().cuda_stream)
    u = T(g.random_vector(2 * p.n, 3))
    y1 = torch.empty_like(u)
    y2 = torch.empty_like(u)
    bp.bipb_matvec(ctx, u, y1)
    bp.bipb_matvec(ctx, u, y2)
    assert torch.equal(y1, y2)  # bitwise reproducible
    ref = oracle.matvec(p, u.cpu().numpy())
    assert _rel(y1.cpu().numpy(), ref) <= 1e-11
    x = torch.zeros(2 * p.n, dtype=torch.float64, device=dev)
    bp.bipb_source(ctx)
    st, rep = bp.bipb_gmres_solve(ctx, x, None, 20, 1e-10, 200)
    x2 = torch.zeros_like(x)
    st2, rep2 = bp.bipb_gmres_solve(ctx, x2, None, 20, 1e-10, 200)
    assert torch.equal(x, x2) and rep["iterations"] == rep2["iterations"]
    ctx.close()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_row_shards_bitwise_equal_single_gpu(bp, world):
    """Each rank's rows (BIPB_DIST_NO_COMM: no communicator, this rank's rows only) equal the
    single-GPU product bitwise: the chunk decomposition depends on N only."""
    p = g.sphere_problem(3, 4.0, g.charges_in_ball(23, 3.0, 5))
    full = _ctx(bp, p)
    full.set_matvec_kernel(0)
    u = g.random_vector(2 * p.n, 9)
    y1 = bp.bipb_matvec(full, u)
    b1 = bp.bipb_source(full)
    phi1 = np.zeros(p.nc)
    e1 = bp.bipb_energy(full, u, phi1)
    full.close()
    y = np.zeros(2 * p.n)
    b = np.zeros(2 * p.n)
    phi = np.zeros(p.nc)
    for r in range(world):
        c = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa,
                          dist=(r, world, None, -1, bp.DIST_NO_COMM))
        c.set_matvec_kernel(0)
        yr = bp.bipb_matvec(c, u)
        br = bp.bipb_source(c)
        ph = np.zeros(p.nc)
        bp.bipb_energy(c, u, ph)
        r0, r1 = bp.bipb_partition(p.n, world, r)
        k0, k1 = bp.bipb_partition(p.nc, world, r)
        mask = np.zeros(2 * p.n, bool)
        mask[r0:r1] = True
        mask[p.n + r0:p.n + r1] = True
        assert np.all(yr[~mask] == 0) and np.all(br[~mask] == 0)
        y[mask] = yr[mask]
        b[mask] = br[mask]
        phi[k0:k1] = ph[k0:k1]
        c.close()
    assert np.array_equal(y, y1) and np.array_equal(b, b1) and np.array_equal(phi, phi1)
    assert e1 == pytest.approx(0.5 * 4 * np.pi * 332.0716 * float(np.dot(p.charges[:, 3], phi)), rel=1e-13)


@pytest.mark.parametrize("flags", [0, 2])
@pytest.mark.parametrize("kind", [0, 1])
def test_nccl_exchange_path_world1(bp, kind, flags):
    """The real NCCL exchange path (dlopen'ed libnccl, unique id, communicator, all-gather
    (row kernel) / all-reduce (symmetric kernel) on the library stream) on a world-1
    communicator equals the unsharded path bitwise; flags = DIST_P2P: the peer-store exchange
    (mailbox, epoch flags, fused epilogue stores) instead of the collective."""
    import torch  # noqa: F401  (torch's libnccl.so.2 is the one the library reuses)
    p = g.sphere_problem(3, 4.0, g.charges_in_ball(23, 3.0, 6))
    ref = _ctx(bp, p)
    ref.set_matvec_kernel(kind)
    u = g.random_vector(2 * p.n, 2)
    y0, b0 = bp.bipb_matvec(ref, u), bp.bipb_source(ref)
    x0 = np.zeros(2 * p.n)
    st0, rep0 = bp.bipb_gmres_solve(ref, x0, None, 20, 1e-10, 300)
    e0 = bp.bipb_energy(ref, x0)
    ref.close()
    uid = bp.bipb_nccl_unique_id()
    assert len(uid) == 128
    c = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa,
                      dist=(0, 1, uid, 0, flags))
    c.set_matvec_kernel(kind)
    y = bp.bipb_matvec(c, u)
    if kind == 0:
        assert np.array_equal(y, y0)
    else:  # sharded symmetric path: partial sums + all-reduce + row epilogue (rounding differs)
        assert _rel(y, y0) <= 1e-15
    assert np.array_equal(bp.bipb_source(c), b0)
    x = np.zeros(2 * p.n)
    st, rep = bp.bipb_gmres_solve(c, x, None, 20, 1e-10, 300)
    assert rep["iterations"] == rep0["iterations"]
    if kind == 0:
        assert np.array_equal(x, x0) and bp.bipb_energy(c, x) == e0
    else:
        assert _rel(x, x0) <= 1e-12 and bp.bipb_energy(c, x) == pytest.approx(e0, rel=1e-12)
    c.close()


@pytest.mark.parametrize("world", [2, 3, 5])
def test_symmetric_shards_sum_to_single_gpu(bp, world):
    """Symmetric kernel sharded by I-blocks (BIPB_DIST_NO_COMM): each rank returns
    d u - P_rank / (4 pi); the rank partials sum to the single-GPU product (to rounding)."""
    p = g.sphere_problem(4, 4.0, g.charges_in_ball(23, 3.0, 5))  # N = 5120 = 10 blocks of 512
    full = _ctx(bp, p)
    full.set_matvec_kernel(1)
    u = g.random_vector(2 * p.n, 9)
    y1 = bp.bipb_matvec(full, u)
    full.close()
    eps = p.eps2 / p.eps1
    du = np.concatenate([0.5 * (1 + eps) * u[:p.n], 0.5 * (1 + 1 / eps) * u[p.n:]])
    acc = np.zeros(2 * p.n)
    for r in range(world):
        c = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa,
                          dist=(r, world, None, -1, bp.DIST_NO_COMM))
        c.set_matvec_kernel(1)
        acc += bp.bipb_matvec(c, u) - du
        c.close()
    assert _rel(acc + du, y1) <= 1e-14


@pytest.mark.parametrize("n_keep", [1, 2, 127, 128, 129, 255, 256, 257, 383, 384, 385, 1151, 1536, 2047, 2560, 5119])
def test_symmetric_block_edges(bp, n_keep):
    """Ragged block counts around the small block B = 128 (the shape every N below ~17k gets, r02):
    nb = 1, 2 with an exactly full / one-row last block, odd and even nb, partial last block."""
    p = _ragged(4, 4.0, n_keep, 3, np.zeros((0, 4))) if n_keep > 1 else g.Problem(
        "n1", np.array([[1.0, 0, 0]]), np.array([[1.0, 0, 0]]), np.array([0.3]), np.zeros((0, 4)))
    ctx = _ctx(bp, p)
    ctx.set_matvec_kernel(1)
    u = g.random_vector(2 * p.n, 4)
    y = bp.bipb_matvec(ctx, u)
    ctx.set_matvec_kernel(0)
    y0 = bp.bipb_matvec(ctx, u)
    ref = oracle.matvec(p, u)
    assert _rel(y, ref) <= 1e-11 and _rel(y0, ref) <= 1e-11
    ctx.close()


@pytest.mark.parametrize("nrhs", [1, 2, 3, 4, 7])
@pytest.mark.parametrize("kappa", [g.KAPPA, 0.0])
def test_matvec_batch(bp, nrhs, kappa):
    """Multi-RHS product (passes of 4/2/1 operands sharing every pair evaluation) equals the
    oracle for every operand, host and device buffers."""
    import torch
    p = g.sphere_problem(4, 4.0, np.zeros((0, 4)), kappa=kappa)
    U = np.stack([g.random_vector(2 * p.n, 100 + r) for r in range(nrhs)])
    ctx = _ctx(bp, p)
    ctx.set_matvec_kernel(1)
    Y = bp.bipb_matvec_batch(ctx, U)
    for r in range(nrhs):
        ref = oracle.matvec(p, U[r])
        assert _rel(Y[r], ref) <= 1e-11
        assert _rel(Y[r], bp.bipb_matvec(ctx, U[r])) <= 1e-14
    Ud = torch.from_numpy(U).cuda()
    Yd = torch.empty_like(Ud)
    bp.bipb_matvec_batch(ctx, Ud, Yd)
    assert _rel(Yd.cpu().numpy(), Y) <= 1e-15
    ctx.set_matvec_kernel(0)  # row kernel loops
    assert _rel(bp.bipb_matvec_batch(ctx, U), Y) <= 1e-14
    ctx.close()


@pytest.mark.parametrize("nrhs", [2, 4])
def test_matvec_batch_large_ragged(bp, nrhs):
    """The multi-RHS symmetric kernels (R = 2: B = 512, R = 4: B = 384, ping-pong record buffers) on
    a ragged N = 45,001 (many blocks, partial last block): every operand element-wise against the
    oracle on >= 2,048 sampled rows per block (block edges of both shapes included) and in full
    against the independently pinned row kernel."""
    p = _ragged(6, 20.0, 45001, 17, g.charges_in_ball(10, 15.0, 6))
    U = np.stack([g.random_vector(2 * p.n, 300 + r) for r in range(nrhs)])
    ctx = _ctx(bp, p)
    ctx.set_matvec_kernel(1)
    Y = bp.bipb_matvec_batch(ctx, U)
    ctx.set_matvec_kernel(0)
    Y0 = bp.bipb_matvec_batch(ctx, U)
    ctx.close()
    edges = np.concatenate([np.arange(0, p.n + 1, 384), np.arange(0, p.n + 1, 512)])
    rows = np.unique(np.clip(np.concatenate([edges - 1, edges, np.linspace(0, p.n - 1, 2100).astype(np.int64)]),
                             0, p.n - 1))
    assert rows.size >= 2048
    for r in range(nrhs):
        assert _rel(Y[r], Y0[r]) <= 1e-13
        yi, yin = oracle.matvec_rows(p, U[r], rows)
        for got, want in ((Y[r][rows], yi), (Y[r][rows + p.n], yin)):
            assert _rel(got, want) <= 1e-11
            assert np.max(np.abs(got - want)) <= 1e-11 * np.max(np.abs(want))


def test_multi_rhs_charge_sets_and_batched_gmres(bp):
    """Several charge sets on one surface (bipb_set_charges): source and energy parity per set,
    and the lockstep multi-RHS GMRES equals the single-system solves (iterations, x, E)."""
    p = g.sphere_problem(5, 4.0, g.charges_in_ball(50, 3.0, 2))  # C2 surface (symmetric kernel)
    sets = [g.charges_in_ball(50, 3.0, s) for s in (2, 12, 13)] + [g.helix_charges()]
    ctx = _ctx(bp, p)
    ctx.set_matvec_kernel(1)
    Bs, singles = [], []
    for ch in sets:
        bp.bipb_set_charges(ctx, ch)
        q = g.Problem("set", p.centroids, p.normals, p.areas, ch, p.eps1, p.eps2, p.kappa)
        b = bp.bipb_source(ctx)
        rows = np.arange(0, p.n, 97)
        sub = g.Problem("sub", p.centroids[rows], p.normals[rows], p.areas[rows], ch, p.eps1, p.eps2, p.kappa)
        bo = oracle.source(sub)
        np.testing.assert_allclose(b[rows], bo[:rows.size], rtol=1e-12)
        x = np.zeros(2 * p.n)
        st, rep = bp.bipb_gmres_solve(ctx, x, None, 20, 1e-10, 300)
        singles.append((x, rep, bp.bipb_energy(ctx, x)))
        Bs.append(b)
        xr = g.random_vector(2 * p.n, 7)
        phi = np.zeros(len(ch))
        bp.bipb_energy(ctx, xr, phi)
        np.testing.assert_allclose(phi, oracle.reaction_potential(q, xr), rtol=1e-11, atol=1e-14 * np.abs(phi).max())
    B = np.stack(Bs)
    X = np.zeros_like(B)
    st, reps = bp.bipb_gmres_solve_batch(ctx, B, X, 20, 1e-10, 300, check_true=True)
    assert st == bp.OK
    for r, ch in enumerate(sets):
        xs, rs, es = singles[r]
        assert abs(reps[r]["iterations"] - rs["iterations"]) <= 1
        assert reps[r]["rel_res_true"] <= 1e-9
        assert _rel(X[r], xs) <= 1e-9
        bp.bipb_set_charges(ctx, ch)
        assert bp.bipb_energy(ctx, X[r]) == pytest.approx(es, rel=1e-9)
    # a singular charge set is rejected
    bad = np.array([[*p.centroids[5], 1.0]])
    with pytest.raises(bp.BipbError) as ei:
        bp.bipb_set_charges(ctx, bad)
    assert ei.value.status == bp.ERR_SINGULAR
    ctx.close()


def test_ingested_msms_pqr_surface(bp):
    """End to end on text inputs (§8(f) item 4): a bumpy star-shaped surface written and read
    back in MSMS .vert/.face format with PQR charges, solved on the GPU vs the oracle."""
    v, f = g.icosphere(3, 1.0)
    u = v / np.linalg.norm(v, axis=1)[:, None]
    rad = 6.0 + 0.6 * np.sin(3 * u[:, 0]) * np.cos(2 * u[:, 1]) + 0.4 * u[:, 2] ** 2
    V0 = u * rad[:, None]
    vert, face = g.write_msms(V0, u, f)
    pqr = "".join(f"ATOM {k} C RES 1 {x:.6f} {y:.6f} {z:.6f} {q:.4f} 1.7\n"
                  for k, (x, y, z, q) in enumerate(g.charges_in_ball(12, 3.5, 4)))
    V, VN, F = g.parse_msms(vert, face)
    c, nrm, a, dropped = g.elements_from_msms(V, VN, F)
    p = g.Problem("msms", c, nrm, a, g.parse_pqr(pqr))
    assert dropped == 0
    ref = oracle.solve(p, restart=20, tol=1e-10)
    ctx = _ctx(bp, p)
    out = bp.solve(ctx, restart_m=20, tol=1e-10)
    ctx.close()
    assert abs(out["report"]["iterations"] - ref["report"]["iterations"]) <= 1
    assert out["energy"] == pytest.approx(ref["energy"], rel=1e-8)


@pytest.mark.parametrize("kind", [0, 1])
def test_gmres_graph_replay_matches_eager(bp, kind):
    """Arnoldi steps replayed as CUDA graphs (BIPB_GRAPHS=1, set for the GPU test session in
    conftest) give bitwise the same solve as the eager path (forced by the timing
    instrumentation)."""
    p = g.sphere_problem(4, 4.0, g.charges_in_ball(20, 3.0, 9))
    ctx = _ctx(bp, p)
    ctx.set_matvec_kernel(kind)
    bp.bipb_source(ctx)
    xs, reps = [], []
    for timing in (False, True, False):
        ctx.timing_enable(timing)
        x = np.zeros(2 * p.n)
        st, rep = bp.bipb_gmres_solve(ctx, x, None, 10, 1e-10, 300)
        xs.append(x)
        reps.append(rep["iterations"])
    assert reps[0] == reps[1] == reps[2]
    assert np.array_equal(xs[0], xs[1]) and np.array_equal(xs[0], xs[2])
    ctx.close()


def test_full_size_c5_sampled_matvec(bp):
    """C5 (N = 1,310,720): >= 2,048 sampled rows of one product ("row-sampled oracle
    matvec (2,048 rows)", block edges included) against the oracle per block, rel-L2 and
    element-wise, and the symmetric and row kernels against each other in full."""
    p = g.config("C5")
    ctx = _ctx(bp, p)
    assert ctx.matvec_kernel == 1
    u = g.random_vector(2 * p.n, 31)
    y = bp.bipb_matvec(ctx, u)
    rows = np.unique(np.concatenate([np.linspace(0, p.n - 1, 2048).astype(np.int64),
                                     [0, 639, 640, 641, p.n - 641, p.n - 640, p.n - 1]]))
    assert rows.size >= 2048
    yi, yin = oracle.matvec_rows(p, u, rows)
    for got, want in ((y[rows], yi), (y[rows + p.n], yin)):
        assert _rel(got, want) <= 1e-11
        assert np.max(np.abs(got - want)) <= 1e-11 * np.max(np.abs(want))
    ctx.set_matvec_kernel(0)
    y0 = bp.bipb_matvec(ctx, u)
    assert _rel(y, y0) <= 1e-13
    ctx.close()


@pytest.mark.parametrize("keep", [4999, 30000])
def test_fused_arnoldi_matches_launches(bp, keep, monkeypatch):
    """The one-cluster Arnoldi kernel (bipb_get_arnoldi > 0: MGS dots reduced through distributed
    shared memory) runs the same algorithm as the multi-launch MGS: same iterations, solutions
    equal to rounding, and the mode follows the 2N <= 65536 rule (bipb.h)."""
    p = _ragged(6 if keep > 20480 else 4, 4.0, keep, 3, g.charges_in_ball(25, 3.0, 4))
    out = {}
    for mode in ("fused", "launches"):
        monkeypatch.setenv("BIPB_ARNOLDI", mode)
        ctx = _ctx(bp, p)
        out[mode] = (ctx.arnoldi,) + tuple(bp.solve(ctx, restart_m=10, tol=1e-10)[k] for k in ("x", "energy", "report"))
        ctx.close()
    ef = {4999: 2, 30000: 8}[keep]
    assert out["fused"][0] == ef and out["launches"][0] == 0
    assert out["fused"][3]["iterations"] == out["launches"][3]["iterations"]
    assert _rel(out["fused"][1], out["launches"][1]) <= 1e-12
    assert out["fused"][2] == pytest.approx(out["launches"][2], rel=1e-12)


def test_fused_arnoldi_size_rule(bp):
    q = g.charges_in_ball(5, 3.0, 2)
    for keep, want in ((32768, 8), (32769, 0)):
        p = _ragged(6, 4.0, keep, 5, q)
        ctx = _ctx(bp, p)
        assert ctx.arnoldi == want
        ctx.close()


@pytest.mark.parametrize("n_keep", [17279, 17280, 17281])
def test_symmetric_block_edges_b384(bp, n_keep):
    """Block edges of the mid-size shape B = 384 (>= 1,024 tasks at B = 384, < 2,048 at B = 640):
    N = 45*384 - 1, 45*384, 45*384 + 1 (nb = 45 with a one-row-short / full last block, nb = 46 with
    a one-row last block).  The whole product against the oracle, per block and element-wise."""
    p = _ragged(6, 20.0, n_keep, 13, np.zeros((0, 4)))
    ctx = _ctx(bp, p)
    assert ctx.matvec_kernel == 1
    u = g.random_vector(2 * p.n, 8)
    y = bp.bipb_matvec(ctx, u)
    ctx.close()
    ref = oracle.matvec(p, u)
    for h in (slice(0, p.n), slice(p.n, 2 * p.n)):
        assert _rel(y[h], ref[h]) <= 1e-11
        assert np.max(np.abs(y[h] - ref[h])) <= 1e-11 * np.max(np.abs(ref[h]))


def test_default_kernel_rule(bp):
    """The default product (r02): the row kernel below 296 small-shape (B = 128) tasks, the symmetric
    kernel from there on (N = 2,560: 220 tasks -> row; N = 3,840: 480 -> symmetric; C1 5,120)."""
    for n_keep, want in ((2560, 0), (3840, 1), (5120, 1)):
        p = _ragged(4, 4.0, n_keep, 5, np.zeros((0, 4))) if n_keep < 5120 else g.config("C1")
        ctx = _ctx(bp, p)
        assert ctx.matvec_kernel == want, n_keep
        ctx.close()


@pytest.mark.parametrize("n_keep", [20000, 45001])
def test_symmetric_block_shapes_ragged(bp, n_keep):
    """Both R = 1 block shapes of the symmetric kernel on ragged sizes: N = 20,000 (mid-size
    shape, B = 384: 53 blocks, 27 offsets, 1,431 tasks < 2,048) and N = 45,001 (B = 640: 71
    blocks, 36 offsets, 2,556 tasks, partial last block).  Sampled rows (block edges included)
    against the oracle, the whole product against the independently pinned row kernel."""
    p = _ragged(6, 20.0, n_keep, 11, g.charges_in_ball(10, 15.0, 6))
    ctx = _ctx(bp, p)
    u = g.random_vector(2 * p.n, 5)
    ctx.set_matvec_kernel(1)
    y1 = bp.bipb_matvec(ctx, u)
    ctx.set_matvec_kernel(0)
    y0 = bp.bipb_matvec(ctx, u)
    ctx.close()
    assert _rel(y1, y0) <= 1e-13
    rows = np.unique(np.array([0, 1, 383, 384, 639, 640, 767, 768, p.n // 2, p.n - 2, p.n - 1]))
    yi, yin = oracle.matvec_rows(p, u, rows)
    assert np.max(np.abs(y1[rows] - yi)) <= 1e-11 * np.max(np.abs(yi))
    assert np.max(np.abs(y1[rows + p.n] - yin)) <= 1e-11 * np.max(np.abs(yin))


# ---- opt-in right preconditioning by the jump-term diagonal (bipb_set_precond; not in the paper) ----

@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("name,make", CASES)
def test_solve_parity_precond(bp, name, make, kind):
    """GPU right-preconditioned GMRES against the oracle's (orc_gmres_bem_jacobi, pinned by its own
    CPU tests): iterations +-1, energy 1e-8, x 1e-8; the energy also equals the plain solve's."""
    p = make(g.KAPPA)
    ref = oracle.solve(p, restart=20, tol=1e-10, precond=True)
    plain = oracle.solve(p, restart=20, tol=1e-10)
    ctx = _ctx(bp, p)
    ctx.set_matvec_kernel(kind)
    ctx.set_precond(1)
    assert ctx.precond == 1
    x = np.zeros(2 * p.n)
    bp.bipb_source(ctx)
    st, rep = bp.bipb_gmres_solve(ctx, x, None, 20, 1e-10, 500, check_true=True)
    e = bp.bipb_energy(ctx, x)
    ctx.close()
    assert st == bp.OK and rep["converged"] and rep["rel_res_true"] <= 1e-9
    assert abs(rep["iterations"] - ref["report"]["iterations"]) <= 1
    assert e == pytest.approx(ref["energy"], rel=1e-8)
    assert e == pytest.approx(plain["energy"], rel=1e-8)
    assert _rel(x, ref["x"]) <= 1e-8


def test_precond_switching_and_launch_path(bp):
    """N = 40,000 (multi-launch MGS, symmetric kernel): precond and plain solves alternated in one
    context (graph replay on in the GPU session: the per-step graphs are keyed by the mode) equal
    fresh-context solves; the preconditioned solve needs fewer than half the iterations."""
    p = _ragged(6, 20.0, 40000, 17, g.charges_in_ball(40, 15.0, 9))
    res = {}
    ctx = _ctx(bp, p)
    assert ctx.arnoldi == 0
    bp.bipb_source(ctx)
    for mode in (0, 1, 0, 1):
        ctx.set_precond(mode)
        x = np.zeros(2 * p.n)
        st, rep = bp.bipb_gmres_solve(ctx, x, None, 20, 1e-10, 500, check_true=True)
        assert st == bp.OK and rep["rel_res_true"] <= 1e-9
        res.setdefault(mode, []).append((x, rep["iterations"], bp.bipb_energy(ctx, x)))
    ctx.close()
    for mode in (0, 1):
        (xa, ia, ea), (xb, ib, eb) = res[mode]
        assert ia == ib and np.array_equal(xa, xb) and ea == eb
    assert res[1][0][1] * 2 < res[0][0][1]
    assert res[1][0][2] == pytest.approx(res[0][0][2], rel=1e-8)


def test_precond_batched_gmres(bp):
    """The lockstep multi-RHS GMRES with the preconditioner equals the preconditioned single solves."""
    p = g.sphere_problem(4, 4.0, g.charges_in_ball(20, 3.0, 2))
    sets = [g.charges_in_ball(20, 3.0, s) for s in (2, 5)] + [g.helix_charges()]
    ctx = _ctx(bp, p)
    ctx.set_precond(1)
    Bs, singles = [], []
    for ch in sets:
        bp.bipb_set_charges(ctx, ch)
        Bs.append(bp.bipb_source(ctx))
        x = np.zeros(2 * p.n)
        st, rep = bp.bipb_gmres_solve(ctx, x, None, 20, 1e-10, 300)
        singles.append((x, rep["iterations"]))
    X = np.zeros((len(sets), 2 * p.n))
    st, reps = bp.bipb_gmres_solve_batch(ctx, np.stack(Bs), X, 20, 1e-10, 300, check_true=True)
    ctx.close()
    assert st == bp.OK
    for r in range(len(sets)):
        assert abs(reps[r]["iterations"] - singles[r][1]) <= 1
        assert reps[r]["rel_res_true"] <= 1e-9
        assert _rel(X[r], singles[r][0]) <= 1e-9


def test_precond_argument_errors(bp):
    p = g.sphere_problem(2, 4.0, g.helix_charges())
    ctx = _ctx(bp, p)
    with pytest.raises(bp.BipbError) as ei:
        ctx.set_precond(2)
    assert ei.value.status == bp.ERR_ARG
    assert ctx.precond == 0
    ctx.close()
