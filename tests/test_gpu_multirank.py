"""The multi-rank code path on one GPU: 2, 3 and 8 processes (8 = one 8-GPU box) share the device
and exchange through a test stand-in for NCCL (tests/fakenccl, selected with BIPB_NCCL_LIB; real
NCCL refuses two ranks on one device), or through the peer-store exchange (CUDA IPC mailboxes,
bipb_p2p.cuh).  Every rank runs the full pipeline (source -> replicated GMRES with one
collective per product -> energy) and must reproduce the single-GPU results: bitwise for the
row kernel (rank-count invariant sums), to rounding for the symmetric kernel (all-reduce of
partial sums)."""
import multiprocessing as mp
import os

import numpy as np
import pytest

import bipb_inputs as g

pytestmark = pytest.mark.gpu
FAKE = os.path.join(os.path.dirname(__file__), "fakenccl", "libfakenccl.so")


def _problem(size="big"):
    if size == "tiny":  # 20 elements, 3 charges: most ranks own no rows, blocks or charges
        return g.sphere_problem(0, 4.0, g.charges_in_ball(3, 2.0, 5))
    return g.sphere_problem(5, 4.0, g.charges_in_ball(30, 3.0, 17))  # N = 20480 (symmetric default)


def _run(rank, world, uid, kind, exchange, q, size="big", sum_mode="fixed"):
    os.environ["BIPB_NCCL_LIB"] = FAKE
    os.environ["BIPB_SUM"] = sum_mode  # exact: integer limb sums (bipb_exact.cuh)
    os.environ["BIPB_GRAPHS"] = "0"  # the stand-in synchronises inside collectives: not capturable
    os.environ["BIPB_EXCHANGE"] = exchange  # nccl: collectives; p2p: peer stores (bipb_p2p.cuh)
    try:
        import paper_1301_5885_b200 as bp
        p = _problem(size)
        dist = None if world == 0 else (rank, world, uid, 0)
        ctx = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa, dist=dist)
        ctx.set_matvec_kernel(kind)
        assert ctx.sum_mode == (1 if sum_mode == "exact" and kind == 1 else 0)
        assert ctx.exchange == ("none" if world == 0 else exchange)
        u = g.random_vector(2 * p.n, 5)
        y = bp.bipb_matvec(ctx, u)
        Y = bp.bipb_matvec_batch(ctx, np.stack([u, 2 * u, -u]))
        b = bp.bipb_source(ctx)
        x = np.zeros(2 * p.n)
        st, rep = bp.bipb_gmres_solve(ctx, x, None, 20, 1e-10, 300)
        phi = np.zeros(p.nc)
        e = bp.bipb_energy(ctx, x, phi)
        ctx.set_precond(1)  # the opt-in preconditioned solve (replicated like the plain one)
        xp = np.zeros(2 * p.n)
        st, repp = bp.bipb_gmres_solve(ctx, xp, None, 20, 1e-10, 300)
        ctx.close()
        q.put((rank, {"y": y, "Y": Y, "b": b, "x": x, "its": rep["iterations"], "e": e, "phi": phi, "xp": xp,
                      "its_p": repp["iterations"]}, None))
    except Exception as ex:  # pragma: no cover
        q.put((rank, None, repr(ex)))


def _spawn(world, kind, exchange="nccl", size="big", sum_mode="fixed"):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    uid = None
    if world:  # the stand-in's unique id is a shared-memory name (made here: the parent process
        # must not load the stand-in into its own copy of the library)
        import time
        uid = f"/bipb_fakenccl_{os.getpid()}_{time.time_ns()}".encode().ljust(128, b"\0")
    procs = [ctx.Process(target=_run, args=(r, world, uid, kind, exchange, q, size, sum_mode))
             for r in range(max(world, 1))]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    for _, _, err in res:
        assert err is None, err
    return [r[1] for r in sorted(res, key=lambda t: t[0])]


@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
@pytest.mark.parametrize("kind", [0, 1])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_multirank_matches_single(world, kind, exchange):
    assert os.path.exists(FAKE), "build tests/fakenccl/libfakenccl.so (__graft_entry__.build())"
    ref = _spawn(0, kind)[0]
    outs = _spawn(world, kind, exchange)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    for o in outs:  # every rank holds the full, identical result
        assert np.array_equal(o["x"], outs[0]["x"]) and o["e"] == outs[0]["e"]
        assert o["its"] == ref["its"] and o["its_p"] == ref["its_p"] < ref["its"]
        assert np.array_equal(o["xp"], outs[0]["xp"])
        assert rel(o["xp"], ref["xp"]) <= (0.0 if kind == 0 else 1e-11)
        if kind == 0:
            assert np.array_equal(o["y"], ref["y"]) and np.array_equal(o["b"], ref["b"])
            assert np.array_equal(o["x"], ref["x"]) and o["e"] == ref["e"]
        else:
            assert rel(o["y"], ref["y"]) <= 1e-14 and rel(o["Y"], ref["Y"]) <= 1e-14
            assert np.array_equal(o["b"], ref["b"])
            assert rel(o["x"], ref["x"]) <= 1e-11 and o["e"] == pytest.approx(ref["e"], rel=1e-12)
        np.testing.assert_allclose(o["phi"], ref["phi"], rtol=1e-13, atol=1e-16)


@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
@pytest.mark.parametrize("kind", [0, 1])
def test_multirank_tiny_problem(kind, exchange):
    """8 ranks on a 20-element surface with 3 charges: ranks without rows, I-blocks or charges
    still take part in every exchange (zero contributions) and end with the single-GPU result."""
    ref = _spawn(0, kind, size="tiny")[0]
    outs = _spawn(8, kind, exchange, size="tiny")
    for o in outs:
        assert o["its"] == ref["its"]
        np.testing.assert_allclose(o["y"], ref["y"], rtol=1e-14, atol=1e-15 * np.abs(ref["y"]).max())
        np.testing.assert_allclose(o["x"], ref["x"], rtol=1e-11, atol=1e-13 * np.abs(ref["x"]).max())
        assert np.array_equal(o["b"], ref["b"])
        assert o["e"] == pytest.approx(ref["e"], rel=1e-12)


@pytest.mark.parametrize("size", ["big", "tiny"])
@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_multirank_exact_sums_bitwise(world, exchange, size):
    """Exact limb sums (bipb_set_sum_mode 1): the symmetric product, the replicated GMRES and the
    energy are bitwise the single-GPU results for every rank count and both exchanges."""
    ref = _spawn(0, 1, size=size, sum_mode="exact")[0]
    outs = _spawn(world, 1, exchange, size=size, sum_mode="exact")
    for o in outs:
        assert np.array_equal(o["y"], ref["y"]) and np.array_equal(o["x"], ref["x"])
        assert o["its"] == ref["its"] and o["e"] == ref["e"]
        assert np.array_equal(o["xp"], ref["xp"])
