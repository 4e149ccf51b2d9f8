"""The multi-rank code path on one GPU: 2, 3 and 8 processes (8 = one 8-GPU box) share the device
and exchange through a test stand-in for NCCL (tests/fakenccl, selected with BIPB_NCCL_LIB; real
NCCL refuses two ranks on one device), or through the peer-store exchange (CUDA IPC mailboxes,
bipb_p2p.cuh).  Every rank runs the full pipeline (source -> replicated GMRES with one
collective per product -> energy) and must reproduce the single-GPU results: bitwise for the
row kernel (rank-count invariant sums), to rounding for the symmetric kernel (all-reduce of
partial sums).  Every rank's results are also checked against the ORACLE (oracle/, computed once
in the parent process; the C2 solve from the stored tests/golden/oracle_C2.json): matvec and
source element-wise and per block, E_sol to 1e-8, iterations +-1, solution rows."""
import json
import multiprocessing as mp
import os
import time

import numpy as np
import pytest

import bipb_inputs as g
import oracle

pytestmark = pytest.mark.gpu
FAKE = os.path.join(os.path.dirname(__file__), "fakenccl", "libfakenccl.so")


def _problem(size="big"):
    if size == "tiny":  # 20 elements, 3 charges: most ranks own no rows, blocks or charges
        return g.sphere_problem(0, 4.0, g.charges_in_ball(3, 2.0, 5))
    if size == "c1":  # N = 5120: the symmetric kernel's small block shape (B = 128, r02)
        return g.config("C1")
    return g.config("C2")  # N = 20480 (symmetric default, B = 384), the stored oracle solve exists


_ORC = {}


def _oracle(size):
    """Oracle values for the pipeline _run executes (u = random_vector(2N, 5), GMRES(20) to 1e-10)."""
    if size not in _ORC:
        p = _problem(size)
        u = g.random_vector(2 * p.n, 5)
        o = {"y": oracle.matvec(p, u), "b": oracle.source(p)}
        if size == "tiny":
            x, st, rep = oracle.gmres(p, o["b"], restart=20, tol=1e-10, max_iters=300)
            o.update(e=oracle.energy(p, x), its=rep["iterations"], rows=np.arange(p.n), x_phi=x[:p.n],
                     x_dphi=x[p.n:], x_norm=float(np.linalg.norm(x)))
        else:
            gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden",
                                               "oracle_C1.json" if size == "c1" else "oracle_C2.json")))
            assert gold["sha256"] == p.sha256()
            s20 = gold["solves"]["20"]
            o.update(e=s20["energy"], its=s20["iterations"], rows=np.array(s20["rows"]),
                     x_phi=np.array(s20["x_phi"]), x_dphi=np.array(s20["x_dphi"]), x_norm=s20["x_norm"])
        _ORC[size] = o
    return _ORC[size]


def _check_oracle(o, orc, n):
    """One rank's outputs against the oracle at the north_star tolerances."""
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    assert rel(o["y"], orc["y"]) <= 1e-11
    for blk in (slice(0, n), slice(n, 2 * n)):
        assert rel(o["y"][blk], orc["y"][blk]) <= 1e-11
        if np.any(orc["b"][blk]):
            assert rel(o["b"][blk], orc["b"][blk]) <= 1e-12
    assert abs(o["its"] - orc["its"]) <= 1
    assert o["e"] == pytest.approx(orc["e"], rel=1e-8)
    rows = orc["rows"]
    np.testing.assert_allclose(o["x"][rows], orc["x_phi"], rtol=1e-7, atol=1e-9 * orc["x_norm"])
    np.testing.assert_allclose(o["x"][rows + n], orc["x_dphi"], rtol=1e-7, atol=1e-9 * orc["x_norm"])


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
        ctx.set_precond(0)
        # lockstep batched GMRES (multi-RHS, one shared product per step): b and 3b -> x and 3x
        XB = np.zeros((2, 2 * p.n))
        stb, repb = bp.bipb_gmres_solve_batch(ctx, np.stack([b, 3.0 * b]), XB, 20, 1e-10, 300)
        ctx.close()
        q.put((rank, {"y": y, "Y": Y, "b": b, "x": x, "its": rep["iterations"], "e": e, "phi": phi, "xp": xp,
                      "its_p": repp["iterations"], "XB": XB, "its_b": [r["iterations"] for r in repb],
                      "st_b": stb}, None))
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
    orc, n = _oracle("big"), _problem().n
    for o in outs:  # every rank holds the full, identical result, equal to the oracle's
        _check_oracle(o, orc, n)
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
        # batched GMRES on P ranks: replicated, equal to the single-GPU batch and to the plain solve
        assert o["st_b"] == 0 and o["its_b"] == ref["its_b"]
        assert np.array_equal(o["XB"], outs[0]["XB"])
        assert rel(o["XB"], ref["XB"]) <= 1e-11
        assert rel(o["XB"][0], o["x"]) <= 1e-9 and rel(o["XB"][1], 3.0 * o["x"]) <= 1e-9


@pytest.mark.parametrize("exchange", ["nccl", "p2p"])
@pytest.mark.parametrize("kind", [0, 1])
def test_multirank_tiny_problem(kind, exchange):
    """8 ranks on a 20-element surface with 3 charges: ranks without rows, I-blocks or charges
    still take part in every exchange (zero contributions) and end with the single-GPU result."""
    ref = _spawn(0, kind, size="tiny")[0]
    outs = _spawn(8, kind, exchange, size="tiny")
    orc, n = _oracle("tiny"), _problem("tiny").n
    for o in outs:
        _check_oracle(o, orc, n)
        assert o["its"] == ref["its"]
        np.testing.assert_allclose(o["y"], ref["y"], rtol=1e-14, atol=1e-15 * np.abs(ref["y"]).max())
        np.testing.assert_allclose(o["x"], ref["x"], rtol=1e-11, atol=1e-13 * np.abs(ref["x"]).max())
        assert np.array_equal(o["b"], ref["b"])
        assert o["e"] == pytest.approx(ref["e"], rel=1e-12)


@pytest.mark.parametrize("world,exchange,size", [(w, x, s) for s in ("big", "tiny") for x in ("nccl", "p2p")
                                                  for w in (2, 3, 8)] + [(8, "p2p", "c1"), (3, "nccl", "c1")])
def test_multirank_exact_sums_bitwise(world, exchange, size):
    """Exact limb sums (bipb_set_sum_mode 1): the symmetric product, the replicated GMRES and the
    energy are bitwise the single-GPU results for every rank count and both exchanges."""
    ref = _spawn(0, 1, size=size, sum_mode="exact")[0]
    outs = _spawn(world, 1, exchange, size=size, sum_mode="exact")
    orc, n = _oracle(size), _problem(size).n
    for o in outs:
        _check_oracle(o, orc, n)
        assert np.array_equal(o["y"], ref["y"]) and np.array_equal(o["x"], ref["x"])
        assert o["its"] == ref["its"] and o["e"] == ref["e"]
        assert np.array_equal(o["xp"], ref["xp"])


def _run_fail(rank, world, uid, mode, q, done):
    """Failure paths of the exchange (bipb.cu p2p_setup / ctx_sync): each mode's expectation."""
    os.environ["BIPB_NCCL_LIB"] = FAKE
    os.environ["BIPB_GRAPHS"] = "0"
    if mode == "timeout":  # rank 1 never takes part in the product: rank 0's wait must time out
        os.environ["BIPB_EXCHANGE"] = "p2p"
        os.environ["BIPB_P2P_TIMEOUT_S"] = "2"
    else:  # rank 1's mapping self-test reports a failure
        os.environ["BIPB_P2P_PROBE_FAIL"] = "1"
        if mode == "probe_required":
            os.environ["BIPB_EXCHANGE"] = "p2p"
    try:
        import paper_1301_5885_b200 as bp
        p = _problem("tiny")
        u = g.random_vector(2 * p.n, 5)
        dist = (rank, world, uid, 0)
        if mode == "probe_required":
            try:
                bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa, dist=dist)
                q.put((rank, None, "setup succeeded although the peer-store exchange was required"))
            except bp.BipbError as ex:
                q.put((rank, {"status": ex.status, "msg": str(ex)}, None))
            return
        ctx = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa, dist=dist)
        if mode == "probe_auto":  # fallback: every rank uses the NCCL collectives, same results
            res = {"exchange": ctx.exchange, "y": bp.bipb_matvec(ctx, u), "b": bp.bipb_source(ctx)}
            ctx.close()
            q.put((rank, res, None))
            return
        res = {"exchange": ctx.exchange}
        if rank == 0:
            t = time.time()
            try:
                bp.bipb_matvec(ctx, u)
                res["first"] = None
            except bp.BipbError as ex:
                res["first"] = (ex.status, str(ex))
            res["seconds"] = time.time() - t
            try:
                bp.bipb_matvec(ctx, u)
                res["second"] = None
            except bp.BipbError as ex:
                res["second"] = (ex.status, str(ex))
            ctx.close()
            # the CUDA context survived: a fresh single-GPU context computes the product
            c1 = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa)
            res["y_fresh"] = bp.bipb_matvec(c1, u)
            c1.close()
            done.set()
            q.put((rank, res, None))
        else:
            done.wait(300)  # keep the mailbox mapped until rank 0 is finished
            # no ctx.close(): rank 0 aborted the communicator, a destroy would wait for it forever
            q.put((rank, res, None))
            q.close()
            q.join_thread()
            os._exit(0)
    except Exception as ex:  # pragma: no cover
        q.put((rank, None, repr(ex)))
        done.set()


def _spawn_fail(mode, world=2):
    ctx = mp.get_context("spawn")
    q, done = ctx.Queue(), ctx.Event()
    uid = f"/bipb_fakenccl_{os.getpid()}_{time.time_ns()}".encode().ljust(128, b"\0")
    procs = [ctx.Process(target=_run_fail, args=(r, world, uid, mode, q, done)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = [q.get(timeout=600) for _ in procs]
    for pr in procs:
        pr.join(timeout=60)
    for _, _, err in res:
        assert err is None, err
    return [r[1] for r in sorted(res, key=lambda t: t[0])]


def test_p2p_timeout_returns_status():
    """A peer that never delivers: the wait kernel gives up after BIPB_P2P_TIMEOUT_S and the call
    returns BIPB_ERR_NCCL (no __trap: the process's CUDA context stays usable); the context is then
    marked failed and later calls return at once."""
    import paper_1301_5885_b200 as bp
    r0, r1 = _spawn_fail("timeout")
    assert r0["exchange"] == r1["exchange"] == "p2p"
    st, msg = r0["first"]
    assert st == bp.ERR_NCCL and "did not deliver" in msg and "rank 1" in msg
    assert 1.5 <= r0["seconds"] < 60
    st2, msg2 = r0["second"]
    assert st2 == bp.ERR_NCCL and "failed earlier" in msg2
    orc = _oracle("tiny")
    assert np.linalg.norm(r0["y_fresh"] - orc["y"]) <= 1e-11 * np.linalg.norm(orc["y"])


def test_p2p_probe_failure_falls_back_to_nccl():
    """One rank's mapping self-test fails: all ranks agree on the NCCL collectives (auto mode) and
    still compute the oracle's product and source term; when peer stores are required, setup fails
    with BIPB_ERR_NCCL on every rank instead."""
    import paper_1301_5885_b200 as bp
    orc, n = _oracle("tiny"), _problem("tiny").n
    for o in _spawn_fail("probe_auto"):
        assert o["exchange"] == "nccl"
        assert np.linalg.norm(o["y"] - orc["y"]) <= 1e-11 * np.linalg.norm(orc["y"])
        np.testing.assert_allclose(o["b"], orc["b"], rtol=1e-12, atol=1e-14 * np.abs(orc["b"]).max())
    for o in _spawn_fail("probe_required"):
        assert o["status"] == bp.ERR_NCCL and "peer-store exchange unavailable" in o["msg"]


def _run_product(rank, world, uid, exchange, cfg, q, kind=1):
    """Product, source, energy and the full GMRES solve of a BASELINE config: the full-size exchange."""
    os.environ["BIPB_NCCL_LIB"] = FAKE
    os.environ["BIPB_GRAPHS"] = "0"
    os.environ["BIPB_EXCHANGE"] = exchange
    try:
        import paper_1301_5885_b200 as bp
        p = g.config(cfg)
        dist = None if world == 0 else (rank, world, uid, 0)
        ctx = bp.bipb_setup(p.centroids, p.normals, p.areas, p.charges, p.eps1, p.eps2, p.kappa, dist=dist)
        assert ctx.matvec_kernel == 1 and ctx.sum_mode == 1
        ctx.set_matvec_kernel(kind)  # 0: the row kernel (rank-count invariant chunk sums)
        u = g.random_vector(2 * p.n, 41)
        y = bp.bipb_matvec(ctx, u)
        b = bp.bipb_source(ctx)
        e = bp.bipb_energy(ctx, u)
        x = np.zeros(2 * p.n)  # the bench's solve: GMRES(20) to 1e-10, one exchange per product
        st, rep = bp.bipb_gmres_solve(ctx, x, None, 20, 1e-10, 500)
        es = bp.bipb_energy(ctx, x)
        ctx.close()
        q.put((rank, {"y": y, "b": b, "e": e, "x": x, "its": rep["iterations"], "es": es, "st": st}, None))
    except Exception as ex:  # pragma: no cover
        q.put((rank, None, repr(ex)))


@pytest.mark.parametrize("kind,exchange", [(1, "p2p"), (1, "nccl"), (0, "p2p")])
def test_multirank_c4_product_bitwise(kind, exchange):
    """The bench workload C4 (N = 327,680) over 8 ranks (an 8-GPU box's decomposition: 64 of the
    512 I-blocks per rank, 625 charges per rank for the energy): every rank's product (exact limb
    sums; the offset runs W come from global sizes, so the partials are the same tiles on every
    rank count) is bitwise the single-GPU product, source and energy are equal to rounding; the
    full GMRES(20) solve on 8 ranks takes the single-GPU iteration count and matches the stored
    oracle solve (tests/golden/oracle_C4.json: E_sol 1e-8, iterations +-1); the single-GPU
    product against the oracle on 256 sampled rows per block."""
    ctx = mp.get_context("spawn")

    def spawn(world):
        q = ctx.Queue()
        uid = f"/bipb_fakenccl_{os.getpid()}_{time.time_ns()}".encode().ljust(128, b"\0") if world else None
        procs = [ctx.Process(target=_run_product, args=(r, world, uid, exchange, "C4", q, kind))
                 for r in range(max(world, 1))]
        for pr in procs:
            pr.start()
        res = [q.get(timeout=900) for _ in procs]
        for pr in procs:
            pr.join(timeout=60)
        for _, _, err in res:
            assert err is None, err
        return [r[1] for r in sorted(res, key=lambda t: t[0])]

    ref = spawn(0)[0]
    outs = spawn(8)
    p = g.config("C4")
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_C4.json")))
    assert gold["sha256"] == p.sha256()
    s20 = gold["solves"]["20"]
    for o in outs:
        assert np.array_equal(o["y"], ref["y"])
        assert np.linalg.norm(o["b"] - ref["b"]) <= 1e-14 * np.linalg.norm(ref["b"])
        assert o["e"] == pytest.approx(ref["e"], rel=1e-13)
        # the full solve on 8 ranks: the single-GPU iteration, and the stored oracle solve
        assert o["st"] == 0 and o["its"] == ref["its"]
        assert np.linalg.norm(o["x"] - ref["x"]) <= 1e-12 * np.linalg.norm(ref["x"])
        assert abs(o["its"] - s20["iterations"]) <= 1
        assert o["es"] == pytest.approx(s20["energy"], rel=1e-8)
    u = g.random_vector(2 * p.n, 41)
    rows = np.unique(np.linspace(0, p.n - 1, 256).astype(np.int64))
    yi, yin = oracle.matvec_rows(p, u, rows)
    for got, want in ((ref["y"][rows], yi), (ref["y"][rows + p.n], yin)):
        assert np.max(np.abs(got - want)) <= 1e-11 * np.max(np.abs(want))
