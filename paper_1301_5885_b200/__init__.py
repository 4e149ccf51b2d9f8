"""paper_1301_5885_b200 — B200-native direct-sum boundary-integral Poisson-Boltzmann hot path.

Thin Python binding (argument marshalling only) over the C ABI in include/bipb.h,
implemented by libbipb.so (hand-written sm_100a CUDA, built in-tree by build.py).
Every step of the path — source term (Eq. (11)), matvec (Eqs. (12)-(13)), GMRES
 and solvation energy (Eq. (14)) of Geng & Jacob, arXiv 1301.5885 —
runs in the library's kernels.  There is no CPU fallback: importing this package fails
loudly if libbipb.so is missing, and every call raises BipbError on a non-OK status.

Array arguments may be numpy arrays (host) or torch tensors (host or CUDA), float64 and
C-contiguous.  CUDA tensors are passed by device pointer (no copies).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("BIPB_LIB") or os.path.join(_HERE, "libbipb.so")  # BIPB_LIB: tuning variants only

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python paper_1301_5885_b200/build.py` "
                      "(or __graft_entry__.build()); there is no fallback path")
_lib = ctypes.CDLL(LIB_PATH)

OK, ERR_ARG, NOT_CONVERGED, ERR_INPUT, ERR_SINGULAR, ERR_CUDA, ERR_NCCL, ERR_OOM = range(8)
_NAMES = {0: "OK", 1: "ERR_ARG", 2: "NOT_CONVERGED", 3: "ERR_INPUT", 4: "ERR_SINGULAR", 5: "ERR_CUDA",
          6: "ERR_NCCL", 7: "ERR_OOM"}


class BipbError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"bipb {_NAMES.get(status, status)}: {msg}")
        self.status = status


DIST_NO_COMM = 1
DIST_P2P = 2  # force the peer-store exchange of the products (bipb.h; default when possible)
DIST_NCCL = 4  # force NCCL collectives for the products


class Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("device", ctypes.c_int32),
                ("flags", ctypes.c_int32), ("nccl_uid", ctypes.c_ubyte * 128)]


class Report(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int64), ("restarts", ctypes.c_int64), ("matvecs", ctypes.c_int64),
                ("converged", ctypes.c_int64), ("rel_res_est", ctypes.c_double),
                ("rel_res_true", ctypes.c_double), ("history", ctypes.POINTER(ctypes.c_double)),
                ("history_cap", ctypes.c_int64), ("history_len", ctypes.c_int64)]


_P = ctypes.c_void_p
_I64, _I32, _D = ctypes.c_int64, ctypes.c_int32, ctypes.c_double
_SIGS = {
    "bipb_setup": ([ctypes.POINTER(_P), _I64, _P, _P, _P, _I64, _P, _D, _D, _D, ctypes.POINTER(Dist), _P], ctypes.c_int),
    "bipb_source": ([_P, _P], ctypes.c_int),
    "bipb_matvec": ([_P, _P, _P], ctypes.c_int),
    "bipb_gmres_solve": ([_P, _P, _P, _I32, _D, _I32, _I32, ctypes.POINTER(Report)], ctypes.c_int),
    "bipb_energy": ([_P, _P, _P, _P], ctypes.c_int),
    "bipb_destroy": ([_P], None),
    "bipb_last_error": ([], ctypes.c_char_p),
    "bipb_partition": ([_I64, _I32, _I32, ctypes.POINTER(_I64), ctypes.POINTER(_I64)], None),
    "bipb_nccl_unique_id": ([_P], ctypes.c_int),
    "bipb_timing_enable": ([_P, _I32], ctypes.c_int),
    "bipb_timing_get": ([_P, _I32, ctypes.POINTER(_D), ctypes.POINTER(_I64)], ctypes.c_int),
    "bipb_timing_reset": ([_P], ctypes.c_int),
    "bipb_version": ([], ctypes.c_char_p),
    "bipb_set_matvec_kernel": ([_P, _I32], ctypes.c_int),
    "bipb_matvec_batch": ([_P, _I32, _P, _P], ctypes.c_int),
    "bipb_gmres_solve_batch": ([_P, _I32, _P, _P, _I32, _D, _I32, _I32, ctypes.POINTER(Report)], ctypes.c_int),
    "bipb_set_charges": ([_P, _I64, _P], ctypes.c_int),
    "bipb_get_matvec_kernel": ([_P], _I32),
    "bipb_get_exchange": ([_P], _I32),
    "bipb_get_arnoldi": ([_P], _I32),
    "bipb_get_graph_cycles": ([_P], _I64),
    "bipb_set_precond": ([_P, _I32], ctypes.c_int),
    "bipb_get_precond": ([_P], _I32),
    "bipb_set_sum_mode": ([_P, _I32], ctypes.c_int),
    "bipb_get_sum_mode": ([_P], _I32),
}
EXPORTS = tuple(_SIGS)
for _name, (_a, _r) in _SIGS.items():
    _f = getattr(_lib, _name)
    _f.argtypes, _f.restype = _a, _r


def _check(st: int):
    if st != OK:
        raise BipbError(st, _lib.bipb_last_error().decode())


def _ptr(a, writable=False, size=None):
    """(pointer, keepalive) for a float64 C-contiguous numpy array or torch tensor holding
    exactly `size` elements when given (the C ABI takes bare pointers)."""
    if a is None:
        return None, None
    if size is not None:
        have = a.size if isinstance(a, np.ndarray) else (a.numel() if hasattr(a, "numel") else None)
        if have != size:
            raise ValueError(f"array has {have} elements, expected {size}")
    if isinstance(a, np.ndarray):
        if a.dtype != np.float64 or not a.flags.c_contiguous or (writable and not a.flags.writeable):
            raise ValueError("arrays must be float64, C-contiguous (and writable for outputs)")
        return a.ctypes.data, a
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(a, torch.Tensor):
        if a.dtype != torch.float64 or not a.is_contiguous():
            raise ValueError("tensors must be float64 and contiguous")
        return a.data_ptr(), a
    raise TypeError(f"unsupported array type {type(a)}")


def _order(ctx, *arrays):
    """Stream ordering for torch CUDA tensors.  The library runs a context's work on
    the stream given at setup (else its own non-blocking stream) and returns after completion, so
    outputs are ready for any stream afterwards.  Inputs produced by torch kernels still queued on
    torch's current stream must be finished first: when the context does not run on that very
    stream, synchronise it before the call."""
    for a in arrays:
        if a is None or isinstance(a, np.ndarray) or not getattr(a, "is_cuda", False):
            continue
        import torch
        cur = torch.cuda.current_stream(a.device)
        if ctx._stream is None or int(ctx._stream) != int(cur.cuda_stream):
            cur.synchronize()
        return


def version() -> str:
    return _lib.bipb_version().decode()


def bipb_partition(n: int, world: int, rank: int) -> tuple[int, int]:
    r0, r1 = _I64(), _I64()
    _lib.bipb_partition(n, world, rank, ctypes.byref(r0), ctypes.byref(r1))
    return r0.value, r1.value


def bipb_nccl_unique_id() -> bytes:
    buf = (ctypes.c_ubyte * 128)()
    _check(_lib.bipb_nccl_unique_id(ctypes.cast(buf, _P)))
    return bytes(buf)


class Context:
    """Owns a bipb_ctx (device geometry, charges, buffers, stream, NCCL comm)."""

    def __init__(self, handle, n, nc, keep, stream=None):
        self._h = handle
        self.n, self.nc = n, nc
        self._keep = keep
        self._stream = stream  # the cudaStream_t the library runs this context on (None: its own)

    @property
    def handle(self):
        if self._h is None:
            raise BipbError(ERR_ARG, "context destroyed")
        return self._h

    def close(self):
        if self._h is not None:
            _lib.bipb_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # matvec kernel selection: 0 = row kernel, 1 = symmetric-pair kernel (default) ----
    def set_matvec_kernel(self, kind: int):
        _check(_lib.bipb_set_matvec_kernel(self.handle, int(kind)))

    @property
    def matvec_kernel(self) -> int:
        return int(_lib.bipb_get_matvec_kernel(self.handle))

    @property
    def exchange(self) -> str:
        """How products are exchanged between ranks: "none", "nccl" or "p2p" (peer stores)."""
        return {0: "none", 1: "nccl", 2: "p2p"}[int(_lib.bipb_get_exchange(self.handle))]

    # GMRES preconditioning: 0 = plain (the paper), 1 = right jump-term diagonal (bipb.h) -------
    def set_precond(self, kind: int):
        _check(_lib.bipb_set_precond(self.handle, int(kind)))

    @property
    def precond(self) -> int:
        return int(_lib.bipb_get_precond(self.handle))

    # partial-sum mode of the symmetric product: 0 fixed-order doubles, 1 exact limbs (bipb.h) ----
    def set_sum_mode(self, mode: int):
        _check(_lib.bipb_set_sum_mode(self.handle, int(mode)))

    @property
    def sum_mode(self) -> int:
        return int(_lib.bipb_get_sum_mode(self.handle))

    @property
    def graph_cycles(self) -> int:
        """GMRES cycles this context ran as one CUDA-graph launch (BIPB_GRAPHS=2; bipb.h)."""
        return int(_lib.bipb_get_graph_cycles(self.handle))

    @property
    def arnoldi(self) -> int:
        """0: one launch per MGS reduction; E > 0: fused cluster kernel, E elements per thread."""
        return int(_lib.bipb_get_arnoldi(self.handle))

    # instrumentation (bench.py) -------------------------------------------------
    def timing_enable(self, on=True):
        _check(_lib.bipb_timing_enable(self.handle, int(on)))

    def timing_reset(self):
        _check(_lib.bipb_timing_reset(self.handle))

    def timing_get(self, which: int) -> tuple[float, int]:
        ms, cnt = _D(), _I64()
        _check(_lib.bipb_timing_get(self.handle, which, ctypes.byref(ms), ctypes.byref(cnt)))
        return ms.value, cnt.value


def bipb_setup(centroids, normals, areas, charges, eps1, eps2, kappa, dist=None, stream=None) -> Context:
    """Table 1 step 4: geometry [n,3] x2, areas [n], charges [nc,4] (x,y,z,Q).
    dist: None or (rank, world, uid_bytes[, device[, flags]]) (flags: DIST_NO_COMM for tests).  stream: None (library stream) or a
    cudaStream_t handle (int), e.g. torch.cuda.current_stream().cuda_stream."""
    n = int(centroids.shape[0])
    nc = int(charges.shape[0]) if charges is not None else 0
    pc, kc = _ptr(centroids, size=3 * n)
    pn, kn = _ptr(normals, size=3 * n)
    pa, ka = _ptr(areas, size=n)
    pq, kq = _ptr(charges, size=4 * nc) if nc > 0 else (None, None)
    d = None
    if dist is not None:
        rank, world, uid = dist[0], dist[1], dist[2]
        dev = dist[3] if len(dist) > 3 else -1
        flags = dist[4] if len(dist) > 4 else 0
        d = Dist(rank=rank, world=world, device=dev, flags=flags)
        if uid is not None:
            ctypes.memmove(d.nccl_uid, bytes(uid), 128)
    h = _P()
    st = _lib.bipb_setup(ctypes.byref(h), n, pc, pn, pa, nc, pq, float(eps1), float(eps2), float(kappa),
                         ctypes.byref(d) if d is not None else None, stream)
    _check(st)
    return Context(h, n, nc, (kc, kn, ka, kq), stream)


def _out_like(ctx_n2, like):
    if like is not None:
        return like
    return np.empty(ctx_n2)


def bipb_source(ctx: Context, b=None):
    """Eq. (11): b = [S1; S2] (2n).  Returns b (a new numpy array if b is None)."""
    b = _out_like(2 * ctx.n, b)
    pb, _ = _ptr(b, writable=True, size=2 * ctx.n)
    _order(ctx, b)
    _check(_lib.bipb_source(ctx.handle, pb))
    return b


def bipb_matvec(ctx: Context, u, y=None):
    """Eqs. (12)-(13): y = A u (2n)."""
    y = _out_like(2 * ctx.n, y)
    pu, _ = _ptr(u, size=2 * ctx.n)
    py, _ = _ptr(y, writable=True, size=2 * ctx.n)
    _order(ctx, u, y)
    _check(_lib.bipb_matvec(ctx.handle, pu, py))
    return y


def bipb_matvec_batch(ctx: Context, U, Y=None):
    """Multi-RHS product: Y[r] = A U[r], U and Y of shape [nrhs, 2n] (C-contiguous)."""
    nrhs = int(U.shape[0])
    if Y is None:
        Y = np.empty((nrhs, 2 * ctx.n))
    pu, _ = _ptr(U, size=nrhs * 2 * ctx.n)
    py, _ = _ptr(Y, writable=True, size=nrhs * 2 * ctx.n)
    _order(ctx, U, Y)
    _check(_lib.bipb_matvec_batch(ctx.handle, nrhs, pu, py))
    return Y


def bipb_set_charges(ctx: Context, charges):
    """Replace the point charges [nc, 4] (x, y, z, Q) on the same surface."""
    nc = int(charges.shape[0])
    pq, _ = _ptr(charges, size=4 * nc) if nc > 0 else (None, None)
    _order(ctx, charges)
    _check(_lib.bipb_set_charges(ctx.handle, nc, pq))
    ctx.nc = nc


def bipb_gmres_solve_batch(ctx: Context, B, X, restart_m=20, tol=1e-10, max_iters=500, check_true=False,
                           history_cap=None):
    """Multi-RHS GMRES: solves A X[r] = B[r] for all r in lockstep (X: initial guesses in, solutions
    out).  Returns (status, [report dict per system])."""
    nrhs = int(B.shape[0])
    cap = max_iters + 1 if history_cap is None else history_cap
    hist = np.zeros((nrhs, max(cap, 1)))
    reps = (Report * nrhs)()
    for r in range(nrhs):
        reps[r].history = hist[r].ctypes.data_as(ctypes.POINTER(ctypes.c_double))
        reps[r].history_cap = cap
    pb, _ = _ptr(B, size=nrhs * 2 * ctx.n)
    px, _ = _ptr(X, writable=True, size=nrhs * 2 * ctx.n)
    _order(ctx, B, X)
    st = _lib.bipb_gmres_solve_batch(ctx.handle, nrhs, pb, px, int(restart_m), float(tol), int(max_iters),
                                     int(check_true), reps)
    if st not in (OK, NOT_CONVERGED):
        _check(st)
    out = []
    for r in range(nrhs):
        rp = reps[r]
        out.append({"iterations": rp.iterations, "restarts": rp.restarts, "matvecs": rp.matvecs,
                    "converged": bool(rp.converged), "rel_res_est": rp.rel_res_est, "rel_res_true": rp.rel_res_true,
                    "history": hist[r, :min(rp.history_len, cap)].copy()})
    return st, out


def bipb_gmres_solve(ctx: Context, x, b=None, restart_m=20, tol=1e-10, max_iters=500, check_true=False,
                     history_cap=None, raise_on_not_converged=False):
    """GMRES(m) on the device.  x holds x0 on entry and the solution on
    return.  Returns (status, report dict)."""
    px, _ = _ptr(x, writable=True, size=2 * ctx.n)
    pb, _ = _ptr(b, size=2 * ctx.n)
    cap = max_iters + 1 if history_cap is None else history_cap
    hist = np.zeros(max(cap, 1))
    rep = Report(history=hist.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), history_cap=cap)
    _order(ctx, x, b)
    st = _lib.bipb_gmres_solve(ctx.handle, pb, px, int(restart_m), float(tol), int(max_iters), int(check_true),
                               ctypes.byref(rep))
    if st not in (OK, NOT_CONVERGED) or (st == NOT_CONVERGED and raise_on_not_converged):
        _check(st)
    return st, {"iterations": rep.iterations, "restarts": rep.restarts, "matvecs": rep.matvecs,
                "converged": bool(rep.converged), "rel_res_est": rep.rel_res_est,
                "rel_res_true": rep.rel_res_true, "history": hist[:min(rep.history_len, cap)].copy()}


def bipb_energy(ctx: Context, x, phi_reac=None) -> float:
    """Eq. (14): E_sol [kcal/mol]; optionally fills phi_reac [nc]."""
    px, _ = _ptr(x, size=2 * ctx.n)
    e = np.zeros(1)
    pp, _ = _ptr(phi_reac, writable=True, size=ctx.nc) if phi_reac is not None else (None, None)
    _order(ctx, x, phi_reac)
    _check(_lib.bipb_energy(ctx.handle, px, e.ctypes.data, pp))
    return float(e[0])


def bipb_set_matvec_kernel(ctx: Context, kind: int):
    """0 = row kernel (bitwise rank-count invariant), 1 = symmetric-pair kernel (bipb.h)."""
    ctx.set_matvec_kernel(kind)


def bipb_get_matvec_kernel(ctx: Context) -> int:
    return ctx.matvec_kernel


def bipb_get_exchange(ctx: Context) -> int:
    """0 none, 1 NCCL collectives, 2 peer stores (bipb.h)."""
    return int(_lib.bipb_get_exchange(ctx.handle))


def bipb_set_precond(ctx: Context, kind: int):
    """0 = plain GMRES (the paper), 1 = right preconditioning by the jump-term diagonal (bipb.h)."""
    ctx.set_precond(kind)


def bipb_get_precond(ctx: Context) -> int:
    return ctx.precond


def bipb_set_sum_mode(ctx: Context, mode: int):
    """1 = exact fixed-point limb sums (the default), 0 = fixed-order double partials (bipb.h)."""
    ctx.set_sum_mode(mode)


def bipb_get_sum_mode(ctx: Context) -> int:
    return ctx.sum_mode


def bipb_get_arnoldi(ctx: Context) -> int:
    """0 multi-launch MGS, E > 0 fused cluster Arnoldi kernel (bipb.h)."""
    return int(_lib.bipb_get_arnoldi(ctx.handle))


def bipb_get_graph_cycles(ctx: Context) -> int:
    """GMRES cycles run as one CUDA-graph launch (BIPB_GRAPHS=2; bipb.h)."""
    return int(_lib.bipb_get_graph_cycles(ctx.handle))


def bipb_destroy(ctx: Context):
    ctx.close()


def solve(ctx: Context, x=None, restart_m=20, tol=1e-10, max_iters=500, check_true=False, precond=None):
    """Table 1 pipeline on the device: source -> GMRES -> energy.  Returns dict.
    precond: None keeps the context's setting; 0 plain GMRES (the paper), 1 the opt-in right
    jump-term diagonal preconditioner (bipb_set_precond) for this call only."""
    prev = ctx.precond
    if precond is not None:
        ctx.set_precond(precond)
    try:
        b = bipb_source(ctx, None if x is None or isinstance(x, np.ndarray) else _zeros_like(x))
        if x is None:
            x = np.zeros(2 * ctx.n)
        st, rep = bipb_gmres_solve(ctx, x, None, restart_m, tol, max_iters, check_true)
        e = bipb_energy(ctx, x)
    finally:
        if precond is not None:
            ctx.set_precond(prev)
    return {"b": b, "x": x, "status": st, "report": rep, "energy": e}


def _zeros_like(t):
    return t.new_zeros(t.shape)
