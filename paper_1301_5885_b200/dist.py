"""Process-group plumbing for the row-sharded multi-GPU path.

torch.distributed is used only to bootstrap: it broadcasts the 128-byte NCCL unique id
created by the library (bipb_nccl_unique_id) and takes maxima over ranks for timing.
The data-path exchange (one all-gather of the 2N-vector per matvec) is done by the
library's own NCCL communicator on its CUDA stream.

Row layout (what every rank's kernels produce and the all-gather reassembles):
  rank p owns element rows [r0_p, r1_p) = bipb_partition(N, P, p), blocks of
  Np = ceil(N / P) rows; its stage buffer is [phi rows (Np) | dphi rows (Np)], the gathered
  buffer is [P][2 Np], and element i of rank p lands at y[i] and y[N + i].
"""
from __future__ import annotations

import os


def env_rank_world():
    return int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)), int(os.environ.get("LOCAL_RANK", 0))


def share_uid(make_uid, rank: int, world: int) -> bytes | None:
    """Rank 0 calls make_uid() (bytes, 128) and every rank returns the same bytes."""
    if world <= 1:
        return None
    import torch.distributed as dist
    obj = [make_uid() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad NCCL unique id broadcast")
    return bytes(uid)


def max_over_ranks(value: float, world: int, device=None) -> float:
    """Maximum of a per-rank scalar (device-timed milliseconds) over all ranks."""
    if world <= 1:
        return float(value)
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def stage_rows(y_rows_phi, y_rows_dphi, np_pad: int):
    """Host model of the per-rank stage buffer [phi | dphi], zero-padded to Np each (tests)."""
    import numpy as np
    st = np.zeros(2 * np_pad)
    st[:len(y_rows_phi)] = y_rows_phi
    st[np_pad:np_pad + len(y_rows_dphi)] = y_rows_dphi
    return st


def unpack_gathered(g, n: int, world: int):
    """Host model of the library's unpack kernel: gathered [world][2 Np] -> y [2n] (tests)."""
    import numpy as np
    np_pad = (n + world - 1) // world
    g = np.asarray(g).reshape(world, 2 * np_pad)
    y = np.empty(2 * n)
    for p in range(world):
        r0 = p * np_pad
        r1 = min(r0 + np_pad, n)
        if r1 <= r0:
            continue
        y[r0:r1] = g[p, :r1 - r0]
        y[n + r0:n + r1] = g[p, np_pad:np_pad + r1 - r0]
    return y
