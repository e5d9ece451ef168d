"""Row-sharded solves over several GPUs of one node (one process per GPU).

SURVEY §8e: rank g holds the contiguous row block [g n / G, (g+1) n / G) of the
cost (or of the source points); u, M, S, w stay local; the only exchange per
evaluation is the all-reduce of the m column partial sums (+ the local <u, a>)
done by libotg over NCCL; the m-vector epilogue runs replicated, so every rank
takes the same stop decision.  This module holds the host side: the row
partition and the NCCL id handshake over an existing torch.distributed group.
"""
from __future__ import annotations

import numpy as np

from . import ot


def shard_rows(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous near-equal row block of `rank` (every row owned exactly once)."""
    if world < 1 or not 0 <= rank < world:
        raise ot.DimensionMismatch("rank outside [0, world)")
    return n * rank // world, n * (rank + 1) // world


def nccl_id_from_group(group=None) -> bytes:
    """Rank 0 draws an ncclUniqueId (libotg) and broadcasts its 128 bytes over
    the torch.distributed group (any backend)."""
    import torch
    import torch.distributed as dist
    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = "cuda" if backend == "nccl" else "cpu"
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(ot.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, 0, group=group)
    return bytes(buf.cpu().numpy())


def gloo_allreduce(group=None):
    """A host all-reduce over a torch.distributed CPU group (gloo) for
    otg_device_opts.allreduce: libotg stages the device buffer through pinned
    memory and calls this from a CUDA host node.  Lets several processes
    exercise the sharded data flow without NCCL (e.g. two ranks on one GPU)."""
    import torch
    import torch.distributed as dist

    def reduce(buf: np.ndarray, op: int) -> None:
        t = torch.from_numpy(buf)  # shares the pinned staging buffer
        dist.all_reduce(t, op=dist.ReduceOp.SUM if op == 0 else dist.ReduceOp.MAX, group=group)

    return reduce


def sharded_points_problem(a, b, x, y, epsilon, world, rank, nccl_id=None, device=None,
                           allreduce=None, **kw):
    """This rank's handle of a row-sharded points problem: only this rank's
    source rows are uploaded (the C-ABI takes the local rows, otg.h)."""
    r0, r1 = shard_rows(len(a), world, rank)
    return ot.TransportProblem.from_points(a, b, np.ascontiguousarray(x[r0:r1]), y, epsilon,
                                           device=rank if device is None else device,
                                           world_size=world, rank=rank, row_begin=r0, row_end=r1,
                                           nccl_unique_id=nccl_id, allreduce=allreduce, **kw)


def sharded_dense_problem(a, b, C, epsilon, world, rank, nccl_id=None, device=None,
                          allreduce=None):
    """This rank's handle of a row-sharded dense problem: C may be the full
    matrix (its rows [r0, r1) are uploaded) -- the C-ABI receives the local
    rows only (otg.h)."""
    r0, r1 = shard_rows(len(a), world, rank)
    p = ot.rescale_problem(ot.make_problem(a, b, C, epsilon))
    return p.to_device(device=rank if device is None else device, world_size=world, rank=rank,
                       row_begin=r0, row_end=r1, nccl_unique_id=nccl_id, allreduce=allreduce)


def gather_u(u_local: np.ndarray, group=None) -> np.ndarray:
    """Concatenate the row potentials of all ranks in rank order."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    t = torch.from_numpy(np.ascontiguousarray(u_local))
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([t.numel()]), group=group)
    mx = int(max(s.item() for s in sizes))
    pad = torch.zeros(mx, dtype=t.dtype)
    pad[: t.numel()] = t
    parts = [torch.zeros(mx, dtype=t.dtype) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return np.concatenate([p[: int(s.item())].numpy() for p, s in zip(parts, sizes)])
