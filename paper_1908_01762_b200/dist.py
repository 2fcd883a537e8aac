"""Process-group plumbing of a slab-decomposed run.

One process per GPU (torchrun).  torch.distributed is plumbing only: it
carries the NCCL unique id from rank 0 to the other ranks and reduces host
scalars (the timing max over ranks).  The data path -- halo exchanges,
migration, the per-sweep allreduce -- runs inside libsisph over NCCL.
"""
from __future__ import annotations

import os

import numpy as np

from .sisph import (Simulation, default_nccl_lib, domain, make_dist, nccl_unique_id, slab_bounds,
                    slab_owner)


def env():
    """(rank, world, local_rank) from the torchrun environment (1 process: 0, 1, 0)."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init_process_group(backend: str):
    import torch.distributed as td
    if not td.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        td.init_process_group(backend)
    return td.get_rank(), td.get_world_size()


def share_nccl_id(rank: int, nccl_lib=None, make=None) -> bytes:
    """Rank 0 draws the NCCL unique id (sisph_nccl_unique_id), every rank gets it."""
    import torch.distributed as td
    box = [None]
    if rank == 0:
        box[0] = (make or nccl_unique_id)(nccl_lib)
    td.broadcast_object_list(box, src=0)
    return box[0]


def max_over_ranks(x: float, device=None) -> float:
    """Max of a host scalar over all ranks (the job's timing is its slowest rank)."""
    import torch
    import torch.distributed as td
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    td.all_reduce(t, op=td.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, device=None) -> float:
    import torch
    import torch.distributed as td
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    td.all_reduce(t, op=td.ReduceOp.SUM)
    return float(t.item())


def owned_ids(case, axis: int, nranks: int, rank: int) -> np.ndarray:
    """Creation ids rank owns at create (sisph_slab_owner on every particle)."""
    dom = domain(case.dim, case.lo, case.hi, case.periodic)
    y = case.x[:, axis]
    return np.array([k for k in range(case.n) if slab_owner(dom, axis, nranks, float(y[k])) == rank], np.int64)


def slab_plan(case, axis: int, nranks: int):
    dom = domain(case.dim, case.lo, case.hi, case.periodic)
    return [slab_bounds(dom, axis, nranks, r) for r in range(nranks)]


def create_rank(case, axis: int, rank: int, world: int, nccl_id: bytes, nccl_lib=None, **overrides) -> Simulation:
    """This rank's handle of the slab-decomposed `case` (every rank passes the global case)."""
    d = make_dist(world, rank, axis, nccl_id=nccl_id, nccl_lib=nccl_lib or default_nccl_lib())
    return Simulation.from_case(case, dist=d, **overrides)
