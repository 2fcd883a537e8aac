"""Host side of the slab-decomposed (N > 1) path on CPU: two processes over
torch.distributed 'gloo' (world size 2), exercising the helpers bench.py's
multi-GPU run uses (paper_1908_01762_b200.dist) and the library's host-only
slab functions (sisph_slab_bounds / sisph_slab_owner, no GPU needed)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    import torch.distributed as td
    td.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1908_01762_b200 import build
    build.build()
    from paper_1908_01762_b200 import dist as D
    out = {}
    for name, case, axis in (("db3d_y", synth.dambreak3d(nfx=12, nfy=8, nfz=10, dx=1.0 / 32, tank_nx=30, wall_nz=14,
                                                         ranks=world), 1),
                             ("db2d_x", synth.dambreak2d(nx=20, ny=40, dx=0.05), 0)):
        own = D.owned_ids(case, axis, world, rank)
        allown = [None] * world
        td.all_gather_object(allown, own.tolist())
        out[name] = (allown, D.slab_plan(case, axis, world), case.n, case.x[:, axis].tolist(),
                     (case.lo[axis], case.hi[axis]))
    # rank 0 draws the id (a stand-in generator here: no NCCL on a CPU box), all receive the same bytes
    uid = D.share_nccl_id(rank, make=lambda lib: bytes((7 * k + 3) % 256 for k in range(128)))
    ids = [None] * world
    td.all_gather_object(ids, uid)
    out["ids"] = ids
    out["max"] = D.max_over_ranks(10.0 + rank)
    out["sum"] = D.sum_over_ranks(1.0)
    q.put((rank, out))
    td.barrier()
    td.destroy_process_group()


@pytest.fixture(scope="module")
def two_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=300) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert all(p.exitcode == 0 for p in ps)
    return res


def test_ownership_is_a_partition(two_ranks):
    for name in ("db3d_y", "db2d_x"):
        allown, plan, n, y, (lo, hi) = two_ranks[0][name]
        assert allown == two_ranks[1][name][0]          # both ranks computed the same sets
        a, b = set(allown[0]), set(allown[1])
        assert not (a & b) and len(a | b) == n          # each particle owned exactly once
        # slabs are contiguous, equal-width and cover the box
        assert plan[0][0] == lo and plan[-1][1] == hi and plan[0][1] == plan[1][0]
        assert plan[0][1] - plan[0][0] == pytest.approx(plan[1][1] - plan[1][0])
        y = np.asarray(y)
        for r in range(2):
            ys = y[np.asarray(allown[r], np.int64)]
            lo_r, hi_r = plan[r]
            inside = (ys >= lo_r) & (ys < hi_r)
            # outside its slab only below the first / above the last slab of a bounded box
            if r == 0:
                assert np.all(inside | (ys < lo_r))
            else:
                assert np.all(inside | (ys >= hi_r))


def test_nccl_id_broadcast_and_reductions(two_ranks):
    for r in (0, 1):
        out = two_ranks[r]
        assert out["ids"][0] == out["ids"][1] and len(out["ids"][0]) == 128
        assert out["max"] == 11.0
        assert out["sum"] == 2.0
