"""N>1 host logic on CPU: world_size-2 gloo process group.

The shard winners' all-gather + position merge (paper_2602_19699_b200.parallel)
must reproduce the single-device stable argsort exactly, and the DP gradient
all-reduce must sum the per-rank partial gradients.  The CUDA kernels are
replaced by NumPy stand-ins here (test scaffolding only): the collective
plumbing around them is what this test covers; the kernels themselves are
covered by tests/test_gpu_parity.py::test_select_merge_of_shards_equals_global.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_19699_b200 import parallel


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _np_topk(scores, k, base):
    s = scores.numpy()
    o = np.argsort(-s, kind="stable")[:k]
    return torch.as_tensor(o + base, dtype=torch.int64), torch.as_tensor(s[o])


def _np_merge(run_scores, run_index, R, keep):
    s = run_scores.numpy()
    idx = run_index.numpy()
    # (same semantics as cacto_select_merge) NaN after numbers, padding (idx < 0) after NaN,
    # ties by the carried index
    key = np.where(idx < 0, 2.0, np.where(np.isnan(s), 1.0, 0.0))
    o = np.lexsort((idx, np.where(np.isnan(s), 0.0, -s), key))[:keep]
    return torch.as_tensor(idx[o], dtype=torch.int64)


def _worker(rank, world, port, scores_all, x_all, keep, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        N = scores_all.shape[0]
        lo, hi = parallel.shard_range(N, rank, world)
        order, kept_x = parallel.sharded_select(torch.as_tensor(scores_all[lo:hi]),
                                                torch.as_tensor(x_all[lo:hi]), lo, keep,
                                                local_topk=_np_topk, merge_fn=_np_merge)
        g = torch.full((5,), float(rank + 1), dtype=torch.float64)
        parallel.allreduce_grads(g)
        out[rank] = (order.numpy(), kept_x.numpy(), g.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N,keep", [(1000, 100), (999, 37), (64, 64)])
def test_sharded_select_equals_global_argsort(N, keep):
    rng = np.random.default_rng(N)
    scores = np.round(rng.normal(0, 1, N), 1)           # heavy ties across shards
    scores[rng.integers(0, N, 5)] = np.nan
    x = rng.normal(size=(N, 3))
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), scores, x, keep, out), nprocs=world,
                       join=True, start_method="fork")
    ref = np.argsort(-scores, kind="stable")[:keep]
    for r in range(world):
        order, kept_x, g = out[r]
        np.testing.assert_array_equal(order, ref)
        np.testing.assert_array_equal(kept_x, x[ref])
        np.testing.assert_array_equal(g, np.full(5, 3.0))


def test_shard_ranges_partition():
    for total in (0, 1, 7, 65536, 1000003):
        for world in (1, 2, 3, 8):
            rs = [parallel.shard_range(total, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == total
            assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
            sizes = [h - l for l, h in rs]
            assert max(sizes) - min(sizes) <= 1


def _dsel_worker(rank, world, port, scores_all, keep, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dselect_standin import NumpyDselect
        N = scores_all.shape[0]
        lo, hi = parallel.shard_range(N, rank, world)
        ds = parallel.DistributedSelect(hi - lo, keep, torch.float32, kernels=NumpyDselect(hi - lo, keep))
        order, _, local, off = ds.run(torch.as_tensor(scores_all[lo:hi]), lo)
        out[rank] = (order.numpy().copy(), local.numpy().copy() + lo, ds.collectives)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("N,keep,kind", [(1000, 100, "ties"), (999, 37, "normal"), (64, 64, "ties"),
                                         (4001, 400, "const"), (10, 1, "normal")])
def test_distributed_select_host_logic(world, N, keep, kind):
    """DistributedSelect's collectives and tie split (4 histogram all-reduces, one
    all-gather of counts, one all-reduce of the winners) with the device phases
    replaced by a NumPy stand-in: every rank gets the global stable argsort and
    exactly its own winners."""
    rng = np.random.default_rng(N + world)
    s = {"ties": np.round(rng.normal(0, 1, N), 1), "normal": rng.normal(0, 1, N), "const": np.full(N, 2.0)}[kind]
    s = s.astype(np.float32)
    s[rng.integers(0, N, 3)] = np.nan
    s[rng.integers(0, N, 3)] = -0.0
    mgr = mp.Manager()
    out = mgr.dict()
    mp.start_processes(_dsel_worker, args=(world, _free_port(), s, keep, out), nprocs=world, join=True,
                       start_method="fork")
    ref = np.argsort(-s, kind="stable")[:keep]
    mine = []
    for r in range(world):
        order, local, ncoll = out[r]
        np.testing.assert_array_equal(order, ref)
        np.testing.assert_array_equal(local, ref[np.isin(ref, local)])
        assert ncoll == 6
        mine.append(local)
    np.testing.assert_array_equal(np.sort(np.concatenate(mine)), np.sort(ref))
