"""N>1 paths on the one available GPU: world-size 2 and 4 gloo process groups
whose ranks share cuda:0 (tests/mp_workers.py).  Every rank runs the real
kernels on its shard; the collectives go through gloo (host-staged).

  * distributed select (csrc/select.cu cacto_dselect_*, parallel.DistributedSelect)
    == np.argsort(-scores, kind="stable")[:keep] over the union of the shards,
    bit-exact (fp32 and fp64 scores, heavy ties, NaN, +-0, uneven shards,
    keep = 1 and keep = N), and each rank's own winners are exactly its shard's
    part of the global set;
  * the sharded rollout+BIC step (BicPipeline.run_sharded) == the single-device
    BicPipeline.run on the same candidates: same global order, and each rank's
    warm starts are the single-device warm starts of its own winners (bitwise);
  * data-parallel UpdateEngine (dp_group) == the 1-rank engine: fp64 losses and
    parameters within 1e-12 rel (only the fold order of the gradient sums
    differs), fp32 within the SURVEY 8(c) loss tolerance 1e-5.
"""

import socket
from pathlib import Path

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

import mp_workers  # noqa: E402


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spawn(fn, world, tmp_path, *args):
    mp.start_processes(fn, args=(world, _port(), str(tmp_path)) + args, nprocs=world, join=True,
                       start_method="spawn")
    return [dict(np.load(Path(tmp_path) / f"rank{r}.npz")) for r in range(world)]


def _scores(kind, N, dtype, seed):
    rng = np.random.default_rng(seed)
    if kind == "ties":
        s = np.round(rng.normal(0, 1, N), 1)
    elif kind == "const":
        s = np.full(N, 0.5)
    else:
        s = rng.normal(0, 1, N)
    s = s.astype(dtype)
    s[rng.integers(0, N, max(1, N // 50))] = np.nan
    s[rng.integers(0, N, max(1, N // 50))] = 0.0
    s[rng.integers(0, N, max(1, N // 50))] = -0.0
    return s


@pytest.mark.parametrize("world", [2, 4])
@pytest.mark.parametrize("dtype", ["f32", "f64"])
@pytest.mark.parametrize("kind,N,keep", [("normal", 100003, 10000), ("ties", 50001, 4999), ("const", 9999, 777),
                                         ("ties", 4097, 4097), ("normal", 3001, 1)])
def test_distributed_select_equals_global_argsort(world, dtype, kind, N, keep, tmp_path):
    s = _scores(kind, N, np.float32 if dtype == "f32" else np.float64, N + world)
    outs = _spawn(mp_workers.dselect_worker, world, tmp_path, s, keep, dtype)
    ref = np.argsort(-s, kind="stable")[:keep]
    mine = []
    for o in outs:
        np.testing.assert_array_equal(o["order"], ref)
        np.testing.assert_array_equal(o["top"].view(np.uint8 if False else o["top"].dtype),
                                      np.where(s[ref] == 0, 0, s[ref]).astype(o["top"].dtype))
        mine.append(o["local"] + int(o["lo"]))
    # every rank holds exactly its own winners, in global order
    got = np.concatenate(mine)
    np.testing.assert_array_equal(np.sort(got), np.sort(ref))
    for o, loc in zip(outs, mine):
        sub = ref[np.isin(ref, loc)]
        np.testing.assert_array_equal(loc, sub)


@pytest.mark.parametrize("name,N", [("dubins", 20000), ("manipulator3", 30001)])
def test_sharded_bic_pipeline_equals_single_device(name, N, tmp_path):
    import paper_2602_19699_b200 as P
    from paper_2602_19699_b200 import specs, trainer
    from bench import make_nets, candidates
    keep = N // 10
    outs = _spawn(mp_workers.bic_worker, 2, tmp_path, name, N, keep)
    P.set_precision("fp32")
    spec, fld = specs.config(name)
    actor, critic, std = make_nets(spec)
    x0 = torch.as_tensor(candidates(spec, 0, N)).cuda()
    pipe = trainer.BicPipeline(spec, fld, actor, critic, std, mode="std_x_gap")
    r = pipe.run(x0, keep)
    order = r["order"].cpu().numpy()
    U = r["U"].cpu().numpy()
    pos = {int(g): i for i, g in enumerate(order)}
    for o in outs:
        # scores are per-candidate (the same kernel on the same start), so the exact
        # select gives the single-device order on every rank
        np.testing.assert_array_equal(o["order"], order)
        glob = o["local"] + int(o["lo"])
        idx = [pos[int(g)] for g in glob]
        np.testing.assert_array_equal(o["U"], U[idx])


@pytest.mark.parametrize("precision,tol", [("fp64", 1e-12), ("fp32", 1e-5)])
def test_dp_update_engine_matches_one_rank(precision, tol, tmp_path):
    import paper_2602_19699_b200 as P
    from dp_setup import engine_setup
    M, B = 5, 50
    outs = _spawn(mp_workers.dp_engine_worker, 2, tmp_path, precision, M, B)
    old = P.get_precision()
    P.set_precision(precision)
    try:
        eng, seed = engine_setup(B)
        closs, sloss = eng.run(M, np.random.default_rng(seed))
        nets = eng.networks()
    finally:
        P.set_precision(old)
    for o in outs:
        np.testing.assert_allclose(o["closs"], closs, rtol=tol)
        np.testing.assert_allclose(o["sloss"], sloss, rtol=tol)
        for i, n in enumerate(nets):
            for j, p in enumerate(n.flat_params()):
                q = o[f"n{i}_{j}"]
                scale = max(np.abs(p).max(), 1e-30)
                assert np.abs(q - p).max() <= 10 * tol * scale, (i, j, np.abs(q - p).max() / scale)
