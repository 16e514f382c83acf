"""Worker bodies for the multi-process GPU tests (tests/test_gpu_multiproc.py).

Each worker is one rank of a gloo process group whose ranks all share cuda:0
(only one GPU is available; gloo collectives stage CUDA tensors through the
host, the rank-local work runs the real sm_100a kernels through the C ABI).
Results go to `<out>/rank<r>.npz`.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def _init(rank, world, port):
    sys.path.insert(0, str(ROOT))
    sys.path.insert(0, str(ROOT / "tests"))
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    return torch, dist


def dselect_worker(rank, world, port, out, scores_all, keep, dtype_name):
    import numpy as np
    torch, dist = _init(rank, world, port)
    try:
        from paper_2602_19699_b200 import parallel
        dt = torch.float32 if dtype_name == "f32" else torch.float64
        N = scores_all.shape[0]
        lo, hi = parallel.shard_range(N, rank, world)
        sc = torch.as_tensor(scores_all[lo:hi]).to("cuda", dt)
        ds = parallel.DistributedSelect(hi - lo, keep, dt)
        order, top, local, off = ds.run(sc, lo)
        np.savez(Path(out) / f"rank{rank}.npz", order=order.cpu().numpy(), top=top.cpu().numpy(),
                 local=local.cpu().numpy(), lo=lo, off=off)
    finally:
        dist.destroy_process_group()


def bic_worker(rank, world, port, out, name, N, keep):
    """BicPipeline.run_sharded on this rank's contiguous shard of N candidates."""
    import numpy as np
    torch, dist = _init(rank, world, port)
    try:
        import paper_2602_19699_b200 as P
        from paper_2602_19699_b200 import parallel, specs, trainer
        from bench import make_nets, candidates
        P.set_precision("fp32")
        spec, fld = specs.config(name)
        actor, critic, std = make_nets(spec)
        lo, hi = parallel.shard_range(N, rank, world)
        x0 = torch.as_tensor(candidates(spec, lo, hi - lo)).cuda()
        pipe = trainer.BicPipeline(spec, fld, actor, critic, std, mode="std_x_gap")
        r = pipe.run_sharded(x0, keep, lo)
        np.savez(Path(out) / f"rank{rank}.npz", order=r["order"].cpu().numpy(), top=r["scores"].cpu().numpy(),
                 local=r["local"].cpu().numpy(), U=r["U"].cpu().numpy(), lo=lo)
    finally:
        dist.destroy_process_group()


def dp_engine_worker(rank, world, port, out, precision, M, B):
    import numpy as np
    torch, dist = _init(rank, world, port)
    try:
        import paper_2602_19699_b200 as P
        from dp_setup import engine_setup
        P.set_precision(precision)
        eng, seed = engine_setup(B, dp_group="world" if world > 1 else None)
        closs, sloss = eng.run(M, np.random.default_rng(seed))
        nets = eng.networks()
        flat = {f"n{i}_{j}": np.asarray(p) for i, n in enumerate(nets) for j, p in enumerate(n.flat_params())}
        np.savez(Path(out) / f"rank{rank}.npz", closs=closs, sloss=sloss, **flat)
    finally:
        dist.destroy_process_group()
