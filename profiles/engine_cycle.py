#!/usr/bin/env python
"""UpdateEngine cycle time (trainer.py:208-234 M-cycle loop, pointmass.ini shapes:
B = 128, 3x64 nets): wall time of run(M) with CUDA-graph replay, per cycle."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2602_19699_b200 import buffer as B_buffer, nets as B_nets, specs  # noqa: E402
from paper_2602_19699_b200.device import set_precision  # noqa: E402
from paper_2602_19699_b200.engine import UpdateEngine  # noqa: E402


def build_engine(B=128):
    set_precision("fp32")
    spec, fld = specs.config("pointmass")
    rng = np.random.default_rng(0)
    c, h = specs.normalisation(spec)
    d = spec.n + 1
    mk = lambda out, **kw: B_nets.init_mlp([d, 64, 64, 64, out], rng, in_center=c, in_half=h, **kw)  # noqa: E731
    actor, critic, target, std = mk(spec.m, head="tanh", out_scale=spec.u_bound), mk(1), mk(1), mk(1, head="std")
    R = 20000
    lo, hi = specs.region_box(spec)
    xa = np.concatenate([rng.uniform(size=(R, spec.n)) * (hi - lo) + lo, rng.integers(0, spec.t_max, (R, 1))], 1)
    xk = np.concatenate([rng.uniform(size=(R, spec.n)) * (hi - lo) + lo, rng.integers(1, spec.t_max + 1, (R, 1))], 1)
    buf = B_buffer.ReplayBuffer(spec.n, spec.m, spec.t_max, capacity=1 << 20)
    buf.push_many(B_buffer.SampleBatch(xa, rng.normal(size=(R, spec.m)), rng.normal(size=R), rng.normal(size=(R, spec.n)),
                                       xk, spec.t_max))
    return UpdateEngine(spec, fld, actor, critic, target, std, buf, minibatch=B)


def main(M=1000, B=128):
    eng = build_engine(B)
    eng.run(M, np.random.default_rng(1))
    torch.cuda.synchronize()
    for rep in range(3):
        t = time.perf_counter()
        eng.run(M, np.random.default_rng(2 + rep))
        torch.cuda.synchronize()
        dt = time.perf_counter() - t
        print(f"M={M} B={B}: {dt * 1e3:.1f} ms  ({dt / M * 1e6:.1f} us per critic+actor+std cycle)")


if __name__ == "__main__":
    main()
