"""Shared set-up of the data-parallel UpdateEngine tests (same nets / ring on every rank)."""

from __future__ import annotations

import numpy as np


def engine_setup(B, dp_group=None, system="pointmass", R=900):
    from paper_2602_19699_b200 import buffer as B_buffer, nets as B_nets, specs as B_specs
    from paper_2602_19699_b200.engine import UpdateEngine
    spec, fld = B_specs.config(system)
    rng = np.random.default_rng(44)
    c, h = B_specs.normalisation(spec)
    d = spec.n + 1
    actor = B_nets.init_mlp([d, 64, 64, 64, spec.m], rng, head="tanh", out_scale=spec.u_bound, in_center=c,
                            in_half=h)
    critic = B_nets.init_mlp([d, 64, 64, 64, 1], rng, in_center=c, in_half=h)
    target = B_nets.init_mlp([d, 64, 64, 64, 1], rng, in_center=c, in_half=h)
    std = B_nets.init_mlp([d, 64, 64, 64, 1], rng, head="std", in_center=c, in_half=h)
    lo, hi = B_specs.region_box(spec)
    # t up to t_max: some rows are past the horizon (skipped by the actor loss, nets.py:310-312)
    xa = np.concatenate([rng.uniform(size=(R, spec.n)) * (hi - lo) + lo, rng.integers(0, spec.t_max + 1, (R, 1))], 1)
    xk = np.concatenate([rng.uniform(size=(R, spec.n)) * (hi - lo) + lo, rng.integers(1, spec.t_max + 1, (R, 1))], 1)
    buf = B_buffer.ReplayBuffer(spec.n, spec.m, spec.t_max, capacity=1 << 12)
    buf.push_many(B_buffer.SampleBatch(xa, rng.normal(size=(R, spec.m)), rng.normal(size=R) * 10,
                                       rng.normal(size=(R, spec.n)), xk, spec.t_max))
    eng = UpdateEngine(spec, fld, actor, critic, target, std, buf, minibatch=B, dp_group=dp_group)
    return eng, 9
