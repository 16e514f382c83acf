"""The tensor-core rollout (csrc/rollout_tc.cu, fp32 via 3xFP16 tcgen05 MMAs)
across network shapes, activations, batch sizes that switch the tile layout,
per-start start times / horizons, and every output, against the float64 oracle
(itself pinned to the reference goldens) and against the SIMT fp32 kernel.

Tolerances (fp32; chaotic amplification makes a few trajectories diverge, so the
bounds are on the distribution): controls / states / step costs median rel 1e-5
and p99 1e-3 of max(1, |ref|); costs median 1e-5, p99 1e-3.  manipulator3 with a
strong actor is chaotic: median 1e-3, p99 0.2.
"""

import os
import zlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2602_19699_b200 as P  # noqa: E402
from paper_2602_19699_b200 import nets as B_nets  # noqa: E402
from paper_2602_19699_b200 import specs as B_specs  # noqa: E402
from oracle import envs as O_envs  # noqa: E402
from oracle import nets as O_nets  # noqa: E402


@pytest.fixture(autouse=True)
def fp32():
    old = P.get_precision()
    P.set_precision("fp32")
    yield
    P.set_precision(old)


def relerr(a, b):
    # both non-finite (a trajectory that blew up in both arithmetics) counts as
    # agreement; exactly one non-finite as infinite error
    # (|x| > 1e30 counts as blown up too: two such values have no meaningful ratio)
    a, b = np.asarray(a, float), np.asarray(b, float)
    with np.errstate(invalid="ignore", over="ignore"):
        e = np.abs(a - b) / np.maximum(1.0, np.abs(b))
        fa, fb = np.isfinite(a) & (np.abs(a) < 1e30), np.isfinite(b) & (np.abs(b) < 1e30)
    e[~fa & ~fb] = 0.0
    e[fa != fb] = np.inf
    return e


def actor_for(spec, hidden, layers, act, rng, gain=3.0):
    c, h = B_specs.normalisation(spec)
    a = B_nets.init_mlp([spec.n + 1, *[hidden] * layers, spec.m], rng, activation=act, head="tanh",
                        out_scale=spec.u_bound, in_center=c, in_half=h)
    p = list(a.flat_params())
    p[-2] = p[-2] * gain
    p = [q + (rng.normal(0, 0.05, q.shape) if i % 2 == 1 else 0) for i, q in enumerate(p)]  # non-zero biases
    return a.with_params(p)


def check(got, ref, med, p99):
    e = relerr(got, ref).ravel()
    q = np.quantile(e, 0.99, method="higher")  # (no interpolation between inf entries)
    assert np.median(e) < med and q < p99, (np.median(e), q)


SHAPES = [(64, 3, "elu"), (32, 2, "tanh"), (64, 1, "elu"), (32, 3, "elu"), (64, 2, "tanh")]


@pytest.mark.parametrize("name", ["toy1d", "pointmass", "dubins", "manipulator3", "aliengo_lipm"])
@pytest.mark.parametrize("shape", SHAPES, ids=lambda s: f"h{s[0]}x{s[1]}{s[2]}")
def test_tc_rollout_shapes_vs_oracle(name, shape):
    spec, fld = B_specs.config(name)
    rng = np.random.default_rng(zlib.crc32(repr((name, shape)).encode()))
    actor = actor_for(spec, *shape, rng, gain=0.5 if name == "manipulator3" else 3.0)
    x0 = O_envs.sample_initial_states(spec, 300, 7)
    r = B_nets.actor_rollout_batch(actor, spec, x0, 0, None, fld)
    X, U, SC, C = O_nets.actor_rollout_batch(actor, spec, x0, 0, spec.t_max, fld)
    # manipulator3 is chaotic: the p99 over every step of every trajectory
    # depends on where rounding pushes the few diverging arms (0.08-0.13 measured across
    # equivalent fp32 formulations); the tail is bounded against the SIMT-FFMA kernel in
    # tests/test_gpu_contract.py
    med, p99 = (1e-3, 0.2) if name == "manipulator3" else (1e-5, 1e-3)
    check(r["U"], U, med, p99)
    check(r["X"], X, med, p99)
    check(r["step_costs"], SC, med, p99)
    check(r["cost"], C, med, p99)


@pytest.mark.parametrize("N", [1, 127, 129, 513, 40000, 80000])
def test_tc_rollout_tile_layouts(N):
    # N switches between 1 tile / CTA (4 warps per lane quadrant), 2 and 4 tiles
    spec, fld = B_specs.config("dubins")
    rng = np.random.default_rng(N)
    actor = actor_for(spec, 64, 3, "elu", rng)
    x0 = O_envs.sample_initial_states(spec, N, 11)
    r = B_nets.actor_rollout_batch(actor, spec, x0, 0, None, fld, emit=("U", "cost"))
    sub = np.linspace(0, N - 1, min(N, 600)).astype(int)
    _, U, _, C = O_nets.actor_rollout_batch(actor, spec, x0[sub], 0, spec.t_max, fld)
    check(r["U"][sub], U, 1e-5, 1e-3)
    check(r["cost"][sub], C, 1e-5, 1e-3)


def test_tc_rollout_per_start_times_and_horizons():
    # eval / warm-start call sites (trainer.py:192-193, 267-268): t0 per start,
    # horizon t_max - t0 per start
    spec, fld = B_specs.config("pointmass")
    rng = np.random.default_rng(3)
    actor = actor_for(spec, 64, 3, "elu", rng)
    x0 = O_envs.sample_initial_states(spec, 400, 12)
    t0 = rng.integers(0, spec.t_max, 400)
    r = B_nets.actor_rollout_batch(actor, spec, x0, t0, None, fld, emit=("U", "cost", "step_costs"))
    for t in np.unique(t0)[:12]:
        sel = np.nonzero(t0 == t)[0]
        T = spec.t_max - int(t)
        _, U, SC, C = O_nets.actor_rollout_batch(actor, spec, x0[sel], int(t), T, fld)
        check(r["U"][sel, :T], U, 1e-5, 1e-3)
        check(r["step_costs"][sel, :T + 1], SC, 1e-5, 1e-3)
        check(r["cost"][sel], C, 1e-5, 1e-3)


def test_tc_rollout_fixed_short_horizon():
    spec, fld = B_specs.config("dubins")
    rng = np.random.default_rng(4)
    actor = actor_for(spec, 64, 3, "elu", rng)
    x0 = O_envs.sample_initial_states(spec, 1000, 13)
    r = B_nets.actor_rollout_batch(actor, spec, x0, 30, 17, fld)
    X, U, SC, C = O_nets.actor_rollout_batch(actor, spec, x0, 30, 17, fld)
    check(r["U"], U, 1e-5, 1e-3)
    check(r["X"], X, 1e-5, 1e-3)
    check(r["cost"], C, 1e-5, 1e-3)


def test_tc_matches_simt_fp32_kernel():
    # the two fp32 kernels (tensor-core 3xFP16 vs CUDA-core FFMA) agree on the bulk
    spec, fld = B_specs.config("dubins")
    rng = np.random.default_rng(5)
    actor = actor_for(spec, 64, 3, "elu", rng)
    x0 = O_envs.sample_initial_states(spec, 20000, 14)
    tc = B_nets.actor_rollout_batch(actor, spec, x0, 0, None, fld, emit=("U", "cost"))
    os.environ["CACTO_ROLLOUT_TC"] = "0"
    try:
        simt = B_nets.actor_rollout_batch(actor, spec, x0, 0, None, fld, emit=("U", "cost"))
    finally:
        os.environ.pop("CACTO_ROLLOUT_TC", None)
    check(tc["cost"], simt["cost"], 1e-5, 1e-3)
    check(tc["U"], simt["U"], 1e-5, 1e-3)
