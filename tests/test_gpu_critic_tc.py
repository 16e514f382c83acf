"""GPU parity of the tensor-core Sobolev critic (csrc/critic_tc.cu: per-sample
tcgen05 layers with A in TMEM + batch-reduction GEMMs) against the float64
oracle critic_loss (nets.py:233-290), which is pinned to the reference goldens.

The path runs for fp32 3 x 64 critics at large batches; CACTO_CRITIC_TC_MIN=0
forces it at test sizes.  Tolerances (fp32): loss 1e-5 rel, gradients 1e-4 of
max |grad| (the reference FD metric, test_nets.py:45-49).
"""

import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_2602_19699_b200 as P  # noqa: E402
from paper_2602_19699_b200 import buffer as B_buffer  # noqa: E402
from paper_2602_19699_b200 import nets as B_nets  # noqa: E402
from paper_2602_19699_b200 import specs as B_specs  # noqa: E402
from oracle import envs as O_envs  # noqa: E402
from oracle import nets as O_nets  # noqa: E402


@pytest.fixture(autouse=True)
def tc_forced():
    old = P.get_precision()
    P.set_precision("fp32")
    os.environ["CACTO_CRITIC_TC_MIN"] = "0"
    yield
    os.environ.pop("CACTO_CRITIC_TC_MIN", None)
    P.set_precision(old)


def grads_close(got, ref, tol):
    scale = max(1e-12, max(np.abs(r).max() for r in ref))
    for g, r in zip(got, ref):
        assert g.shape == r.shape
        assert np.abs(g - r).max() / scale < tol, (np.abs(g - r).max() / scale)


def nets(spec, rng, act="elu"):
    c, h = B_specs.normalisation(spec)
    d = spec.n + 1
    mk = lambda: B_nets.init_mlp([d, 64, 64, 64, 1], rng, activation=act, in_center=c, in_half=h)  # noqa: E731
    critic, target = mk(), mk()
    jit = lambda n: n.with_params([p + (rng.normal(0, 0.05, p.shape) if i % 2 else 0)  # noqa: E731
                                   for i, p in enumerate(n.flat_params())])
    return jit(critic), jit(target)


def batch(spec, R, rng):
    lo, hi = O_envs.region_box(spec)
    t = rng.integers(0, spec.t_max, (R, 1)).astype(float)
    xa = np.concatenate([rng.uniform(size=(R, spec.n)) * (hi - lo) + lo, t], 1)
    xk = np.concatenate([rng.uniform(size=(R, spec.n)) * (hi - lo) + lo, rng.integers(1, spec.t_max + 1, (R, 1))], 1)
    return B_buffer.SampleBatch(xa, rng.normal(size=(R, spec.m)), rng.normal(size=R) * 10,
                                rng.normal(size=(R, spec.n)), xk, spec.t_max)


@pytest.mark.parametrize("name", ["toy1d", "pointmass", "dubins", "manipulator3", "aliengo_lipm"])
@pytest.mark.parametrize("boot", [False, True])
def test_critic_tc_vs_oracle(name, boot):
    spec, _ = B_specs.config(name)
    rng = np.random.default_rng(31)
    critic, target = nets(spec, rng)
    b = batch(spec, 1000, rng)
    loss, grads = B_nets.critic_loss(critic, target, b, 0.7, boot)
    ref, ref_g = O_nets.critic_loss(critic, target, b, 0.7, boot)
    assert loss == pytest.approx(ref, rel=1e-5)
    grads_close(grads, ref_g, 1e-4)


@pytest.mark.parametrize("R", [1, 127, 129, 20000])
def test_critic_tc_batch_sizes(R):
    spec, _ = B_specs.config("manipulator3")
    rng = np.random.default_rng(R)
    critic, target = nets(spec, rng)
    b = batch(spec, R, rng)
    loss, grads = B_nets.critic_loss(critic, target, b, 1.0, True)
    ref, ref_g = O_nets.critic_loss(critic, target, b, 1.0, True)
    assert loss == pytest.approx(ref, rel=1e-5)
    grads_close(grads, ref_g, 1e-4)


def test_critic_tc_tanh():
    spec, _ = B_specs.config("dubins")
    rng = np.random.default_rng(33)
    critic, target = nets(spec, rng, act="tanh")
    b = batch(spec, 700, rng)
    loss, grads = B_nets.critic_loss(critic, target, b, 0.5, True)
    ref, ref_g = O_nets.critic_loss(critic, target, b, 0.5, True)
    assert loss == pytest.approx(ref, rel=1e-5)
    grads_close(grads, ref_g, 1e-4)


def test_critic_tc_matches_simt_kernel():
    spec, _ = B_specs.config("dubins")
    rng = np.random.default_rng(34)
    critic, target = nets(spec, rng)
    b = batch(spec, 9000, rng)
    lt, gt = B_nets.critic_loss(critic, target, b, 1.0, True)
    os.environ["CACTO_CRITIC_TC"] = "0"
    try:
        ls, gs = B_nets.critic_loss(critic, target, b, 1.0, True)
    finally:
        os.environ.pop("CACTO_CRITIC_TC", None)
    assert lt == pytest.approx(ls, rel=1e-5)
    grads_close(gt, gs, 1e-4)
